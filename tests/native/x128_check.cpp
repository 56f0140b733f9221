// Host check of the 128-bit window conversions (fixed192.cuh) against the
// 192-bit fixed-point path on random values, including exact ties.
// Built and run by tests/test_fixed_window.py.
#include <cstdint>
#include <cstdio>
#include <random>

#include "../../paper_2111_00655_b200/csrc/fixed192.cuh"

int main(int argc, char** argv) {
  const long iters = argc > 1 ? atol(argv[1]) : 200000;
  std::mt19937_64 rng(1);
  long bad = 0;
  for (long it = 0; it < iters; ++it) {
    const int s = 40 + (int)(rng() % 60);
    int nbits = 1 + (int)(rng() % 125);
    if (nbits + s > 190) nbits = 190 - s;  // the plan's window keeps X * 2^s below 2^192
    uint64_t lo = rng(), hi = rng();
    if (nbits < 64) {
      hi = 0;
      lo &= (1ull << nbits) - 1ull;
    } else if (nbits < 128) {
      hi &= nbits == 64 ? 0ull : ((1ull << (nbits - 64)) - 1ull);
    }
    if (rng() % 3 == 0) lo &= ~((1ull << (rng() % 60)) - 1ull);  // exact ties and short values
    const fx192 v = fx_shl(fx192{{lo, hi, 0ull}}, s);
    const double ref = fx_to_double(v);
    const double got = x128_to_double(lo, hi, s);
    if (ref != got) ++bad;
    fx192 t;
    bool ok_ref = fx_from_double(ref, t) && !fx_any_below(t, s);
    const fx192 tx = fx_shr(t, s);
    ok_ref = ok_ref && tx.w[2] == 0ull && (tx.w[1] >> 62) == 0ull;
    uint64_t l2, h2;
    const bool ok = x128_from_double(ref, s, l2, h2);
    if (ok != ok_ref || (ok && (l2 != tx.w[0] || h2 != tx.w[1]))) ++bad;
  }
  printf("%ld %ld\n", iters, bad);
  return bad != 0;
}
