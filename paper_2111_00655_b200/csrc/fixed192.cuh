// Exact fixed-point accumulator shared by host plan builders and device kernels.
//
// The reference prices every placement with math.fsum, i.e. the exactly
// rounded sum of its double terms (tensorplace/cost.py:300-305, :370-373).
// Sums here are carried exactly in a 192-bit unsigned fixed-point number
// (value = w[2]:w[1]:w[0] * 2^-128, range [0, 2^64)), which makes addition
// associative, and are rounded to the nearest double (ties to even) once at
// the end -- the same result fsum produces.  A double converts exactly when
// its least significant bit is >= 2^-128 and it is < 2^64; anything else sets
// the caller's `inexact` flag instead of silently losing bits.
#pragma once
#ifdef __CUDACC_RTC__  // NVRTC (jit.cu): no host headers
typedef unsigned long long uint64_t;
typedef unsigned int uint32_t;
typedef int int32_t;
typedef long long int64_t;
#else
#include <stdint.h>
#endif

#ifdef __CUDACC__
#define FXI __host__ __device__ __forceinline__
#else
#define FXI inline
#endif

struct fx192 {
  uint64_t w[3];
};

FXI fx192 fx_zero() {
  fx192 r;
  r.w[0] = r.w[1] = r.w[2] = 0;
  return r;
}

FXI bool fx_is_zero(const fx192& a) { return (a.w[0] | a.w[1] | a.w[2]) == 0; }

// a += b (mod 2^192)
FXI void fx_add(fx192& a, const fx192& b) {
#ifdef __CUDA_ARCH__
  // one carry chain (IADD3 with carry predicates) instead of compare-based carries
  asm("add.cc.u64 %0, %0, %3;\n\t"
      "addc.cc.u64 %1, %1, %4;\n\t"
      "addc.u64 %2, %2, %5;"
      : "+l"(a.w[0]), "+l"(a.w[1]), "+l"(a.w[2])
      : "l"(b.w[0]), "l"(b.w[1]), "l"(b.w[2]));
  return;
#endif
  uint64_t s0 = a.w[0] + b.w[0];
  uint64_t c0 = s0 < a.w[0];
  uint64_t t1 = a.w[1] + b.w[1];
  uint64_t c1 = t1 < a.w[1];
  uint64_t s1 = t1 + c0;
  c1 += s1 < t1;
  a.w[0] = s0;
  a.w[1] = s1;
  a.w[2] = a.w[2] + b.w[2] + c1;
}

// a -= b (mod 2^192); exact whenever the true result is non-negative
FXI void fx_sub(fx192& a, const fx192& b) {
#ifdef __CUDA_ARCH__
  asm("sub.cc.u64 %0, %0, %3;\n\t"
      "subc.cc.u64 %1, %1, %4;\n\t"
      "subc.u64 %2, %2, %5;"
      : "+l"(a.w[0]), "+l"(a.w[1]), "+l"(a.w[2])
      : "l"(b.w[0]), "l"(b.w[1]), "l"(b.w[2]));
  return;
#endif
  uint64_t d0 = a.w[0] - b.w[0];
  uint64_t br0 = a.w[0] < b.w[0];
  uint64_t t1 = a.w[1] - b.w[1];
  uint64_t br1 = a.w[1] < b.w[1];
  uint64_t d1 = t1 - br0;
  br1 += t1 < br0;
  a.w[0] = d0;
  a.w[1] = d1;
  a.w[2] = a.w[2] - b.w[2] - br1;
}

FXI int fx_cmp(const fx192& a, const fx192& b) {
  if (a.w[2] != b.w[2]) return a.w[2] < b.w[2] ? -1 : 1;
  if (a.w[1] != b.w[1]) return a.w[1] < b.w[1] ? -1 : 1;
  if (a.w[0] != b.w[0]) return a.w[0] < b.w[0] ? -1 : 1;
  return 0;
}

FXI bool fx_eq(const fx192& a, const fx192& b) {
  return a.w[0] == b.w[0] && a.w[1] == b.w[1] && a.w[2] == b.w[2];
}

FXI uint64_t fx_bits_of(double d) {
#ifdef __CUDA_ARCH__
  return (uint64_t)__double_as_longlong(d);
#else
  union { double d; uint64_t u; } c;
  c.d = d;
  return c.u;
#endif
}

FXI double fx_double_of(uint64_t u) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)u);
#else
  union { double d; uint64_t u; } c;
  c.u = u;
  return c.d;
#endif
}

// Exact conversion of a non-negative finite double.  Returns false (and
// leaves the best truncated value in `out`) if bits would be lost or the
// value is negative, non-finite or >= 2^64.
FXI bool fx_from_double(double d, fx192& out) {
  out = fx_zero();
  uint64_t bits = fx_bits_of(d);
  if (bits == 0) return true;                        // +0.0
  if (bits >> 63) return bits == 0x8000000000000000ull;  // -0.0 ok, negatives not
  int ex = (int)((bits >> 52) & 0x7ff);
  uint64_t mant = bits & ((1ull << 52) - 1);
  if (ex == 0x7ff) return false;                     // inf / nan
  int e;
  if (ex == 0) {
    e = -1074;
  } else {
    mant |= 1ull << 52;
    e = ex - 1075;
  }
  int s = e + 128;  // bit position of the mantissa LSB inside the 192-bit word
  bool exact = true;
  if (s < 0) {
    int sh = -s;
    if (sh >= 64) {
      return false;  // everything (non-zero) would be lost
    }
    if (mant & ((1ull << sh) - 1)) exact = false;
    mant >>= sh;
    s = 0;
  }
  if (s + 53 > 192) return false;  // >= 2^64
  // static-index placement (no dynamic limb indexing -> stays in registers)
  const int limb = s >> 6;
  const int off = s & 63;
  const uint64_t lo = mant << off;
  const uint64_t hi = off ? (mant >> (64 - off)) : 0ull;
  out.w[0] = limb == 0 ? lo : 0ull;
  out.w[1] = limb == 0 ? hi : (limb == 1 ? lo : 0ull);
  out.w[2] = limb == 1 ? hi : (limb == 2 ? lo : 0ull);
  return exact;
}

FXI int fx_clz64(uint64_t x) {
#ifdef __CUDA_ARCH__
  return __clzll((long long)x);
#else
  return x ? __builtin_clzll(x) : 64;
#endif
}

// bits [s, s+64) of the 192-bit value (s in [0, 192)); static indexing only
FXI uint64_t fx_window(const fx192& a, int s) {
  const int l = s >> 6, o = s & 63;
  const uint64_t x0 = l == 0 ? a.w[0] : (l == 1 ? a.w[1] : a.w[2]);
  const uint64_t x1 = l == 0 ? a.w[1] : (l == 1 ? a.w[2] : 0ull);
  return o ? ((x0 >> o) | (x1 << (64 - o))) : x0;
}

// any bit strictly below position s (s in [0, 192])
FXI bool fx_any_below(const fx192& a, int s) {
  const uint64_t m0 = s >= 64 ? ~0ull : ((1ull << s) - 1);
  const uint64_t m1 = s >= 128 ? ~0ull : (s <= 64 ? 0ull : ((1ull << (s - 64)) - 1));
  const uint64_t m2 = s >= 192 ? ~0ull : (s <= 128 ? 0ull : ((1ull << (s - 128)) - 1));
  return ((a.w[0] & m0) | (a.w[1] & m1) | (a.w[2] & m2)) != 0ull;
}

// Round to the nearest double, ties to even (what math.fsum returns).
FXI double fx_to_double(const fx192& a) {
  const int limb = a.w[2] ? 2 : (a.w[1] ? 1 : (a.w[0] ? 0 : -1));
  if (limb < 0) return 0.0;
  const uint64_t top = limb == 2 ? a.w[2] : (limb == 1 ? a.w[1] : a.w[0]);
  int p = limb * 64 + 63 - fx_clz64(top);  // index of the MSB
  uint64_t m;
  if (p <= 52) {
    m = a.w[0];  // fits exactly; p <= 52 implies limb 0
  } else {
    const int sh = p - 52;  // drop `sh` low bits (1 <= sh <= 139)
    const uint64_t win = fx_window(a, sh - 1);  // round bit at bit 0, mantissa above
    m = (win >> 1) & ((1ull << 53) - 1);
    const bool round_bit = win & 1ull;
    const bool sticky = fx_any_below(a, sh - 1);
    if (round_bit && (sticky || (m & 1ull))) {
      m += 1;
      if (m == (1ull << 53)) {
        m >>= 1;
        p += 1;
      }
    }
  }
  if (p <= 52) {
    // value = m * 2^-128 with m < 2^53: exact, normalised below
    int q = 63 - fx_clz64(m);  // MSB of m
    int ex = q - 128;          // unbiased exponent of the result
    uint64_t frac = (m << (52 - q)) & ((1ull << 52) - 1);
    return fx_double_of(((uint64_t)(ex + 1023) << 52) | frac);
  }
  int ex = p - 128;
  uint64_t frac = m & ((1ull << 52) - 1);
  if (ex > 1023) return fx_double_of(0x7ff0000000000000ull);
  return fx_double_of(((uint64_t)(ex + 1023) << 52) | frac);
}

// ---------------------------------------------------------------- windows
// Plans whose every value is a multiple of 2^(s-128) and small enough can be
// carried as 128-bit integers X = v >> s (value X * 2^(s-128)); these move
// between the two forms exactly.

// a << s (0 <= s < 192), bits past 2^192 dropped; static indexing only
FXI fx192 fx_shl(const fx192& a, int s) {
  const int q = s >> 6, r = s & 63;
  const uint64_t b0 = q == 0 ? a.w[0] : 0ull;
  const uint64_t b1 = q == 0 ? a.w[1] : (q == 1 ? a.w[0] : 0ull);
  const uint64_t b2 = q == 0 ? a.w[2] : (q == 1 ? a.w[1] : a.w[0]);
  fx192 o;
  o.w[0] = b0 << r;
  o.w[1] = (b1 << r) | (r ? b0 >> (64 - r) : 0ull);
  o.w[2] = (b2 << r) | (r ? b1 >> (64 - r) : 0ull);
  return o;
}

// a >> s (0 <= s < 192), logical
FXI fx192 fx_shr(const fx192& a, int s) {
  const int q = s >> 6, r = s & 63;
  const uint64_t b0 = q == 0 ? a.w[0] : (q == 1 ? a.w[1] : a.w[2]);
  const uint64_t b1 = q == 0 ? a.w[1] : (q == 1 ? a.w[2] : 0ull);
  const uint64_t b2 = q == 0 ? a.w[2] : 0ull;
  fx192 o;
  o.w[0] = (b0 >> r) | (r ? b1 << (64 - r) : 0ull);
  o.w[1] = (b1 >> r) | (r ? b2 << (64 - r) : 0ull);
  o.w[2] = b2 >> r;
  return o;
}

// index of the lowest set bit (192 if zero) / highest set bit (-1 if zero)
FXI int fx_lowest_bit(const fx192& a) {
  for (int l = 0; l < 3; ++l)
    if (a.w[l]) {
      uint64_t x = a.w[l];
      int b = 0;
      while (!(x & 1ull)) {
        x >>= 1;
        ++b;
      }
      return l * 64 + b;
    }
  return 192;
}
FXI int fx_highest_bit(const fx192& a) {
  for (int l = 2; l >= 0; --l)
    if (a.w[l]) return l * 64 + 63 - fx_clz64(a.w[l]);
  return -1;
}

// ------------------------------------------------------ 128-bit window
// A value carried in a plan's 128-bit window is X * 2^(s-128) with X a
// non-negative integer below 2^126 (region sums and terms).  These convert
// it to and from double directly, without the 192-bit detour: round to
// nearest, ties to even (as fx_to_double); the reverse conversion reports
// bits that would be lost.

FXI double fx_pow2(int k) {  // 2^k for -1022 <= k <= 1023
  return fx_double_of((uint64_t)(k + 1023) << 52);
}

// low 64 bits of (hi:lo) >> k, 0 <= k < 128
FXI uint64_t x128_shr64(uint64_t lo, uint64_t hi, int k) {
  if (k == 0) return lo;
  if (k < 64) return (lo >> k) | (hi << (64 - k));
  if (k == 64) return hi;
  return hi >> (k - 64);
}

// any of the low k bits of hi:lo set, 0 <= k <= 128
FXI bool x128_low_nonzero(uint64_t lo, uint64_t hi, int k) {
  if (k == 0) return false;
  if (k < 64) return (lo & ((1ull << k) - 1ull)) != 0ull;
  if (k == 64) return lo != 0ull;
  if (k < 128) return lo != 0ull || (hi & ((1ull << (k - 64)) - 1ull)) != 0ull;
  return (lo | hi) != 0ull;
}

// X = hi:lo (X < 2^126), value X * 2^(s-128), rounded to the nearest double
FXI double x128_to_double(uint64_t lo, uint64_t hi, int s) {
  if ((lo | hi) == 0ull) return 0.0;
  const int msb = hi ? 127 - fx_clz64(hi) : 63 - fx_clz64(lo);
  if (msb <= 52) return (double)lo * fx_pow2(s - 128);  // exact: X < 2^53
  const int sh = msb - 52;                                // 1 .. 73 bits dropped
  uint64_t m = x128_shr64(lo, hi, sh) & ((1ull << 53) - 1ull);
  const bool round_bit = (x128_shr64(lo, hi, sh - 1) & 1ull) != 0ull;
  const bool sticky = x128_low_nonzero(lo, hi, sh - 1);
  int e = sh;
  if (round_bit && (sticky || (m & 1ull))) {
    m += 1ull;
    if (m == (1ull << 53)) {
      m >>= 1;
      e += 1;
    }
  }
  return (double)m * fx_pow2(e + s - 128);
}

// d (non-negative, finite) as X with value X * 2^(s-128); false when bits
// below 2^(s-128) would be lost or X would reach 2^126
FXI bool x128_from_double(double d, int s, uint64_t& lo, uint64_t& hi) {
  lo = hi = 0ull;
  const uint64_t bits = fx_bits_of(d);
  if ((bits << 1) == 0ull) return true;  // +0.0 / -0.0
  if (bits >> 63) return false;
  const int ex = (int)((bits >> 52) & 0x7ff);
  if (ex == 0x7ff) return false;
  uint64_t m = bits & ((1ull << 52) - 1ull);
  int e;
  if (ex == 0) {
    e = -1074;
  } else {
    m |= 1ull << 52;
    e = ex - 1075;
  }
  const int t = e + 128 - s;  // X = m * 2^t
  if (t < 0) {
    if (t <= -64) return false;  // m != 0: all bits would be lost
    if (m & ((1ull << -t) - 1ull)) return false;
    lo = m >> -t;
    return true;
  }
  if (t + 53 > 126) return false;
  if (t == 0) {
    lo = m;
  } else if (t < 64) {
    lo = m << t;
    hi = m >> (64 - t);
  } else {
    hi = m << (t - 64);
  }
  return true;
}
