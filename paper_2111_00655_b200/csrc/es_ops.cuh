// Device-side ES operators shared by the breed kernels (es.cu) and the fused
// breed + fitness kernel (fitness_packed128.cu): Philox4x32-10 draws,
// two-point crossover segment masks, and the thread-per-child generation of
// one child row (tournament selection on 32-bit order keys, crossover,
// mutation by geometric gaps) -- see es.cu for the reference semantics.
#pragma once
#include "cb_internal.cuh"

// Philox4x32-10
struct Philox {
  uint32_t k0, k1;
  uint32_t c[4];
  uint32_t out[4];
  int used;
  __device__ Philox(uint64_t seed, uint32_t c0, uint32_t c1, uint32_t c2) {
    k0 = (uint32_t)seed;
    k1 = (uint32_t)(seed >> 32);
    c[0] = c0;
    c[1] = c1;
    c[2] = c2;
    c[3] = 0;
    used = 4;
  }
  __device__ void refill() {
    uint32_t x0 = c[0], x1 = c[1], x2 = c[2], x3 = c[3];
    uint32_t a0 = k0, a1 = k1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      uint32_t hi0 = __umulhi(0xD2511F53u, x0), lo0 = 0xD2511F53u * x0;
      uint32_t hi1 = __umulhi(0xCD9E8D57u, x2), lo1 = 0xCD9E8D57u * x2;
      uint32_t y0 = hi1 ^ x1 ^ a0, y1 = lo1, y2 = hi0 ^ x3 ^ a1, y3 = lo0;
      x0 = y0;
      x1 = y1;
      x2 = y2;
      x3 = y3;
      a0 += 0x9E3779B9u;
      a1 += 0xBB67AE85u;
    }
    out[0] = x0;
    out[1] = x1;
    out[2] = x2;
    out[3] = x3;
    c[3] += 1;
    used = 0;
  }
  __device__ uint32_t next() {
    if (used == 4) refill();
    // select instead of out[used] so the state stays in registers
    const uint32_t r = used == 0 ? out[0] : (used == 1 ? out[1] : (used == 2 ? out[2] : out[3]));
    ++used;
    return r;
  }
  // uniform in [0, n) (Lemire, with rejection)
  __device__ uint32_t below(uint32_t n) {
    uint64_t m = (uint64_t)next() * n;
    uint32_t l = (uint32_t)m;
    if (l < n) {
      uint32_t t = (uint32_t)(-n) % n;
      while (l < t) {
        m = (uint64_t)next() * n;
        l = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
  // uniform double in (0, 1]
  __device__ double unit() {
    uint64_t hi = next(), lo = next();
    uint64_t v = ((hi << 21) ^ lo) & ((1ull << 53) - 1);
    return ((double)v + 1.0) * (1.0 / 9007199254740992.0);
  }
};

__device__ __forceinline__ uint64_t seg_mask(int64_t lo, int64_t hi, int64_t w) {
  // bits of word w that fall inside [lo, hi)
  int64_t b0 = w * 64, b1 = b0 + 64;
  int64_t s = lo > b0 ? lo : b0, e = hi < b1 ? hi : b1;
  if (s >= e) return 0ull;
  int sb = (int)(s - b0), eb = (int)(e - b0);
  uint64_t upto = eb == 64 ? ~0ull : ((1ull << eb) - 1ull);
  uint64_t from = ~((1ull << sb) - 1ull);
  return upto & from;
}


// Tournament order keys: the fitness quantised to 16 bits against the
// population's finite [min, max] (65535 = infinite), non-decreasing in the
// fitness, so a key order decides a comparison exactly and only equal keys
// read the doubles.  32 MB for 16.7 M parents (vs 64 MB of 32-bit keys).
typedef uint16_t cb_key_t;

// Row of W words (8-byte aligned) in as few requests as its alignment
// allows: 16-byte streaming loads for every aligned word pair, so a 24-byte
// row is two requests instead of three (each request to a sector that is
// still in flight counts as another L2 miss).
template <int W>
__device__ __forceinline__ void load_row_cs(const uint64_t* __restrict__ row, uint64_t (&v)[W]) {
  const bool odd = (reinterpret_cast<uintptr_t>(row) & 8u) != 0u;
  if (W == 1) {
    v[0] = __ldcs(row);
    return;
  }
  if (odd) {
    v[0] = __ldcs(row);
#pragma unroll
    for (int w = 1; w + 1 < W; w += 2) {
      const ulonglong2 x = __ldcs(reinterpret_cast<const ulonglong2*>(row + w));
      v[w] = x.x;
      v[w + 1] = x.y;
    }
    if (W % 2 == 0) v[W - 1] = __ldcs(row + W - 1);
  } else {
#pragma unroll
    for (int w = 0; w + 1 < W; w += 2) {
      const ulonglong2 x = __ldcs(reinterpret_cast<const ulonglong2*>(row + w));
      v[w] = x.x;
      v[w + 1] = x.y;
    }
    if (W % 2 == 1) v[W - 1] = __ldcs(row + W - 1);
  }
}

// Tournament key gather with an L2 evict-last hint: the parent rows and
// child rows stream past with evict-first, the keys are re-read ~128 times
// per 32-byte sector within one generation.
__device__ __forceinline__ uint32_t ld_key(const cb_key_t* p) {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  unsigned short v;
  asm("ld.global.nc.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(pol));
  return v;
}

// Parameters of one generation's breeding (device pointers).
struct BreedArgs {
  int32_t k;
  const uint64_t* parents;
  const double* fit;
  const cb_key_t* keys;
  int64_t n_parents;
  const uint64_t* keep;
  int64_t n_keep;
  uint64_t seed;
  uint32_t generation, stream_id;
  int32_t tournament;
  double rate, log1m_rate;
};

// Two tournaments of size TOUR (same draws and winners as the loop form:
// first draw leads, a challenger wins only when strictly fitter).
template <int TOUR>
__device__ __forceinline__ void tournament_pair(Philox& rng, int64_t n_parents, const cb_key_t* __restrict__ keys,
                                                const double* __restrict__ fit, int64_t& pa, int64_t& pb) {
  uint32_t idx[2 * TOUR], kv[2 * TOUR];
#pragma unroll
  for (int q = 0; q < 2 * TOUR; ++q) idx[q] = rng.below((uint32_t)n_parents);
#pragma unroll
  for (int q = 0; q < 2 * TOUR; ++q) kv[q] = ld_key(keys + idx[q]);
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    uint32_t best = idx[t * TOUR], bk = kv[t * TOUR];
#pragma unroll
    for (int j = 1; j < TOUR; ++j) {
      const uint32_t i = idx[t * TOUR + j], ki = kv[t * TOUR + j];
      if (ki < bk || (ki == bk && __ldg(fit + i) < __ldg(fit + best))) {
        best = i;
        bk = ki;
      }
    }
    if (t == 0) pa = best;
    else pb = best;
  }
}

// Child row `child` of a generation into v[0..W): the kept elite rows first,
// then tournament / crossover / mutation children (Philox keyed by seed,
// countered by child, generation and stream).
template <int W>
__device__ __forceinline__ void make_child(uint64_t (&v)[W], int32_t k, const uint64_t* __restrict__ parents,
                                           const double* __restrict__ fit, const cb_key_t* __restrict__ keys,
                                           int64_t n_parents, int64_t child, const uint64_t* __restrict__ keep,
                                           int64_t n_keep, uint64_t seed, uint32_t generation, uint32_t stream_id,
                                           int32_t tournament, double rate, double log1m_rate) {
  if (child < n_keep) {
#pragma unroll
    for (int w = 0; w < W; ++w) v[w] = keep[child * W + w];
  } else {
    Philox rng(seed, (uint32_t)child, (uint32_t)(child >> 32) ^ (generation * 0x9E3779B9u),
               stream_id);
    int64_t pa = 0, pb = 0;
    // tournaments compare the 16-bit order keys (an L2-resident array), the
    // full doubles only on a key tie; the default size draws all indices
    // first so the key gathers are in flight together
    if (tournament == 4) {
      tournament_pair<4>(rng, n_parents, keys, fit, pa, pb);
    } else {
      for (int t = 0; t < 2; ++t) {
        int64_t best = rng.below((uint32_t)n_parents);
        uint32_t bk = ld_key(keys + best);
        for (int j = 1; j < tournament; ++j) {
          const int64_t i = rng.below((uint32_t)n_parents);
          const uint32_t ki = ld_key(keys + i);
          if (ki < bk || (ki == bk && __ldg(fit + i) < __ldg(fit + best))) {
            best = i;
            bk = ki;
          }
        }
        if (t == 0) pa = best;
        else pb = best;
      }
    }
    int64_t ci = 0, cj = 0;
    if (k >= 2) {
      const int64_t x = rng.below((uint32_t)(k + 1)), y = rng.below((uint32_t)(k + 1));
      ci = x < y ? x : y;
      cj = x < y ? y : x;
    }
    // parent rows and child rows stream through L2 with evict-first
    // priority so the tournament keys stay resident
    uint64_t ra[W], rb[W];
    load_row_cs<W>(parents + pa * W, ra);
    load_row_cs<W>(parents + pb * W, rb);
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint64_t mb = seg_mask(ci, cj, w);
      v[w] = (ra[w] & ~mb) | (rb[w] & mb);
    }
    if (rate >= 1.0 || rate * (double)k > 8.0) {
      for (int64_t bit = 0; bit < k; ++bit) {
        const double u = ((double)(rng.next() >> 8) + 0.5) * (1.0 / 16777216.0);
        if (u < rate) {
#pragma unroll
          for (int w = 0; w < W; ++w)
            if (w == (bit >> 6)) v[w] ^= 1ull << (bit & 63);
        }
      }
    } else if (rate > 0.0) {
      int64_t pos = -1;
      while (true) {
        const double gap = floor(log(rng.unit()) / log1m_rate);
        if (!(gap < (double)k)) break;
        pos += 1 + (int64_t)gap;
        if (pos >= k) break;
#pragma unroll
        for (int w = 0; w < W; ++w)
          if (w == (pos >> 6)) v[w] ^= 1ull << (pos & 63);
      }
    }
    if (k % 64) {  // clear padding bits past the genome (static indexing keeps v in registers)
#pragma unroll
      for (int w = 0; w < W; ++w)
        if (w == ((k - 1) >> 6)) v[w] &= (1ull << (k % 64)) - 1ull;
    }
  }
}
