// Sparse warp-per-genome walk of the frontier program, for plans whose
// frontier is too wide for the thread-per-genome kernels (17..128 slots;
// e.g. the 100k-op random DAG needs 36).
//
// Same semantics as the other fitness kernels (tensorplace/evolution.py:
// 256-371 decode, tensorplace/cost.py:320-373 graph-level pricing): the
// on units of a genome form regions = connected components of the dynamic
// unit graph restricted to on units; the fitness is the exact sum of the
// plan constant, minus the removed op-kernel terms of on units, plus one
// term round(round(sum) * r(cnt)) + eps per region, rounded once.
//
// One warp evaluates one genome.  Lane l owns frontier slots l, l+32, ...
// (SPL slots per lane) and keeps their state in registers: the slot's
// component label, the program position after which its unit has no
// neighbour left ("end"), and -- for a component's anchor slot -- the exact
// component sum, kernel count and single-unit id.  Control flow is warp
// uniform (one genome), so nothing diverges.
//
// Only ON units are visited: the warp jumps from one set genome bit (or
// fixed unit) to the next.  Slots whose unit ended before the visited
// position are released lazily, all lanes at once.  A component's data
// lives at its anchor = the member slot with the latest end, so a
// component is complete exactly when its anchor is released; releasing any
// other member is a bit clear.  On a merge the anchor with the later end
// survives and the loser's lanes relabel in parallel.  Closed multi-unit
// regions are queued per warp and priced 32 at a time, one per lane; every
// lane accumulates its own partial total and a shuffle reduction finishes
// the genome.
#include "fitness_plan.cuh"

#define WD_THREADS 128
#define WD_QCAP (32 + 32)  // < 32 queued before a batch of <= 32 insertions

namespace {

struct WideArgs {
  int32_t M, words, k;
  fx192 base_const, eps;
  const UnitRec* __restrict__ prog;
  const uint8_t* __restrict__ slots;
  const int32_t* __restrict__ last;
  const int32_t* __restrict__ pos_of_bit;
  const int32_t* __restrict__ fixed_pos;
  const uint64_t* __restrict__ infeas;
  const double* __restrict__ rt;
  unsigned long long* flags;
};

__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src) {
  return (uint64_t)__shfl_sync(0xffffffffu, (long long)v, src);
}

__device__ __forceinline__ fx192 shfl_xor_fx(const fx192& v, int m) {
  fx192 r;
  r.w[0] = (uint64_t)__shfl_xor_sync(0xffffffffu, (long long)v.w[0], m);
  r.w[1] = (uint64_t)__shfl_xor_sync(0xffffffffu, (long long)v.w[1], m);
  r.w[2] = (uint64_t)__shfl_xor_sync(0xffffffffu, (long long)v.w[2], m);
  return r;
}

// Slot state of one lane: SPL slots, statically indexed.
template <int SPL>
struct Lane {
  int32_t lab[SPL];     // component label (anchor slot) of each owned slot
  int32_t endp[SPL];    // end position of the slot's unit
  int32_t cnt[SPL];     // kernels of the component (anchor slots)
  int32_t single[SPL];  // program position of a one-unit component, -1 merged
  uint64_t s0[SPL], s1[SPL], s2[SPL];  // exact component sum (anchor slots)
};

template <int SPL>
__device__ __forceinline__ int32_t pick(const int32_t (&a)[SPL], int h) {
  int32_t v = a[0];
#pragma unroll
  for (int i = 1; i < SPL; ++i)
    if (h == i) v = a[i];
  return v;
}
template <int SPL>
__device__ __forceinline__ uint64_t pick(const uint64_t (&a)[SPL], int h) {
  uint64_t v = a[0];
#pragma unroll
  for (int i = 1; i < SPL; ++i)
    if (h == i) v = a[i];
  return v;
}

// Price queued regions [0, n) (lane i takes entry i) into the lanes' totals.
__device__ __forceinline__ void wd_price(const uint64_t* q, int n, int lane, const WideArgs& a,
                                         fx192& tacc, bool& inexact) {
  if (lane < n) {
    const fx192 sum = {{q[lane], q[WD_QCAP + lane], q[2 * WD_QCAP + lane]}};
    const int32_t c = (int32_t)q[3 * WD_QCAP + lane];
    const double prod = __dmul_rn(fx_to_double(sum), __ldg(a.rt + c));
    fx192 term;
    inexact |= !fx_from_double(prod, term);
    fx_add(term, a.eps);
    fx_add(tacc, term);
  }
}

// Release every owned active slot whose unit ended before position `p`;
// anchors close their region (one-unit regions add their precomputed term,
// multi-unit regions go to the warp queue).
template <int SPL>
__device__ __forceinline__ void wd_release(Lane<SPL>& L, uint32_t (&act)[SPL], int32_t p, int lane,
                                           uint64_t* q, int& qn, const WideArgs& a, fx192& tacc,
                                           bool& inexact) {
#pragma unroll
  for (int h = 0; h < SPL; ++h) {
    const bool mine = ((act[h] >> lane) & 1u) && L.endp[h] < p;
    const unsigned rel = __ballot_sync(0xffffffffu, mine);
    if (!rel) continue;
    act[h] &= ~rel;
    const bool anchor = mine && L.lab[h] == lane + 32 * h;
    const bool multi = anchor && L.single[h] < 0;
    if (anchor && !multi) {
      const UnitRec* r = a.prog + L.single[h];
      const fx192 t = {{__ldg(&r->term1.w[0]), __ldg(&r->term1.w[1]), __ldg(&r->term1.w[2])}};
      fx_add(tacc, t);
    }
    const unsigned em = __ballot_sync(0xffffffffu, multi);
    if (em) {
      if (multi) {
        const int at = qn + __popc(em & ((1u << lane) - 1u));
        q[at] = L.s0[h];
        q[WD_QCAP + at] = L.s1[h];
        q[2 * WD_QCAP + at] = L.s2[h];
        q[3 * WD_QCAP + at] = (uint64_t)(uint32_t)L.cnt[h];
      }
      qn += __popc(em);
      if (qn >= 32) {
        __syncwarp();
        wd_price(q, 32, lane, a, tacc, inexact);
        __syncwarp();
        if (lane < qn - 32) {
          q[lane] = q[32 + lane];
          q[WD_QCAP + lane] = q[WD_QCAP + 32 + lane];
          q[2 * WD_QCAP + lane] = q[2 * WD_QCAP + 32 + lane];
          q[3 * WD_QCAP + lane] = q[3 * WD_QCAP + 32 + lane];
        }
        qn -= 32;
      }
      __syncwarp();
    }
  }
}

template <int SPL>
__global__ void __launch_bounds__(WD_THREADS)
fitness_wide_kernel(WideArgs a, const uint64_t* __restrict__ pop, int64_t n, double* __restrict__ fit,
                    const int64_t* __restrict__ list, const int32_t* __restrict__ list_count) {
  // list != nullptr: evaluate genomes list[0 .. *list_count) only
  if (list) n = *list_count;
  __shared__ uint64_t queue[WD_THREADS / 32][4 * WD_QCAP];
  const int lane = threadIdx.x & 31;
  uint64_t* q = queue[threadIdx.x >> 5];
  bool inexact = false;
  const int64_t warps = (int64_t)gridDim.x * (WD_THREADS / 32);
  for (int64_t gi = (int64_t)blockIdx.x * (WD_THREADS / 32) + (threadIdx.x >> 5); gi < n; gi += warps) {
    const int64_t g = list ? list[gi] : gi;
    const uint64_t* gen = pop + g * a.words;
    bool dead = false;
    for (int32_t w = lane; w < a.words; w += 32) dead |= (gen[w] & __ldg(a.infeas + w)) != 0ull;
    if (__any_sync(0xffffffffu, dead)) {
      if (lane == 0) fit[g] = __longlong_as_double(0x7ff0000000000000ll);
      continue;
    }
    Lane<SPL> L;
    uint32_t act[SPL];
#pragma unroll
    for (int h = 0; h < SPL; ++h) {
      act[h] = 0u;
      L.lab[h] = -1;
      L.endp[h] = 0;
      L.cnt[h] = 0;
      L.single[h] = -1;
      L.s0[h] = L.s1[h] = L.s2[h] = 0ull;
    }
    fx192 tacc = fx_zero();
    int qn = 0;
    int32_t wi = 0;
    uint64_t cur = a.words > 0 ? gen[0] : 0ull;
    int32_t fi = 0;
    int32_t next_fixed = __ldg(a.fixed_pos);
    for (;;) {
      // next visited position: the next set genome bit or the next fixed unit
      while (cur == 0ull && wi + 1 < a.words) cur = gen[++wi];
      int32_t pb = a.M;
      if (cur) {
        const int32_t b = wi * 64 + __ffsll((long long)cur) - 1;
        if (b < a.k)
          pb = __ldg(a.pos_of_bit + b);
        else
          cur = 0ull;  // padding bits past the genome are ignored
      }
      int32_t p;
      if (pb < next_fixed) {
        p = pb;
        cur &= cur - 1ull;
      } else {
        p = next_fixed;
        if (p >= a.M) break;
        next_fixed = __ldg(a.fixed_pos + ++fi);
      }
      wd_release<SPL>(L, act, p, lane, q, qn, a, tacc, inexact);
      // open the unit in its slot
      const UnitRec* r = a.prog + p;
      const uint4 meta = __ldg(reinterpret_cast<const uint4*>(&r->back_off));
      // meta.x = back_off, meta.y = end_off, meta.z = slot | nback << 8 | nend << 16, meta.w = bit
      const int S = meta.z & 0xff;
      const int nback = (meta.z >> 8) & 0xff;
      const int hS = S >> 5, oS = S & 31;
      if (lane == oS) {
        const int32_t endp = __ldg(a.last + p);
        const int32_t c = __ldg(&r->cnt);
        const uint64_t r0 = __ldg(&r->rep.w[0]), r1 = __ldg(&r->rep.w[1]), r2 = __ldg(&r->rep.w[2]);
#pragma unroll
        for (int h = 0; h < SPL; ++h)
          if (h == hS) {
            L.lab[h] = S;
            L.endp[h] = endp;
            L.cnt[h] = c;
            L.single[h] = p;
            L.s0[h] = r0;
            L.s1[h] = r1;
            L.s2[h] = r2;
          }
        if ((int32_t)meta.w >= 0) {
          const fx192 off = {{__ldg(&r->off.w[0]), __ldg(&r->off.w[1]), __ldg(&r->off.w[2])}};
          fx_sub(tacc, off);
        }
      }
#pragma unroll
      for (int h = 0; h < SPL; ++h)
        if (h == hS) act[h] |= 1u << oS;
      int A = S;  // current label of the new unit's component (uniform)
      for (int j = 0; j < nback; ++j) {
        const int b = __ldg(a.slots + meta.x + j);
        const int hb = b >> 5, ob = b & 31;
        uint32_t ab = act[0];
#pragma unroll
        for (int h = 1; h < SPL; ++h)
          if (h == hb) ab = act[h];
        if (!((ab >> ob) & 1u)) continue;  // neighbour is off
        const int B = __shfl_sync(0xffffffffu, pick<SPL>(L.lab, hb), ob);
        if (B == A) continue;
        const int hA = A >> 5, oA = A & 31, hB = B >> 5, oB = B & 31;
        const int32_t eA = __shfl_sync(0xffffffffu, pick<SPL>(L.endp, hA), oA);
        const int32_t eB = __shfl_sync(0xffffffffu, pick<SPL>(L.endp, hB), oB);
        const bool keepA = eA >= eB;  // the later-ending anchor survives
        const int W = keepA ? A : B, X = keepA ? B : A;
        const int hX = X >> 5, oX = X & 31, hW = W >> 5, oW = W & 31;
        const uint64_t x0 = shfl64(pick<SPL>(L.s0, hX), oX);
        const uint64_t x1 = shfl64(pick<SPL>(L.s1, hX), oX);
        const uint64_t x2 = shfl64(pick<SPL>(L.s2, hX), oX);
        const int32_t xc = __shfl_sync(0xffffffffu, pick<SPL>(L.cnt, hX), oX);
        if (lane == oW) {
#pragma unroll
          for (int h = 0; h < SPL; ++h)
            if (h == hW) {
              fx192 s = {{L.s0[h], L.s1[h], L.s2[h]}};
              const fx192 x = {{x0, x1, x2}};
              fx_add(s, x);
              L.s0[h] = s.w[0];
              L.s1[h] = s.w[1];
              L.s2[h] = s.w[2];
              L.cnt[h] += xc;
              L.single[h] = -1;
            }
        }
#pragma unroll
        for (int h = 0; h < SPL; ++h)
          if (L.lab[h] == X) L.lab[h] = W;
        A = W;
      }
    }
    wd_release<SPL>(L, act, a.M, lane, q, qn, a, tacc, inexact);
    __syncwarp();
    wd_price(q, qn, lane, a, tacc, inexact);
    __syncwarp();
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      const fx192 o = shfl_xor_fx(tacc, m);
      fx_add(tacc, o);
    }
    if (lane == 0) {
      fx192 total = a.base_const;
      fx_add(total, tacc);
      fit[g] = fx_to_double(total);
    }
  }
  if (__any_sync(0xffffffffu, inexact) && lane == 0) atomicAdd(a.flags, 1ull);
}

template <int SPL>
int launch_wide_t(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit, cudaStream_t stream,
                  const int64_t* list = nullptr, const int32_t* list_count = nullptr) {
  WideArgs a;
  a.M = p->M;
  a.words = p->words;
  a.k = p->k;
  a.base_const = p->base_const;
  a.eps = p->eps;
  a.prog = p->d_prog.p;
  a.slots = p->d_prog_slots.p;
  a.last = p->d_prog_last.p;
  a.pos_of_bit = p->d_pos_of_bit.p;
  a.fixed_pos = p->d_fixed_pos.p;
  a.infeas = p->d_infeas.p;
  a.rt = p->d_rt.p;
  a.flags = p->d_flags.p;
  int per_sm = 0;
  CB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fitness_wide_kernel<SPL>, WD_THREADS, 0));
  if (per_sm < 1) per_sm = 1;
  const int64_t want = (n + WD_THREADS / 32 - 1) / (WD_THREADS / 32);
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)per_sm * cb_sm_count()));
  fitness_wide_kernel<SPL><<<(unsigned)grid, WD_THREADS, 0, stream>>>(a, d_pop, n, d_fit, list, list_count);
  CB_CUDA_TRY(cudaGetLastError());
  return CB_OK;
}

}  // namespace

int launch_fitness_wide(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit,
                        cudaStream_t stream) {
  if (p->F <= 32) return launch_wide_t<1>(p, d_pop, n, d_fit, stream);
  if (p->F <= 64) return launch_wide_t<2>(p, d_pop, n, d_fit, stream);
  return launch_wide_t<4>(p, d_pop, n, d_fit, stream);
}
