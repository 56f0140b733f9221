// ON-unit walk for wide frontier programs (up to 64 slots): the fitness
// kernel of the random 100k-op DAG (36 slots, 99 446-bit genomes),
// BASELINE.json configs[4].
//
// Semantics are those of every fitness kernel here (tensorplace/
// evolution.py:65-135 decode, tensorplace/cost.py:320-373 graph-level
// pricing): the genome's ON units (offloaded kernels, plus the always-on
// fixed components) form regions = connected components over the unit graph;
// each region costs round(sum) * r(n) + eps, every other kernel its own term.
//
// One thread per genome; unlike the lockstep frontier walks, a lane visits
// only ITS ON units, in program order (set genome bits, merged with the fixed
// positions), so the work per genome follows its density instead of the
// program length:
//
// * Visiting ON unit q adds its one-unit region term minus its own kernel
//   term (term1 - off): correct while q stays alone.  Merging a one-unit
//   component into a bigger one takes that back (- term1) and contributes its
//   replacement sum to the region.
// * Components live in frontier slots (the plan gives every unit a slot from
//   its position to its last neighbour's).  Labels are per-lane words in
//   shared memory: a non-anchor slot points to a slot of its component that
//   ends no earlier (path-compressed), an anchor holds either its unit's
//   program position (one-unit component) or a pool entry (merged).  A back
//   neighbour's slot label is read only when the neighbour is ON (its genome
//   bit), so slots of skipped units never matter.
// * Merged components keep an exact sum with the kernel count packed in bits
//   108-127 (plan-checked 128-bit window) and their end (latest last
//   neighbour of a member) in a pool of 64 entries per lane: C in shared
//   memory, the rest spilled to global memory.  A merged component is
//   complete once the walk passes its end; it is then queued and priced in
//   warp batches of up to 32 (round, __dmul_rn by r(n), + eps).
// * Per ON unit a lane gathers one 48-byte record (slot, last neighbour,
//   back neighbours as (slot, genome bit), term1 - off) from the L2-resident
//   plan; merges gather the 32-byte (rep | count, term1) records.
#include <algorithm>
#include <climits>
#include <cstring>

#include "fitness_plan.cuh"

#define OW_THREADS 128
#define OW_QCAP 32

namespace {

constexpr uint32_t L_ANCHOR = 0x80000000u;
constexpr uint32_t L_MERGED = 0x40000000u;
constexpr uint32_t L_PAYLOAD = 0x00FFFFFFu;  // parent slot / unit position / pool entry
constexpr int CNT_SHIFT = 44;                // count at bit 64 + 44 = 108 of a packed sum
constexpr uint64_t VAL_HI_MASK = (1ull << CNT_SHIFT) - 1ull;
constexpr uint32_t NO_BIT = 0xFFFFFFu;

struct X128 {
  uint64_t lo, hi;
};
__device__ __forceinline__ void x_add(X128& a, const X128& b) {
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(a.lo), "+l"(a.hi) : "l"(b.lo), "l"(b.hi));
}
__device__ __forceinline__ void x_sub(X128& a, const X128& b) {
  asm("sub.cc.u64 %0, %0, %2;\n\tsubc.u64 %1, %1, %3;" : "+l"(a.lo), "+l"(a.hi) : "l"(b.lo), "l"(b.hi));
}
__device__ __forceinline__ X128 ld_x(const ulonglong2* p) {
  const ulonglong2 v = __ldg(p);
  return {v.x, v.y};
}

// 48-byte per-position record (three 16-byte loads)
struct __align__(16) OwRec {
  uint32_t meta;     // slot | nback << 6 | long << 15 (back list in `lists` at back[0])
  int32_t last;      // position of the unit's last neighbour
  uint32_t back[4];  // back neighbour j: slot | genome bit << 6 (bit NO_BIT: fixed, always on)
  uint32_t pad[2];
  uint64_t t1lo, t1hi;  // term1 - off (two's complement X)
};
static_assert(sizeof(OwRec) == 48, "OwRec layout");

struct OwArgs {
  int32_t M, words, shift, n_infeas, n_fixed;
  bool seq;  // genome bit b is program position b (no fixed units)
  fx192 base_const;
  X128 eps;
  const OwRec* __restrict__ rec;
  const ulonglong2* __restrict__ mrec;  // [M][2]: rep | cnt << 108, term1
  const uint32_t* __restrict__ lists;   // long back lists (same encoding as OwRec::back)
  const int32_t* __restrict__ pos_of_bit;
  const int32_t* __restrict__ fixed_pos;  // ascending, sentinel M
  const int32_t* __restrict__ infeas_word;
  const uint64_t* __restrict__ infeas_mask;
  const double* __restrict__ rt;
  unsigned long long* flags;
  int32_t* ovf_count;
  int64_t* ovf_list;
  ulonglong2* spill;    // [64 - C][resident threads] sums
  int32_t* spill_end;   // [64 - C][resident threads] ends
};

// 32-bit shared-memory accesses
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ X128 lds_x(uint32_t a) {
  X128 v;
  asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(v.lo), "=l"(v.hi) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_x(uint32_t a, const X128& v) {
  asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(a), "l"(v.lo), "l"(v.hi));
}

struct OwLane {
  uint32_t lab;   // shared address of slot 0's label (slot s at + 4 s T)
  uint32_t psum;  // shared address of pool entry 0's sum (entry e < C at + 16 e T)
  uint32_t pend;  // shared address of pool entry 0's end (+ 4 e T)
  ulonglong2* spill;
  int32_t* spill_end;
  int64_t spill_stride;
  uint64_t pfree;   // free pool entries
  uint64_t pused;   // live merged components (pool entries)
  int32_t next_close;  // smallest end of a live merged component (INT_MAX: none)
  bool ovf;
  X128 total;
};

template <int C>
__device__ __forceinline__ X128 pool_sum(const OwLane& L, uint32_t e) {
  if (e < (uint32_t)C) return lds_x(L.psum + e * (16 * OW_THREADS));
  const ulonglong2 v = L.spill[(int64_t)(e - C) * L.spill_stride];
  return {v.x, v.y};
}
template <int C>
__device__ __forceinline__ int32_t pool_end(const OwLane& L, uint32_t e) {
  if (e < (uint32_t)C) return (int32_t)lds_u32(L.pend + e * (4 * OW_THREADS));
  return L.spill_end[(int64_t)(e - C) * L.spill_stride];
}
template <int C>
__device__ __forceinline__ void pool_put(const OwLane& L, uint32_t e, const X128& s, int32_t end) {
  if (e < (uint32_t)C) {
    sts_x(L.psum + e * (16 * OW_THREADS), s);
    sts_u32(L.pend + e * (4 * OW_THREADS), (uint32_t)end);
  } else {
    L.spill[(int64_t)(e - C) * L.spill_stride] = make_ulonglong2(s.lo, s.hi);
    L.spill_end[(int64_t)(e - C) * L.spill_stride] = end;
  }
}

// Price the queued regions (one per lane) into their owners' accumulators.
__device__ __forceinline__ void ow_flush(const ulonglong2* qx, const uint8_t* qown, int qn, int lane,
                                         const OwArgs& a, unsigned long long* tacc, bool& inexact) {
  __syncwarp();
  if (lane < qn) {
    const ulonglong2 q = qx[lane];
    const uint32_t cnt = (uint32_t)(q.y >> CNT_SHIFT);
    const double prod = __dmul_rn(x128_to_double(q.x, q.y & VAL_HI_MASK, a.shift), __ldg(a.rt + cnt));
    X128 term;
    inexact |= !x128_from_double(prod, a.shift, term.lo, term.hi);
    x_add(term, a.eps);
    unsigned long long* w = tacc + 2 * qown[lane];
    const unsigned long long o0 = atomicAdd(w, (unsigned long long)term.lo);
    atomicAdd(w + 1, (unsigned long long)(term.hi + ((o0 + term.lo) < o0)));
  }
  __syncwarp();
}

// Close (queue) the lane's merged components that end before `limit`, one
// per lane per round; every lane takes part in every round.
template <int C>
__device__ __forceinline__ void ow_close_before(OwLane& L, int32_t limit, int lane, ulonglong2* qx,
                                                uint8_t* qown, int& qn, const OwArgs& a,
                                                unsigned long long* tacc, bool& inexact) {
  while (__any_sync(0xffffffffu, L.next_close < limit)) {
    bool emit = false;
    X128 ev = {0ull, 0ull};
    if (L.next_close < limit) {
      // the live entry with the smallest end, and the new smallest end
      uint32_t pick = 0;
      int32_t best = INT_MAX, second = INT_MAX;
      for (uint64_t m = L.pused; m; m &= m - 1ull) {
        const uint32_t e = (uint32_t)(__ffsll((long long)m) - 1);
        const int32_t end = pool_end<C>(L, e);
        if (end < best) {
          second = best;
          best = end;
          pick = e;
        } else if (end < second) {
          second = end;
        }
      }
      if (best < limit) {
        ev = pool_sum<C>(L, pick);
        L.pused &= ~(1ull << pick);
        L.pfree |= 1ull << pick;
        L.next_close = second;
        emit = true;
      } else {
        L.next_close = best;  // the smallest end was absorbed by a merge
      }
    }
    const unsigned closing = __ballot_sync(0xffffffffu, emit);
    const int cnt = __popc(closing);
    if (qn + cnt > OW_QCAP) {
      ow_flush(qx, qown, qn, lane, a, tacc, inexact);
      qn = 0;
    }
    if (emit) {
      const int at = qn + __popc(closing & ((1u << lane) - 1u));
      qx[at] = make_ulonglong2(ev.lo, ev.hi);
      qown[at] = (uint8_t)lane;
    }
    qn += cnt;
  }
}

// Genome bit test of a back neighbour (fixed units are always on).
__device__ __forceinline__ bool bit_on(const uint64_t* gen, uint32_t bit) {
  if (bit == NO_BIT) return true;
  return (__ldg(gen + (bit >> 6)) >> (bit & 63u)) & 1ull;
}

template <int C>
__device__ __forceinline__ void ow_merge(OwLane& L, const OwArgs& a, int b, int& A, uint32_t& lA_cache) {
  constexpr int T = OW_THREADS;
  int x = b;
  uint32_t lx = lds_u32(L.lab + 4u * T * b);
  while (!(lx & L_ANCHOR)) {
    x = (int)(lx & L_PAYLOAD);
    lx = lds_u32(L.lab + 4u * T * x);
  }
  if (x != b) sts_u32(L.lab + 4u * T * b, (uint32_t)x);  // path compression
  if (x == A) return;
  const uint32_t lA = lA_cache;
  // ends: one-unit components from the plan, merged ones from the pool
  const bool mA = (lA & L_MERGED) != 0u, mX = (lx & L_MERGED) != 0u;
  const int32_t endA = mA ? pool_end<C>(L, lA & 63u) : __ldg(&a.rec[lA & L_PAYLOAD].last);
  const int32_t endX = mX ? pool_end<C>(L, lx & 63u) : __ldg(&a.rec[lx & L_PAYLOAD].last);
  const bool keepA = endA >= endX;  // the later-ending anchor survives
  const int Wn = keepA ? A : x, Xn = keepA ? x : A;
  const uint32_t lW = keepA ? lA : lx, lX = keepA ? lx : lA;
  const bool mW = keepA ? mA : mX, mXX = keepA ? mX : mA;
  X128 sW, sX;
  if (mW) {
    sW = pool_sum<C>(L, lW & 63u);
  } else {
    const uint32_t u = lW & L_PAYLOAD;
    sW = ld_x(a.mrec + 2 * u);
    x_sub(L.total, ld_x(a.mrec + 2 * u + 1));  // no longer a one-unit region
  }
  if (mXX) {
    sX = pool_sum<C>(L, lX & 63u);
  } else {
    const uint32_t u = lX & L_PAYLOAD;
    sX = ld_x(a.mrec + 2 * u);
    x_sub(L.total, ld_x(a.mrec + 2 * u + 1));
  }
  x_add(sW, sX);
  uint32_t e;
  if (mW) {
    e = lW & 63u;
    if (mXX) {
      L.pfree |= 1ull << (lX & 63u);
      L.pused &= ~(1ull << (lX & 63u));
    }
  } else if (mXX) {
    e = lX & 63u;
  } else if (L.pfree) {
    e = (uint32_t)(__ffsll((long long)L.pfree) - 1);
    L.pfree &= L.pfree - 1ull;
    L.pused |= 1ull << e;
  } else {
    L.ovf = true;  // 64 live merged components: the genome goes to the fallback kernel
    e = 0;
  }
  const int32_t end = keepA ? endA : endX;
  pool_put<C>(L, e, sW, end);
  L.next_close = min(L.next_close, end);
  const uint32_t lnew = L_ANCHOR | L_MERGED | e;
  sts_u32(L.lab + 4u * T * Wn, lnew);
  sts_u32(L.lab + 4u * T * Xn, (uint32_t)Wn);
  A = Wn;
  lA_cache = lnew;
}

template <int C>
__global__ void __launch_bounds__(OW_THREADS)
fitness_onwalk_kernel(OwArgs a, const uint64_t* __restrict__ pop, int64_t n, double* __restrict__ fit) {
  constexpr int T = OW_THREADS, W = OW_THREADS / 32;
  extern __shared__ __align__(16) unsigned char ow_smem[];
  ulonglong2* psum = reinterpret_cast<ulonglong2*>(ow_smem);                   // [C][T]
  ulonglong2* qx_all = psum + C * T;                                           // [W][QCAP]
  unsigned long long* tacc_all = reinterpret_cast<unsigned long long*>(qx_all + W * OW_QCAP);  // [W][64]
  uint32_t* pend = reinterpret_cast<uint32_t*>(tacc_all + W * 64);           // [C][T]
  uint8_t* qown_all = reinterpret_cast<uint8_t*>(pend + C * T);               // [W][QCAP]
  uint32_t* LAB = reinterpret_cast<uint32_t*>(qown_all + W * OW_QCAP);        // [F][T]
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  ulonglong2* qx = qx_all + warp * OW_QCAP;
  uint8_t* qown = qown_all + warp * OW_QCAP;
  unsigned long long* tacc = tacc_all + warp * 64;
  OwLane L;
  L.lab = (uint32_t)__cvta_generic_to_shared(LAB + t);
  L.psum = (uint32_t)__cvta_generic_to_shared(psum + t);
  L.pend = (uint32_t)__cvta_generic_to_shared(pend + t);
  L.spill_stride = (int64_t)gridDim.x * T;
  L.spill = a.spill + (int64_t)blockIdx.x * T + t;
  L.spill_end = a.spill_end + (int64_t)blockIdx.x * T + t;
  tacc[2 * lane] = tacc[2 * lane + 1] = 0ull;
  __syncwarp();
  bool inexact = false;
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t base = (int64_t)blockIdx.x * T + (t & ~31); base < n; base += stride) {
    const int64_t i = base + lane;
    const bool in_range = i < n;
    const uint64_t* gen = pop + (in_range ? i : 0) * a.words;
    bool dead = !in_range;
    for (int32_t j = 0; j < a.n_infeas; ++j)
      dead |= (__ldg(gen + __ldg(a.infeas_word + j)) & __ldg(a.infeas_mask + j)) != 0ull;
    L.pfree = ~0ull;
    L.pused = 0ull;
    L.next_close = INT_MAX;
    L.ovf = false;
    L.total = {0ull, 0ull};
    int qn = 0;
    // streams of ON positions: set genome bits (in bit order = program order)
    // and the fixed positions
    int32_t wi = 0;
    uint64_t word = (!dead && a.words > 0) ? __ldg(gen) : 0ull;
    int32_t fi = 0;
    int32_t fpos = a.n_fixed > 0 && !dead ? __ldg(a.fixed_pos) : INT_MAX;
    while (true) {
      while (word == 0ull && wi + 1 < a.words) word = __ldg(gen + ++wi);
      int32_t bpos = INT_MAX;
      if (word) {
        const int32_t bit = wi * 64 + __ffsll((long long)word) - 1;
        bpos = a.seq ? bit : __ldg(a.pos_of_bit + bit);
      }
      const int32_t q = min(bpos, fpos);
      // merged components that end before q are complete
      ow_close_before<C>(L, q, lane, qx, qown, qn, a, tacc, inexact);
      if (!__any_sync(0xffffffffu, q != INT_MAX)) break;
      if (q != INT_MAX) {
        if (q == bpos) {
          word &= word - 1ull;
        } else {
          fpos = ++fi < a.n_fixed ? __ldg(a.fixed_pos + fi) : INT_MAX;
        }
        const uint4* rp = reinterpret_cast<const uint4*>(a.rec + q);
        const uint4 r0 = __ldg(rp), r2 = __ldg(rp + 2);
        const int S = (int)(r0.x & 63u);
        const int nb = (int)((r0.x >> 6) & 0x1FFu);
        const bool lng = (r0.x >> 15) & 1u;
        x_add(L.total, X128{((uint64_t)r2.y << 32) | r2.x, ((uint64_t)r2.w << 32) | r2.z});
        uint32_t lA = L_ANCHOR | (uint32_t)q;
        sts_u32(L.lab + 4u * T * S, lA);
        int A = S;
        if (nb) {
          const uint4 r1 = __ldg(rp + 1);
          if (!lng) {
            const uint32_t bk[4] = {r0.z, r0.w, r1.x, r1.y};
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (j < nb && bit_on(gen, bk[j] >> 6)) ow_merge<C>(L, a, (int)(bk[j] & 63u), A, lA);
          } else {
            const uint32_t off = r0.z;
            for (int j = 0; j < nb; ++j) {
              const uint32_t bkj = __ldg(a.lists + off + j);
              if (bit_on(gen, bkj >> 6)) ow_merge<C>(L, a, (int)(bkj & 63u), A, lA);
            }
          }
        }
      }
    }
    ow_flush(qx, qown, qn, lane, a, tacc, inexact);
    X128 total = L.total;
    x_add(total, X128{tacc[2 * lane], tacc[2 * lane + 1]});
    tacc[2 * lane] = tacc[2 * lane + 1] = 0ull;
    __syncwarp();
    if (in_range) {
      if (L.ovf && !dead) {
        fit[i] = __longlong_as_double(0x7ff8000000000000ll);
        const int32_t at = atomicAdd(a.ovf_count, 1);
        a.ovf_list[at] = i;
      } else if (dead) {
        fit[i] = __longlong_as_double(0x7ff0000000000000ll);
      } else {
        // sign-extend the 128-bit dynamic part, scale back, add the constant
        const uint64_t sx = (uint64_t)((int64_t)total.hi >> 63);
        fx192 v = fx_shl(fx192{{total.lo, total.hi, sx}}, a.shift);
        fx_add(v, a.base_const);
        fit[i] = fx_to_double(v);
      }
    }
  }
  if (inexact) atomicAdd(a.flags, 1ull);
}

size_t onwalk_smem(int C, int F) {
  constexpr int T = OW_THREADS, W = OW_THREADS / 32;
  return (size_t)C * T * 16 + (size_t)W * (OW_QCAP * 16 + 64 * 8) + (size_t)C * T * 4 + (size_t)W * OW_QCAP +
         (size_t)F * T * 4;
}

template <int C>
int launch_onwalk_t(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit, cudaStream_t stream) {
  const size_t smem = onwalk_smem(C, p->F);
  if (cb_smem_claim((const void*)fitness_onwalk_kernel<C>, smem))
    CB_CUDA_TRY(cudaFuncSetAttribute(fitness_onwalk_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  int per_sm = 0;
  CB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fitness_onwalk_kernel<C>, OW_THREADS,
                                                            smem));
  if (per_sm < 1) per_sm = 1;
  if (p->d_ovf_list.n < (size_t)std::max<int64_t>(n, 1)) CB_CUDA_TRY(p->d_ovf_list.alloc((size_t)n));
  if (p->d_ovf_count.n < 1) CB_CUDA_TRY(p->d_ovf_count.alloc(1));
  CB_CUDA_TRY(cudaMemsetAsync(p->d_ovf_count.p, 0, sizeof(int32_t), stream));
  OwArgs a;
  a.M = p->M;
  a.words = p->words;
  a.shift = p->anchor_shift;
  a.n_infeas = (int32_t)p->d_an_infeas_word.n;
  a.n_fixed = (int32_t)p->fixed_pos.size() - 1;  // without the sentinel
  a.seq = p->ow_seq;
  a.base_const = p->base_const;
  const fx192 ex = fx_shr(p->eps, p->anchor_shift);
  a.eps = {ex.w[0], ex.w[1]};
  a.rec = reinterpret_cast<const OwRec*>(p->d_owrec.p);
  a.mrec = reinterpret_cast<const ulonglong2*>(p->d_owmrec.p);
  a.lists = p->d_owlists.p;
  a.pos_of_bit = p->d_pos_of_bit.p;
  a.fixed_pos = p->d_fixed_pos.p;
  a.infeas_word = p->d_an_infeas_word.p;
  a.infeas_mask = p->d_an_infeas_mask.p;
  a.rt = p->d_rt.p;
  a.flags = p->d_flags.p;
  a.ovf_count = p->d_ovf_count.p;
  a.ovf_list = p->d_ovf_list.p;
  const int64_t want = (n + OW_THREADS - 1) / OW_THREADS;
  const int64_t grid = std::min<int64_t>(want, (int64_t)per_sm * cb_sm_count());
  const size_t spill = (size_t)(64 - C) * grid * OW_THREADS;
  DBuf<uint64_t>* sp;
  {
    std::lock_guard<std::mutex> lock(p->aspill_mu);
    auto& slot = p->aspill[stream];
    if (!slot) slot.reset(new DBuf<uint64_t>());
    sp = slot.get();
  }
  // sums (2 words) then ends (one int32 each, half a word)
  const size_t words_needed = spill * 2 + (spill + 1) / 2;
  if (sp->n < words_needed) CB_CUDA_TRY(sp->alloc(words_needed));
  a.spill = reinterpret_cast<ulonglong2*>(sp->p);
  a.spill_end = reinterpret_cast<int32_t*>(sp->p + spill * 2);
  fitness_onwalk_kernel<C><<<(unsigned)grid, OW_THREADS, smem, stream>>>(a, d_pop, n, d_fit);
  CB_CUDA_TRY(cudaGetLastError());
  // genomes with 64 live merged components: warp-per-genome kernel over the list
  return launch_fitness_wide_list(p, d_pop, n, d_fit, p->d_ovf_list.p, p->d_ovf_count.p, stream);
}

}  // namespace

// Plan time: the per-position records (needs the anchor plan's 128-bit
// window, build_anchor_plan runs first).
int build_onwalk_plan(cb_es_plan* P) {
  P->ow_ok = false;
  if (!P->anchor_wide_ok || P->F > 64 || P->M >= (1 << 24)) return CB_OK;
  const int32_t M = P->M;
  const int lo = P->anchor_shift;
  std::vector<OwRec> rec(M);
  std::vector<uint64_t> mrec((size_t)M * 4);
  std::vector<uint32_t> lists;
  // genome bit of every position (NO_BIT for fixed units)
  std::vector<uint32_t> bit_at(M);
  bool seq = P->fixed_pos.size() == 1;
  for (int32_t p = 0; p < M; ++p) {
    const int32_t b = P->prog[p].bit;
    bit_at[p] = b >= 0 ? (uint32_t)b : NO_BIT;
    if (b != p) seq = false;
  }
  for (int32_t p = 0; p < M; ++p) {
    const UnitRec& r = P->prog[p];
    OwRec h;
    std::memset(&h, 0, sizeof(h));
    // back neighbours: the units at earlier positions sharing an edge; the
    // plan's back list holds their slots in the same order as `nbr`
    std::vector<uint32_t> bk;
    for (int j = 0; j < r.nback; ++j) {
      const int32_t q = P->prog_back_pos[r.back_off + j];
      bk.push_back((uint32_t)P->prog_slots[r.back_off + j] | (bit_at[q] << 6));
    }
    if (r.nback > 0x1FF) return CB_OK;
    h.meta = (uint32_t)r.slot | ((uint32_t)r.nback << 6);
    if (r.nback <= 4) {
      uint32_t* dst[4] = {&h.back[0], &h.back[1], &h.back[2], &h.back[3]};
      for (int j = 0; j < r.nback; ++j) *dst[j] = bk[j];
    } else {
      h.meta |= 1u << 15;
      h.back[0] = (uint32_t)lists.size();
      lists.insert(lists.end(), bk.begin(), bk.end());
    }
    h.last = P->prog_last[p];
    const fx192 xo = fx_shr(r.off, lo), xr = fx_shr(r.rep, lo), xt = fx_shr(r.term1, lo);
    fx192 t1m = xt;
    fx_sub(t1m, xo);  // term1 - off, two's complement in the low 128 bits
    h.t1lo = t1m.w[0];
    h.t1hi = t1m.w[1];
    rec[p] = h;
    mrec[4 * p] = xr.w[0];
    mrec[4 * p + 1] = xr.w[1] | ((uint64_t)r.cnt << 44);
    mrec[4 * p + 2] = xt.w[0];
    mrec[4 * p + 3] = xt.w[1];
  }
  if (lists.empty()) lists.push_back(0);
  P->ow_seq = seq;
  cudaError_t e;
  if ((e = P->d_owrec.upload(reinterpret_cast<const uint8_t*>(rec.data()), rec.size() * sizeof(OwRec))) !=
          cudaSuccess ||
      (e = P->d_owmrec.upload(mrec)) != cudaSuccess || (e = P->d_owlists.upload(lists)) != cudaSuccess) {
    cb_set_error(std::string("CUDA error in plan upload: ") + cudaGetErrorString(e));
    return CB_ERR_CUDA;
  }
  P->ow_ok = true;
  return CB_OK;
}

int launch_fitness_onwalk(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit, cudaStream_t stream) {
  const int C = p->pool_entries;
  if (C <= 4) return launch_onwalk_t<4>(p, d_pop, n, d_fit, stream);
  if (C <= 8) return launch_onwalk_t<8>(p, d_pop, n, d_fit, stream);
  return launch_onwalk_t<16>(p, d_pop, n, d_fit, stream);
}
