// Frontier walk as a finite-state machine (thread per genome, <= 8 slots).
//
// Same semantics as every fitness kernel here (tensorplace/evolution.py:
// 256-371 decode, tensorplace/cost.py:320-373 graph-level pricing).  The
// packed-label kernels recompute, for every genome and step, which frontier
// slots are occupied and how they are grouped into components -- the
// connectivity part of the walk, which is most of its instructions.  That
// part depends only on the frontier *state* (the partition of the occupied
// slots into components, plus whether each component already holds more
// than one unit) and on the step's genome bit, and the number of reachable
// states is small (BERT-base: at most 62 per step, 5 798 transitions in
// all; NasNet-A: 2 784 per step).  So the plan enumerates the reachable
// states step by step and tabulates every transition: next state plus the
// arithmetic it implies -- store the unit's sum in its slot, add component
// sums into the surviving anchor slot, queue closed multi-unit regions for
// pricing -- and one exact delta folding every genome-independent term of
// the transition (closed one-unit regions, the removed kernel term).  The
// kernel then does per step: one 32-byte table load indexed by (state, bit),
// one 128-bit add, and only the listed sum moves.  Components keep their data at their anchor (the
// member whose unit ends last), as in fitness_pa_kernel.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <numeric>
#include <unordered_map>

#include "fitness_plan.cuh"

#define FSM_THREADS 256
#ifndef FSM_MINB
#define FSM_MINB 4  // resident blocks per SM the registers are budgeted for (1 024 threads)
#endif
#ifndef FSM_BITS_IN_REGS
#define FSM_BITS_IN_REGS 1
#endif
#define FSM_QCAP 64

namespace {

struct FsmArgs {
  int32_t M, words, shift;
  fx192 base_const;
  uint64_t eps_lo, eps_hi;
  // [M][2]: {table offset, bit info, slot | nend << 8, max merges | max emits << 8},
  // then the unit's packed sum (128-bit X, kernel count in bits 112..127)
  const uint4* __restrict__ hdr;
  const uint4* __restrict__ table;     // transitions (32-byte layout)
  const uint2* __restrict__ ctable;    // transitions (8-byte layout)
  const uint4* __restrict__ mtable;    // transitions (16-byte layout)
  const uint32_t* __restrict__ xtable;  // mixed layout: 8-byte steps and 16-byte steps, word offsets
  const uint4* __restrict__ dtab;      // distinct deltas of the 8- / 16-byte layouts
  int32_t n_delta;
  const uint64_t* __restrict__ infeas;
  const double* __restrict__ rt;
  unsigned long long* flags;
};

// Packed sums: a component's 128-bit sum X (non-negative, < 2^101 by the
// plan's window check) with its kernel count in the top 16 bits, so one
// 128-bit add merges both; queued entries carry the owner lane in bits 104..111.
#define FSM_LANE_SHIFT 40
#define FSM_CNT_SHIFT 48
#define FSM_BIT_FORCED 0x80u  // bit info: the unit has no genome bit (always on)
#define FSM_WIDE_STEP 0x10000u  // header .w: the step's transitions use the 16-byte form (mixed layout)
#define FSM_BIT_NEWWORD 0x40u   // bit info: the step's genome word differs from the previous step's

// merge / emit counts as thermometer bits: merge k at bit 13 + k, emit k at bit 18 + k
static inline uint32_t fsm_therm(int n_merge, int n_emit) {
  return (((1u << n_merge) - 1u) << 13) | (((1u << n_emit) - 1u) << 18);
}

__device__ __forceinline__ ulonglong2 lds_u2(uint32_t a) {
  ulonglong2 v;
  asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u2(uint32_t a, const ulonglong2& v) {
  asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(a), "l"(v.x), "l"(v.y));
}
__device__ __forceinline__ void sts_u4(uint32_t a, const uint4& v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
}

template <typename U>
__device__ __forceinline__ void fadd2(U& lo, U& hi, uint64_t blo, uint64_t bhi) {
  static_assert(sizeof(U) == 8, "64-bit words");
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(lo), "+l"(hi) : "l"(blo), "l"(bhi));
}

// Delta `idx` of the shared delta table as a 128-bit value (x..w, low word
// first): 16-byte entries, or 8-byte entries sign-extended (D64).
template <bool D64>
__device__ __forceinline__ uint4 load_delta(uint32_t base, uint32_t idx) {
  uint4 dv;
  if (D64) {
    uint32_t lo, hi;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(base + idx * 8u));
    const uint32_t sx = (uint32_t)((int32_t)hi >> 31);
    dv = make_uint4(lo, hi, sx, sx);
  } else {
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(dv.x), "=r"(dv.y), "=r"(dv.z), "=r"(dv.w)
                 : "r"(base + idx * 16u));
  }
  return dv;
}

// Price queue entry `idx` and add its term to the owner lane's accumulator.
__device__ __forceinline__ void fsm_price(const ulonglong2* q, int idx, const FsmArgs& a, uint64_t* tlo,
                                          uint64_t* thi, bool& inexact) {
  const ulonglong2 v = q[idx];
  const uint32_t cnt = (uint32_t)(v.y >> FSM_CNT_SHIFT);
  const int owner = (int)((v.y >> FSM_LANE_SHIFT) & 0xFFu);
  const uint64_t xhi = v.y & ((1ull << FSM_LANE_SHIFT) - 1ull);
  const double prod = __dmul_rn(x128_to_double(v.x, xhi, a.shift), __ldg(a.rt + cnt));
  uint64_t lo, hi;
  inexact |= !x128_from_double(prod, a.shift, lo, hi);
  fadd2(lo, hi, a.eps_lo, a.eps_hi);
  const unsigned long long o0 = atomicAdd(reinterpret_cast<unsigned long long*>(tlo + owner), lo);
  atomicAdd(reinterpret_cast<unsigned long long*>(thi + owner), hi + ((o0 + lo) < o0));
}

template <int F, int W>
struct FsmSmemBase {  // packed sums [F][T], per-warp queues and lane totals, genome words [W + 1][T]
  static constexpr size_t wtab_off =
      (size_t)F * FSM_THREADS * 16 + (size_t)(FSM_THREADS / 32) * (FSM_QCAP * 16 + 64 * 8);
  // per-warp slot table: packed sum of the unit in each slot (8 x 16 bytes)
  static constexpr size_t words_off = wtab_off + (size_t)(FSM_THREADS / 32) * 8 * 16;
  // (the words only when the walk reads its bits from shared memory: with
  // FSM_BITS_IN_REGS the freed 8 (W + 1) KB per block go to L1, where the
  // transition table lives)
  static constexpr size_t bytes = words_off + (W > 0 && !FSM_BITS_IN_REGS ? (size_t)(W + 1) * FSM_THREADS * 8 : 0);
};

// Transition entry (32 bytes, layout 0): x = next | open << 16 | n_merge << 17 |
// n_emit << 20, y = merges (src 3 bits | dst 3 bits) x 5, z = emit anchor
// slots (3 bits) x 5, w = merge / emit thermometers (bits 13 + k / 18 + k)
// | one-unit operand bits (source m at bit m < 3 / m + 1, merge 0's
// destination at bit 3); then the transition's exact 128-bit delta: the
// terms of the one-unit regions it closes minus the removed op-kernel term of
// an offloaded unit.
//
// 16-byte layout (2; the wide steps of the mixed layout 3 use the 8-byte x):
// x = next (16 bits) | open | counts | delta index << 24, y = merges, z =
// emit slots, w as above.
//
// Compact layout (8 bytes, 1): x = next (12 bits) | open << 12 | merge
// thermometer (3 bits) << 13 | emit thermometer (3 bits) << 18 | delta index
// (8 bits) << 24, y = merges (6 bits) x 3 | emit slots (3 bits) x 3 << 18 |
// one-unit operand bits (4) << 27; the deltas (at most 256 distinct values;
// BERT-base has 22) sit in shared memory.  Used when every transition fits:
// a quarter of the table's cache footprint.
template <int F, int W, int L>
__global__ void __launch_bounds__(FSM_THREADS, FSM_MINB)
fitness_fsm_kernel(FsmArgs a, const uint64_t* __restrict__ pop, int64_t n, double* __restrict__ fit) {
  constexpr int T = FSM_THREADS;
  // L = layout (0: 32-byte entries, 1: 8, 2: 16, 3: mixed) + 4 when every
  // distinct delta fits a signed 64-bit word: the shared delta table then
  // holds 8-byte entries (half the shared wavefronts of the per-step read)
  constexpr int LL = L & 3;
  constexpr bool D64 = L >= 4;
  // WT: one-unit components' sums from the per-warp slot table instead of a
  // per-lane store at every open (W > 0: BERT-base +2 %, NasRNN +5 %;
  // NasNet-A's W = 0 walk, F = 8, lost 4 % to it and keeps the store)
  constexpr bool WT = W > 0;
  extern __shared__ __align__(16) unsigned char fsm_smem[];
  // deltas after the per-thread arrays (dynamic size: n_delta entries)
  uint4* sdelta = reinterpret_cast<uint4*>(fsm_smem + FsmSmemBase<F, W>::bytes);
  const uint32_t sdelta_base = (uint32_t)__cvta_generic_to_shared(sdelta);
  if (LL != 0) {
    for (int k = threadIdx.x; k < a.n_delta; k += T) {
      const uint4 d = __ldg(a.dtab + k);
      if (D64)
        reinterpret_cast<uint64_t*>(sdelta)[k] = ((uint64_t)d.y << 32) | d.x;
      else
        sdelta[k] = d;
    }
    __syncthreads();
  }
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  ulonglong2* sv = reinterpret_cast<ulonglong2*>(fsm_smem);  // [F][T] packed anchor sums
  ulonglong2* mine = sv + t;                                  // slot s at mine[s * T]
  // 32-bit shared addresses of this thread's slot sums (slot s at + s * 16 T)
  // and genome words (word w at + 8 w T): no generic-to-shared conversion
  // inside the step loop
  const uint32_t mine_a = (uint32_t)__cvta_generic_to_shared(mine);
  // one-unit components keep no per-lane sum: merges read it from the
  // warp's slot table (written once per step by lane 0)
  const uint32_t wtab_a = (uint32_t)__cvta_generic_to_shared(fsm_smem + FsmSmemBase<F, W>::wtab_off) + warp * 128u;
  ulonglong2* q = sv + F * T + warp * FSM_QCAP;               // pricing queue of this warp
  uint64_t* tlo = reinterpret_cast<uint64_t*>(sv + F * T + (T / 32) * FSM_QCAP) + warp * 64;
  uint64_t* thi = tlo + 32;
  tlo[lane] = thi[lane] = 0ull;
  // W > 0: the genome's words, then an all-ones word for units without a
  // genome bit; a step's header holds its word's byte offset and bit, so the
  // bit is one shared load + shift (no per-step word select)
  uint64_t* swd = reinterpret_cast<uint64_t*>(fsm_smem + FsmSmemBase<F, W>::words_off) + t;
  if (W > 0 && !FSM_BITS_IN_REGS) swd[W * T] = ~0ull;
  const uint32_t swd_a = (uint32_t)__cvta_generic_to_shared(swd);
  __syncwarp();
  int qn = 0;
  bool inexact = false;
  const int64_t stride = (int64_t)gridDim.x * T;
  constexpr int WR = W > 0 ? W : 1;
  uint64_t pre[WR];
  if (W > 0) {
    const int64_t i0 = (int64_t)blockIdx.x * T + t;
#pragma unroll
    for (int w = 0; w < WR; ++w) pre[w] = i0 < n ? __ldcs(pop + i0 * W + w) : 0ull;
  }
  for (int64_t base = (int64_t)blockIdx.x * T + (t & ~31); base < n; base += stride) {
    const int64_t i = base + lane;
    const bool in_range = i < n;
    const uint64_t* gen = pop + (in_range ? i : 0) * a.words;
    bool dead = !in_range;
    uint64_t cur[WR];
    if (W > 0) {
#pragma unroll
      for (int w = 0; w < WR; ++w) {
        cur[w] = pre[w];
        dead |= (cur[w] & __ldg(a.infeas + w)) != 0ull;
      }
      const int64_t inext = i + stride;  // prefetch the next genome of this thread
#pragma unroll
      for (int w = 0; w < WR; ++w) pre[w] = inext < n ? __ldcs(pop + inext * W + w) : 0ull;
      // an infeasible genome walks all-zero bits (its result is discarded)
#pragma unroll
      for (int w = 0; w < WR; ++w)  // asm like the step loop's loads (volatile asm keeps their order)
        if (!FSM_BITS_IN_REGS)
          asm volatile("st.shared.u64 [%0], %1;" ::"r"(swd_a + w * (8u * T)), "l"(dead ? 0ull : cur[w]));
    } else if (in_range) {
      for (int32_t w = 0; w < a.words; ++w) dead |= (__ldg(gen + w) & __ldg(a.infeas + w)) != 0ull;
    }
    uint32_t state = 0u;
    uint64_t tot_lo = 0ull, tot_hi = 0ull;
    int32_t cached_word = -1;
    uint64_t word = 0ull, next_word = W == 0 && a.words > 0 ? __ldg(gen) : 0ull;
    // step headers are warp uniform: prefetched one step ahead (the plan
    // pads the header array with a dummy step M, so no bound check)
    const uint4* hp = a.hdr;
    uint4 hn = __ldg(hp);
    // the 16-byte layout (an L2-resident table) also prefetches the unit's
    // packed sum (NasNet-A +3 %; the L1-resident walks lose ~0.5 % to it)
    constexpr bool PRE_REP = LL >= 2;
    uint4 rn = PRE_REP ? __ldg(hp + 1) : make_uint4(0u, 0u, 0u, 0u);
#if FSM_BITS_IN_REGS
    uint64_t gw[WR];
#pragma unroll
    for (int w = 0; w < WR; ++w) gw[w] = dead ? 0ull : cur[w];
    // W > 0: the step's genome bit from the current word, reselected from
    // the registers only when the word changes (warp uniform: consecutive
    // steps mostly read one word; the integer pipe is what binds)
    uint64_t cwd = 0ull;
    auto bit_of = [&](uint32_t hy) {
      if (hy & FSM_BIT_NEWWORD) {
        const uint32_t wi = hy >> 8;
        cwd = ~0ull;  // word W: units without a genome bit
#pragma unroll
        for (int w = 0; w < WR; ++w) cwd = wi == (uint32_t)w ? gw[w] : cwd;
      }
      return (uint32_t)(cwd >> (hy & 63u)) & 1u;
    };
#else
    auto bit_of = [&](uint32_t hy) {  // W > 0: the step's genome bit from shared memory
      uint64_t wd;
      asm volatile("ld.shared.u64 %0, [%1];" : "=l"(wd) : "r"(swd_a + (hy >> 8) * (8u * T)));
      return (uint32_t)(wd >> (hy & 63u)) & 1u;
    };
#endif
    uint32_t on_next = W > 0 ? bit_of(hn.y) : 0u;
    // ACC64: the deltas (|d| < 2^57, plan-checked) add into a 64-bit
    // accumulator folded into the 128-bit total every 64 steps (NasNet-A's
    // W = 0 walk, F = 8, lost 4 % to it: sign-extended 128-bit adds there)
    constexpr bool ACC64 = D64 && W > 0;
    constexpr int32_t CHUNK = ACC64 ? 64 : 0x40000000;
    for (int32_t p0 = 0; p0 < a.M; p0 += CHUNK) {
    const int32_t pe = min(a.M, p0 + CHUNK);
    int64_t dacc = 0;
    for (int32_t p = p0; p < pe; ++p) {
      const uint4 h = hn, rp = rn;
      hp += 2;
      hn = __ldg(hp);
      if (PRE_REP) rn = __ldg(hp + 1);
      bool on;
      if (W > 0) {
        on = on_next != 0u;
      } else {
        on = true;
        if (!(h.y & FSM_BIT_FORCED)) {
          const int32_t wi = (int32_t)(h.y >> 8);
          if (wi != cached_word) {  // warp uniform
            word = wi == cached_word + 1 ? next_word : __ldg(gen + wi);
            next_word = wi + 1 < a.words ? __ldg(gen + wi + 1) : 0ull;
            cached_word = wi;
          }
          on = (word >> (h.y & 63u)) & 1ull;
        }
      }
      if (W == 0) on = on && !dead;
      const uint32_t onb = W > 0 ? on_next : (on ? 1u : 0u);  // (W > 0: the bit as is, no select)
      const uint32_t idx = h.x + 2u * state + onb;  // 32-bit index math
      // th: merge / emit counts as thermometers (bit 13 + k: the transition
      // has merge k, bit 18 + k: emit k), tested in place -- no field extraction
      uint32_t open, th, merges, emits, sg;  // sg: merge operands that are one-unit components
      uint32_t didx = 0u, dbyte = 0u;  // shared delta table index (layouts 1-3: the entry's top byte)
      uint4 dv = make_uint4(0u, 0u, 0u, 0u);  // exact delta: closed one-unit regions' terms - removed term
      if (LL == 3) {
        // mixed: the step's header says whether its transitions take 8 or
        // 16 bytes (warp-uniform); h.x is a word offset
        if (h.w & FSM_WIDE_STEP) {
          const uint4 e = __ldg(reinterpret_cast<const uint4*>(a.xtable + h.x + 4u * (2u * state + onb)));
          state = e.x & 0xFFFu;  // (mixed layouts keep <= 4096 states per step)
          open = (e.x >> 12) & 1u;
          th = e.x;
          didx = e.x >> 24;
          if (!ACC64) dv = load_delta<D64>(sdelta_base, didx);  // in the branch (NasNet-A: 4 % faster)
          merges = e.y;
          emits = e.z;
          sg = e.w;
        } else {
          const uint2 e = __ldg(reinterpret_cast<const uint2*>(a.xtable + h.x + 2u * (2u * state + onb)));
          state = e.x & 0xFFFu;
          open = (e.x >> 12) & 1u;
          th = e.x;
          didx = e.x >> 24;
          if (!ACC64) dv = load_delta<D64>(sdelta_base, didx);  // in the branch (NasNet-A: 4 % faster)
          merges = e.y & 0x3FFFFu;
          emits = e.y >> 18;
          sg = e.y >> 27;
        }
      } else if (LL == 1) {
        const uint2 e = __ldg(a.ctable + idx);
        state = e.x & 0xFFFu;
        open = (e.x >> 12) & 1u;
        th = e.x;
        didx = e.x >> 24;
        dbyte = e.x >> 21;
        merges = e.y;
        emits = e.y >> 18;
        sg = e.y >> 27;
      } else if (LL == 2) {
        const uint4 e = __ldg(a.mtable + idx);
        state = e.x & 0xFFFFu;
        open = (e.x >> 16) & 1u;
        th = e.w;
        didx = e.x >> 24;
        merges = e.y;
        emits = e.z;
        sg = e.w;
      } else {
        const uint4 e = __ldg(a.table + 2u * idx);
        dv = __ldg(a.table + 2u * idx + 1u);
        state = e.x & 0xFFFFu;
        open = (e.x >> 16) & 1u;
        th = e.w;
        merges = e.y;
        emits = e.z;
        sg = e.w;
      }
      if (ACC64) {
        int64_t d;
        // layout 1: bits 21-23 of the entry are zero (emit thermometer <= 3
        // bits), so the byte offset is one shift
        const uint32_t doff = LL == 1 ? dbyte : didx * 8u;
        asm volatile("ld.shared.s64 %0, [%1];" : "=l"(d) : "r"(sdelta_base + doff));
        dacc += d;
      } else {
        if (LL != 0 && LL != 3) dv = load_delta<D64>(sdelta_base, didx);
        fadd2(tot_lo, tot_hi, ((uint64_t)dv.y << 32) | dv.x, ((uint64_t)dv.w << 32) | dv.z);
      }
      if (WT) {  // the step's unit takes its slot: its packed sum into the warp's slot table
        const uint4 r = PRE_REP ? rp : __ldg(hp - 1);
        __syncwarp();  // every lane is past the slot's previous occupant
        if (lane == 0) sts_u4(wtab_a + (h.z >> 8), r);  // h.z: slot x 16 T; the table: slot x 16
        __syncwarp();
      } else if (open) {  // the unit opens its slot with its packed sum (per lane)
        const uint4 r = PRE_REP ? rp : __ldg(hp - 1);
        sts_u4(mine_a + h.z, r);
      }
      if (h.w & 0x1Fu) {  // some transition of the step merges (thermometer of the step's maximum)
        constexpr int MAXM = LL == 1 ? 3 : 5;
#pragma unroll
        for (int k = 0; k < MAXM; ++k) {  // component sums into the surviving anchor
          if (!(th & (1u << (13 + k)))) break;
          const uint32_t src = (merges >> (6 * k)) & 7u, dst = (merges >> (6 * k + 3)) & 7u;
          const uint32_t da = mine_a + dst * (16u * T);
          // sg: bit k (k < 3) / k + 1: source k is a one-unit component,
          // bit 3: merge 0's destination is (later merges' never is)
          const bool s1 = WT && ((sg >> (k < 3 ? k : k + 1)) & 1u), d1 = WT && k == 0 && ((sg >> 3) & 1u);
          ulonglong2 d = lds_u2(d1 ? wtab_a + dst * 16u : da);
          const ulonglong2 v = lds_u2(s1 ? wtab_a + src * 16u : mine_a + src * (16u * T));
          fadd2(d.x, d.y, v.x, v.y);
          sts_u2(da, d);
        }
      }
      // the step's largest emit count (uniform, a thermometer at header bit
      // 8): later iterations of lanes with fewer emits see an empty ballot
      constexpr int MAXE = LL == 1 ? 3 : 5;
#pragma unroll
      for (int k = 0; k < MAXE; ++k) {  // multi-unit regions close: queued for pricing
        if (!(h.w & (0x100u << k))) break;
        const bool emit = (th >> (18 + k)) & 1u;
        const unsigned closing = __ballot_sync(0xffffffffu, emit);
        if (closing) {
          if (emit) {
            ulonglong2 v = lds_u2(mine_a + ((emits >> (3 * k)) & 7u) * (16u * T));
            v.y |= (uint64_t)lane << FSM_LANE_SHIFT;
            q[qn + __popc(closing & ((1u << lane) - 1u))] = v;
          }
          qn += __popc(closing);
          if (qn >= 32) {
            __syncwarp();
            fsm_price(q, lane, a, tlo, thi, inexact);
            __syncwarp();
            if (lane < qn - 32) q[lane] = q[32 + lane];
            __syncwarp();
            qn -= 32;
          }
        }
      }
      if (W > 0) on_next = bit_of(hn.y);  // next step's bit, off the state chain
    }
    if (ACC64) fadd2(tot_lo, tot_hi, (uint64_t)dacc, (uint64_t)(dacc >> 63));
    }
    __syncwarp();
    if (lane < qn) fsm_price(q, lane, a, tlo, thi, inexact);
    qn = 0;
    __syncwarp();
    fadd2(tot_lo, tot_hi, tlo[lane], thi[lane]);
    tlo[lane] = thi[lane] = 0ull;
    __syncwarp();
    if (in_range) {
      if (dead) {
        fit[i] = __longlong_as_double(0x7ff0000000000000ll);
      } else {
        const uint64_t sx = (uint64_t)((int64_t)tot_hi >> 63);
        fx192 v = fx_shl(fx192{{tot_lo, tot_hi, sx}}, a.shift);
        fx_add(v, a.base_const);
        fit[i] = fx_to_double(v);
      }
    }
  }
  if (inexact) atomicAdd(a.flags, 1ull);
}

template <int F, int W, int L>
int launch_fsm_t(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit, cudaStream_t stream) {
  const size_t smem = FsmSmemBase<F, W>::bytes + ((L & 3) != 0 ? (size_t)p->fsm_deltas * (L >= 4 ? 8 : 16) : 0);
  if (cb_smem_claim((const void*)fitness_fsm_kernel<F, W, L>, smem)) {
    CB_CUDA_TRY(cudaFuncSetAttribute(fitness_fsm_kernel<F, W, L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    // the smallest shared-memory configuration holding 1024 threads (8
    // blocks: the register limit); the rest of the 256 KB stays L1 for the transition
    // table (BERT-base, F = 6: 164 KB, +4% over the maximal carveout).  The
    // percentage is rounded down so it maps back onto that configuration.
    const char* cv = getenv("CB_FSM_CARVEOUT");
    int pct = 100;
    for (int kb : {100, 132, 164, 196})
      if ((size_t)kb * 1024 >= (size_t)FSM_MINB * (smem + 1024)) {
        pct = kb * 100 / 228;
        break;
      }
    CB_CUDA_TRY(cudaFuncSetAttribute(fitness_fsm_kernel<F, W, L>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cv ? atoi(cv) : pct));
  }
  int per_sm = 0;
  CB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fitness_fsm_kernel<F, W, L>, FSM_THREADS, smem));
  if (per_sm < 1) per_sm = 1;
  if (const char* cb = getenv("CB_FSM_BLOCKS")) per_sm = std::min(per_sm, std::max(1, atoi(cb)));
  FsmArgs a;
  a.M = p->M;
  a.words = p->words;
  a.shift = p->anchor_shift;
  a.base_const = p->base_const;
  const fx192 ex = fx_shr(p->eps, p->anchor_shift);
  a.eps_lo = ex.w[0];
  a.eps_hi = ex.w[1];
  a.hdr = reinterpret_cast<const uint4*>(p->d_fsm_hdr.p);
  a.table = reinterpret_cast<const uint4*>(p->d_fsm_table.p);
  a.ctable = reinterpret_cast<const uint2*>(p->d_fsm_ctable.p);
  a.mtable = reinterpret_cast<const uint4*>(p->d_fsm_ctable.p);
  a.xtable = p->d_fsm_ctable.p;
  a.dtab = reinterpret_cast<const uint4*>(p->d_fsm_dtab.p);
  a.n_delta = p->fsm_deltas;
  a.infeas = p->d_infeas.p;
  a.rt = p->d_rt.p;
  a.flags = p->d_flags.p;
  const int64_t want = (n + FSM_THREADS - 1) / FSM_THREADS;
  const int64_t grid = std::min<int64_t>(want, (int64_t)per_sm * cb_sm_count());
  fitness_fsm_kernel<F, W, L><<<(unsigned)grid, FSM_THREADS, smem, stream>>>(a, d_pop, n, d_fit);
  CB_CUDA_TRY(cudaGetLastError());
  return CB_OK;
}

template <int F>
int launch_fsm_w(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit, cudaStream_t stream) {
  // 64-bit deltas (L + 4) when the plan found every delta within a signed 64-bit word
  if (p->fsm_d64 && p->fsm_layout != 0) {
    switch (p->fsm_layout * 8 + (p->words <= 4 ? p->words : 0)) {
      case 8 + 1: return launch_fsm_t<F, 1, 5>(p, d_pop, n, d_fit, stream);
      case 8 + 2: return launch_fsm_t<F, 2, 5>(p, d_pop, n, d_fit, stream);
      case 8 + 3: return launch_fsm_t<F, 3, 5>(p, d_pop, n, d_fit, stream);
      case 8 + 4: return launch_fsm_t<F, 4, 5>(p, d_pop, n, d_fit, stream);
      case 8 + 0: return launch_fsm_t<F, 0, 5>(p, d_pop, n, d_fit, stream);
      case 16 + 1: return launch_fsm_t<F, 1, 6>(p, d_pop, n, d_fit, stream);
      case 16 + 2: return launch_fsm_t<F, 2, 6>(p, d_pop, n, d_fit, stream);
      case 16 + 3: return launch_fsm_t<F, 3, 6>(p, d_pop, n, d_fit, stream);
      case 16 + 4: return launch_fsm_t<F, 4, 6>(p, d_pop, n, d_fit, stream);
      case 16 + 0: return launch_fsm_t<F, 0, 6>(p, d_pop, n, d_fit, stream);
      case 24 + 1: return launch_fsm_t<F, 1, 7>(p, d_pop, n, d_fit, stream);
      case 24 + 2: return launch_fsm_t<F, 2, 7>(p, d_pop, n, d_fit, stream);
      case 24 + 3: return launch_fsm_t<F, 3, 7>(p, d_pop, n, d_fit, stream);
      case 24 + 4: return launch_fsm_t<F, 4, 7>(p, d_pop, n, d_fit, stream);
      default: return launch_fsm_t<F, 0, 7>(p, d_pop, n, d_fit, stream);
    }
  }
  switch (p->fsm_layout * 8 + (p->words <= 4 ? p->words : 0)) {
    case 8 + 1: return launch_fsm_t<F, 1, 1>(p, d_pop, n, d_fit, stream);
    case 8 + 2: return launch_fsm_t<F, 2, 1>(p, d_pop, n, d_fit, stream);
    case 8 + 3: return launch_fsm_t<F, 3, 1>(p, d_pop, n, d_fit, stream);
    case 8 + 4: return launch_fsm_t<F, 4, 1>(p, d_pop, n, d_fit, stream);
    case 8 + 0: return launch_fsm_t<F, 0, 1>(p, d_pop, n, d_fit, stream);
    case 16 + 1: return launch_fsm_t<F, 1, 2>(p, d_pop, n, d_fit, stream);
    case 16 + 2: return launch_fsm_t<F, 2, 2>(p, d_pop, n, d_fit, stream);
    case 16 + 3: return launch_fsm_t<F, 3, 2>(p, d_pop, n, d_fit, stream);
    case 16 + 4: return launch_fsm_t<F, 4, 2>(p, d_pop, n, d_fit, stream);
    case 16 + 0: return launch_fsm_t<F, 0, 2>(p, d_pop, n, d_fit, stream);
    case 24 + 1: return launch_fsm_t<F, 1, 3>(p, d_pop, n, d_fit, stream);
    case 24 + 2: return launch_fsm_t<F, 2, 3>(p, d_pop, n, d_fit, stream);
    case 24 + 3: return launch_fsm_t<F, 3, 3>(p, d_pop, n, d_fit, stream);
    case 24 + 4: return launch_fsm_t<F, 4, 3>(p, d_pop, n, d_fit, stream);
    case 24 + 0: return launch_fsm_t<F, 0, 3>(p, d_pop, n, d_fit, stream);
    case 1: return launch_fsm_t<F, 1, 0>(p, d_pop, n, d_fit, stream);
    case 2: return launch_fsm_t<F, 2, 0>(p, d_pop, n, d_fit, stream);
    case 3: return launch_fsm_t<F, 3, 0>(p, d_pop, n, d_fit, stream);
    case 4: return launch_fsm_t<F, 4, 0>(p, d_pop, n, d_fit, stream);
    default: return launch_fsm_t<F, 0, 0>(p, d_pop, n, d_fit, stream);
  }

}

// ------------------------------------------------------------ plan time

// A state: component label per slot (4 bits, 0 = free) and a multi-unit flag
// per component (bit c-1 for label c); labels numbered by first slot.
struct FsmState {
  uint32_t lab = 0, multi = 0;
  uint64_t key() const { return (uint64_t)lab | ((uint64_t)multi << 32); }
};

FsmState canonical(const int* lab, const bool* multi_of_label, int F) {
  int remap[16];
  for (int i = 0; i < 16; ++i) remap[i] = 0;
  int next = 0;
  FsmState s;
  for (int slot = 0; slot < F; ++slot) {
    const int l = lab[slot];
    if (!l) continue;
    if (!remap[l]) {
      remap[l] = ++next;
      if (multi_of_label[l]) s.multi |= 1u << (next - 1);
    }
    s.lab |= (uint32_t)remap[l] << (4 * slot);
  }
  return s;
}

struct FsmTrans {  // one computed transition before its next-state id is assigned
  FsmState ns;
  uint32_t open = 0, merges = 0, emits = 0, singles = 0;
  int n_merge = 0, n_emit = 0;
  fx192 dx;
  bool ok = false;
};

}  // namespace

static int fsm_entry_bytes(const cb_es_plan* P) {
  return P->fsm_layout == 1 || P->fsm_layout == 3 ? 8 : P->fsm_layout == 2 ? 16 : 32;
}

// Enumerate the reachable frontier states step by step and tabulate every
// (state, bit) transition.  Leaves fsm_ok false when the program is wider
// than 8 slots, a transition needs more actions than an entry encodes, or
// the table would exceed 64 MB.
int build_fsm_plan(cb_es_plan* P) {
  P->fsm_ok = false;
  if (!P->anchor_ok || P->F <= 0 || P->F > 8 || P->M == 0) return CB_OK;
  const auto t_build0 = std::chrono::steady_clock::now();
  const int32_t M = P->M, F = P->F;
  // packed sums: non-negative unit sums below 2^101 (window span <= 100) and
  // kernel counts that fit 16 bits
  if (P->anchor_span > 100) return CB_OK;
  int64_t cnt_total = 0;
  for (int32_t q = 0; q < M; ++q) {
    if ((P->prog[q].rep.w[2] >> 63) != 0 || P->prog[q].cnt < 0) return CB_OK;
    cnt_total += P->prog[q].cnt;
  }
  if (cnt_total > 0xFFFF) return CB_OK;
  std::vector<std::vector<int32_t>> ends(M);
  for (int32_t q = 0; q < M; ++q) ends[P->prog_last[q]].push_back(q);
  std::vector<uint4> table;
  std::vector<uint4> hdr(M);
  std::vector<int32_t> occ_end(F, -1);
  // genome word a step's bit lies in (W > 0 kernels reselect the word only
  // when it changes: FSM_BIT_NEWWORD); units without a bit read word `words`
  auto word_of = [&](int32_t q) -> int32_t {
    if (q < 0) return -1;
    return P->prog[q].bit >= 0 ? (int32_t)(P->prog[q].bit >> 6) : P->words;
  };
  std::vector<FsmState> cur(1);  // the empty frontier
  std::vector<uint64_t> hkey;
  std::vector<int32_t> hval;
  std::vector<FsmState> nxt;
  std::vector<FsmTrans> tr;
  const size_t cap = (size_t)64 << 20;
  for (int32_t p = 0; p < M; ++p) {
    const UnitRec& r = P->prog[p];
    const int S = r.slot;
    occ_end[S] = P->prog_last[p];
    if ((int)ends[p].size() != r.nend) return CB_OK;  // program / end lists disagree
    // bit | word << 8; a unit without a genome bit reads bit 0 of word
    // `words` (the kernel's all-ones word when W > 0) and is flagged for W = 0
    const uint32_t bitinfo = r.bit >= 0 ? ((uint32_t)r.bit & 63u) | ((uint32_t)(r.bit >> 6) << 8)
                                        : FSM_BIT_FORCED | ((uint32_t)P->words << 8);
    // z: the slot's byte offset in the kernel's per-thread slot sums
    hdr[p] = make_uint4((uint32_t)(table.size() / 2), bitinfo | (word_of(p) != word_of(p - 1) ? FSM_BIT_NEWWORD : 0u),
                        (uint32_t)S * 16u * FSM_THREADS, 0u);
    if ((table.size() + 4 * cur.size()) * sizeof(uint4) > cap) return CB_OK;
    // next-state ids: open addressing on key + 1 (0 = empty), sized for
    // every transition of the step
    size_t hsize = 16;
    int hbits = 4;
    while (hsize < 4 * cur.size()) {
      hsize <<= 1;
      ++hbits;
    }
    hkey.assign(hsize, 0ull);
    hval.resize(hsize);
    nxt.clear();
    // every (state, bit) transition of the step, in parallel over states;
    // next-state ids are then assigned in order, so the table is the same
    // for every thread count
    tr.resize(2 * cur.size());
    auto compute = [&](const FsmState& st, int on, FsmTrans& out) -> bool {
      int lab[8];
      bool multi[17];
      for (int i = 0; i < 17; ++i) multi[i] = false;
      for (int s = 0; s < F; ++s) {
        lab[s] = (st.lab >> (4 * s)) & 0xF;
        if (lab[s]) multi[lab[s]] = (st.multi >> (lab[s] - 1)) & 1u;
      }
      uint32_t open = 0, merges = 0, emits = 0, singles = 0;
      int n_merge = 0, n_emit = 0;
      fx192 delta = fx_zero();  // terms of the one-unit regions closed by this transition
      auto anchor_of = [&](int label) {  // member whose unit ends last (ties: larger slot)
        int best = -1;
        for (int s = 0; s < F; ++s)
          if (lab[s] == label && (best < 0 || occ_end[s] > occ_end[best] || (occ_end[s] == occ_end[best] && s > best)))
            best = s;
        return best;
      };
      if (on) {
        int join[8], nj = 0;
        for (int j = 0; j < r.nback; ++j) {
          const int b = P->prog_slots[r.back_off + j];
          const int l = lab[b];
          if (!l) continue;
          bool seen = false;
          for (int k = 0; k < nj; ++k) seen |= join[k] == l;
          if (!seen) join[nj++] = l;
        }
        int anchors[8];
        bool single[8];  // the joined component had one unit before this step
        for (int k = 0; k < nj; ++k) {
          anchors[k] = anchor_of(join[k]);
          single[k] = !multi[join[k]];
        }
        const int L = 16;  // temporary label of the new component
        lab[S] = L;
        multi[L] = nj > 0;
        for (int k = 0; k < nj; ++k)
          for (int s = 0; s < F; ++s)
            if (lab[s] == join[k]) lab[s] = L;
        const int Wn = anchor_of(L);
        open = 1;
        // one-unit operands (their sums come from the kernel's slot table):
        // the surviving anchor until the first merge writes it, every source
        // that is the new unit or a joined single.  singles: source m at bit
        // m (m < 3) / m + 1, merge 0's destination at bit 3
        bool dst_single = Wn == S;
        for (int k = 0; k < nj; ++k)
          if (anchors[k] == Wn) dst_single = single[k];
        auto add_merge = [&](int src, bool src_single) {
          if (n_merge >= 5) return false;
          merges |= ((uint32_t)src | ((uint32_t)Wn << 3)) << (6 * n_merge);
          if (src_single) singles |= 1u << (n_merge < 3 ? n_merge : n_merge + 1);
          if (n_merge == 0 && dst_single) singles |= 1u << 3;
          ++n_merge;
          return true;
        };
        for (int k = 0; k < nj; ++k)
          if (anchors[k] != Wn && !add_merge(anchors[k], single[k])) return false;
        if (S != Wn && !add_merge(S, true)) return false;
      }
      // releases: a component closes when its last member leaves; its data
      // is at the anchor it had when the step's releases began (the anchor
      // ends last, so members still present then end at this step too)
      int anchor_at[17];
      for (int l = 0; l < 17; ++l) anchor_at[l] = -1;
      for (int s = 0; s < F; ++s)
        if (lab[s] && anchor_at[lab[s]] < 0) anchor_at[lab[s]] = anchor_of(lab[s]);
      for (int j = 0; j < r.nend; ++j) {
        const int e = P->prog_slots[r.end_off + j];
        const int l = lab[e];
        if (!l) continue;
        const int A = anchor_at[l];
        lab[e] = 0;
        bool left = false;
        for (int s = 0; s < F; ++s) left |= lab[s] == l;
        if (left) continue;
        if (multi[l]) {
          if (n_emit >= 5) return false;
          emits |= (uint32_t)A << (3 * n_emit);
          ++n_emit;
        } else {
          fx_add(delta, P->prog[ends[p][j]].term1);  // its unit: end-list entry j
        }
      }
      // the new component's label may be 16: remap before canonicalising
      int lab2[8];
      bool multi2[17];
      for (int i = 0; i < 17; ++i) multi2[i] = multi[i];
      for (int s = 0; s < F; ++s) lab2[s] = lab[s];
      if (on) {
        int freel = 1;
        bool used[17] = {false};
        for (int s = 0; s < F; ++s) used[lab2[s]] = true;
        while (used[freel]) ++freel;
        for (int s = 0; s < F; ++s)
          if (lab2[s] == 16) lab2[s] = freel;
        multi2[freel] = multi[16];
      }
      const FsmState ns = canonical(lab2, multi2, F);
      // exact delta of the transition: terms of the one-unit regions it
      // closes minus the removed op-kernel term of an offloaded unit
      if (on && r.bit >= 0) fx_sub(delta, r.off);
      // to the 128-bit window: shift the magnitude, then restore the sign
      const bool neg = (delta.w[2] >> 63) != 0;
      fx192 mag = delta;
      if (neg) {
        mag = fx_zero();
        fx_sub(mag, delta);
      }
      fx192 dx = fx_shr(mag, P->anchor_shift);
      if (dx.w[2] != 0 || (dx.w[1] >> 62) != 0) return false;  // outside the window
      if (neg) {
        const fx192 m2 = dx;
        dx = fx_zero();
        fx_sub(dx, m2);
      }
      out.ns = ns;
      out.open = open;
      out.merges = merges;
      out.singles = singles;
      out.emits = emits;
      out.n_merge = n_merge;
      out.n_emit = n_emit;
      out.dx = dx;
      return true;
    };
    const int64_t n_states = (int64_t)cur.size();
#pragma omp parallel for schedule(static) if (n_states >= 64)
    for (int64_t si = 0; si < n_states; ++si)
      for (int on = 0; on < 2; ++on) tr[2 * si + on].ok = compute(cur[si], on, tr[2 * si + on]);
    for (const FsmTrans& t_ : tr) {
      if (!t_.ok) return CB_OK;
      const FsmState& ns = t_.ns;
      const uint32_t open = t_.open, merges = t_.merges, emits = t_.emits;
      const int n_merge = t_.n_merge, n_emit = t_.n_emit;
      const fx192& dx = t_.dx;
      const uint64_t hk = ns.key() + 1ull;
      size_t h = (size_t)((hk * 0x9E3779B97F4A7C15ull) >> (64 - hbits));  // Fibonacci hashing: top bits
      while (hkey[h] != 0ull && hkey[h] != hk) h = (h + 1) & (hsize - 1);
      int32_t nid;
      if (hkey[h] == 0ull) {
        nid = (int32_t)nxt.size();
        if (nid > 0xFFFF) return CB_OK;
        hkey[h] = hk;
        hval[h] = nid;
        nxt.push_back(ns);
      } else {
        nid = hval[h];
      }
      table.push_back(make_uint4((uint32_t)nid | (open << 16) | ((uint32_t)n_merge << 17) |
                                     ((uint32_t)n_emit << 20),
                                 merges, emits, fsm_therm(n_merge, n_emit) | t_.singles));
      table.push_back(make_uint4((uint32_t)dx.w[0], (uint32_t)(dx.w[0] >> 32), (uint32_t)dx.w[1],
                                 (uint32_t)(dx.w[1] >> 32)));
    }
    // step-level maxima: the kernel skips the emit / merge loops when no
    // transition of the step has any (warp-uniform)
    uint32_t max_emit = 0, max_merge = 0;
    for (size_t k = hdr[p].x * 2; k < table.size(); k += 2) {
      max_merge = std::max(max_merge, (table[k].x >> 17) & 7u);
      max_emit = std::max(max_emit, (table[k].x >> 20) & 7u);
    }
    hdr[p].w = ((1u << max_merge) - 1u) | (((1u << max_emit) - 1u) << 8);  // thermometers
    cur.swap(nxt);
  }
  // Renumber every step's states by visit frequency (most visited first),
  // estimated by walking 2 048 uniformly random genomes through the table:
  // the transitions a warp gathers then crowd into fewer cache lines.
  // CB_FSM_ORDER=0 keeps discovery order (A/B).  Only for cache-resident
  // tables (<= 64 K entries): on NasNet-A's 864 K it gained 1 % of the walk
  // for ~50 ms of plan time.
  if ((!getenv("CB_FSM_ORDER") || atoi(getenv("CB_FSM_ORDER")) != 0) && table.size() / 2 <= 65536) {
    const size_t n_ent = table.size() / 2;
    std::vector<uint32_t> base(M + 1);
    for (int32_t q = 0; q < M; ++q) base[q] = hdr[q].x / 2;
    base[M] = (uint32_t)(n_ent / 2);
    std::vector<uint32_t> visits(n_ent / 2, 0u);
    uint64_t x = 0x9E3779B97F4A7C15ull;
    for (int smp = 0; smp < 2048; ++smp) {
      uint32_t st = 0;
      for (int32_t q = 0; q < M; ++q) {
        ++visits[base[q] + st];
        x ^= x << 13;
        x ^= x >> 7;
        x ^= x << 17;
        const uint32_t bit = P->prog[q].bit >= 0 ? (uint32_t)(x >> 63) : 1u;
        st = table[2 * (hdr[q].x + 2 * st + bit)].x & 0xFFFFu;
      }
    }
    std::vector<uint32_t> newid(n_ent / 2), old_of(n_ent / 2);
    for (int32_t q = 0; q < M; ++q) {
      const uint32_t b0 = base[q], ns = base[q + 1] - b0;
      std::vector<uint32_t> ord(ns);
      std::iota(ord.begin(), ord.end(), 0u);
      // the walk starts in state 0 of step 0: keep it there
      std::stable_sort(ord.begin() + (q == 0 ? 1 : 0), ord.end(),
                       [&](uint32_t a2, uint32_t b2) { return visits[b0 + a2] > visits[b0 + b2]; });
      for (uint32_t j = 0; j < ns; ++j) {
        old_of[b0 + j] = ord[j];
        newid[b0 + ord[j]] = j;
      }
    }
    std::vector<uint4> t2(table.size());
    for (int32_t q = 0; q < M; ++q) {
      const uint32_t b0 = base[q], ns = base[q + 1] - b0;
      for (uint32_t j = 0; j < ns; ++j)
        for (uint32_t bit = 0; bit < 2; ++bit) {
          const size_t src = hdr[q].x + 2 * old_of[b0 + j] + bit, dst = hdr[q].x + 2 * j + bit;
          t2[2 * dst] = table[2 * src];
          t2[2 * dst + 1] = table[2 * src + 1];
          if (q + 1 < M) {
            const uint32_t nx = t2[2 * dst].x & 0xFFFFu;
            t2[2 * dst].x = (t2[2 * dst].x & ~0xFFFFu) | newid[base[q + 1] + nx];
          }
        }
    }
    table.swap(t2);
  }
  if (getenv("CB_FSM_STATS")) {
    int smax = 0, mm = 0, me = 0, dbits = 0, zero = 0;
    size_t wide_entries = 0, wide_steps = 0;  // entries / steps beyond the 8-byte layout
    for (int32_t q = 0; q < M; ++q) {
      const size_t b = hdr[q].x * 2, e = q + 1 < M ? hdr[q + 1].x * 2 : table.size();
      bool any = false;
      for (size_t k2 = b; k2 < e; k2 += 2) {
        const uint32_t xx = table[k2].x;
        const bool w = (xx & 0xFFFFu) > 0xFFFu || ((xx >> 17) & 7u) > 3 || ((xx >> 20) & 7u) > 3;
        wide_entries += w;
        any |= w;
      }
      wide_steps += any;
    }
    fprintf(stderr, "fsm stats: %zu of %zu entries and %zu of %d steps need more than 8 bytes\n", wide_entries,
            table.size() / 2, wide_steps, M);
    std::unordered_map<uint64_t, int> dd;
    for (int32_t q = 0; q < M; ++q) {
      const size_t b = hdr[q].x * 2, e = q + 1 < M ? hdr[q + 1].x * 2 : table.size();
      smax = std::max<int>(smax, (int)((e - b) / 4));
      for (size_t k = b; k < e; k += 2) {
        mm = std::max<int>(mm, (table[k].x >> 17) & 7);
        me = std::max<int>(me, (table[k].x >> 20) & 7);
        const uint64_t lo = ((uint64_t)table[k + 1].y << 32) | table[k + 1].x;
        const uint64_t hi = ((uint64_t)table[k + 1].w << 32) | table[k + 1].z;
        const bool neg = hi >> 63;
        uint64_t ml = lo, mh = hi;
        if (neg) { ml = ~lo + 1; mh = ~hi + (ml == 0); }
        const int bits = mh ? 128 - __builtin_clzll(mh) : (ml ? 64 - __builtin_clzll(ml) : 0);
        dbits = std::max(dbits, bits);
        zero += !lo && !hi;
        dd[lo * 1000003ull ^ hi] = 1;
      }
    }
    fprintf(stderr, "fsm stats: M %d F %d entries %zu states/step max %d merges max %d emits max %d delta bits max %d zero %d distinct %zu window span %d enumeration %.1f ms\n",
            M, F, table.size() / 2, smax, mm, me, dbits, zero, dd.size(), P->anchor_span,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_build0).count());
  }
  const size_t n_entries = table.size() / 2;
  // the smallest layout every transition fits: 8 bytes (12-bit next state,
  // <= 3 merges / emits), 16 bytes (<= 5), else 32; both short layouts index
  // <= 256 distinct deltas.  CB_FSM_ENTRY_BYTES (8 / 16 / 32) sets the
  // smallest layout tried (tests), CB_FSM_WIDE_ENTRIES forces 32.
  std::vector<uint32_t> stab;
  std::vector<uint4> dtab;
  P->fsm_layout = 0;
  {
    int min_bytes = getenv("CB_FSM_ENTRY_BYTES") ? atoi(getenv("CB_FSM_ENTRY_BYTES")) : 8;
    if (getenv("CB_FSM_WIDE_ENTRIES")) min_bytes = 32;
    std::unordered_map<std::string, uint32_t> didx;
    bool deltas_fit = true;
    std::vector<uint32_t> dref(n_entries);
    for (size_t k = 0; k < n_entries && deltas_fit; ++k) {
      const uint4 dv = table[2 * k + 1];
      const std::string key(reinterpret_cast<const char*>(&dv), sizeof(dv));
      auto it = didx.find(key);
      if (it == didx.end()) {
        if (dtab.size() >= 256) {
          deltas_fit = false;
          break;
        }
        it = didx.emplace(key, (uint32_t)dtab.size()).first;
        dtab.push_back(dv);
      }
      dref[k] = it->second;
    }
    bool fits8 = deltas_fit && min_bytes <= 8, fits16 = deltas_fit && min_bytes <= 16;
    for (int32_t q = 0; fits8 && q < M; ++q) {
      const size_t b = hdr[q].x, e = q + 1 < M ? hdr[q + 1].x : n_entries;
      if (e - b > 2 * 4096) fits8 = false;  // next-state ids take 12 bits
    }
    for (size_t k = 0; fits8 && k < n_entries; ++k) {
      const uint32_t x = table[2 * k].x;
      if ((x & 0xFFFFu) > 0xFFFu || ((x >> 17) & 7u) > 3 || ((x >> 20) & 7u) > 3) fits8 = false;
    }
    // mixed layout: 8-byte transitions for every step whose entries fit,
    // 16-byte ones for the rest (NasNet-A: 16 of 620 steps)
    std::vector<uint8_t> step_wide(M, 0);
    bool mixed = !fits8 && fits16 && min_bytes <= 8 &&
                 !(getenv("CB_FSM_MIXED") && atoi(getenv("CB_FSM_MIXED")) == 0);
    size_t narrow_steps = 0;
    for (int32_t q = 0; mixed && q < M; ++q) {
      const size_t b = hdr[q].x, e = q + 1 < M ? hdr[q + 1].x : n_entries;
      bool w = e - b > 2 * 4096;
      for (size_t k = b; k < e && !w; ++k) {
        const uint32_t x = table[2 * k].x;
        w = (x & 0xFFFFu) > 0xFFFu || ((x >> 17) & 7u) > 3 || ((x >> 20) & 7u) > 3;
      }
      step_wide[q] = w;
      narrow_steps += !w;
    }
    if (mixed && narrow_steps == 0) mixed = false;
    // wide steps of the mixed layout share the 8-byte field positions (12-bit next state)
    for (int32_t q = 0; mixed && q < M; ++q) {
      const size_t b = hdr[q].x, e = q + 1 < M ? hdr[q + 1].x : n_entries;
      for (size_t k = b; step_wide[q] && k < e; ++k)
        if ((table[2 * k].x & 0xFFFFu) > 0xFFFu) mixed = false;
    }
    if (mixed) {
      P->fsm_layout = 3;
      std::vector<uint32_t> offs(M);
      size_t words = 0;
      for (int32_t q = 0; q < M; ++q) {
        const size_t b = hdr[q].x, e = q + 1 < M ? hdr[q + 1].x : n_entries;
        if (step_wide[q]) words = (words + 3) & ~(size_t)3;  // 16-byte aligned
        offs[q] = (uint32_t)words;
        words += (e - b) * (step_wide[q] ? 4 : 2);
      }
      stab.assign(words, 0u);
      for (int32_t q = 0; q < M; ++q) {
        const size_t b = hdr[q].x, e = q + 1 < M ? hdr[q + 1].x : n_entries;
        for (size_t k = b; k < e; ++k) {
          const uint4 t0 = table[2 * k];
          uint32_t* dst = stab.data() + offs[q] + (k - b) * (step_wide[q] ? 4 : 2);
          if (step_wide[q]) {
            dst[0] = (t0.x & 0xFFFu) | (((t0.x >> 16) & 1u) << 12) | (t0.w & ~0x3Fu) | (dref[k] << 24);
            dst[1] = t0.y;
            dst[2] = t0.z;
            dst[3] = t0.w & 0x3Fu;  // singles
          } else {
            const uint32_t nxt = t0.x & 0xFFFFu, open = (t0.x >> 16) & 1u, nm = (t0.x >> 17) & 7u,
                           ne = (t0.x >> 20) & 7u;
            dst[0] = nxt | (open << 12) | fsm_therm(nm, ne) | (dref[k] << 24);
            dst[1] = (t0.y & 0x3FFFFu) | ((t0.z & 0x1FFu) << 18) | ((t0.w & 0xFu) << 27);
          }
        }
        hdr[q].x = offs[q];
        if (step_wide[q]) hdr[q].w |= FSM_WIDE_STEP;
      }
    } else if (fits8) {
      P->fsm_layout = 1;
      stab.resize(2 * n_entries);
      for (size_t k = 0; k < n_entries; ++k) {
        const uint4 t0 = table[2 * k];
        const uint32_t nxt = t0.x & 0xFFFFu, open = (t0.x >> 16) & 1u, nm = (t0.x >> 17) & 7u, ne = (t0.x >> 20) & 7u;
        stab[2 * k] = nxt | (open << 12) | fsm_therm(nm, ne) | (dref[k] << 24);
        stab[2 * k + 1] = (t0.y & 0x3FFFFu) | ((t0.z & 0x1FFu) << 18) | ((t0.w & 0xFu) << 27);
      }
    } else if (fits16) {
      P->fsm_layout = 2;
      stab.resize(4 * n_entries);
      for (size_t k = 0; k < n_entries; ++k) {
        const uint4 t0 = table[2 * k];
        stab[4 * k] = (t0.x & 0xFFFFFFu) | (dref[k] << 24);
        stab[4 * k + 1] = t0.y;
        stab[4 * k + 2] = t0.z;
        stab[4 * k + 3] = t0.w;  // thermometers
      }
    } else {
      dtab.clear();
    }
  }
  // step headers interleaved with the units' packed sums
  // (+ one dummy step: the kernel prefetches step p + 1's header unguarded)
  std::vector<uint4> hdr2((size_t)2 * M + 2, make_uint4(0u, 0u, 0u, 0u));
  for (int32_t q = 0; q < M; ++q) {
    const fx192 x = fx_shr(P->prog[q].rep, P->anchor_shift);
    const uint64_t hi = x.w[1] | ((uint64_t)P->prog[q].cnt << FSM_CNT_SHIFT);
    hdr2[2 * q] = hdr[q];
    hdr2[2 * q + 1] = make_uint4((uint32_t)x.w[0], (uint32_t)(x.w[0] >> 32), (uint32_t)hi, (uint32_t)(hi >> 32));
  }
  cudaError_t e;
  if (P->fsm_layout != 0) {
    if ((e = P->d_fsm_ctable.upload(stab.data(), stab.size())) != cudaSuccess ||
        (e = P->d_fsm_dtab.upload(reinterpret_cast<const uint32_t*>(dtab.data()), dtab.size() * 4)) != cudaSuccess) {
      cb_set_error(std::string("CUDA error in plan upload: ") + cudaGetErrorString(e));
      return CB_ERR_CUDA;
    }
    P->fsm_deltas = (int32_t)dtab.size();
    // 8-byte shared deltas when every distinct delta is a sign-extended
    // 64-bit value below 2^57 in magnitude (all BASELINE models: <= 57 bits); CB_FSM_D64=0 keeps
    // the 16-byte table (A/B, tests)
    P->fsm_d64 = !(getenv("CB_FSM_D64") && atoi(getenv("CB_FSM_D64")) == 0);
    for (const uint4& d : dtab) {
      const uint64_t lo = ((uint64_t)d.y << 32) | d.x, hi = ((uint64_t)d.w << 32) | d.z;
      // |d| < 2^57: 64 steps' deltas sum within the kernel's 64-bit accumulator
      const int64_t top = (int64_t)lo >> 57;
      P->fsm_d64 = P->fsm_d64 && hi == ((lo >> 63) ? ~0ull : 0ull) && (top == 0 || top == -1) &&
                   (int64_t)lo != -(int64_t)(1ull << 57);
    }
    table.resize(2);  // only the short copy is kept on the device
  }
  if ((e = P->d_fsm_hdr.upload(reinterpret_cast<const uint32_t*>(hdr2.data()), hdr2.size() * 4)) != cudaSuccess ||
      (e = P->d_fsm_table.upload(reinterpret_cast<const uint32_t*>(table.data()), table.size() * 4)) !=
          cudaSuccess) {
    cb_set_error(std::string("CUDA error in plan upload: ") + cudaGetErrorString(e));
    return CB_ERR_CUDA;
  }
  P->fsm_states_max = 0;
  P->fsm_entries = (int64_t)n_entries;
  P->fsm_ok = true;
  // automatic selection while the table stays cache-resident: in L1 for
  // BERT-base (46 KB), in L2 for NasNet-A (13.8 MB at 16 bytes, still faster
  // than the packed-label walk); `set_path("fsm")` forces it beyond
  const size_t table_bytes = P->fsm_layout == 3 ? P->d_fsm_ctable.n * sizeof(uint32_t)
                                                 : n_entries * (size_t)fsm_entry_bytes(P);
  P->fsm_auto = table_bytes <= ((size_t)32 << 20);
  return CB_OK;
}

int launch_fitness_fsm(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit, cudaStream_t stream) {
  if (p->F <= 4) return launch_fsm_w<4>(p, d_pop, n, d_fit, stream);
  if (p->F <= 6) return launch_fsm_w<6>(p, d_pop, n, d_fit, stream);
  return launch_fsm_w<8>(p, d_pop, n, d_fit, stream);
}
