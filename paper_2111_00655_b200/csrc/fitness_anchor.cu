// Thread-per-genome frontier walk for wide programs (up to 64 slots): the
// kernel for the random 100k-op DAG (36 slots), BASELINE.json configs[4].
//
// Semantics are those of every fitness kernel here (tensorplace/
// evolution.py:65-135 decode, tensorplace/cost.py:320-373 graph-level
// pricing): the genome's ON units form regions = connected components of
// the unit graph; a region of one unit costs its precomputed term1, a larger
// one round(sum) * r(n) + eps, every OFF unit its own kernel term.
//
// Lanes walk the frontier program in lockstep, one genome each, so every
// per-step record is a warp-uniform (broadcast) load; only the component
// structure of the occupied slots and the merged components' sums are
// per-lane data:
//
// * Anchors.  A component's data lives at its ANCHOR: the member slot whose
//   unit has the latest end (last neighbour position).  Merging two
//   components keeps the later-ending anchor, so no member outlives its
//   anchor and no data ever moves between slots.
// * Byte labels.  A non-anchor slot holds a parent slot of its component
//   (path-compressed on lookup; a pointer always targets a slot that ends no
//   earlier); an anchor holds a flag, plus a pool entry when merged.
// * Visiting ON unit p adds term1(p) - off(p) to the lane's total (right
//   while p stays alone); merging a one-unit component takes its term1 back
//   and contributes its replacement sum to the merged component's pool
//   entry (128-bit window sum with the kernel count in bits 108-127).
// * Closing without end lists.  The plan hands a slot to a later unit only
//   after its unit's last neighbour, and an anchor ends last in its
//   component, so a merged component is complete exactly when its anchor
//   slot is handed on: the step reading the slot's old label queues the
//   sum for pricing (round, __dmul_rn by r(n), + eps: warp batches of 32).
//   Every pool entry is named by one anchor label, so a lane never holds
//   more than F entries (C in shared memory, the rest in local memory).
// * Per-warp slot table.  The unit currently in each slot is the same for
//   all lanes: (end, replacement sum | count, term1) per slot, written by
//   three lanes per step from the unit's 48-byte slot record, so merges
//   read everything from shared memory.
// * Genome words are read per lane one word ahead (rows are read once).
//
// Shared memory per thread: one byte per slot + 16 bytes per pool entry; per
// warp the slot table, the region queue and the owner accumulators.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "fitness_plan.cuh"

#define AN_QCAP 32

namespace {

// 80-byte step record (five 16-byte chunks): the step header, term1 - off
// (added when the unit is ON) and the unit's slot-table entry
struct __align__(16) AStep {
  uint32_t bs;     // genome bit (bits 0-23; 0xFFFFFF: always-on fixed unit) | slot << 24 | long << 31
  uint32_t lists;  // short: nback (3 bits) | back slot j at 3 + 6 j (j < 4); long: nback
  uint32_t off;    // long: offset of the back list
  uint32_t pad;
};
static_assert(sizeof(AStep) == 16, "AStep layout");
constexpr int REC_CHUNKS = 5;             // AStep | term1 - off | end | rep, count | term1
constexpr int REC_BYTES = 16 * REC_CHUNKS;
constexpr int WT_OFF = 32;                // slot-table part of a record
constexpr uint32_t WT_BYTES = 48;         // slot table entry: end | rep, count | term1
constexpr int CH = 32;                    // steps per staged record chunk

// labels (one byte per slot and lane): 0 = no ON unit, 0x80 = anchor of a
// one-unit component, 0xC0 | e = anchor of a merged component (pool entry
// e), 0x40 | s = member pointing to slot s (which ends no earlier)
constexpr uint32_t L_ANCHOR = 0x80u;
constexpr uint32_t L_MERGED = 0x40u;
constexpr uint32_t L_PTR = 0x40u;
constexpr int CNT_SHIFT = 44;  // count at bit 64 + 44 = 108 of a packed sum
constexpr uint64_t VAL_HI_MASK = (1ull << CNT_SHIFT) - 1ull;

struct X128 {
  uint64_t lo, hi;
};

__device__ __forceinline__ void x_add(X128& a, const X128& b) {
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(a.lo), "+l"(a.hi) : "l"(b.lo), "l"(b.hi));
}
__device__ __forceinline__ void x_sub(X128& a, const X128& b) {
  asm("sub.cc.u64 %0, %0, %2;\n\tsubc.u64 %1, %1, %3;" : "+l"(a.lo), "+l"(a.hi) : "l"(b.lo), "l"(b.hi));
}

struct AnArgs {
  int32_t M, words, shift, n_infeas, Fp, F;
  fx192 base_const;
  X128 eps;
  const uint4* __restrict__ rec;        // [M][5] step records
  const uint8_t* __restrict__ lists;    // long back lists
  const int32_t* __restrict__ infeas_word;
  const uint64_t* __restrict__ infeas_mask;
  const double* __restrict__ rt;
  unsigned long long* flags;
};

// Price the queued regions (one per lane) and add each term to its owner's
// 128-bit accumulator (shared atomics: an owner can have several entries).
__device__ __forceinline__ void an_flush(const ulonglong2* qx, const uint8_t* qown, int qn, int lane,
                                         const AnArgs& a, unsigned long long* tacc, bool& inexact) {
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

// 32-bit shared-memory addressing (addresses stay in registers)
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u8(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ int32_t lds_s32(uint32_t a) {
  int32_t v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ X128 lds_x(uint32_t a) {
  X128 v;
  asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(v.lo), "=l"(v.hi) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds_v4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_x(uint32_t a, const X128& v) {
  asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(a), "l"(v.lo), "l"(v.hi));
}
__device__ __forceinline__ void sts_v4(uint32_t a, const uint4& v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// Stage the records of chunk c (steps [c * CH, c * CH + CH) clipped to M)
// into buffer `buf` -- the block's threads copy 16 bytes each, asynchronously.
__device__ __forceinline__ void stage_chunk(const AnArgs& a, int32_t c, uint32_t buf, int t, int T) {
  const int32_t p0 = c * CH;
  const int32_t n16 = max(0, min(CH, a.M - p0)) * REC_CHUNKS;
  const uint4* src = a.rec + (int64_t)p0 * REC_CHUNKS;
  for (int k = t; k < n16; k += T) cp_async16(buf + 16 * k, src + k);
  cp_async_commit();
}

// Per-lane walk state.
struct AnLane {
  uint32_t lab;    // shared address of this lane's label for slot 0 (slot s at + 4 s)
  uint32_t pool;   // shared address of this lane's pool entry 0 (entry e < C at + e * 16 T)
  uint32_t wtab;   // shared address of the warp's slot table (slot s at + 48 s)
  uint64_t pfree;  // free pool entries
  X128 total;      // genome-dependent part of the cost (two's complement)
};

// pool entries e >= C live in the thread's local memory (lane-interleaved,
// L1-cached; at most F <= 64 entries are ever held)
template <int C, int T>
__device__ __forceinline__ X128 pool_ld(const AnLane& L, const ulonglong2* spill, uint32_t e) {
  if (e < (uint32_t)C) return lds_x(L.pool + e * (16 * T));
  const ulonglong2 v = spill[e - C];
  return {v.x, v.y};
}
template <int C, int T>
__device__ __forceinline__ void pool_st(const AnLane& L, ulonglong2* spill, uint32_t e, const X128& v) {
  if (e < (uint32_t)C)
    sts_x(L.pool + e * (16 * T), v);
  else
    spill[e - C] = make_ulonglong2(v.lo, v.hi);
}

// Back edge to slot b (label lb) of the new unit whose component is
// anchored at A: find b's anchor, merge the two components at the
// later-ending anchor.
template <int C, int T>
__device__ __forceinline__ void an_merge(AnLane& L, ulonglong2* spill, bool need, uint32_t b, uint32_t lb,
                                         uint32_t& A) {
  uint32_t x = b, lx = need ? lb : L_ANCHOR;
  if (!(lx & L_ANCHOR)) {
    x = lx & 63u;
    lx = lds_u8(L.lab + 4 * x);
  }
  while (__any_sync(0xffffffffu, !(lx & L_ANCHOR))) {  // rare deeper chains
    if (!(lx & L_ANCHOR)) {
      x = lx & 63u;
      lx = lds_u8(L.lab + 4 * x);
    }
  }
  if (x != b) sts_u8(L.lab + 4 * b, L_PTR | x);  // path compression (x == b when !need)
  if (!need || x == A) return;
  const uint32_t lA = lds_u8(L.lab + 4 * A);
  const bool keepA = lds_s32(L.wtab + WT_BYTES * A) >= lds_s32(L.wtab + WT_BYTES * x);
  const uint32_t Wn = keepA ? A : x, Xn = keepA ? x : A;
  const uint32_t lW = keepA ? lA : lx, lX = keepA ? lx : lA;
  const bool mW = (lW & L_MERGED) != 0u, mX = (lX & L_MERGED) != 0u;
  const uint32_t eW = lW & 63u, eX = lX & 63u;
  // sums: a merged component's pool entry, a one-unit component's
  // replacement sum from the slot table (whose one-unit term leaves the
  // total) -- selects, not branches; pool entries >= C (rare) from local memory
  const uint32_t wW = L.wtab + WT_BYTES * Wn, wX = L.wtab + WT_BYTES * Xn;
  X128 sW = lds_x(mW && eW < (uint32_t)C ? L.pool + eW * (16 * T) : wW + 16);
  X128 sX = lds_x(mX && eX < (uint32_t)C ? L.pool + eX * (16 * T) : wX + 16);
  if (mW && eW >= (uint32_t)C) sW = pool_ld<C, T>(L, spill, eW);
  if (mX && eX >= (uint32_t)C) sX = pool_ld<C, T>(L, spill, eX);
  const X128 tW = lds_x(wW + 32), tX = lds_x(wX + 32);
  x_sub(L.total, X128{mW ? 0ull : tW.lo, mW ? 0ull : tW.hi});
  x_sub(L.total, X128{mX ? 0ull : tX.lo, mX ? 0ull : tX.hi});
  x_add(sW, sX);
  // the surviving entry: W's, else X's, else a fresh one (at most F <= 64
  // entries are ever named by anchor labels; the low 32 nearly always)
  const uint32_t lo = (uint32_t)L.pfree;
  const uint32_t fresh = lo ? (uint32_t)(__ffs(lo) - 1) : 32u + (uint32_t)(__ffs((uint32_t)(L.pfree >> 32)) - 1);
  const uint32_t e = mW ? eW : (mX ? eX : fresh);
  L.pfree = (!mW && !mX) ? (L.pfree & (L.pfree - 1ull)) : L.pfree;
  L.pfree |= (mW && mX) ? (1ull << eX) : 0ull;
  pool_st<C, T>(L, spill, e, sW);
  sts_u8(L.lab + 4 * Wn, L_ANCHOR | L_MERGED | e);
  sts_u8(L.lab + 4 * Xn, L_PTR | Wn);
  A = Wn;
}

// an_merge with branches instead of selects (A/B: CB_ANCHOR_MERGE=1)
template <int C, int T>
__device__ __forceinline__ void an_merge_br(AnLane& L, ulonglong2* spill, bool need, uint32_t b, uint32_t lb,
                                         uint32_t& A) {
  uint32_t x = b, lx = need ? lb : L_ANCHOR;
  if (!(lx & L_ANCHOR)) {
    x = lx & 63u;
    lx = lds_u8(L.lab + 4 * x);
  }
  while (__any_sync(0xffffffffu, !(lx & L_ANCHOR))) {  // rare deeper chains
    if (!(lx & L_ANCHOR)) {
      x = lx & 63u;
      lx = lds_u8(L.lab + 4 * x);
    }
  }
  if (x != b) sts_u8(L.lab + 4 * b, L_PTR | x);  // path compression (x == b when !need)
  if (!need || x == A) return;
  const uint32_t lA = lds_u8(L.lab + 4 * A);
  const bool keepA = lds_s32(L.wtab + WT_BYTES * A) >= lds_s32(L.wtab + WT_BYTES * x);
  const uint32_t Wn = keepA ? A : x, Xn = keepA ? x : A;
  const uint32_t lW = keepA ? lA : lx, lX = keepA ? lx : lA;
  X128 sW, sX;
  // merged components: their pool sums; one-unit components: the unit's
  // replacement sum, and its one-unit term leaves the total
  if (lW & L_MERGED) {
    sW = pool_ld<C, T>(L, spill, lW & 63u);
  } else {
    sW = lds_x(L.wtab + WT_BYTES * Wn + 16);
    x_sub(L.total, lds_x(L.wtab + WT_BYTES * Wn + 32));
  }
  if (lX & L_MERGED) {
    sX = pool_ld<C, T>(L, spill, lX & 63u);
  } else {
    sX = lds_x(L.wtab + WT_BYTES * Xn + 16);
    x_sub(L.total, lds_x(L.wtab + WT_BYTES * Xn + 32));
  }
  x_add(sW, sX);
  uint32_t e;
  if (lW & L_MERGED) {
    e = lW & 63u;
    if (lX & L_MERGED) L.pfree |= 1ull << (lX & 63u);
  } else if (lX & L_MERGED) {
    e = lX & 63u;
  } else {
    // at most F <= 64 entries are ever named by anchor labels
    e = (uint32_t)(__ffsll((long long)L.pfree) - 1);
    L.pfree &= L.pfree - 1ull;
  }
  pool_st<C, T>(L, spill, e, sW);
  sts_u8(L.lab + 4 * Wn, L_ANCHOR | L_MERGED | e);
  sts_u8(L.lab + 4 * Xn, L_PTR | Wn);
  A = Wn;
}

// The label a slot held before it is handed on (or the program ends): a
// merged anchor's region is complete -- queue it; all lanes take part.
template <int C, int T>
__device__ __forceinline__ void an_close(AnLane& L, const ulonglong2* spill, uint32_t old, int lane, int owner,
                                         ulonglong2* qx, uint8_t* qown,
                                         int& qn, const AnArgs& a, unsigned long long* tacc, bool& inexact) {
  const bool emit = (old & (L_ANCHOR | L_MERGED)) == (L_ANCHOR | L_MERGED);
  const unsigned closing = __ballot_sync(0xffffffffu, emit);
  if (!closing) return;
  X128 ev = {0ull, 0ull};
  if (emit) {
    ev = pool_ld<C, T>(L, spill, old & 63u);
    L.pfree |= 1ull << (old & 63u);
  }
  const int cnt = __popc(closing);
  if (qn + cnt > AN_QCAP) {
    an_flush(qx, qown, qn, lane, a, tacc, inexact);
    qn = 0;
  }
  if (emit) {
    const int at = qn + __popc(closing & ((1u << lane) - 1u));
    qx[at] = make_ulonglong2(ev.lo, ev.hi);
    qown[at] = (uint8_t)owner;
  }
  qn += cnt;
}

// Block-lockstep walk: the warps of a block step through the program
// together, so each 32-step chunk of records is staged once per block
// (cp.async, double-buffered) and every per-step record read is a
// broadcast shared-memory load.  Each thread walks G genomes at once
// (independent instruction streams that hide each other's latency, one
// record decode for both).
template <int C, int T, int G, int MB>
__global__ void __launch_bounds__(T, (G == 1 ? 768 : 512) / T)
fitness_anchor_kernel(AnArgs a, const uint64_t* __restrict__ pop, int64_t n, double* __restrict__ fit) {
  constexpr int W = T / 32;
  extern __shared__ __align__(16) unsigned char an_smem[];
  unsigned char* chunks = an_smem;                                            // [2][CH][80]
  ulonglong2* pool = reinterpret_cast<ulonglong2*>(chunks + 2 * CH * REC_BYTES);  // [G][C][T]
  ulonglong2* qx_all = pool + G * C * T;                                      // [W][QCAP]
  unsigned long long* tacc_all = reinterpret_cast<unsigned long long*>(qx_all + W * AN_QCAP);  // [W][32 G][2]
  unsigned char* wtab_all = reinterpret_cast<unsigned char*>(tacc_all + W * 64 * G);  // [W][F][48]
  uint8_t* qown_all = wtab_all + (size_t)W * a.F * WT_BYTES;                 // [W][QCAP]
  uint8_t* LAB = qown_all + W * AN_QCAP;                                      // [G][T / 4][Fp][4]
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  ulonglong2* qx = qx_all + warp * AN_QCAP;
  uint8_t* qown = qown_all + warp * AN_QCAP;
  unsigned long long* tacc = tacc_all + warp * 64 * G;
  const uint32_t chunk0 = (uint32_t)__cvta_generic_to_shared(chunks);
  const uint32_t wtab0 = (uint32_t)__cvta_generic_to_shared(wtab_all + (size_t)warp * a.F * WT_BYTES);
  AnLane L[G];
  ulonglong2 spill[G][64 - C];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    L[g].lab = (uint32_t)__cvta_generic_to_shared(LAB + (size_t)g * (T / 4) * a.Fp * 4 + (t >> 2) * a.Fp * 4 + (t & 3));
    L[g].pool = (uint32_t)__cvta_generic_to_shared(pool + (size_t)g * C * T + t);
    L[g].wtab = wtab0;
    for (int s = 0; s < a.F; ++s) sts_u8(L[g].lab + 4 * s, 0u);
    tacc[2 * (G * lane + g)] = tacc[2 * (G * lane + g) + 1] = 0ull;
  }
  __syncwarp();
  bool inexact = false;
  const int32_t n_chunks = (a.M + CH - 1) / CH;
  const int64_t stride = (int64_t)gridDim.x * T * G;
  // every warp of the block runs the same number of genome rounds (block syncs)
  for (int64_t base = (int64_t)blockIdx.x * T * G; base < n; base += stride) {
    int64_t gi[G];
    const uint64_t* gen[G];
    bool dead[G];
    uint64_t w0[G], w1[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      gi[g] = base + (int64_t)g * T + t;
      const bool in_range = gi[g] < n;
      gen[g] = pop + (in_range ? gi[g] : 0) * a.words;
      dead[g] = !in_range;
      for (int32_t j = 0; j < a.n_infeas; ++j)
        dead[g] |= (__ldg(gen[g] + __ldg(a.infeas_word + j)) & __ldg(a.infeas_mask + j)) != 0ull;
      L[g].pfree = ~0ull;
      L[g].total = {0ull, 0ull};
      w0[g] = w1[g] = 0ull;
    }
    int qn = 0;
    int32_t cur_w = -2;  // genome words: w0 = word cur_w, w1 = word cur_w + 1 (loaded ahead)
    __syncthreads();  // the previous round is done with both buffers
    stage_chunk(a, 0, chunk0, t, T);
    stage_chunk(a, 1, chunk0 + CH * REC_BYTES, t, T);
    for (int32_t c = 0; c < n_chunks; ++c) {
      cp_async_wait1();  // chunk c has landed (c + 1 may be in flight)
      __syncthreads();
      const uint32_t buf = chunk0 + (uint32_t)(c & 1) * (CH * REC_BYTES);
      const int32_t steps = min(CH, a.M - c * CH);
      for (int32_t k = 0; k < steps; ++k) {
        const uint32_t r = buf + k * REC_BYTES;
        const uint4 h = lds_v4(r);
        const uint32_t bitf = h.x & 0xFFFFFFu;
        const uint32_t S = (h.x >> 24) & 63u;
        // the unit's slot-table entry (three lanes, 16 bytes each); the slot's
        // previous unit may still be read by lanes finishing the last step's merges
        __syncwarp();
        if (lane < 3) sts_v4(wtab0 + WT_BYTES * S + 16 * lane, lds_v4(r + WT_OFF + 16 * lane));
        bool on[G];
#pragma unroll
        for (int g = 0; g < G; ++g) on[g] = !dead[g];
        if (bitf != 0xFFFFFFu) {
          const int32_t wi = (int32_t)(bitf >> 6);
          if (wi != cur_w) {  // warp uniform
#pragma unroll
            for (int g = 0; g < G; ++g) {
              w0[g] = (wi == cur_w + 1) ? w1[g] : (dead[g] ? 0ull : __ldg(gen[g] + wi));
              w1[g] = (!dead[g] && wi + 1 < a.words) ? __ldg(gen[g] + wi + 1) : 0ull;
            }
            cur_w = wi;
          }
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const uint32_t half = (bitf & 32u) ? (uint32_t)(w0[g] >> 32) : (uint32_t)w0[g];
            on[g] = on[g] && ((half >> (bitf & 31u)) & 1u);
          }
        }
        const X128 tm = lds_x(r + 16);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          // the slot's previous owner is complete
          const uint32_t labS = L[g].lab + 4 * S;
          an_close<C, T>(L[g], spill[g], lds_u8(labS), lane, G * lane + g, qx, qown, qn, a, tacc, inexact);
          sts_u8(labS, on[g] ? L_ANCHOR : 0u);
          if (on[g]) x_add(L[g].total, tm);
        }
        __syncwarp();  // slot table entry visible to every lane
        uint32_t A[G];
#pragma unroll
        for (int g = 0; g < G; ++g) A[g] = S;  // anchor of the new unit's component
        // back neighbours (warp uniform); one call site per genome keeps the loop small
        const bool lng = (h.x >> 31) != 0u;
        const int nb = lng ? (int)h.y : (int)(h.y & 7u);
#pragma unroll 1
        for (int j = 0; j < nb; ++j) {
          const uint32_t b = lng ? (uint32_t)__ldg(a.lists + h.z + j) : (h.y >> (3 + 6 * j)) & 63u;
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const uint32_t lb = lds_u8(L[g].lab + 4 * b);
            const bool need = on[g] && lb != 0u;  // b's unit is ON
            if (__any_sync(0xffffffffu, need)) {
              if (MB)
                an_merge_br<C, T>(L[g], spill[g], need, b, lb, A[g]);
              else
                an_merge<C, T>(L[g], spill[g], need, b, lb, A[g]);
            }
          }
        }
      }
      __syncthreads();  // every warp is done with buffer c & 1
      stage_chunk(a, c + 2, buf, t, T);
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      // regions open at the end of the program; labels cleared for the next genome
      for (int s = 0; s < a.F; ++s) {
        const uint32_t la = L[g].lab + 4 * s;
        an_close<C, T>(L[g], spill[g], lds_u8(la), lane, G * lane + g, qx, qown, qn, a, tacc, inexact);
        sts_u8(la, 0u);
      }
    }
    an_flush(qx, qown, qn, lane, a, tacc, inexact);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int o = G * lane + g;
      X128 total = L[g].total;
      x_add(total, X128{tacc[2 * o], tacc[2 * o + 1]});
      tacc[2 * o] = tacc[2 * o + 1] = 0ull;
      if (gi[g] < n) {
        if (dead[g]) {
          fit[gi[g]] = __longlong_as_double(0x7ff0000000000000ll);
        } else {
          // sign-extend the 128-bit dynamic part, scale back, add the constant
          const uint64_t sx = (uint64_t)((int64_t)total.hi >> 63);
          fx192 v = fx_shl(fx192{{total.lo, total.hi, sx}}, a.shift);
          fx_add(v, a.base_const);
          fit[gi[g]] = fx_to_double(v);
        }
      }
    }
    __syncwarp();
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (inexact) atomicAdd(a.flags, 1ull);
}

size_t anchor_smem(int C, int F, int Fp, int T, int G) {
  const int W = T / 32;
  return (size_t)2 * CH * REC_BYTES + (size_t)G * C * T * 16 +
         (size_t)W * (AN_QCAP * 16 + 64 * 8 * G + (size_t)F * WT_BYTES + AN_QCAP) +
         (size_t)G * (T / 4) * Fp * 4;
}

template <int C, int T, int G, int MB>
int launch_anchor_tt(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit, cudaStream_t stream) {
  const int Fp = p->F | 1;  // odd row stride: a uniform slot hits 8 distinct banks
  const size_t smem = anchor_smem(C, p->F, Fp, T, G);
  if (cb_smem_claim((const void*)fitness_anchor_kernel<C, T, G, MB>, smem))
    CB_CUDA_TRY(cudaFuncSetAttribute(fitness_anchor_kernel<C, T, G, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  int per_sm = 0;
  CB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fitness_anchor_kernel<C, T, G, MB>, T, smem));
  if (per_sm < 1) per_sm = 1;
  AnArgs a;
  a.M = p->M;
  a.words = p->words;
  a.shift = p->anchor_shift;
  a.n_infeas = (int32_t)p->d_an_infeas_word.n;
  a.Fp = Fp;
  a.F = p->F;
  a.base_const = p->base_const;
  const fx192 ex = fx_shr(p->eps, p->anchor_shift);
  a.eps = {ex.w[0], ex.w[1]};
  a.rec = reinterpret_cast<const uint4*>(p->d_arec.p);
  a.lists = p->d_alists.p;
  a.infeas_word = p->d_an_infeas_word.p;
  a.infeas_mask = p->d_an_infeas_mask.p;
  a.rt = p->d_rt.p;
  a.flags = p->d_flags.p;
  const int64_t want = (n + (int64_t)T * G - 1) / ((int64_t)T * G);
  const int64_t grid = std::min<int64_t>(want, (int64_t)per_sm * cb_sm_count());
  fitness_anchor_kernel<C, T, G, MB><<<(unsigned)grid, T, smem, stream>>>(a, d_pop, n, d_fit);
  CB_CUDA_TRY(cudaGetLastError());
  return CB_OK;
}

// 128-thread blocks (four warps share each staged record chunk) when the
// population fills the GPU; 64-thread blocks for smaller (search-sized)
// populations, where fewer warps per block barrier wait less on the slowest
template <int C>
int launch_anchor_t(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit, cudaStream_t stream) {
  // (G = 2 genomes per thread measured 25-55 % slower: fewer resident
  // blocks, twice the code in the step loop; the kernel keeps G as a parameter)
  const char* bt = getenv("CB_ANCHOR_BLOCK");
  const int want = bt ? atoi(bt) : (n < (int64_t)cb_sm_count() * 6 * 128 ? 64 : 128);
  // merge form (A/B on one ES population, tools/ab_probe.py): with branches
  // 10 % faster on a full 1 M-genome launch, with selects 3.5 % faster on a
  // latency-bound 65 536-genome one; CB_ANCHOR_MERGE=0/1 forces one
  const char* mb = getenv("CB_ANCHOR_MERGE");
  const int merge_br = mb ? atoi(mb) : (want == 64 ? 0 : 1);
  if (merge_br)
    return want == 64 ? launch_anchor_tt<C, 64, 1, 1>(p, d_pop, n, d_fit, stream)
                      : launch_anchor_tt<C, 128, 1, 1>(p, d_pop, n, d_fit, stream);
  return want == 64 ? launch_anchor_tt<C, 64, 1, 0>(p, d_pop, n, d_fit, stream)
                    : launch_anchor_tt<C, 128, 1, 0>(p, d_pop, n, d_fit, stream);
}

}  // namespace

// Plan time: choose the 128-bit window and build the step headers.  Leaves
// anchor_ok false (other kernels are used) when the program is wider than
// 64 slots or a value / partial sum does not fit the window.
int build_anchor_plan(cb_es_plan* P) {
  P->anchor_ok = false;
  const int32_t M = P->M;
  if (P->F <= 0 || P->F > 64 || M == 0) return CB_OK;
  // lowest bit any carried value can have, highest bit any partial sum can reach
  int lo = fx_lowest_bit(P->eps);
  fx192 bound = fx_zero();
  double min_pos_rep = INFINITY;
  for (int32_t p = 0; p < M; ++p) {
    const UnitRec& r = P->prog[p];
    for (const fx192* v : {&r.rep, &r.off, &r.term1}) {
      lo = std::min(lo, fx_lowest_bit(*v));
      fx_add(bound, *v);
    }
    fx_add(bound, P->eps);
    const double rd = fx_to_double(r.rep);
    if (rd > 0.0) min_pos_rep = std::min(min_pos_rep, rd);
  }
  if (std::isfinite(min_pos_rep)) {
    // smallest non-zero multi-unit region term: round(S) * r with S >= min_pos_rep
    double rmin = INFINITY;
    for (double r : P->rt)
      if (r > 0.0) rmin = std::min(rmin, r);
    if (!std::isfinite(rmin)) return CB_OK;
    volatile double tmin = min_pos_rep * rmin;
    if (!(tmin > 0.0)) return CB_OK;
    lo = std::min(lo, std::ilogb(tmin) - 52 + 128);
  }
  fx_add(bound, bound);  // region terms are at most their sums (r <= 1)
  if (lo >= 192) lo = 0;
  if (lo < 0) return CB_OK;
  const int hb = fx_highest_bit(bound);
  if (hb - lo > 125) return CB_OK;  // partial sums need more than 127 bits
  P->anchor_shift = lo;
  P->anchor_span = hb - lo;
  // wide anchor walk: packed sums need values below 2^108 and region kernel
  // counts below 2^20
  int64_t cnt_total = 0;
  for (int32_t p = 0; p < M; ++p) cnt_total += P->prog[p].cnt;
  P->anchor_wide_ok = P->anchor_span <= 106 && cnt_total < (1 << 20) && P->k < 0xFFFFFF;
  // per-position constants of the packed-label walks (fitness_packed128.cu)
  std::vector<uint64_t> cold((size_t)M * 6);
  std::vector<int32_t> cnt(M);
  for (int32_t p = 0; p < M; ++p) {
    const UnitRec& r = P->prog[p];
    const fx192* vals[3] = {&r.rep, &r.off, &r.term1};
    for (int k = 0; k < 3; ++k) {
      const fx192 x = fx_shr(*vals[k], lo);
      cold[(size_t)p * 6 + 2 * k] = x.w[0];
      cold[(size_t)p * 6 + 2 * k + 1] = x.w[1];
    }
    cnt[p] = r.cnt;
  }
  // per position: the 80-byte step record (header, term1 - off, and the
  // slot-table entry: end, replacement sum | count << 108, term1)
  std::vector<uint64_t> rec((size_t)M * 10);
  std::vector<uint8_t> lists;
  for (int32_t p = 0; p < M && P->anchor_wide_ok; ++p) {
    const UnitRec& r = P->prog[p];
    AStep h;
    std::memset(&h, 0, sizeof(h));
    h.bs = (r.bit >= 0 ? (uint32_t)r.bit : 0xFFFFFFu) | ((uint32_t)r.slot << 24);
    if (r.nback <= 4) {
      h.lists = (uint32_t)r.nback;
      for (int j = 0; j < r.nback; ++j) h.lists |= (uint32_t)P->prog_slots[r.back_off + j] << (3 + 6 * j);
    } else {
      h.bs |= 1u << 31;
      h.lists = (uint32_t)r.nback;
      h.off = (uint32_t)lists.size();
      for (int j = 0; j < r.nback; ++j) lists.push_back(P->prog_slots[r.back_off + j]);
    }
    const fx192 xo = fx_shr(r.off, lo), xr = fx_shr(r.rep, lo), xt = fx_shr(r.term1, lo);
    fx192 xtm = xt;
    fx_sub(xtm, xo);  // two's complement in the low 128 bits
    uint64_t* q = rec.data() + (size_t)p * 10;
    std::memcpy(q, &h, sizeof(h));
    q[2] = xtm.w[0];
    q[3] = xtm.w[1];
    q[4] = (uint64_t)(uint32_t)P->prog_last[p];
    q[5] = 0;
    q[6] = xr.w[0];
    q[7] = xr.w[1] | ((uint64_t)r.cnt << 44);
    q[8] = xt.w[0];
    q[9] = xt.w[1];
  }
  if (lists.empty()) lists.push_back(0);
  std::vector<int32_t> iw;
  std::vector<uint64_t> im;
  for (int32_t w = 0; w < (int32_t)P->infeas_mask.size(); ++w)
    if (P->infeas_mask[w]) {
      iw.push_back(w);
      im.push_back(P->infeas_mask[w]);
    }
  // packed anchor headers (F <= 8): bit | slot | nback | nend, back / end
  // slot nibbles, and the end rank of every slot's current unit (slots
  // ordered by their unit's last neighbour, ties by slot)
  P->pa_ok = P->F <= 8 && P->k < 0xFFFFF;
  std::vector<uint32_t> pah;
  if (P->pa_ok) {
    pah.resize((size_t)M * 4);
    std::vector<int32_t> occ_last(P->F, -1);
    for (int32_t p = 0; p < M && P->pa_ok; ++p) {
      const UnitRec& r = P->prog[p];
      if (r.nback > 8 || r.nend > 8) {
        P->pa_ok = false;
        break;
      }
      occ_last[r.slot] = P->prog_last[p];
      uint32_t x = (r.bit >= 0 ? (uint32_t)r.bit : 0xFFFFFu) | ((uint32_t)r.slot << 20) |
                   ((uint32_t)r.nback << 24) | ((uint32_t)r.nend << 28);
      uint32_t yb = 0, ze = 0, wr = 0;
      for (int j = 0; j < r.nback; ++j) yb |= (uint32_t)(P->prog_slots[r.back_off + j] & 0xF) << (4 * j);
      for (int j = 0; j < r.nend; ++j) ze |= (uint32_t)(P->prog_slots[r.end_off + j] & 0xF) << (4 * j);
      for (int s = 0; s < P->F; ++s) {
        int rank = 0;
        for (int q = 0; q < P->F; ++q)
          if (occ_last[q] < occ_last[s] || (occ_last[q] == occ_last[s] && q < s)) ++rank;
        wr |= (uint32_t)rank << (4 * s);
      }
      pah[(size_t)p * 4 + 0] = x;
      pah[(size_t)p * 4 + 1] = yb;
      pah[(size_t)p * 4 + 2] = ze;
      pah[(size_t)p * 4 + 3] = wr;
    }
  }
  cudaError_t e;
  if (P->pa_ok && (e = P->d_pahdr.upload(pah)) != cudaSuccess) {
    cb_set_error(std::string("CUDA error in plan upload: ") + cudaGetErrorString(e));
    return CB_ERR_CUDA;
  }
  if ((e = P->d_acold.upload(cold)) != cudaSuccess || (e = P->d_acnt.upload(cnt)) != cudaSuccess) {
    cb_set_error(std::string("CUDA error in plan upload: ") + cudaGetErrorString(e));
    return CB_ERR_CUDA;
  }
  if (P->anchor_wide_ok &&
      ((e = P->d_arec.upload(rec)) != cudaSuccess || (e = P->d_alists.upload(lists)) != cudaSuccess ||
       (e = P->d_an_infeas_word.upload(iw)) != cudaSuccess ||
       (e = P->d_an_infeas_mask.upload(im)) != cudaSuccess)) {
    cb_set_error(std::string("CUDA error in plan upload: ") + cudaGetErrorString(e));
    return CB_ERR_CUDA;
  }
  P->anchor_ok = true;
  return CB_OK;
}

int launch_fitness_anchor(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit,
                          cudaStream_t stream) {
  if (!p->anchor_wide_ok) return launch_fitness_wide(p, d_pop, n, d_fit, stream);
  // C pool entries per lane live in shared memory, the other F - C (at most
  // F entries are ever held) in the thread's local memory
  const int C = p->pool_entries;
  if (C <= 4) return launch_anchor_t<4>(p, d_pop, n, d_fit, stream);
  if (C <= 8) return launch_anchor_t<8>(p, d_pop, n, d_fit, stream);
  if (C <= 12) return launch_anchor_t<12>(p, d_pop, n, d_fit, stream);
  return launch_anchor_t<16>(p, d_pop, n, d_fit, stream);
}
