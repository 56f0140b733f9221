// Thread-per-genome frontier walk for wide programs (up to 64 slots), with
// slot state small enough for shared memory at useful occupancy.
//
// Semantics are those of every fitness kernel here (tensorplace/evolution.py:
// 256-371 decode, tensorplace/cost.py:320-373 graph-level pricing).  The
// walk visits every program position in lockstep across the warp (like
// fitness_frontier2_kernel), but represents the components differently:
//
// * Anchors.  A component's data lives at its ANCHOR: the member slot whose
//   unit has the latest end (last neighbour position).  Merging two
//   components keeps the later-ending anchor, so no member ever outlives
//   its anchor: releasing a non-anchor slot is a bit clear, releasing an
//   anchor closes the region, and no data ever moves between slots.
// * Union-find labels.  A non-anchor slot points to another slot of its
//   component (path-compressed on lookup); an absorbed anchor points to the
//   survivor.  A pointer always targets a slot that ends no earlier, so no
//   active slot ever points to a released one.
// * Sums only where needed.  A one-unit component is described by its unit
//   (rep, cnt, term1 come from its program position, kept in the label).
//   Only merged components hold an exact sum, in a per-thread pool;
//   the anchor's label word carries the pool index and the kernel count.  A
//   genome that needs more live merged components than the pool holds is
//   listed for the warp-per-genome kernel (fitness_wide.cu) instead.
// * 128-bit window.  When every plan value is a multiple of 2^(s-128) and
//   all partial sums stay below 2^(253-s) (checked when the plan is built,
//   including the smallest possible region term), values are carried as
//   128-bit integers X = v >> s; the 192-bit form is rebuilt only to round
//   a region sum and to add the plan constant at the end.
//
// Shared memory per thread: 4 B label per slot + 16 B per pool entry.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "fitness_plan.cuh"

#define AN_THREADS 64
#define AN_QCAP 64

namespace {

// Per-position step header, one 32-byte uniform load per step.
struct __align__(16) AHot {
  int32_t bit;       // genome bit, -1 for fixed units
  int32_t last;      // position of the unit's last neighbour
  uint32_t hdr;      // slot | nback << 8 | nend << 16 | long_list << 31
  uint8_t list[20];  // back slots then end slots (or int32 offset into prog_slots)
};
static_assert(sizeof(AHot) == 32, "AHot layout");

// label word: non-anchor:    parent slot (bit 31 clear)
//             single anchor: bit 31 | bit 30 | program position of its unit
//             merged anchor: bit 31 | cnt << 8 | pool entry
constexpr uint32_t L_ANCHOR = 0x80000000u;
constexpr uint32_t L_SINGLE = 0x40000000u;
constexpr uint32_t L_CNT_MAX = (1u << 22) - 1u;
constexpr uint32_t L_POS_MASK = (1u << 30) - 1u;  // single anchors: program position of the unit

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
  int32_t M, words, shift;
  fx192 base_const;
  X128 eps;
  const AHot* __restrict__ hot;
  const uint64_t* __restrict__ cold;  // [M][6] rep, off, term1
  const int32_t* __restrict__ cnt;
  const uint8_t* __restrict__ slots;
  const uint64_t* __restrict__ infeas;
  const double* __restrict__ rt;
  unsigned long long* flags;
  int32_t* ovf_count;
  int64_t* ovf_list;
};

__device__ __forceinline__ X128 ld_x(const uint64_t* p) {
  const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(p));
  return {v.x, v.y};
}

// Price queue entry `idx` (region sum X, kernel count, owner lane) and add
// its term to the owner's 128-bit accumulator (shared atomics: an owner can
// have several entries in one batch).
__device__ __forceinline__ void an_price(const uint64_t* ql, const uint64_t* qh, const uint64_t* qm, int idx,
                                         const AnArgs& a, uint64_t* tlo, uint64_t* thi, bool& inexact) {
  const uint64_t m = qm[idx];
  const double prod = __dmul_rn(x128_to_double(ql[idx], qh[idx], a.shift), __ldg(a.rt + (uint32_t)m));
  X128 term;
  inexact |= !x128_from_double(prod, a.shift, term.lo, term.hi);
  x_add(term, a.eps);
  const int owner = (int)(m >> 32);
  unsigned long long* w0 = reinterpret_cast<unsigned long long*>(tlo + owner);
  unsigned long long* w1 = reinterpret_cast<unsigned long long*>(thi + owner);
  const unsigned long long o0 = atomicAdd(w0, (unsigned long long)term.lo);
  atomicAdd(w1, (unsigned long long)(term.hi + ((o0 + term.lo) < o0)));
}

// slot j of a short back+end list: byte j of the header's list (word 3 + j / 4)
__device__ __forceinline__ int hdr_slot(const uint4& h0, const uint4& h1, int j) {
  const int k = j >> 2;
  const uint32_t w = k == 0 ? h0.w : (k == 1 ? h1.x : (k == 2 ? h1.y : (k == 3 ? h1.z : h1.w)));
  return (int)((w >> (8 * (j & 3))) & 0xffu);
}

template <int C>
__global__ void __launch_bounds__(AN_THREADS)
fitness_anchor_kernel(AnArgs a, const uint64_t* __restrict__ pop, int64_t n, double* __restrict__ fit) {
  constexpr int T = AN_THREADS, W = AN_THREADS / 32;
  extern __shared__ __align__(16) unsigned char an_smem[];
  uint64_t* PL = reinterpret_cast<uint64_t*>(an_smem);  // [C][T] pool sums, low word
  uint64_t* PH = PL + C * T;                             // [C][T] high word
  uint64_t* qall = PH + C * T;                           // [W][3][QCAP] region queue
  uint64_t* tall = qall + W * 3 * AN_QCAP;               // [W][2][32] owner accumulators
  int32_t* end_all = reinterpret_cast<int32_t*>(tall + W * 64);  // [W][64] end of the slot's unit
  uint32_t* LAB = reinterpret_cast<uint32_t*>(end_all + W * 64);  // [F][T] labels
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  uint64_t* ql = qall + warp * 3 * AN_QCAP;
  uint64_t* qh = ql + AN_QCAP;
  uint64_t* qm = qh + AN_QCAP;
  uint64_t* tlo = tall + warp * 64;
  uint64_t* thi = tlo + 32;
  int32_t* endw = end_all + warp * 64;
  uint32_t* lab = LAB + t;  // this thread's column: lab[slot * T]
  uint64_t* pl = PL + t;
  uint64_t* ph = PH + t;
  tlo[lane] = thi[lane] = 0ull;
  __syncwarp();
  int qn = 0;
  bool inexact = false;
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t base = (int64_t)blockIdx.x * T + (t & ~31); base < n; base += stride) {
    const int64_t i = base + lane;
    const bool in_range = i < n;
    const uint64_t* gen = pop + (in_range ? i : 0) * a.words;
    bool dead = !in_range;
    if (in_range)
      for (int32_t w = 0; w < a.words; ++w) dead |= (__ldg(gen + w) & __ldg(a.infeas + w)) != 0ull;
    uint64_t act = 0ull;
    uint32_t pfree = C >= 32 ? 0xffffffffu : ((1u << C) - 1u);
    bool ovf = false;
    X128 total = {0ull, 0ull};
    int32_t cached_word = -1;
    uint64_t word = 0ull, next_word = a.words > 0 ? __ldg(gen) : 0ull;
    // the step header and the unit's removed-kernel term are loaded one step
    // ahead: a wide program lives in L2, not L1, and its loads head every
    // step's dependency chain
    uint4 nh0 = __ldg(reinterpret_cast<const uint4*>(a.hot));
    uint4 nh1 = __ldg(reinterpret_cast<const uint4*>(a.hot) + 1);
    X128 noff = ld_x(a.cold + 2);
    for (int32_t p = 0; p < a.M; ++p) {
      const AHot* hp = a.hot + p;
      const uint4 h0 = nh0, h1 = nh1;
      const X128 off = noff;
      if (p + 1 < a.M) {
        nh0 = __ldg(reinterpret_cast<const uint4*>(hp + 1));
        nh1 = __ldg(reinterpret_cast<const uint4*>(hp + 1) + 1);
        noff = ld_x(a.cold + (size_t)(p + 1) * 6 + 2);
      }
      const int32_t bit = (int32_t)h0.x;
      const int S = h0.z & 0xff;
      const int nback = (h0.z >> 8) & 0xff;
      const int nend = (h0.z >> 16) & 0xff;
      const bool long_list = (h0.z >> 31) != 0u;
      const uint8_t* lst = a.slots + h0.w;  // long lists only
      bool on = !dead;
      if (bit >= 0) {
        const int32_t wi = bit >> 6;
        if (wi != cached_word) {  // warp uniform; the next word is loaded one word ahead
          word = wi == cached_word + 1 ? next_word : __ldg(gen + wi);
          if (dead) word = 0ull;
          next_word = wi + 1 < a.words ? __ldg(gen + wi + 1) : 0ull;
          cached_word = wi;
        }
        on = (word >> (bit & 63)) & 1ull;
      }
      if (lane == 0) endw[S] = (int32_t)h0.y;
      __syncwarp();
      if (on) {
        if (bit >= 0) x_sub(total, off);
        act |= 1ull << S;
        lab[S * T] = L_ANCHOR | L_SINGLE | (uint32_t)p;
      }
      int A = S;  // root slot of the new unit's component
      for (int j = 0; j < nback; ++j) {
        const int b = long_list ? __ldg(lst + j) : hdr_slot(h0, h1, j);
        if (!on || !((act >> b) & 1ull)) continue;
        int x = b;
        uint32_t lx = lab[x * T];
        while (!(lx & L_ANCHOR)) {
          x = (int)(lx & 0xff);
          lx = lab[x * T];
        }
        if (x != b) lab[b * T] = (uint32_t)x;  // path compression
        if (x == A) continue;
        const uint32_t lA = lab[A * T];
        const bool keepA = endw[A] >= endw[x];  // the later-ending anchor survives
        const int Wn = keepA ? A : x, Xn = keepA ? x : A;
        const uint32_t lW = keepA ? lA : lx, lX = keepA ? lx : lA;
        X128 sW, sX;
        uint32_t cW, cX;
        if (lW & L_SINGLE) {
          const uint32_t u = lW & L_POS_MASK;
          sW = ld_x(a.cold + (size_t)u * 6);
          cW = (uint32_t)__ldg(a.cnt + u);
        } else {
          const int e = lW & 0x3f;
          sW = {pl[e * T], ph[e * T]};
          cW = (lW >> 8) & L_CNT_MAX;
        }
        if (lX & L_SINGLE) {
          const uint32_t u = lX & L_POS_MASK;
          sX = ld_x(a.cold + (size_t)u * 6);
          cX = (uint32_t)__ldg(a.cnt + u);
        } else {
          const int e = lX & 0x3f;
          sX = {pl[e * T], ph[e * T]};
          cX = (lX >> 8) & L_CNT_MAX;
        }
        x_add(sW, sX);
        const uint32_t c = cW + cX;
        int e;
        if (!(lW & L_SINGLE)) {
          e = lW & 0x3f;
          if (!(lX & L_SINGLE)) pfree |= 1u << (lX & 0x3f);
        } else if (!(lX & L_SINGLE)) {
          e = lX & 0x3f;
        } else if (pfree) {
          e = __ffs(pfree) - 1;
          pfree &= pfree - 1u;
        } else {
          ovf = true;  // pool exhausted: the genome goes to the fallback kernel
          e = 0;
        }
        ovf |= c > L_CNT_MAX;
        pl[e * T] = sW.lo;
        ph[e * T] = sW.hi;
        lab[Wn * T] = L_ANCHOR | ((c & L_CNT_MAX) << 8) | (uint32_t)e;
        lab[Xn * T] = (uint32_t)Wn;
        A = Wn;
      }
      for (int j = 0; j < nend; ++j) {
        const int e = long_list ? __ldg(lst + nback + j) : hdr_slot(h0, h1, nback + j);
        bool emit = false;
        uint32_t le = 0u;
        if ((act >> e) & 1ull) {
          act &= ~(1ull << e);
          le = lab[e * T];
          if (le & L_ANCHOR) {  // the anchor leaves: its region is complete
            if (le & L_SINGLE) {
              x_add(total, ld_x(a.cold + (size_t)(le & L_POS_MASK) * 6 + 4));
            } else {
              emit = true;
              pfree |= 1u << (le & 0x3f);
            }
          }
        }
        // closed multi-unit regions of all lanes are priced 32 at a time
        const unsigned closing = __ballot_sync(0xffffffffu, emit);
        if (closing) {
          if (emit) {
            const int at = qn + __popc(closing & ((1u << lane) - 1u));
            const int pe = le & 0x3f;
            ql[at] = pl[pe * T];
            qh[at] = ph[pe * T];
            qm[at] = ((uint64_t)lane << 32) | ((le >> 8) & L_CNT_MAX);
          }
          qn += __popc(closing);
          if (qn >= 32) {
            __syncwarp();
            an_price(ql, qh, qm, lane, a, tlo, thi, inexact);
            __syncwarp();
            if (lane < qn - 32) {
              ql[lane] = ql[32 + lane];
              qh[lane] = qh[32 + lane];
              qm[lane] = qm[32 + lane];
            }
            __syncwarp();
            qn -= 32;
          }
        }
      }
    }
    __syncwarp();
    if (lane < qn) an_price(ql, qh, qm, lane, a, tlo, thi, inexact);
    qn = 0;
    __syncwarp();
    x_add(total, X128{tlo[lane], thi[lane]});
    tlo[lane] = thi[lane] = 0ull;
    __syncwarp();
    if (in_range) {
      if (ovf && !dead) {
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

size_t anchor_smem(int C, int F) {
  constexpr int T = AN_THREADS, W = AN_THREADS / 32;
  return (size_t)2 * C * T * 8 + (size_t)W * (3 * AN_QCAP + 64) * 8 + (size_t)W * 64 * 4 +
         (size_t)F * T * 4;
}

template <int C>
int launch_anchor_t(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit, cudaStream_t stream) {
  const size_t smem = anchor_smem(C, p->F);
  CB_CUDA_TRY(cudaFuncSetAttribute(fitness_anchor_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
  int per_sm = 0;
  CB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fitness_anchor_kernel<C>, AN_THREADS,
                                                            smem));
  if (per_sm < 1) per_sm = 1;
  if (p->d_ovf_list.n < (size_t)std::max<int64_t>(n, 1)) CB_CUDA_TRY(p->d_ovf_list.alloc((size_t)n));
  if (p->d_ovf_count.n < 1) CB_CUDA_TRY(p->d_ovf_count.alloc(1));
  CB_CUDA_TRY(cudaMemsetAsync(p->d_ovf_count.p, 0, sizeof(int32_t), stream));
  AnArgs a;
  a.M = p->M;
  a.words = p->words;
  a.shift = p->anchor_shift;
  a.base_const = p->base_const;
  const fx192 ex = fx_shr(p->eps, p->anchor_shift);
  a.eps = {ex.w[0], ex.w[1]};
  a.hot = reinterpret_cast<const AHot*>(p->d_ahot.p);
  a.cold = p->d_acold.p;
  a.cnt = p->d_acnt.p;
  a.slots = p->d_prog_slots.p;
  a.infeas = p->d_infeas.p;
  a.rt = p->d_rt.p;
  a.flags = p->d_flags.p;
  a.ovf_count = p->d_ovf_count.p;
  a.ovf_list = p->d_ovf_list.p;
  const int64_t want = (n + AN_THREADS - 1) / AN_THREADS;
  const int64_t grid = std::min<int64_t>(want, (int64_t)per_sm * cb_sm_count());
  fitness_anchor_kernel<C><<<(unsigned)grid, AN_THREADS, smem, stream>>>(a, d_pop, n, d_fit);
  CB_CUDA_TRY(cudaGetLastError());
  if (p->pool_auto) {  // let the next launch see this one's overflow count
    if (!p->h_ovf) {
      CB_CUDA_TRY(cudaHostAlloc((void**)&p->h_ovf, sizeof(int32_t), cudaHostAllocDefault));
      *p->h_ovf = 0;
    }
    CB_CUDA_TRY(cudaMemcpyAsync(p->h_ovf, p->d_ovf_count.p, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
    p->last_anchor_n = n;
  }
  // genomes that ran out of pool entries: warp-per-genome kernel over the list
  return launch_fitness_wide_list(p, d_pop, n, d_fit, p->d_ovf_list.p, p->d_ovf_count.p, stream);
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
  std::vector<AHot> hot(M);
  std::vector<uint64_t> cold((size_t)M * 6);
  std::vector<int32_t> cnt(M);
  for (int32_t p = 0; p < M; ++p) {
    const UnitRec& r = P->prog[p];
    AHot h;
    std::memset(&h, 0, sizeof(h));
    h.bit = r.bit;
    h.last = P->prog_last[p];
    h.hdr = (uint32_t)r.slot | ((uint32_t)r.nback << 8) | ((uint32_t)r.nend << 16);
    const int nl = r.nback + r.nend;  // back list and end list are contiguous in prog_slots
    if (nl <= 20) {
      for (int j = 0; j < nl; ++j) h.list[j] = P->prog_slots[r.back_off + j];
    } else {
      h.hdr |= 1u << 31;
      const int32_t off = r.back_off;
      std::memcpy(h.list, &off, sizeof(off));  // read as hot.w by the kernel
    }
    hot[p] = h;
    const fx192* vals[3] = {&r.rep, &r.off, &r.term1};
    for (int k = 0; k < 3; ++k) {
      const fx192 x = fx_shr(*vals[k], lo);
      cold[(size_t)p * 6 + 2 * k] = x.w[0];
      cold[(size_t)p * 6 + 2 * k + 1] = x.w[1];
    }
    cnt[p] = r.cnt;
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
  if ((e = P->d_ahot.upload(reinterpret_cast<const uint8_t*>(hot.data()), hot.size() * sizeof(AHot))) !=
          cudaSuccess ||
      (e = P->d_acold.upload(cold)) != cudaSuccess || (e = P->d_acnt.upload(cnt)) != cudaSuccess) {
    cb_set_error(std::string("CUDA error in plan upload: ") + cudaGetErrorString(e));
    return CB_ERR_CUDA;
  }
  P->anchor_ok = true;
  return CB_OK;
}

int launch_fitness_anchor(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit,
                          cudaStream_t stream) {
  int C = p->pool_entries;
  if (p->pool_auto) {
    // 14 entries fit 8 CTAs of 64 threads per SM on a 36-slot program; when
    // more than 1 % of the previous launch's genomes overflowed (dense
    // populations) use 16.  The count is read without synchronising: it is
    // the last launch that finished, a hint only -- results never depend on C.
    const volatile int32_t* h = p->h_ovf;
    if (h && p->last_anchor_n > 0)
      p->auto_pool = (int64_t)*h * 100 > p->last_anchor_n ? 16 : 14;
    C = std::min(p->pool_entries, p->auto_pool);
  }
  if (C <= 8) return launch_anchor_t<8>(p, d_pop, n, d_fit, stream);
  if (C <= 12) return launch_anchor_t<12>(p, d_pop, n, d_fit, stream);
  if (C <= 14) return launch_anchor_t<14>(p, d_pop, n, d_fit, stream);
  if (C <= 16) return launch_anchor_t<16>(p, d_pop, n, d_fit, stream);
  return launch_anchor_t<24>(p, d_pop, n, d_fit, stream);
}
