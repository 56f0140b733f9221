// Thread-per-genome frontier walk for wide programs (up to 64 slots): the
// kernel for the random 100k-op DAG (36 slots), BASELINE.json configs[4].
//
// Semantics are those of every fitness kernel here (tensorplace/
// evolution.py:65-135 decode, tensorplace/cost.py:320-373 graph-level
// pricing).  Lanes walk the frontier program in lockstep, one genome each;
// only the component structure of the occupied slots and the merged
// components' sums are per-lane data, everything else is uniform:
//
// * Anchors.  A component's data lives at its ANCHOR: the member slot whose
//   unit has the latest end (last neighbour position).  Merging two
//   components keeps the later-ending anchor, so no member ever outlives
//   its anchor: releasing a non-anchor slot is a bit clear, releasing an
//   anchor closes the region, and no data ever moves between slots.
// * Byte labels.  A non-anchor slot holds a parent slot of its component
//   (path-compressed on lookup; a pointer always targets a slot that ends no
//   earlier).  An anchor holds a flag, plus a pool entry when the component
//   has merged.  A one-unit component needs no data of its own: the unit in
//   a slot, its end and its constants are the same for every lane, kept per
//   warp in shared memory (program position, end) and read from the plan.
// * Packed sums.  A merged component's exact sum is carried in the plan's
//   128-bit window (X = v >> s, checked at plan time) with its kernel count
//   in bits 108-127, so a merge is one 128-bit add; pool entries live in
//   shared memory ([entry][thread], 16 bytes).  A genome needing more live
//   merged components than the pool holds is listed for the warp-per-genome
//   kernel (fitness_wide.cu) instead.
// * Region pricing (round(sum) * r(n) + eps) happens in warp batches: a
//   closing region is queued with its owner lane, and the queue (32 entries)
//   is priced one entry per lane, adding into the owner's accumulator.
// * Step records are 16 bytes (genome bit, slot, end position, up to four
//   back and four end slots inline), prefetched one step ahead.
//
// Shared memory per thread: one byte per slot + 16 bytes per pool entry, and
// per warp the slot tables, the region queue and the owner accumulators.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "fitness_plan.cuh"

#define AN_THREADS 128
#define AN_QCAP 32

namespace {

// 16-byte step record
struct __align__(16) AStep {
  uint32_t bs;     // genome bit (bits 0-23; 0xFFFFFF: always-on fixed unit) | slot << 24 | long << 31
  int32_t last;    // program position of the unit's last neighbour
  uint32_t lists;  // short: nback (3 bits) | nend << 3 | back slot j at 6 + 6 j (j < 4)
                   // long:  nback (16 bits) | nend << 16
  uint32_t ends;   // short: end slot j at 6 j (j < 4); long: offset of back + end lists
};
static_assert(sizeof(AStep) == 16, "AStep layout");

constexpr uint32_t L_ANCHOR = 0x80u;
constexpr uint32_t L_MERGED = 0x40u;
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
__device__ __forceinline__ X128 ld_x(const ulonglong2* p) {
  const ulonglong2 v = __ldg(p);
  return {v.x, v.y};
}

struct AnArgs {
  int32_t M, words, shift, n_infeas, Fp;
  fx192 base_const;
  X128 eps;
  const AStep* __restrict__ step;
  const ulonglong2* __restrict__ off;    // [M] own kernel cost + eps (removed when on)
  const ulonglong2* __restrict__ repc;   // [M] replacement sum | count << 108
  const ulonglong2* __restrict__ term1;  // [M] one-unit region term
  const uint8_t* __restrict__ lists;     // long back / end lists
  const int32_t* __restrict__ infeas_word;
  const uint64_t* __restrict__ infeas_mask;
  const double* __restrict__ rt;
  unsigned long long* flags;
  int32_t* ovf_count;
  int64_t* ovf_list;
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

template <int C>
__global__ void __launch_bounds__(AN_THREADS, 8)
fitness_anchor_kernel(AnArgs a, const uint64_t* __restrict__ pop, int64_t n, double* __restrict__ fit) {
  constexpr int T = AN_THREADS, W = AN_THREADS / 32;
  extern __shared__ __align__(16) unsigned char an_smem[];
  ulonglong2* pool = reinterpret_cast<ulonglong2*>(an_smem);         // [C][T]
  ulonglong2* qx_all = pool + C * T;                                 // [W][QCAP]
  unsigned long long* tacc_all = reinterpret_cast<unsigned long long*>(qx_all + W * AN_QCAP);  // [W][32][2]
  int2* wtab_all = reinterpret_cast<int2*>(tacc_all + W * 64);      // [W][64] (position, end) per slot
  uint8_t* qown_all = reinterpret_cast<uint8_t*>(wtab_all + W * 64);  // [W][QCAP]
  uint8_t* LAB = qown_all + W * AN_QCAP;                             // [T / 4][Fp][4]
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  ulonglong2* pl = pool + t;                                   // pl[e * T]
  uint8_t* lab = LAB + (t >> 2) * a.Fp * 4 + (t & 3);          // lab[s * 4]
  ulonglong2* qx = qx_all + warp * AN_QCAP;
  uint8_t* qown = qown_all + warp * AN_QCAP;
  unsigned long long* tacc = tacc_all + warp * 64;
  int2* wtab = wtab_all + warp * 64;
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
    uint64_t act = 0ull;
    uint32_t pfree = C >= 32 ? 0xffffffffu : ((1u << C) - 1u);
    bool ovf = false;
    X128 total = {0ull, 0ull};
    int qn = 0;
    int32_t cur_w = -1;
    uint64_t word = 0ull, next_word = a.words > 0 ? __ldg(gen) : 0ull;
    uint4 nh = __ldg(reinterpret_cast<const uint4*>(a.step));
    X128 noff = ld_x(a.off);
    for (int32_t p = 0; p < a.M; ++p) {
      const uint4 h = nh;
      const X128 off = noff;
      if (p + 1 < a.M) {
        nh = __ldg(reinterpret_cast<const uint4*>(a.step + p + 1));
        noff = ld_x(a.off + p + 1);
      }
      const uint32_t bitf = h.x & 0xFFFFFFu;
      const int S = (int)((h.x >> 24) & 63u);
      const bool lng = (h.x >> 31) != 0u;
      if (lane == 0) wtab[S] = make_int2(p, (int32_t)h.y);
      bool on = !dead;
      if (bitf != 0xFFFFFFu) {
        const int32_t wi = (int32_t)(bitf >> 6);
        if (wi != cur_w) {  // warp uniform; the next word is loaded one word ahead
          word = wi == cur_w + 1 ? next_word : __ldg(gen + wi);
          next_word = wi + 1 < a.words ? __ldg(gen + wi + 1) : 0ull;
          cur_w = wi;
        }
        on = on && ((word >> (bitf & 63u)) & 1ull);
      }
      __syncwarp();
      if (on) {
        x_sub(total, off);
        act |= 1ull << S;
        lab[S * 4] = (uint8_t)L_ANCHOR;
      }
      const int nb = lng ? (int)(h.z & 0xFFFFu) : (int)(h.z & 7u);
      const int ne = lng ? (int)(h.z >> 16) : (int)((h.z >> 3) & 7u);
      int A = S;  // anchor of the new unit's component
      for (int j = 0; j < nb; ++j) {
        const int b = lng ? (int)__ldg(a.lists + h.w + j) : (int)((h.z >> (6 + 6 * j)) & 63u);
        if (!on || !((act >> b) & 1ull)) continue;
        int x = b;
        uint32_t lx = lab[x * 4];
        while (!(lx & L_ANCHOR)) {
          x = (int)lx;
          lx = lab[x * 4];
        }
        if (x != b) lab[b * 4] = (uint8_t)x;  // path compression
        if (x == A) continue;
        const uint32_t lA = lab[A * 4];
        const int2 tA = wtab[A], tX = wtab[x];
        const bool keepA = tA.y >= tX.y;  // the later-ending anchor survives
        const int Wn = keepA ? A : x, Xn = keepA ? x : A;
        const uint32_t lW = keepA ? lA : lx, lX = keepA ? lx : lA;
        X128 sW = (lW & L_MERGED) ? X128{pl[(lW & 63u) * T].x, pl[(lW & 63u) * T].y}
                                  : ld_x(a.repc + (keepA ? tA.x : tX.x));
        const X128 sX = (lX & L_MERGED) ? X128{pl[(lX & 63u) * T].x, pl[(lX & 63u) * T].y}
                                        : ld_x(a.repc + (keepA ? tX.x : tA.x));
        x_add(sW, sX);
        int e;
        if (lW & L_MERGED) {
          e = (int)(lW & 63u);
          if (lX & L_MERGED) pfree |= 1u << (lX & 63u);
        } else if (lX & L_MERGED) {
          e = (int)(lX & 63u);
        } else if (pfree) {
          e = __ffs(pfree) - 1;
          pfree &= pfree - 1u;
        } else {
          ovf = true;  // pool exhausted: the genome goes to the fallback kernel
          e = 0;
        }
        pl[e * T] = make_ulonglong2(sW.lo, sW.hi);
        lab[Wn * 4] = (uint8_t)(L_ANCHOR | L_MERGED | (uint32_t)e);
        lab[Xn * 4] = (uint8_t)Wn;
        A = Wn;
      }
      for (int j = 0; j < ne; ++j) {
        const int e = lng ? (int)__ldg(a.lists + h.w + nb + j) : (int)((h.w >> (6 * j)) & 63u);
        bool emit = false;
        ulonglong2 ev = make_ulonglong2(0ull, 0ull);
        if ((act >> e) & 1ull) {
          act &= ~(1ull << e);
          const uint32_t le = lab[e * 4];
          if (le & L_ANCHOR) {  // the anchor leaves: its region is complete
            if (le & L_MERGED) {
              emit = true;
              ev = pl[(le & 63u) * T];
              pfree |= 1u << (le & 63u);
            } else {
              x_add(total, ld_x(a.term1 + wtab[e].x));
            }
          }
        }
        // closed multi-unit regions of all lanes are priced 32 at a time
        const unsigned closing = __ballot_sync(0xffffffffu, emit);
        if (closing) {
          const int cnt = __popc(closing);
          if (qn + cnt > AN_QCAP) {
            an_flush(qx, qown, qn, lane, a, tacc, inexact);
            qn = 0;
          }
          if (emit) {
            const int at = qn + __popc(closing & ((1u << lane) - 1u));
            qx[at] = ev;
            qown[at] = (uint8_t)lane;
          }
          qn += cnt;
        }
      }
    }
    an_flush(qx, qown, qn, lane, a, tacc, inexact);
    x_add(total, X128{tacc[2 * lane], tacc[2 * lane + 1]});
    tacc[2 * lane] = tacc[2 * lane + 1] = 0ull;
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

size_t anchor_smem(int C, int Fp) {
  constexpr int T = AN_THREADS, W = AN_THREADS / 32;
  return (size_t)C * T * 16 + (size_t)W * (AN_QCAP * 16 + 64 * 8 + 64 * 8 + AN_QCAP) +
         (size_t)(T / 4) * Fp * 4;
}

template <int C>
int launch_anchor_t(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit, cudaStream_t stream) {
  const int Fp = p->F | 1;  // odd row stride: a uniform slot hits 8 distinct banks
  const size_t smem = anchor_smem(C, Fp);
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
  a.n_infeas = (int32_t)p->d_an_infeas_word.n;
  a.Fp = Fp;
  a.base_const = p->base_const;
  const fx192 ex = fx_shr(p->eps, p->anchor_shift);
  a.eps = {ex.w[0], ex.w[1]};
  a.step = reinterpret_cast<const AStep*>(p->d_astep.p);
  a.off = reinterpret_cast<const ulonglong2*>(p->d_aoff.p);
  a.repc = reinterpret_cast<const ulonglong2*>(p->d_arepc.p);
  a.term1 = reinterpret_cast<const ulonglong2*>(p->d_aterm.p);
  a.lists = p->d_alists.p;
  a.infeas_word = p->d_an_infeas_word.p;
  a.infeas_mask = p->d_an_infeas_mask.p;
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
  std::vector<AStep> steps(M);
  std::vector<uint64_t> off((size_t)M * 2), repc((size_t)M * 2), term((size_t)M * 2);
  std::vector<uint8_t> lists;
  for (int32_t p = 0; p < M && P->anchor_wide_ok; ++p) {
    const UnitRec& r = P->prog[p];
    AStep h;
    std::memset(&h, 0, sizeof(h));
    h.bs = (r.bit >= 0 ? (uint32_t)r.bit : 0xFFFFFFu) | ((uint32_t)r.slot << 24);
    h.last = P->prog_last[p];
    if (r.nback <= 4 && r.nend <= 4) {
      h.lists = (uint32_t)r.nback | ((uint32_t)r.nend << 3);
      for (int j = 0; j < r.nback; ++j) h.lists |= (uint32_t)P->prog_slots[r.back_off + j] << (6 + 6 * j);
      for (int j = 0; j < r.nend; ++j) h.ends |= (uint32_t)P->prog_slots[r.end_off + j] << (6 * j);
    } else {
      h.bs |= 1u << 31;
      h.lists = (uint32_t)r.nback | ((uint32_t)r.nend << 16);
      h.ends = (uint32_t)lists.size();
      for (int j = 0; j < r.nback; ++j) lists.push_back(P->prog_slots[r.back_off + j]);
      for (int j = 0; j < r.nend; ++j) lists.push_back(P->prog_slots[r.end_off + j]);
    }
    steps[p] = h;
    const fx192 xo = fx_shr(r.off, lo), xr = fx_shr(r.rep, lo), xt = fx_shr(r.term1, lo);
    off[2 * p] = xo.w[0];
    off[2 * p + 1] = xo.w[1];
    repc[2 * p] = xr.w[0];
    repc[2 * p + 1] = xr.w[1] | ((uint64_t)r.cnt << 44);
    term[2 * p] = xt.w[0];
    term[2 * p + 1] = xt.w[1];
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
      ((e = P->d_astep.upload(reinterpret_cast<const uint8_t*>(steps.data()), steps.size() * sizeof(AStep))) !=
           cudaSuccess ||
       (e = P->d_aoff.upload(off)) != cudaSuccess || (e = P->d_arepc.upload(repc)) != cudaSuccess ||
       (e = P->d_aterm.upload(term)) != cudaSuccess || (e = P->d_alists.upload(lists)) != cudaSuccess ||
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
  int C = p->pool_entries;
  if (p->pool_auto) {
    // 8 entries fit 8 CTAs of 128 threads per SM on a 36-slot program; when
    // more than 1 % of the previous launch's genomes overflowed (dense
    // populations) use 12, above 5 % 16.  The count is read without
    // synchronising: it is the last launch that finished, a hint only --
    // results never depend on C.
    const volatile int32_t* h = p->h_ovf;
    if (h && p->last_anchor_n > 0) {
      const int64_t pct = (int64_t)*h * 100 / p->last_anchor_n;
      p->auto_pool = pct >= 5 ? 16 : (pct >= 1 ? 12 : 8);
    }
    C = std::min(p->pool_entries, p->auto_pool);
  }
  if (C <= 8) return launch_anchor_t<8>(p, d_pop, n, d_fit, stream);
  if (C <= 12) return launch_anchor_t<12>(p, d_pop, n, d_fit, stream);
  if (C <= 16) return launch_anchor_t<16>(p, d_pop, n, d_fit, stream);
  return launch_anchor_t<24>(p, d_pop, n, d_fit, stream);
}
