// Packed-label frontier walk (thread per genome, <= 16 slots) carrying the
// plan's values in its 128-bit window.
//
// Same walk as fitness_frontier2_kernel (fitness.cu): the component labels
// of all slots are 4-bit fields of one register, occupancy a nibble mask,
// merges / member tests / releases are SWAR operations, and closed
// multi-unit regions are priced 32 at a time through a per-warp queue.
// The difference is the arithmetic: when the plan's values fit a 128-bit
// window (build_anchor_plan, fitness_anchor.cu: every value a multiple of
// 2^(s-128), every partial sum below 2^(253-s), including the smallest
// possible region term), sums are 2-limb integers X = v >> s instead of
// 192-bit fixed point -- one add fewer per merge, one shared-memory word
// fewer per slot.  Results are bit-identical (tests/test_gpu_wide.py,
// tests/test_gpu_parity.py).
#include <type_traits>

#include "es_ops.cuh"
#include "fitness_plan.cuh"

#define PK_THREADS 128
#define PK_QCAP 64

namespace {

template <int V>
using IC = std::integral_constant<int, V>;

template <typename LT>
struct Nib2;
template <>
struct Nib2<uint32_t> {
  static constexpr uint32_t ONE = 0x11111111u, LOW3 = 0x77777777u;
};
template <>
struct Nib2<uint64_t> {
  static constexpr uint64_t ONE = 0x1111111111111111ull, LOW3 = 0x7777777777777777ull;
};

// nibble mask (0xF) of the nibbles of x equal to v
template <typename LT>
__device__ __forceinline__ LT nibeq(LT x, uint32_t v) {
  const LT y = x ^ ((LT)v * Nib2<LT>::ONE);
  const LT z = ~(((y & Nib2<LT>::LOW3) + Nib2<LT>::LOW3) | y | Nib2<LT>::LOW3);
  return (z >> 3) * (LT)0xF;
}

template <typename LT>
__device__ __forceinline__ int nibfirst(LT m) {
  if (sizeof(LT) == 8) return __ffsll((long long)m) - 1 >> 2;
  return __ffs((int)m) - 1 >> 2;
}

__device__ __forceinline__ void add2(uint64_t& lo, uint64_t& hi, uint64_t blo, uint64_t bhi) {
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(lo), "+l"(hi) : "l"(blo), "l"(bhi));
}
__device__ __forceinline__ void sub2(uint64_t& lo, uint64_t& hi, uint64_t blo, uint64_t bhi) {
  asm("sub.cc.u64 %0, %0, %2;\n\tsubc.u64 %1, %1, %3;" : "+l"(lo), "+l"(hi) : "l"(blo), "l"(bhi));
}

struct PkArgs {
  int32_t M, words, shift;
  fx192 base_const;
  uint64_t eps_lo, eps_hi;
  const UnitRec* __restrict__ prog;   // hot headers
  const uint64_t* __restrict__ cold;  // [M][6] rep, off, term1 as 128-bit X
  const int32_t* __restrict__ cnt;
  const uint64_t* __restrict__ infeas;
  const double* __restrict__ rt;
  unsigned long long* flags;
};

// Price queue entry `idx` and add its term to the owner lane's accumulator.
__device__ __forceinline__ void pk_price(const uint64_t* ql, const uint64_t* qh, const uint64_t* qm, int idx,
                                         const PkArgs& a, uint64_t* tlo, uint64_t* thi, bool& inexact) {
  const uint64_t m = qm[idx];
  const double prod = __dmul_rn(x128_to_double(ql[idx], qh[idx], a.shift), __ldg(a.rt + (uint32_t)m));
  uint64_t lo, hi;
  inexact |= !x128_from_double(prod, a.shift, lo, hi);
  add2(lo, hi, a.eps_lo, a.eps_hi);
  const int owner = (int)(m >> 32);
  const unsigned long long o0 = atomicAdd(reinterpret_cast<unsigned long long*>(tlo + owner), lo);
  atomicAdd(reinterpret_cast<unsigned long long*>(thi + owner), hi + ((o0 + lo) < o0));
}

template <typename LT, int F>
__global__ void __launch_bounds__(PK_THREADS)
fitness_packed128_kernel(PkArgs a, const uint64_t* __restrict__ pop, int64_t n, double* __restrict__ fit) {
  constexpr int T = PK_THREADS;
  extern __shared__ __align__(16) unsigned char pk_smem[];
  uint64_t(*sl)[T] = reinterpret_cast<uint64_t(*)[T]>(pk_smem);  // [F][T] sum, low word
  uint64_t(*sh)[T] = sl + F;                                       // high word
  uint64_t(*cs)[T] = sh + F;  // low 32: kernel count, high 32: single unit or -1
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  uint64_t* ql = reinterpret_cast<uint64_t*>(cs + F) + (size_t)warp * 3 * PK_QCAP;
  uint64_t* qh = ql + PK_QCAP;
  uint64_t* qm = qh + PK_QCAP;  // low 32: kernel count, high 32: owner lane
  uint64_t* tlo = reinterpret_cast<uint64_t*>(cs + F) + (size_t)(T / 32) * 3 * PK_QCAP + (size_t)warp * 64;
  uint64_t* thi = tlo + 32;
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
    LT lab = 0;  // nibble s: label of slot s
    LT act = 0;  // 0xF in nibble s while slot s is occupied
    uint64_t tot_lo = 0ull, tot_hi = 0ull;  // dynamic part of the total (two's complement)
    int32_t cached_word = -1;
    uint64_t word = 0;
    for (int32_t p = 0; p < a.M; ++p) {
      const uint4 hot = __ldg(&a.prog[p].hot);  // bit, slot|nback|nend, back nibbles, end nibbles
      const int32_t bit = (int32_t)hot.x;
      bool on = !dead;
      if (bit >= 0) {
        const int32_t wi = bit >> 6;
        if (wi != cached_word) {
          word = dead ? 0ull : __ldg(gen + wi);
          cached_word = wi;
        }
        on = (word >> (bit & 63)) & 1ull;
      }
      const int S = hot.y & 0xff;
      const int nback = (hot.y >> 8) & 0xff;
      const int nend = (hot.y >> 16) & 0xff;
      const LT nibS = (LT)0xF << (4 * S);
      if (on) {
        const uint64_t* c = a.cold + (size_t)p * 6;
        if (bit >= 0) {
          const ulonglong2 off = __ldg(reinterpret_cast<const ulonglong2*>(c + 2));
          sub2(tot_lo, tot_hi, off.x, off.y);
        }
        const ulonglong2 rep = __ldg(reinterpret_cast<const ulonglong2*>(c));
        sl[S][t] = rep.x;
        sh[S][t] = rep.y;
        cs[S][t] = ((uint64_t)(uint32_t)p << 32) | (uint32_t)__ldg(a.cnt + p);
        act |= nibS;
        lab = (lab & ~nibS) | ((LT)S << (4 * S));
      }
      for (int j = 0; j < nback; ++j) {
        const int b = (hot.z >> (4 * j)) & 0xF;
        const uint32_t B = (uint32_t)(lab >> (4 * b)) & 0xF;
        const bool merge = on && ((act >> (4 * b)) & 1) && B != (uint32_t)S;
        if (merge) {
          uint64_t lo = sl[S][t], hi = sh[S][t];
          add2(lo, hi, sl[B][t], sh[B][t]);
          sl[S][t] = lo;
          sh[S][t] = hi;
          const uint32_t c = (uint32_t)cs[S][t] + (uint32_t)cs[B][t];
          cs[S][t] = 0xffffffff00000000ull | c;
          const LT m = nibeq<LT>(lab, B) & act;
          lab = (lab & ~m) | (((LT)S * Nib2<LT>::ONE) & m);
        }
      }
      for (int j = 0; j < nend; ++j) {
        const int e = (hot.w >> (4 * j)) & 0xF;
        const LT nibE = (LT)0xF << (4 * e);
        int emit_slot = -1;
        if (act & nibE) {
          const uint32_t X = (uint32_t)(lab >> (4 * e)) & 0xF;
          act &= ~nibE;
          const LT others = nibeq<LT>(lab, X) & act;
          if (others == 0) {  // last member leaves: the region is complete
            const int32_t one = (int32_t)(cs[e][t] >> 32);
            if (one >= 0) {
              const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(a.cold + (size_t)one * 6 + 4));
              add2(tot_lo, tot_hi, v.x, v.y);
            } else {
              emit_slot = e;  // multi-unit region: queued for warp-wide pricing
            }
          } else if (X == (uint32_t)e) {  // data moves to a member that stays
            const int tgt = nibfirst<LT>(others);
            sl[tgt][t] = sl[e][t];
            sh[tgt][t] = sh[e][t];
            cs[tgt][t] = cs[e][t];
            lab = (lab & ~others) | (((LT)tgt * Nib2<LT>::ONE) & others);
          }
        }
        const unsigned closing = __ballot_sync(0xffffffffu, emit_slot >= 0);
        if (closing) {
          if (emit_slot >= 0) {
            const int at = qn + __popc(closing & ((1u << lane) - 1u));
            ql[at] = sl[emit_slot][t];
            qh[at] = sh[emit_slot][t];
            qm[at] = ((uint64_t)lane << 32) | (uint32_t)cs[emit_slot][t];
          }
          qn += __popc(closing);
          if (qn >= 32) {
            __syncwarp();
            pk_price(ql, qh, qm, lane, a, tlo, thi, inexact);
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
    if (lane < qn) pk_price(ql, qh, qm, lane, a, tlo, thi, inexact);
    qn = 0;
    __syncwarp();
    add2(tot_lo, tot_hi, tlo[lane], thi[lane]);
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

// Anchor form (F <= 8): the component label is the member slot whose unit
// ends last (the header's end-rank nibbles order the slots' current units by
// their last neighbour), so a non-anchor release is a bit clear and an
// anchor release closes the region -- no member test, no data move.
// W in 1..4: the genome's words are held in registers and loaded one genome
// ahead (the next row's loads overlap the current walk); W = 0 loads words
// on demand (longer genomes).
template <int F, int W>
__global__ void __launch_bounds__(PK_THREADS)
fitness_pa_kernel(PkArgs a, const uint4* __restrict__ hdr, const uint64_t* __restrict__ pop, int64_t n,
                  double* __restrict__ fit) {
  using LT = uint32_t;
  constexpr int T = PK_THREADS;
  extern __shared__ __align__(16) unsigned char pk_smem[];
  uint64_t(*sl)[T] = reinterpret_cast<uint64_t(*)[T]>(pk_smem);  // [F][T] sum, low word
  uint64_t(*sh)[T] = sl + F;                                       // high word
  uint64_t(*cs)[T] = sh + F;  // low 32: kernel count, high 32: single unit or -1
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  uint64_t* ql = reinterpret_cast<uint64_t*>(cs + F) + (size_t)warp * 3 * PK_QCAP;
  uint64_t* qh = ql + PK_QCAP;
  uint64_t* qm = qh + PK_QCAP;  // low 32: kernel count, high 32: owner lane
  uint64_t* tlo = reinterpret_cast<uint64_t*>(cs + F) + (size_t)(T / 32) * 3 * PK_QCAP + (size_t)warp * 64;
  uint64_t* thi = tlo + 32;
  tlo[lane] = thi[lane] = 0ull;
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
    } else if (in_range) {
      for (int32_t w = 0; w < a.words; ++w) dead |= (__ldg(gen + w) & __ldg(a.infeas + w)) != 0ull;
    }
    LT lab = 0;  // nibble s: label (anchor slot) of slot s
    LT act = 0;  // 0xF in nibble s while slot s is occupied
    uint64_t tot_lo = 0ull, tot_hi = 0ull;  // dynamic part of the total (two's complement)
    int32_t cached_word = -1;
    uint64_t word = 0, next_word = W == 0 && a.words > 0 ? __ldg(gen) : 0ull;
    for (int32_t p = 0; p < a.M; ++p) {
      // x = bit (20 bits, all ones = fixed unit) | slot << 20 | nback << 24 | nend << 28,
      // y = back slot nibbles, z = end slot nibbles, w = end rank of each slot's unit
      const uint4 h = __ldg(hdr + p);
      const uint32_t bitf = h.x & 0xFFFFFu;
      bool on = !dead;
      if (bitf != 0xFFFFFu) {
        const int32_t wi = (int32_t)(bitf >> 6);
        if (wi != cached_word) {  // warp uniform: the lanes walk the same program
          if (W > 0) {
            word = cur[0];
#pragma unroll
            for (int w = 1; w < WR; ++w)
              if (wi == w) word = cur[w];
            if (dead) word = 0ull;
          } else {  // long genomes: the next word is loaded one word ahead
            word = wi == cached_word + 1 ? next_word : __ldg(gen + wi);
            if (dead) word = 0ull;
            next_word = wi + 1 < a.words ? __ldg(gen + wi + 1) : 0ull;
          }
          cached_word = wi;
        }
        on = (word >> (bitf & 63)) & 1ull;
      }
      const int S = (h.x >> 20) & 0xF;
      const int nback = (h.x >> 24) & 0xF;
      const int nend = h.x >> 28;
      const LT nibS = (LT)0xF << (4 * S);
      if (on) {
        const uint64_t* c = a.cold + (size_t)p * 6;
        if (bitf != 0xFFFFFu) {
          const ulonglong2 off = __ldg(reinterpret_cast<const ulonglong2*>(c + 2));
          sub2(tot_lo, tot_hi, off.x, off.y);
        }
        const ulonglong2 rep = __ldg(reinterpret_cast<const ulonglong2*>(c));
        sl[S][t] = rep.x;
        sh[S][t] = rep.y;
        cs[S][t] = ((uint64_t)(uint32_t)p << 32) | (uint32_t)__ldg(a.cnt + p);
        act |= nibS;
        lab = (lab & ~nibS) | ((LT)S << (4 * S));
      }
      // back / end lists: straight-line code for the common (nback, nend)
      // shapes (warp-uniform switch on the header), a loop otherwise
      auto step_lists = [&](auto nb_c, auto ne_c) {
        constexpr int NB = decltype(nb_c)::value, NE = decltype(ne_c)::value;
        uint32_t A = (uint32_t)S;  // anchor of the new unit's component
        for (int j = 0; j < (NB >= 0 ? NB : nback); ++j) {  // constant trip counts unroll
          const int b = (h.y >> (4 * j)) & 0xF;
          const uint32_t B = (uint32_t)(lab >> (4 * b)) & 0xF;
          const bool merge = on && ((act >> (4 * b)) & 1) && B != A;
          if (merge) {
            // the anchor whose unit ends later survives
            const bool keepA = ((h.w >> (4 * A)) & 0xF) >= ((h.w >> (4 * B)) & 0xF);
            const uint32_t win = keepA ? A : B, los = keepA ? B : A;
            uint64_t lo = sl[win][t], hi = sh[win][t];
            add2(lo, hi, sl[los][t], sh[los][t]);
            sl[win][t] = lo;
            sh[win][t] = hi;
            const uint32_t c = (uint32_t)cs[win][t] + (uint32_t)cs[los][t];
            cs[win][t] = 0xffffffff00000000ull | c;
            const LT m = nibeq<LT>(lab, los) & act;
            lab = (lab & ~m) | (((LT)win * Nib2<LT>::ONE) & m);
            A = win;
          }
        }
        for (int j = 0; j < (NE >= 0 ? NE : nend); ++j) {
          const int e = (h.z >> (4 * j)) & 0xF;
          const LT nibE = (LT)0xF << (4 * e);
          int emit_slot = -1;
          if (act & nibE) {
            act &= ~nibE;
            if (((lab >> (4 * e)) & 0xF) == (uint32_t)e) {  // the anchor leaves: region complete
              const int32_t one = (int32_t)(cs[e][t] >> 32);
              if (one >= 0) {
                const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(a.cold + (size_t)one * 6 + 4));
                add2(tot_lo, tot_hi, v.x, v.y);
              } else {
                emit_slot = e;  // multi-unit region: queued for warp-wide pricing
              }
            }
          }
          const unsigned closing = __ballot_sync(0xffffffffu, emit_slot >= 0);
          if (closing) {
            if (emit_slot >= 0) {
              const int at = qn + __popc(closing & ((1u << lane) - 1u));
              ql[at] = sl[emit_slot][t];
              qh[at] = sh[emit_slot][t];
              qm[at] = ((uint64_t)lane << 32) | (uint32_t)cs[emit_slot][t];
            }
            qn += __popc(closing);
            if (qn >= 32) {
              __syncwarp();
              pk_price(ql, qh, qm, lane, a, tlo, thi, inexact);
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
      };
      switch ((nback << 4) | nend) {
        case 0x11: step_lists(IC<1>{}, IC<1>{}); break;
        case 0x10: step_lists(IC<1>{}, IC<0>{}); break;
        case 0x22: step_lists(IC<2>{}, IC<2>{}); break;
        case 0x21: step_lists(IC<2>{}, IC<1>{}); break;
        case 0x00: step_lists(IC<0>{}, IC<0>{}); break;
        case 0x32: step_lists(IC<3>{}, IC<2>{}); break;
        case 0x33: step_lists(IC<3>{}, IC<3>{}); break;
        default: step_lists(IC<-1>{}, IC<-1>{}); break;
      }
    }
    __syncwarp();
    if (lane < qn) pk_price(ql, qh, qm, lane, a, tlo, thi, inexact);
    qn = 0;
    __syncwarp();
    add2(tot_lo, tot_hi, tlo[lane], thi[lane]);
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

// Fused generation: each thread breeds its child (make_child, same draws as
// breed_thread_kernel), streams the row out, and prices it from registers
// with the packed anchor walk -- the breed's random parent / key gathers
// overlap the walk of other warps instead of running as a separate
// memory-bound launch, and the fitness pass needs no genome loads.
template <int F, int W>
__global__ void __launch_bounds__(PK_THREADS)
fitness_pa_breed_kernel(PkArgs a, const uint4* __restrict__ hdr, BreedArgs br, uint64_t* __restrict__ children,
                        int64_t n, double* __restrict__ fit) {
  using LT = uint32_t;
  constexpr int T = PK_THREADS;
  extern __shared__ __align__(16) unsigned char pk_smem[];
  uint64_t(*sl)[T] = reinterpret_cast<uint64_t(*)[T]>(pk_smem);  // [F][T] sum, low word
  uint64_t(*sh)[T] = sl + F;                                       // high word
  uint64_t(*cs)[T] = sh + F;  // low 32: kernel count, high 32: single unit or -1
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  uint64_t* ql = reinterpret_cast<uint64_t*>(cs + F) + (size_t)warp * 3 * PK_QCAP;
  uint64_t* qh = ql + PK_QCAP;
  uint64_t* qm = qh + PK_QCAP;  // low 32: kernel count, high 32: owner lane
  uint64_t* tlo = reinterpret_cast<uint64_t*>(cs + F) + (size_t)(T / 32) * 3 * PK_QCAP + (size_t)warp * 64;
  uint64_t* thi = tlo + 32;
  tlo[lane] = thi[lane] = 0ull;
  __syncwarp();
  int qn = 0;
  bool inexact = false;
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t base = (int64_t)blockIdx.x * T + (t & ~31); base < n; base += stride) {
    const int64_t i = base + lane;
    const bool in_range = i < n;
    uint64_t v[W];
    if (in_range) {
      make_child<W>(v, br.k, br.parents, br.fit, br.keys, br.n_parents, i, br.keep, br.n_keep, br.seed,
                    br.generation, br.stream_id, br.tournament, br.rate, br.log1m_rate);
#pragma unroll
      for (int w = 0; w < W; ++w) __stcs(children + i * W + w, v[w]);
    } else {
#pragma unroll
      for (int w = 0; w < W; ++w) v[w] = 0ull;
    }
    bool dead = !in_range;
#pragma unroll
    for (int w = 0; w < W; ++w) dead |= (v[w] & __ldg(a.infeas + w)) != 0ull;
    LT lab = 0;  // nibble s: label (anchor slot) of slot s
    LT act = 0;  // 0xF in nibble s while slot s is occupied
    uint64_t tot_lo = 0ull, tot_hi = 0ull;  // dynamic part of the total (two's complement)
    for (int32_t p = 0; p < a.M; ++p) {
      // x = bit (20 bits, all ones = fixed unit) | slot << 20 | nback << 24 | nend << 28,
      // y = back slot nibbles, z = end slot nibbles, w = end rank of each slot's unit
      const uint4 h = __ldg(hdr + p);
      const uint32_t bitf = h.x & 0xFFFFFu;
      bool on = !dead;
      if (bitf != 0xFFFFFu) {
        const int32_t wi = (int32_t)(bitf >> 6);
        uint64_t word = v[0];
#pragma unroll
        for (int w = 1; w < W; ++w)
          if (wi == w) word = v[w];
        on = !dead && ((word >> (bitf & 63)) & 1ull);
      }
      const int S = (h.x >> 20) & 0xF;
      const int nback = (h.x >> 24) & 0xF;
      const int nend = h.x >> 28;
      const LT nibS = (LT)0xF << (4 * S);
      if (on) {
        const uint64_t* c = a.cold + (size_t)p * 6;
        if (bitf != 0xFFFFFu) {
          const ulonglong2 off = __ldg(reinterpret_cast<const ulonglong2*>(c + 2));
          sub2(tot_lo, tot_hi, off.x, off.y);
        }
        const ulonglong2 rep = __ldg(reinterpret_cast<const ulonglong2*>(c));
        sl[S][t] = rep.x;
        sh[S][t] = rep.y;
        cs[S][t] = ((uint64_t)(uint32_t)p << 32) | (uint32_t)__ldg(a.cnt + p);
        act |= nibS;
        lab = (lab & ~nibS) | ((LT)S << (4 * S));
      }
      uint32_t A = (uint32_t)S;  // anchor of the new unit's component
      for (int j = 0; j < nback; ++j) {
        const int b = (h.y >> (4 * j)) & 0xF;
        const uint32_t B = (uint32_t)(lab >> (4 * b)) & 0xF;
        const bool merge = on && ((act >> (4 * b)) & 1) && B != A;
        if (merge) {
          // the anchor whose unit ends later survives
          const bool keepA = ((h.w >> (4 * A)) & 0xF) >= ((h.w >> (4 * B)) & 0xF);
          const uint32_t win = keepA ? A : B, los = keepA ? B : A;
          uint64_t lo = sl[win][t], hi = sh[win][t];
          add2(lo, hi, sl[los][t], sh[los][t]);
          sl[win][t] = lo;
          sh[win][t] = hi;
          const uint32_t c = (uint32_t)cs[win][t] + (uint32_t)cs[los][t];
          cs[win][t] = 0xffffffff00000000ull | c;
          const LT m = nibeq<LT>(lab, los) & act;
          lab = (lab & ~m) | (((LT)win * Nib2<LT>::ONE) & m);
          A = win;
        }
      }
      for (int j = 0; j < nend; ++j) {
        const int e = (h.z >> (4 * j)) & 0xF;
        const LT nibE = (LT)0xF << (4 * e);
        int emit_slot = -1;
        if (act & nibE) {
          act &= ~nibE;
          if (((lab >> (4 * e)) & 0xF) == (uint32_t)e) {  // the anchor leaves: region complete
            const int32_t one = (int32_t)(cs[e][t] >> 32);
            if (one >= 0) {
              const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(a.cold + (size_t)one * 6 + 4));
              add2(tot_lo, tot_hi, v.x, v.y);
            } else {
              emit_slot = e;  // multi-unit region: queued for warp-wide pricing
            }
          }
        }
        const unsigned closing = __ballot_sync(0xffffffffu, emit_slot >= 0);
        if (closing) {
          if (emit_slot >= 0) {
            const int at = qn + __popc(closing & ((1u << lane) - 1u));
            ql[at] = sl[emit_slot][t];
            qh[at] = sh[emit_slot][t];
            qm[at] = ((uint64_t)lane << 32) | (uint32_t)cs[emit_slot][t];
          }
          qn += __popc(closing);
          if (qn >= 32) {
            __syncwarp();
            pk_price(ql, qh, qm, lane, a, tlo, thi, inexact);
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
    if (lane < qn) pk_price(ql, qh, qm, lane, a, tlo, thi, inexact);
    qn = 0;
    __syncwarp();
    add2(tot_lo, tot_hi, tlo[lane], thi[lane]);
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

PkArgs make_pk_args(cb_es_plan* p) {
  PkArgs a;
  a.M = p->M;
  a.words = p->words;
  a.shift = p->anchor_shift;
  a.base_const = p->base_const;
  const fx192 ex = fx_shr(p->eps, p->anchor_shift);
  a.eps_lo = ex.w[0];
  a.eps_hi = ex.w[1];
  a.prog = p->d_prog.p;
  a.cold = p->d_acold.p;
  a.cnt = p->d_acnt.p;
  a.infeas = p->d_infeas.p;
  a.rt = p->d_rt.p;
  a.flags = p->d_flags.p;
  return a;
}

template <typename LT, int F>
int launch_pk_t(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit, cudaStream_t stream) {
  const size_t smem = ((size_t)3 * F * PK_THREADS + (size_t)(PK_THREADS / 32) * (3 * PK_QCAP + 64)) *
                      sizeof(uint64_t);
  if (cb_smem_claim((const void*)fitness_packed128_kernel<LT, F>, smem))
    CB_CUDA_TRY(cudaFuncSetAttribute(fitness_packed128_kernel<LT, F>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  CB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fitness_packed128_kernel<LT, F>,
                                                            PK_THREADS, smem));
  if (per_sm < 1) per_sm = 1;
  PkArgs a = make_pk_args(p);
  const int64_t want = (n + PK_THREADS - 1) / PK_THREADS;
  const int64_t grid = std::min<int64_t>(want, (int64_t)per_sm * cb_sm_count());
  fitness_packed128_kernel<LT, F><<<(unsigned)grid, PK_THREADS, smem, stream>>>(a, d_pop, n, d_fit);
  CB_CUDA_TRY(cudaGetLastError());
  return CB_OK;
}

template <int F, int W>
int launch_pa_t(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit, cudaStream_t stream) {
  const size_t smem = ((size_t)3 * F * PK_THREADS + (size_t)(PK_THREADS / 32) * (3 * PK_QCAP + 64)) *
                      sizeof(uint64_t);
  if (cb_smem_claim((const void*)fitness_pa_kernel<F, W>, smem))
    CB_CUDA_TRY(cudaFuncSetAttribute(fitness_pa_kernel<F, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  int per_sm = 0;
  CB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fitness_pa_kernel<F, W>, PK_THREADS, smem));
  if (per_sm < 1) per_sm = 1;
  PkArgs a = make_pk_args(p);
  const int64_t want = (n + PK_THREADS - 1) / PK_THREADS;
  const int64_t grid = std::min<int64_t>(want, (int64_t)per_sm * cb_sm_count());
  fitness_pa_kernel<F, W><<<(unsigned)grid, PK_THREADS, smem, stream>>>(
      a, reinterpret_cast<const uint4*>(p->d_pahdr.p), d_pop, n, d_fit);
  CB_CUDA_TRY(cudaGetLastError());
  return CB_OK;
}

template <int F>
int launch_pa_w(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit, cudaStream_t stream) {
  switch (p->words) {
    case 1: return launch_pa_t<F, 1>(p, d_pop, n, d_fit, stream);
    case 2: return launch_pa_t<F, 2>(p, d_pop, n, d_fit, stream);
    case 3: return launch_pa_t<F, 3>(p, d_pop, n, d_fit, stream);
    case 4: return launch_pa_t<F, 4>(p, d_pop, n, d_fit, stream);
    default: return launch_pa_t<F, 0>(p, d_pop, n, d_fit, stream);
  }
}

template <int F, int W>
int launch_pab_t(cb_es_plan* p, const BreedArgs& br, uint64_t* d_children, int64_t n, double* d_fit,
                 cudaStream_t stream) {
  const size_t smem = ((size_t)3 * F * PK_THREADS + (size_t)(PK_THREADS / 32) * (3 * PK_QCAP + 64)) *
                      sizeof(uint64_t);
  if (cb_smem_claim((const void*)fitness_pa_breed_kernel<F, W>, smem))
    CB_CUDA_TRY(cudaFuncSetAttribute(fitness_pa_breed_kernel<F, W>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  CB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fitness_pa_breed_kernel<F, W>,
                                                            PK_THREADS, smem));
  if (per_sm < 1) per_sm = 1;
  PkArgs a = make_pk_args(p);
  const int64_t want = (n + PK_THREADS - 1) / PK_THREADS;
  const int64_t grid = std::min<int64_t>(want, (int64_t)per_sm * cb_sm_count());
  fitness_pa_breed_kernel<F, W><<<(unsigned)grid, PK_THREADS, smem, stream>>>(
      a, reinterpret_cast<const uint4*>(p->d_pahdr.p), br, d_children, n, d_fit);
  CB_CUDA_TRY(cudaGetLastError());
  return CB_OK;
}

template <int F>
int launch_pab_f(cb_es_plan* p, const BreedArgs& br, uint64_t* c, int64_t n, double* f, cudaStream_t s) {
  switch (p->words) {
    case 1: return launch_pab_t<F, 1>(p, br, c, n, f, s);
    case 2: return launch_pab_t<F, 2>(p, br, c, n, f, s);
    case 3: return launch_pab_t<F, 3>(p, br, c, n, f, s);
    default: return launch_pab_t<F, 4>(p, br, c, n, f, s);
  }
}

}  // namespace

bool fused_generation_ok(const cb_es_plan* p) {
  return p->F > 0 && p->pa_ok && p->anchor_ok && p->words <= 4 && (p->force_path == -1 || p->force_path == 6);
}

int launch_fused_generation(cb_es_plan* p, const BreedArgs& br, uint64_t* d_children, int64_t n,
                            double* d_fit, cudaStream_t stream) {
  if (p->F <= 4) return launch_pab_f<4>(p, br, d_children, n, d_fit, stream);
  if (p->F <= 6) return launch_pab_f<6>(p, br, d_children, n, d_fit, stream);
  return launch_pab_f<8>(p, br, d_children, n, d_fit, stream);
}

int launch_fitness_packed_anchor(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit,
                                 cudaStream_t stream) {
  if (p->F <= 4) return launch_pa_w<4>(p, d_pop, n, d_fit, stream);
  if (p->F <= 6) return launch_pa_w<6>(p, d_pop, n, d_fit, stream);
  return launch_pa_w<8>(p, d_pop, n, d_fit, stream);
}

int launch_fitness_packed128(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit,
                             cudaStream_t stream) {
  if (p->F <= 4) return launch_pk_t<uint32_t, 4>(p, d_pop, n, d_fit, stream);
  if (p->F <= 6) return launch_pk_t<uint32_t, 6>(p, d_pop, n, d_fit, stream);
  if (p->F <= 8) return launch_pk_t<uint32_t, 8>(p, d_pop, n, d_fit, stream);
  if (p->F <= 12) return launch_pk_t<uint64_t, 12>(p, d_pop, n, d_fit, stream);
  return launch_pk_t<uint64_t, 16>(p, d_pop, n, d_fit, stream);
}
