// Operator-level placement DP on the device.
//
// The reference (tensorplace/dp.py:71-179) keeps one state per covered node
// set and relaxes every stored state for every candidate match; its optimum
// is the cheapest partition of the graph into registry matches, ties broken
// by the canonical key (sorted (registration index, sorted node ids) pairs,
// tensorplace/placement.py:78-82).  Because a match may only expose its
// root (matching.py:93-101), every non-root member of a kernel is
// post-dominated by the kernel root, so the kernels of any partition nest
// along the post-dominator tree.  That turns the covered-set DP into an
// exact DP over post-dominator subtrees:
//
//   OPT(r) = min over matches m rooted at r of
//            cost(m) + eps + sum_{x not in m, ipdom(x) in m} OPT(x)
//
// and the answer is the sum of OPT over nodes whose ipdom is the virtual
// sink.  OPT(x) only depends on DAG ancestors of r, so all nodes of one
// topological frontier level (the reference's pop order (depth, id)) are
// relaxed in parallel: one warp per node, one lane per candidate match.
// Costs are exact 192-bit fixed-point sums (fixed192.cuh) so equal
// partitions compare equal; the warp minimum uses shuffles, and exact ties
// are settled by the reference's key order: the winner is the side holding
// the smallest kernel of the symmetric difference, found by walking the two
// candidate solutions down the post-dominator tree until they agree.
#include <algorithm>
#include <climits>
#include <cstring>

#include <cmath>

#include "cb_internal.cuh"

#define DP_NARROW_WARPS 16
#define DP_WIDE_WARPS 8
#define DP_STAGE_MAX (200 * 1024)
#define DP_WSTACK 64  // per-warp tie-walk stack entries in shared memory

struct DPArgs {
  // graph
  const int32_t* level_nodes;
  const int32_t* pch_ptr;
  const int32_t* pch;
  // matches grouped by root
  const int32_t* group_ptr;
  const int32_t* pat;
  const int32_t* mem_ptr;
  const int32_t* members;
  const double* cost;
  fx192 eps;
  // state
  fx192* opt;
  uint8_t* feas;
  int32_t* choice;
  fx192* regret;  // min positive regret per node (all-ones = none)
  // tie walks
  int* lock;
  int4* stack;
  unsigned long long* counters;  // [0] ties, [1] walk steps, [2] inexact
};

__device__ __forceinline__ fx192 shfl_fx(const fx192& v, int src) {
  fx192 r;
  r.w[0] = __shfl_sync(0xffffffffu, v.w[0], src);
  r.w[1] = __shfl_sync(0xffffffffu, v.w[1], src);
  r.w[2] = __shfl_sync(0xffffffffu, v.w[2], src);
  return r;
}

__device__ __forceinline__ fx192 fx_max() {
  fx192 r;
  r.w[0] = r.w[1] = r.w[2] = ~0ull;
  return r;
}

__device__ __forceinline__ bool is_member(const DPArgs& a, int32_t m, int32_t u) {
  int32_t lo = a.mem_ptr[m], hi = a.mem_ptr[m + 1];
  while (lo < hi) {
    int32_t mid = (lo + hi) >> 1;
    int32_t v = a.members[mid];
    if (v < u) lo = mid + 1;
    else if (v > u) hi = mid;
    else return true;
  }
  return false;
}

// Kernel key order: (registration index, sorted node tuple).
__device__ bool elem_less(const DPArgs& a, int32_t k1, int32_t k2) {
  if (a.pat[k1] != a.pat[k2]) return a.pat[k1] < a.pat[k2];
  int32_t i = a.mem_ptr[k1], ie = a.mem_ptr[k1 + 1];
  int32_t j = a.mem_ptr[k2], je = a.mem_ptr[k2 + 1];
  for (; i < ie && j < je; ++i, ++j)
    if (a.members[i] != a.members[j]) return a.members[i] < a.members[j];
  return (ie - i) < (je - j);
}

__device__ bool same_members(const DPArgs& a, int32_t k1, int32_t k2) {
  int32_t n1 = a.mem_ptr[k1 + 1] - a.mem_ptr[k1];
  if (n1 != a.mem_ptr[k2 + 1] - a.mem_ptr[k2]) return false;
  for (int32_t i = 0; i < n1; ++i)
    if (a.members[a.mem_ptr[k1] + i] != a.members[a.mem_ptr[k2] + i]) return false;
  return true;
}

// True when the subtree solution that roots r with k1 sorts before the one
// rooting r with k2 (both equal in cost).  Executed by a single thread: a
// depth-first walk of the post-dominator subtree that only descends where the
// two solutions' owning kernels differ, tracking the smallest kernel each side
// holds outside the other.  The walk uses the warp's own shared-memory stack;
// a walk deeper than that restarts on the global stack under a lock.
__device__ bool solution_walk(const DPArgs& a, int32_t r, int32_t k1, int32_t k2, int4* stack,
                              int64_t cap, bool& overflow) {
  int32_t best1 = k1, best2 = k2;
  int64_t top = 0;
  unsigned long long steps = 0;
  stack[top++] = make_int4(r, k1, k2, 0);
  overflow = false;
  while (top > 0) {
    int4 e = stack[--top];
    for (int32_t j = a.pch_ptr[e.x]; j < a.pch_ptr[e.x + 1]; ++j) {
      const int32_t u = a.pch[j];
      ++steps;
      const bool in1 = is_member(a, e.y, u);
      const bool in2 = is_member(a, e.z, u);
      const int32_t cu = a.choice[u];
      const int32_t o1 = in1 ? e.y : cu;
      const int32_t o2 = in2 ? e.z : cu;
      if (o1 == o2) continue;
      if (!in1 && cu >= 0 && elem_less(a, cu, best1)) best1 = cu;
      if (!in2 && cu >= 0 && elem_less(a, cu, best2)) best2 = cu;
      if (top == cap) {
        overflow = true;
        return false;
      }
      stack[top++] = make_int4(u, o1, o2, 0);
    }
  }
  atomicAdd(a.counters + 1, steps);
  return elem_less(a, best1, best2);
}

__device__ bool solution_less(const DPArgs& a, int32_t r, int32_t k1, int32_t k2, int4* wstack) {
  if (same_members(a, k1, k2)) return a.pat[k1] < a.pat[k2];
  bool overflow = false;
  const bool less = solution_walk(a, r, k1, k2, wstack, DP_WSTACK, overflow);
  if (!overflow) return less;
  while (atomicCAS(a.lock, 0, 1) != 0) {
  }
  __threadfence();
  const bool res = solution_walk(a, r, k1, k2, a.stack, INT64_MAX, overflow);
  __threadfence();
  atomicExch(a.lock, 0);
  return res;
}

// Value of candidate c for root r; returns false when some required
// sub-solution is infeasible.
__device__ __forceinline__ bool candidate_value(const DPArgs& a, int32_t c, fx192& val,
                                                bool& inexact) {
  if (!fx_from_double(a.cost[c], val)) inexact = true;
  fx_add(val, a.eps);
  const int32_t i0 = a.mem_ptr[c], i1 = a.mem_ptr[c + 1];
  for (int32_t i = i0; i < i1; ++i) {
    const int32_t u = a.members[i];
    for (int32_t j = a.pch_ptr[u]; j < a.pch_ptr[u + 1]; ++j) {
      const int32_t x = a.pch[j];
      if (is_member(a, c, x)) continue;
      // plain loads: values come from earlier launches or, inside one CTA,
      // from earlier levels separated by __syncthreads (opt/feas may live in
      // shared memory in the narrow-segment kernel)
      if (!a.feas[x]) return false;
      const fx192 o = a.opt[x];
      fx_add(val, o);
    }
  }
  return true;
}

// Whole warp relaxes node r (`wstack`: the warp's tie-walk stack).
__device__ void dp_node(const DPArgs& a, int32_t r, int4* wstack) {
  const int lane = threadIdx.x & 31;
  const int32_t c0 = a.group_ptr[r], c1 = a.group_ptr[r + 1];
  bool inexact = false;
  // pass 1: minimum and second minimum (distinct) over feasible candidates
  fx192 best = fx_max(), second = fx_max();
  bool any = false;
  fx192 last_v = fx_max();
  bool last_ok = false;
  for (int32_t base = c0; base < c1; base += 32) {
    const int32_t c = base + lane;
    fx192 v = fx_max();
    bool ok = false;
    if (c < c1) ok = candidate_value(a, c, v, inexact);
    if (!ok) v = fx_max();
    last_v = v;
    last_ok = ok;
    // warp min of v
    fx192 mn = v;
    for (int off = 16; off > 0; off >>= 1) {
      fx192 o = shfl_fx(mn, lane ^ off);
      if (fx_cmp(o, mn) < 0) mn = o;
    }
    const bool chunk_any = __any_sync(0xffffffffu, ok);
    // second candidate within this chunk: smallest v > mn
    fx192 sv = (ok && fx_cmp(v, mn) > 0) ? v : fx_max();
    for (int off = 16; off > 0; off >>= 1) {
      fx192 o = shfl_fx(sv, lane ^ off);
      if (fx_cmp(o, sv) < 0) sv = o;
    }
    if (chunk_any) {
      if (!any) {
        best = mn;
        second = sv;
      } else {
        const int cmpv = fx_cmp(mn, best);
        if (cmpv < 0) {  // the old best is now the runner-up candidate
          second = (fx_cmp(best, sv) < 0) ? best : sv;
          best = mn;
        } else if (cmpv > 0) {
          if (fx_cmp(mn, second) < 0) second = mn;
        } else if (fx_cmp(sv, second) < 0) {
          second = sv;
        }
      }
      any = true;
    }
  }
  if (__any_sync(0xffffffffu, inexact) && lane == 0) atomicAdd(a.counters + 2, 1ull);
  if (!any) {
    if (lane == 0) {
      a.feas[r] = 0;
      a.choice[r] = -1;
      a.regret[r] = fx_max();
    }
    return;
  }
  // pass 2: candidates attaining the minimum, settled by the key order
  // (a single chunk reuses its pass-1 values instead of recomputing them)
  int32_t winner = -1;
  int ties = 0;
  const bool one_chunk = c1 - c0 <= 32;
  for (int32_t base = c0; base < c1; base += 32) {
    const int32_t c = base + lane;
    fx192 v = last_v;
    bool ok = last_ok;
    bool dummy = false;
    if (!one_chunk) {
      ok = false;
      if (c < c1) ok = candidate_value(a, c, v, dummy);
    }
    const bool hit = ok && fx_eq(v, best);
    unsigned mask = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) {
      while (mask) {
        const int bit = __ffs(mask) - 1;
        mask &= mask - 1;
        const int32_t cand = base + bit;
        if (winner < 0) {
          winner = cand;
        } else {
          ++ties;
          if (solution_less(a, r, cand, winner, wstack)) winner = cand;
        }
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    a.opt[r] = best;
    a.feas[r] = 1;
    a.choice[r] = winner;
    fx192 reg = second;
    if (!(reg.w[0] == ~0ull && reg.w[1] == ~0ull && reg.w[2] == ~0ull)) fx_sub(reg, best);
    a.regret[r] = reg;
    if (ties) atomicAdd(a.counters + 0, (unsigned long long)ties);
  }
}

// One CTA walks a run of narrow levels.  When the graph is small enough the
// per-node DP values (OPT, feasibility) are staged in shared memory for the
// whole run, so each level's dependent reads of its post-dominator
// children's values hit shared memory instead of L2; they are written back
// to global memory for the nodes of this run at the end.
// Sizes of the read-only arrays a narrow run may stage in shared memory.
struct DPStage {
  int32_t n_stage;     // nodes whose OPT / feasibility are staged (0 = none)
  int32_t n_groups;    // graph nodes (group_ptr has n_groups + 1 entries)
  int32_t n_matches;   // 0 = match tables not staged
  int32_t n_members;
  int32_t n_pch;
};

__global__ void __launch_bounds__(DP_NARROW_WARPS * 32)
dp_narrow_kernel(DPArgs a, const int32_t* __restrict__ level_ptr, int32_t lvl_begin, int32_t lvl_end,
                 DPStage st) {
  extern __shared__ __align__(16) unsigned char dp_smem[];
  __shared__ int4 s_stack[DP_WSTACK * DP_NARROW_WARPS];
  const int warp = threadIdx.x >> 5;
  DPArgs b = a;
  unsigned char* cur = dp_smem;
  if (st.n_stage > 0) {
    fx192* s_opt = reinterpret_cast<fx192*>(cur);
    uint8_t* s_feas = reinterpret_cast<uint8_t*>(s_opt + st.n_stage);
    for (int32_t v = threadIdx.x; v < st.n_stage; v += blockDim.x) {
      s_opt[v] = a.opt[v];
      s_feas[v] = a.feas[v];
    }
    b.opt = s_opt;
    b.feas = s_feas;
    cur = reinterpret_cast<unsigned char*>(s_feas) + ((st.n_stage + 15) & ~15);
  }
  if (st.n_matches > 0) {
    // the match tables and the post-dominator tree are read by every
    // relaxation of the run: stage them so the dependent chains of a
    // candidate's value (group -> members -> children -> OPT) stay on chip
    auto stage_i32 = [&](const int32_t* src, int32_t count) -> const int32_t* {
      int32_t* dst = reinterpret_cast<int32_t*>(cur);
      for (int32_t i = threadIdx.x; i < count; i += blockDim.x) dst[i] = src[i];
      cur += ((size_t)count * 4 + 15) & ~(size_t)15;
      return dst;
    };
    double* s_cost = reinterpret_cast<double*>(cur);
    for (int32_t i = threadIdx.x; i < st.n_matches; i += blockDim.x) s_cost[i] = a.cost[i];
    cur += ((size_t)st.n_matches * 8 + 15) & ~(size_t)15;
    b.cost = s_cost;
    b.group_ptr = stage_i32(a.group_ptr, st.n_groups + 1);
    b.pat = stage_i32(a.pat, st.n_matches);
    b.mem_ptr = stage_i32(a.mem_ptr, st.n_matches + 1);
    b.members = stage_i32(a.members, st.n_members);
    b.pch_ptr = stage_i32(a.pch_ptr, st.n_groups + 1);
    b.pch = stage_i32(a.pch, st.n_pch);
  }
  __syncthreads();
  for (int32_t l = lvl_begin; l < lvl_end; ++l) {
    const int32_t i0 = level_ptr[l], i1 = level_ptr[l + 1];
    for (int32_t i = i0 + warp; i < i1; i += DP_NARROW_WARPS)
      dp_node(b, a.level_nodes[i], s_stack + warp * DP_WSTACK);
    __syncthreads();
  }
  if (st.n_stage > 0) {
    const int32_t i0 = level_ptr[lvl_begin], i1 = level_ptr[lvl_end];
    for (int32_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
      const int32_t v = a.level_nodes[i];
      a.opt[v] = b.opt[v];
      a.feas[v] = b.feas[v];
    }
  }
}

__global__ void __launch_bounds__(DP_WIDE_WARPS * 32)
dp_wide_kernel(DPArgs a, int32_t i0, int32_t i1) {
  __shared__ int4 s_stack[DP_WIDE_WARPS * DP_WSTACK];
  const int32_t i = i0 + blockIdx.x * DP_WIDE_WARPS + (threadIdx.x >> 5);
  if (i < i1) dp_node(a, a.level_nodes[i], s_stack + (threadIdx.x >> 5) * DP_WSTACK);
}

// Sum of OPT over post-dominator-tree roots + global minimum regret.
__global__ void dp_total_kernel(int32_t n, const int32_t* __restrict__ ipdom, const fx192* opt,
                                const uint8_t* feas, const fx192* regret, fx192* out_total,
                                fx192* out_regret, int32_t* out_feasible) {
  __shared__ fx192 s_tot[256];
  __shared__ fx192 s_reg[256];
  __shared__ int s_feas[256];
  fx192 tot = fx_zero(), reg = fx_max();
  int f = 1;
  for (int32_t v = threadIdx.x; v < n; v += blockDim.x) {
    if (ipdom[v] < 0) {
      if (!feas[v]) f = 0;
      else fx_add(tot, opt[v]);
    }
    if (feas[v] && fx_cmp(regret[v], reg) < 0) reg = regret[v];
  }
  s_tot[threadIdx.x] = tot;
  s_reg[threadIdx.x] = reg;
  s_feas[threadIdx.x] = f;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int t = 1; t < blockDim.x; ++t) {
      fx_add(tot, s_tot[t]);
      if (fx_cmp(s_reg[t], reg) < 0) reg = s_reg[t];
      f &= s_feas[t];
    }
    *out_total = tot;
    *out_regret = reg;
    *out_feasible = f;
  }
}

// True when the reference's rounded comparisons cannot choose differently
// from the exact ones.  The reference keeps one state per covered set and
// compares states by their rounded costs (dp.py:128-147, cost.py:300-305).
// Any two states of one cover differ by a sum of decision regrets (the
// cover is a union of post-dominator subtrees, solved independently), so
// a state that is exactly worse is worse by at least the minimum positive
// regret `gap`.  States that matter cost at most the total T (costs are
// non-negative); an exactly-worse one can share T's rounded value only if
// it is within about one ulp of the binade above T.  gap >= 4 ulp(T) rules
// that out (the same test as oracle/oracle.py window_safe).
static bool rounding_window_safe(const fx192& total, const fx192& gap) {
  const double t = fx_to_double(total);
  const double ulp = std::nextafter(t, INFINITY) - t;
  fx192 lim;
  if (!fx_from_double(4.0 * ulp, lim)) return false;
  return fx_cmp(gap, lim) >= 0;
}

extern "C" int cb_dp_solve(cb_graph* g, cb_matches* m, double epsilon, int32_t* kernel_match,
                           cb_dp_result* res) {
  return cb_dp_solve_stream(g, m, epsilon, kernel_match, res, nullptr);
}

extern "C" int cb_dp_solve_stream(cb_graph* g, cb_matches* m, double epsilon, int32_t* kernel_match,
                                  cb_dp_result* res, void* stream) {
  cudaStream_t strm = (cudaStream_t)stream;
  CB_ARG_CHECK(g && m && res, "cb_dp_solve: null argument");
  CB_ARG_CHECK(m->by_root && m->n_groups == g->n, "cb_dp_solve: matches must come from cb_match_all");
  if (!m->costs_set) {
    cb_set_error("cb_dp_solve: kernel costs have not been set");
    return CB_ERR_STATE;
  }
  int rc = cb_graph_ensure_device(g);
  if (rc != CB_OK) return rc;
  std::memset(res, 0, sizeof(*res));
  res->first_zero_candidate = -1;
  const int32_t n = g->n;
  fx192 eps_fx;
  if (!fx_from_double(epsilon, eps_fx)) {
    cb_set_error("epsilon is negative, non-finite or outside the exact accumulator range");
    return CB_ERR_INEXACT;
  }
  rc = cb_matches_ensure_host(m);
  if (rc != CB_OK) return rc;
  for (int32_t i = 0; i < n; ++i) {
    int32_t v = g->level_nodes[i];
    if (m->group_ptr[v + 1] == m->group_ptr[v]) {
      res->first_zero_candidate = v;
      break;
    }
  }
  res->candidates = m->n_matches;
  if (n == 0) {
    res->feasible = 1;
    res->cost_ms = 0.0;
    return CB_OK;
  }
  DBuf<fx192> opt, regret, d_tot, d_reg;
  DBuf<uint8_t> feas;
  DBuf<int32_t> choice, d_feas_out, d_level_ptr;
  DBuf<int> lock;
  DBuf<int4> stack;
  DBuf<unsigned long long> counters;
  CB_CUDA_TRY(opt.alloc(n));
  CB_CUDA_TRY(regret.alloc(n));
  CB_CUDA_TRY(feas.alloc(n));
  CB_CUDA_TRY(choice.alloc(n));
  CB_CUDA_TRY(d_tot.alloc(1));
  CB_CUDA_TRY(d_reg.alloc(1));
  CB_CUDA_TRY(d_feas_out.alloc(1));
  CB_CUDA_TRY(lock.alloc(1));
  CB_CUDA_TRY(stack.alloc((size_t)n + 1));
  CB_CUDA_TRY(counters.alloc(4));
  CB_CUDA_TRY(d_level_ptr.upload(g->level_ptr));
  CB_CUDA_TRY(cudaMemsetAsync(lock.p, 0, sizeof(int), strm));
  CB_CUDA_TRY(cudaMemsetAsync(counters.p, 0, 4 * sizeof(unsigned long long), strm));
  CB_CUDA_TRY(cudaMemsetAsync(feas.p, 0, n, strm));

  DPArgs a;
  a.level_nodes = g->d_level_nodes.p;
  a.pch_ptr = g->d_pch_ptr.p;
  a.pch = g->d_pch.p;
  a.group_ptr = m->d_group_ptr.p;
  a.pat = m->d_pat.p;
  a.mem_ptr = m->d_mem_ptr.p;
  a.members = m->d_members.p;
  a.cost = m->d_cost.p;
  a.eps = eps_fx;
  a.opt = opt.p;
  a.feas = feas.p;
  a.choice = choice.p;
  a.regret = regret.p;
  a.lock = lock.p;
  a.stack = stack.p;
  a.counters = counters.p;

  cudaEvent_t ev0, ev1;
  cudaEventCreate(&ev0);
  cudaEventCreate(&ev1);
  cudaEventRecord(ev0, strm);
  std::vector<LevelSegment> segs = cb_plan_levels(g, 2 * DP_NARROW_WARPS);
  if (cb_smem_claim((const void*)dp_narrow_kernel, DP_STAGE_MAX))
    CB_CUDA_TRY(cudaFuncSetAttribute(dp_narrow_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)DP_STAGE_MAX));
  for (const LevelSegment& s : segs) {
    if (s.narrow) {
      auto al = [](size_t b) { return (b + 15) & ~(size_t)15; };
      DPStage st{};
      size_t bytes = 0;
      const size_t opt_bytes = (size_t)n * sizeof(fx192) + al((size_t)n);
      if (opt_bytes <= DP_STAGE_MAX) {
        st.n_stage = n;
        bytes = opt_bytes;
      }
      const size_t tab_bytes = al((size_t)m->n_matches * 8) + al(((size_t)n + 1) * 4) * 2 +
                               al((size_t)m->n_matches * 4) + al(((size_t)m->n_matches + 1) * 4) +
                               al((size_t)m->n_members * 4) + al(g->pch.size() * 4);
      if (st.n_stage && bytes + tab_bytes <= DP_STAGE_MAX) {
        st.n_groups = n;
        st.n_matches = (int32_t)m->n_matches;
        st.n_members = (int32_t)m->n_members;
        st.n_pch = (int32_t)g->pch.size();
        bytes += tab_bytes;
      }
      dp_narrow_kernel<<<1, DP_NARROW_WARPS * 32, bytes, strm>>>(a, d_level_ptr.p, s.lvl_begin, s.lvl_end, st);
    } else {
      int32_t i0 = g->level_ptr[s.lvl_begin], i1 = g->level_ptr[s.lvl_end];
      int32_t blocks = (i1 - i0 + DP_WIDE_WARPS - 1) / DP_WIDE_WARPS;
      dp_wide_kernel<<<blocks, DP_WIDE_WARPS * 32, 0, strm>>>(a, i0, i1);
    }
    CB_CUDA_TRY(cudaGetLastError());
  }
  dp_total_kernel<<<1, 256, 0, strm>>>(n, g->d_ipdom.p, opt.p, feas.p, regret.p, d_tot.p, d_reg.p,
                              d_feas_out.p);
  cudaEventRecord(ev1, strm);
  CB_CUDA_TRY(cudaEventSynchronize(ev1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ev0, ev1);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  CB_CUDA_TRY(cudaGetLastError());
  res->device_ms = ms;
  res->n_levels = (int32_t)g->level_ptr.size() - 1;
  res->n_launches = (int32_t)segs.size() + 1;

  fx192 tot, reg;
  int32_t feasible = 0;
  unsigned long long cnt[4];
  CB_CUDA_TRY(cudaMemcpy(&tot, d_tot.p, sizeof(fx192), cudaMemcpyDeviceToHost));
  CB_CUDA_TRY(cudaMemcpy(&reg, d_reg.p, sizeof(fx192), cudaMemcpyDeviceToHost));
  CB_CUDA_TRY(cudaMemcpy(&feasible, d_feas_out.p, sizeof(int32_t), cudaMemcpyDeviceToHost));
  CB_CUDA_TRY(cudaMemcpy(cnt, counters.p, sizeof(cnt), cudaMemcpyDeviceToHost));
  res->ties = (int64_t)cnt[0];
  res->walk_steps = (int64_t)cnt[1];
  if (cnt[2]) {
    cb_set_error("a kernel cost falls outside the exact accumulator range [2^-75, 2^64)");
    return CB_ERR_INEXACT;
  }
  res->feasible = feasible;
  if (!feasible) return CB_OK;
  res->cost_ms = fx_to_double(tot);
  bool no_regret = reg.w[0] == ~0ull && reg.w[1] == ~0ull && reg.w[2] == ~0ull;
  res->window_safe = (no_regret || rounding_window_safe(tot, reg)) ? 1 : 0;

  // Extract the kernels top-down along the post-dominator tree (host; O(n)).
  std::vector<int32_t> hchoice;
  CB_CUDA_TRY(choice.download(hchoice));
  std::vector<int32_t> owner(n, -1);
  auto member = [&](int32_t k, int32_t u) {
    auto b = m->members.begin() + m->mem_ptr[k];
    auto e = m->members.begin() + m->mem_ptr[k + 1];
    return std::binary_search(b, e, u);
  };
  std::vector<uint8_t> is_root(n, 0);
  for (int32_t i = n - 1; i >= 0; --i) {
    const int32_t v = g->level_nodes[i];
    const int32_t p = g->ipdom[v];
    if (p >= 0 && owner[p] >= 0 && member(owner[p], v)) {
      owner[v] = owner[p];
    } else {
      owner[v] = hchoice[v];
      is_root[v] = 1;
      if (owner[v] < 0) {
        cb_set_error("internal: infeasible root inside a feasible solution");
        return CB_ERR_STATE;
      }
    }
  }
  int32_t k = 0;
  for (int32_t i = 0; i < n; ++i) {
    const int32_t v = g->level_nodes[i];
    if (is_root[v]) {
      if (kernel_match) kernel_match[k] = owner[v];
      ++k;
    }
  }
  res->n_kernels = k;
  return CB_OK;
}
