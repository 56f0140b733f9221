// Backend pattern matcher: every (anchor node, candidate pattern) pair.
//
// Semantics follow tensorplace/matching.py:53-103 (match_at): the pattern
// root binds the anchor, pattern argument i descends to the producer of the
// bound node's i-th input, wildcards bind edges only, a zero-argument op
// pattern accepts any arity, two positions may bind one node only when their
// sub-patterns are structurally equal, and every non-root bound node must be
// neither a graph output nor consumed outside the match.  Candidate patterns
// per anchor are the registry's root index in registration order
// (tensorplace/registry.py:135-145).
//
// Device layout: one warp per anchor (group), one lane per candidate
// pattern.  Pass 1 decides every pair and counts members; warp ballots give
// the per-anchor match count; device-wide exclusive scans (CUB) turn the
// per-pair sizes into output offsets; pass 2 re-walks the matching pairs and
// writes the compacted, deterministic CSR (group -> matches in candidate
// order).  The anchor's input row is staged in shared memory because every
// lane's first descent reads it.
#include <cub/cub.cuh>

#include <algorithm>

#include "cb_internal.cuh"

#define CB_MAXPOS 128
#define MATCH_WARPS 8
#define STAGE_IN 32

extern "C" int cb_patterns_create(int32_t n_pat, int32_t n_kinds, const int32_t* pat_pos_ptr,
                                  const int32_t* pos_kind, const int32_t* pos_nargs,
                                  const int32_t* pos_parent, const int32_t* pos_argidx,
                                  const int32_t* pos_sid, const int32_t* pos_con_ptr,
                                  const int32_t* con_key, const int8_t* con_op,
                                  const int32_t* con_val_ptr, const int8_t* val_tag,
                                  const int64_t* val_ival, const double* val_fval,
                                  const int64_t* con_lo, const int64_t* con_hi,
                                  const int32_t* pat_backend, const int32_t* kind_pat_ptr,
                                  const int32_t* kind_pat, cb_patterns** out) {
  CB_ARG_CHECK(out && n_pat >= 0 && n_kinds >= 0, "cb_patterns_create: bad arguments");
  cb_patterns* p = new cb_patterns();
  p->n_pat = n_pat;
  p->n_kinds = n_kinds;
  p->pat_pos_ptr.assign(pat_pos_ptr, pat_pos_ptr + n_pat + 1);
  int32_t n_pos = p->pat_pos_ptr[n_pat];
  p->n_pos = n_pos;
  for (int32_t i = 0; i < n_pat; ++i) {
    int32_t sz = p->pat_pos_ptr[i + 1] - p->pat_pos_ptr[i];
    p->max_pos = std::max(p->max_pos, sz);
    if (sz < 1) {
      delete p;
      cb_set_error("cb_patterns_create: pattern without an op root");
      return CB_ERR_ARG;
    }
  }
  if (p->max_pos > CB_MAXPOS) {
    delete p;
    cb_set_error("pattern has more than 128 op positions (device matcher limit)");
    return CB_ERR_LIMIT;
  }
  p->pos_kind.assign(pos_kind, pos_kind + n_pos);
  p->pos_nargs.assign(pos_nargs, pos_nargs + n_pos);
  p->pos_parent.assign(pos_parent, pos_parent + n_pos);
  p->pos_argidx.assign(pos_argidx, pos_argidx + n_pos);
  p->pos_sid.assign(pos_sid, pos_sid + n_pos);
  p->pos_con_ptr.assign(pos_con_ptr, pos_con_ptr + n_pos + 1);
  int32_t n_con = n_pos ? p->pos_con_ptr[n_pos] : 0;
  if (n_pos == 0) p->pos_con_ptr.assign(1, 0);
  p->con_key.assign(con_key, con_key + n_con);
  p->con_op.assign(con_op, con_op + n_con);
  p->con_val_ptr.assign(con_val_ptr, con_val_ptr + n_con + 1);
  int32_t n_val = p->con_val_ptr[n_con];
  p->val_tag.assign(val_tag, val_tag + n_val);
  p->val_ival.assign(val_ival, val_ival + n_val);
  p->val_fval.assign(val_fval, val_fval + n_val);
  p->con_lo.assign(con_lo, con_lo + n_con);
  p->con_hi.assign(con_hi, con_hi + n_con);
  p->pat_backend.assign(pat_backend, pat_backend + n_pat);
  p->kind_pat_ptr.assign(kind_pat_ptr, kind_pat_ptr + n_kinds + 1);
  if (n_kinds == 0) p->kind_pat_ptr.assign(1, 0);
  p->kind_pat.assign(kind_pat, kind_pat + p->kind_pat_ptr[n_kinds]);
  *out = p;
  return CB_OK;
}

extern "C" void cb_patterns_destroy(cb_patterns* p) { delete p; }

static int patterns_to_device(cb_patterns* p) {
  if (p->on_device) return CB_OK;
  CB_CUDA_TRY(p->d_pat_pos_ptr.upload(p->pat_pos_ptr));
  CB_CUDA_TRY(p->d_pos_kind.upload(p->pos_kind));
  CB_CUDA_TRY(p->d_pos_nargs.upload(p->pos_nargs));
  CB_CUDA_TRY(p->d_pos_parent.upload(p->pos_parent));
  CB_CUDA_TRY(p->d_pos_argidx.upload(p->pos_argidx));
  CB_CUDA_TRY(p->d_pos_sid.upload(p->pos_sid));
  CB_CUDA_TRY(p->d_pos_con_ptr.upload(p->pos_con_ptr));
  CB_CUDA_TRY(p->d_con_key.upload(p->con_key));
  CB_CUDA_TRY(p->d_con_op.upload(p->con_op));
  CB_CUDA_TRY(p->d_con_val_ptr.upload(p->con_val_ptr));
  CB_CUDA_TRY(p->d_val_tag.upload(p->val_tag));
  CB_CUDA_TRY(p->d_val_ival.upload(p->val_ival));
  CB_CUDA_TRY(p->d_val_fval.upload(p->val_fval));
  CB_CUDA_TRY(p->d_con_lo.upload(p->con_lo));
  CB_CUDA_TRY(p->d_con_hi.upload(p->con_hi));
  CB_CUDA_TRY(p->d_pat_backend.upload(p->pat_backend));
  p->on_device = true;
  return CB_OK;
}

// ------------------------------------------------------------- device side
struct MatchArgs {
  // graph
  const int32_t* kind;
  const int32_t* in_ptr;
  const int32_t* in_src;
  const int32_t* out_ptr;
  const int32_t* out_dst;
  const uint8_t* is_output;
  const int32_t* attr_ptr;
  const int32_t* attr_key;
  const int8_t* attr_tag;
  const int64_t* attr_ival;
  const double* attr_fval;
  // patterns
  const int32_t* pat_pos_ptr;
  const int32_t* pos_kind;
  const int32_t* pos_nargs;
  const int32_t* pos_parent;
  const int32_t* pos_argidx;
  const int32_t* pos_sid;
  const int32_t* pos_con_ptr;
  const int32_t* con_key;
  const int8_t* con_op;
  const int32_t* con_val_ptr;
  const int8_t* val_tag;
  const int64_t* val_ival;
  const double* val_fval;
  const int64_t* con_lo;
  const int64_t* con_hi;
  const int32_t* pat_backend;
  // groups
  int64_t n_groups;
  const int32_t* group_anchor;
  const int32_t* cand_ptr;  // n_groups+1
  const int32_t* cand_pat;
};

__device__ __forceinline__ bool int_like(int8_t t) { return t == TAG_INT || t == TAG_BOOL; }

// Python `==` between an attribute value and a pattern literal.
__device__ __forceinline__ bool py_equal(int8_t ta, int64_t ia, double fa, int8_t tb, int64_t ib,
                                         double fb) {
  if (ta == TAG_STR || tb == TAG_STR) return ta == tb && ia == ib;
  if (ta == TAG_OTHER || tb == TAG_OTHER) return false;
  if (int_like(ta) && int_like(tb)) return ia == ib;
  if (ta == TAG_FLOAT && tb == TAG_FLOAT) return fa == fb;
  // int vs float: exact comparison (Python compares the mathematical values)
  double f = int_like(ta) ? fb : fa;
  int64_t i = int_like(ta) ? ia : ib;
  if (!(f == f)) return false;
  if (f != floor(f)) return false;
  if (f < -9223372036854775808.0 || f >= 9223372036854775808.0) return false;
  return (int64_t)f == i;
}

__device__ bool constraints_hold(const MatchArgs& a, int32_t P, int32_t node) {
  const int32_t c0 = a.pos_con_ptr[P], c1 = a.pos_con_ptr[P + 1];
  if (c0 == c1) return true;
  const int32_t a0 = a.attr_ptr[node], a1 = a.attr_ptr[node + 1];
  for (int32_t c = c0; c < c1; ++c) {
    const int32_t key = a.con_key[c];
    int32_t slot = -1;
    for (int32_t j = a0; j < a1; ++j)
      if (a.attr_key[j] == key) {
        slot = j;
        break;
      }
    if (slot < 0) return false;
    const int8_t tag = a.attr_tag[slot];
    const int64_t iv = a.attr_ival[slot];
    const double fv = a.attr_fval[slot];
    const int8_t op = a.con_op[c];
    if (op == CON_RANGE) {
      if (tag != TAG_INT) return false;
      if (iv < a.con_lo[c] || iv > a.con_hi[c]) return false;
      continue;
    }
    bool any = false;
    for (int32_t v = a.con_val_ptr[c]; v < a.con_val_ptr[c + 1] && !any; ++v)
      any = py_equal(tag, iv, fv, a.val_tag[v], a.val_ival[v], a.val_fval[v]);
    if (!any) return false;
  }
  return true;
}

// Walk pattern `p` anchored at `root`.  On success fills bind[0..npos) and
// members[0..nmem) (sorted, unique) and returns true.
__device__ bool match_walk(const MatchArgs& a, int32_t root, int32_t p, int32_t* bind,
                           int32_t* members, int32_t& npos, int32_t& nmem,
                           const int32_t* s_row, int32_t s_deg) {
  const int32_t base = a.pat_pos_ptr[p];
  npos = a.pat_pos_ptr[p + 1] - base;
  nmem = 0;
  for (int32_t i = 0; i < npos; ++i) {
    const int32_t P = base + i;
    int32_t node;
    if (i == 0) {
      node = root;
    } else {
      const int32_t pp = a.pos_parent[P];
      const int32_t slot = a.pos_argidx[P];
      if (pp == 0 && slot < s_deg) {
        node = s_row[slot];  // the anchor's input row, staged by the warp
      } else {
        const int32_t par = bind[pp];
        node = __ldg(a.in_src + a.in_ptr[par] + slot);
      }
      if (node < 0) return false;  // graph input where an op is required
    }
    if (__ldg(a.kind + node) != a.pos_kind[P]) return false;
    const int32_t nargs = a.pos_nargs[P];
    if (nargs && nargs != a.in_ptr[node + 1] - a.in_ptr[node]) return false;
    if (!constraints_hold(a, P, node)) return false;
    const int32_t sid = a.pos_sid[P];
    for (int32_t q = 0; q < i; ++q)
      if (bind[q] == node && a.pos_sid[base + q] != sid) return false;
    bind[i] = node;
  }
  // sorted unique member list (insertion sort; patterns are small)
  for (int32_t i = 0; i < npos; ++i) {
    const int32_t v = bind[i];
    int32_t j = nmem;
    bool dup = false;
    while (j > 0 && members[j - 1] >= v) {
      if (members[j - 1] == v) {
        dup = true;
        break;
      }
      --j;
    }
    if (dup) continue;
    for (int32_t k = nmem; k > j; --k) members[k] = members[k - 1];
    members[j] = v;
    ++nmem;
  }
  // single exit: only the root's value may leave the match
  for (int32_t i = 0; i < nmem; ++i) {
    const int32_t u = members[i];
    if (u == root) continue;
    if (a.is_output[u]) return false;
    for (int32_t j = a.out_ptr[u]; j < a.out_ptr[u + 1]; ++j) {
      const int32_t c = __ldg(a.out_dst + j);
      int32_t lo = 0, hi = nmem;
      while (lo < hi) {
        int32_t mid = (lo + hi) >> 1;
        if (members[mid] < c) lo = mid + 1;
        else hi = mid;
      }
      if (lo >= nmem || members[lo] != c) return false;
    }
  }
  return true;
}

// Pass 1: decide every pair.  One warp per group (anchor).
__global__ void __launch_bounds__(MATCH_WARPS * 32)
match_count_kernel(MatchArgs a, uint8_t* pair_ok, int32_t* pair_mem, int32_t* pair_bind,
                   int32_t* group_cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * MATCH_WARPS + (threadIdx.x >> 5);
  if (g >= a.n_groups) return;
  const int32_t root = a.group_anchor[g];
  const int32_t c0 = a.cand_ptr[g], c1 = a.cand_ptr[g + 1];
  __shared__ int32_t s_in[MATCH_WARPS][STAGE_IN];
  int32_t* s_row = s_in[threadIdx.x >> 5];
  const int32_t s_deg = min(a.in_ptr[root + 1] - a.in_ptr[root], STAGE_IN);
  if (lane < s_deg) s_row[lane] = a.in_src[a.in_ptr[root] + lane];
  __syncwarp();
  int32_t bind[CB_MAXPOS];
  int32_t members[CB_MAXPOS];
  int32_t count = 0;
  for (int32_t base = c0; base < c1; base += 32) {
    const int32_t c = base + lane;
    bool ok = false;
    int32_t npos = 0, nmem = 0;
    if (c < c1) {
      ok = match_walk(a, root, a.cand_pat[c], bind, members, npos, nmem, s_row, s_deg);
      pair_ok[c] = ok ? 1 : 0;
      pair_mem[c] = ok ? nmem : 0;
      pair_bind[c] = ok ? npos : 0;
    }
    const unsigned mask = __ballot_sync(0xffffffffu, ok);
    count += __popc(mask);
  }
  if (lane == 0) group_cnt[g] = count;
}

// Pass 2: write the compacted CSR.
__global__ void __launch_bounds__(MATCH_WARPS * 32)
match_fill_kernel(MatchArgs a, const uint8_t* pair_ok, const int32_t* mem_off,
                  const int32_t* bind_off, const int32_t* group_ptr, int32_t* out_pat,
                  int32_t* out_root, int32_t* out_backend, int32_t* out_mem_ptr,
                  int32_t* out_members, int32_t* out_bind_ptr, int32_t* out_binds) {
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * MATCH_WARPS + (threadIdx.x >> 5);
  if (g >= a.n_groups) return;
  const int32_t root = a.group_anchor[g];
  const int32_t c0 = a.cand_ptr[g], c1 = a.cand_ptr[g + 1];
  __shared__ int32_t s_in[MATCH_WARPS][STAGE_IN];
  int32_t* s_row = s_in[threadIdx.x >> 5];
  const int32_t s_deg = min(a.in_ptr[root + 1] - a.in_ptr[root], STAGE_IN);
  if (lane < s_deg) s_row[lane] = a.in_src[a.in_ptr[root] + lane];
  __syncwarp();
  int32_t bind[CB_MAXPOS];
  int32_t members[CB_MAXPOS];
  int32_t rank_base = group_ptr[g];
  for (int32_t base = c0; base < c1; base += 32) {
    const int32_t c = base + lane;
    const bool ok = c < c1 && pair_ok[c];
    const unsigned mask = __ballot_sync(0xffffffffu, ok);
    if (ok) {
      int32_t npos, nmem;
      const int32_t p = a.cand_pat[c];
      match_walk(a, root, p, bind, members, npos, nmem, s_row, s_deg);
      const int32_t m = rank_base + __popc(mask & ((1u << lane) - 1u));
      out_pat[m] = p;
      out_root[m] = root;
      out_backend[m] = a.pat_backend[p];
      const int32_t mo = mem_off[c], bo = bind_off[c];
      out_mem_ptr[m] = mo;
      out_bind_ptr[m] = bo;
      for (int32_t i = 0; i < nmem; ++i) out_members[mo + i] = members[i];
      for (int32_t i = 0; i < npos; ++i) out_binds[bo + i] = bind[i];
    }
    rank_base += __popc(mask);
  }
}

__global__ void finish_ptrs_kernel(int32_t* mem_ptr, int32_t* bind_ptr, int64_t n_matches,
                                   int32_t n_members, int32_t n_binds) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    mem_ptr[n_matches] = n_members;
    bind_ptr[n_matches] = n_binds;
  }
}

template <typename T>
static cudaError_t exclusive_scan(const T* in, T* out, int64_t n, DBuf<uint8_t>& tmp) {
  size_t bytes = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, (int)n);
  if (e != cudaSuccess) return e;
  if (tmp.n < bytes) {
    e = tmp.alloc(bytes);
    if (e != cudaSuccess) return e;
  }
  return cub::DeviceScan::ExclusiveSum(tmp.p, bytes, in, out, (int)n);
}

__global__ void widen_u8(const uint8_t* in, int32_t* out, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}

static int run_match(cb_graph* g, cb_patterns* p, const std::vector<int32_t>& anchors,
                     const std::vector<int32_t>& cand_ptr, const std::vector<int32_t>& cand_pat,
                     bool by_root, cb_matches** out) {
  int rc = cb_graph_ensure_device(g);
  if (rc != CB_OK) return rc;
  rc = patterns_to_device(p);
  if (rc != CB_OK) return rc;
  const int64_t n_groups = (int64_t)anchors.size();
  const int64_t n_pairs = cand_pat.size();
  DBuf<int32_t> d_anchor, d_cand_ptr, d_cand_pat;
  CB_CUDA_TRY(d_anchor.upload(anchors));
  CB_CUDA_TRY(d_cand_ptr.upload(cand_ptr));
  CB_CUDA_TRY(d_cand_pat.upload(cand_pat));

  MatchArgs a;
  a.kind = g->d_kind.p;
  a.in_ptr = g->d_in_ptr.p;
  a.in_src = g->d_in_src.p;
  a.out_ptr = g->d_out_ptr.p;
  a.out_dst = g->d_out_dst.p;
  a.is_output = g->d_is_output.p;
  a.attr_ptr = g->d_attr_ptr.p;
  a.attr_key = g->d_attr_key.p;
  a.attr_tag = g->d_attr_tag.p;
  a.attr_ival = g->d_attr_ival.p;
  a.attr_fval = g->d_attr_fval.p;
  a.pat_pos_ptr = p->d_pat_pos_ptr.p;
  a.pos_kind = p->d_pos_kind.p;
  a.pos_nargs = p->d_pos_nargs.p;
  a.pos_parent = p->d_pos_parent.p;
  a.pos_argidx = p->d_pos_argidx.p;
  a.pos_sid = p->d_pos_sid.p;
  a.pos_con_ptr = p->d_pos_con_ptr.p;
  a.con_key = p->d_con_key.p;
  a.con_op = p->d_con_op.p;
  a.con_val_ptr = p->d_con_val_ptr.p;
  a.val_tag = p->d_val_tag.p;
  a.val_ival = p->d_val_ival.p;
  a.val_fval = p->d_val_fval.p;
  a.con_lo = p->d_con_lo.p;
  a.con_hi = p->d_con_hi.p;
  a.pat_backend = p->d_pat_backend.p;
  a.n_groups = n_groups;
  a.group_anchor = d_anchor.p;
  a.cand_ptr = d_cand_ptr.p;
  a.cand_pat = d_cand_pat.p;

  cb_matches* m = new cb_matches();
  m->by_root = by_root;
  m->n_groups = n_groups;
  DBuf<uint8_t> ok, tmp;
  DBuf<int32_t> okw, pmem, pbind, mem_off, bind_off, gcnt, pair_idx;
  auto fail = [&](cudaError_t e) {
    delete m;
    cb_set_error(std::string("CUDA error in matcher: ") + cudaGetErrorString(e));
    return CB_ERR_CUDA;
  };
  cudaError_t e;
  if ((e = ok.alloc(n_pairs + 1)) != cudaSuccess) return fail(e);
  if ((e = pmem.alloc(n_pairs + 1)) != cudaSuccess) return fail(e);
  if ((e = pbind.alloc(n_pairs + 1)) != cudaSuccess) return fail(e);
  if ((e = mem_off.alloc(n_pairs + 1)) != cudaSuccess) return fail(e);
  if ((e = bind_off.alloc(n_pairs + 1)) != cudaSuccess) return fail(e);
  if ((e = gcnt.alloc(n_groups + 1)) != cudaSuccess) return fail(e);
  if ((e = m->d_group_ptr.alloc(n_groups + 1)) != cudaSuccess) return fail(e);
  cudaMemset(pmem.p, 0, (n_pairs + 1) * sizeof(int32_t));
  cudaMemset(pbind.p, 0, (n_pairs + 1) * sizeof(int32_t));
  cudaMemset(gcnt.p, 0, (n_groups + 1) * sizeof(int32_t));
  const int64_t blocks = (n_groups + MATCH_WARPS - 1) / MATCH_WARPS;
  if (blocks > 0) {
    match_count_kernel<<<(unsigned)blocks, MATCH_WARPS * 32>>>(a, ok.p, pmem.p, pbind.p, gcnt.p);
    if ((e = cudaGetLastError()) != cudaSuccess) return fail(e);
  }
  if ((e = exclusive_scan(gcnt.p, m->d_group_ptr.p, n_groups + 1, tmp)) != cudaSuccess) return fail(e);
  if ((e = exclusive_scan(pmem.p, mem_off.p, n_pairs + 1, tmp)) != cudaSuccess) return fail(e);
  if ((e = exclusive_scan(pbind.p, bind_off.p, n_pairs + 1, tmp)) != cudaSuccess) return fail(e);
  int32_t n_matches = 0, n_members = 0, n_binds = 0;
  cudaMemcpy(&n_matches, m->d_group_ptr.p + n_groups, sizeof(int32_t), cudaMemcpyDeviceToHost);
  cudaMemcpy(&n_members, mem_off.p + n_pairs, sizeof(int32_t), cudaMemcpyDeviceToHost);
  if ((e = cudaMemcpy(&n_binds, bind_off.p + n_pairs, sizeof(int32_t), cudaMemcpyDeviceToHost)) !=
      cudaSuccess)
    return fail(e);
  m->n_matches = n_matches;
  m->n_members = n_members;
  m->n_binds = n_binds;
  if ((e = m->d_pat.alloc(n_matches + 1)) != cudaSuccess) return fail(e);
  if ((e = m->d_root.alloc(n_matches + 1)) != cudaSuccess) return fail(e);
  if ((e = m->d_backend.alloc(n_matches + 1)) != cudaSuccess) return fail(e);
  if ((e = m->d_mem_ptr.alloc(n_matches + 1)) != cudaSuccess) return fail(e);
  if ((e = m->d_bind_ptr.alloc(n_matches + 1)) != cudaSuccess) return fail(e);
  if ((e = m->d_members.alloc(n_members + 1)) != cudaSuccess) return fail(e);
  if ((e = m->d_binds.alloc(n_binds + 1)) != cudaSuccess) return fail(e);
  if ((e = m->d_cost.alloc(n_matches + 1)) != cudaSuccess) return fail(e);
  if (blocks > 0) {
    match_fill_kernel<<<(unsigned)blocks, MATCH_WARPS * 32>>>(
        a, ok.p, mem_off.p, bind_off.p, m->d_group_ptr.p, m->d_pat.p, m->d_root.p,
        m->d_backend.p, m->d_mem_ptr.p, m->d_members.p, m->d_bind_ptr.p, m->d_binds.p);
    if ((e = cudaGetLastError()) != cudaSuccess) return fail(e);
  }
  finish_ptrs_kernel<<<1, 1>>>(m->d_mem_ptr.p, m->d_bind_ptr.p, n_matches, n_members, n_binds);
  if ((e = cudaDeviceSynchronize()) != cudaSuccess) return fail(e);
  *out = m;
  return CB_OK;
}

extern "C" int cb_match_all(cb_graph* g, cb_patterns* p, cb_matches** out) {
  CB_ARG_CHECK(g && p && out, "cb_match_all: null argument");
  const int32_t n = g->n;
  std::vector<int32_t> anchors(n), cand_ptr(n + 1, 0), cand_pat;
  for (int32_t v = 0; v < n; ++v) {
    anchors[v] = v;
    const int32_t k = g->kind[v];
    if (k >= 0 && k < p->n_kinds)
      for (int32_t j = p->kind_pat_ptr[k]; j < p->kind_pat_ptr[k + 1]; ++j)
        cand_pat.push_back(p->kind_pat[j]);
    cand_ptr[v + 1] = (int32_t)cand_pat.size();
  }
  return run_match(g, p, anchors, cand_ptr, cand_pat, true, out);
}

extern "C" int cb_match_pairs(cb_graph* g, cb_patterns* p, int32_t n_pairs, const int32_t* roots,
                              const int32_t* pats, cb_matches** out) {
  CB_ARG_CHECK(g && p && out && n_pairs >= 0, "cb_match_pairs: bad arguments");
  std::vector<int32_t> anchors(roots, roots + n_pairs), cand_ptr(n_pairs + 1), cand_pat(pats, pats + n_pairs);
  for (int32_t i = 0; i <= n_pairs; ++i) cand_ptr[i] = i;
  for (int32_t i = 0; i < n_pairs; ++i) {
    CB_ARG_CHECK(anchors[i] >= 0 && anchors[i] < g->n, "cb_match_pairs: root out of range");
    CB_ARG_CHECK(cand_pat[i] >= 0 && cand_pat[i] < p->n_pat, "cb_match_pairs: pattern out of range");
  }
  return run_match(g, p, anchors, cand_ptr, cand_pat, false, out);
}

extern "C" int cb_matches_counts(const cb_matches* m, int64_t* n_groups, int64_t* n_matches,
                                 int64_t* n_members, int64_t* n_binds) {
  CB_ARG_CHECK(m, "cb_matches_counts: null matches");
  if (n_groups) *n_groups = m->n_groups;
  if (n_matches) *n_matches = m->n_matches;
  if (n_members) *n_members = m->n_members;
  if (n_binds) *n_binds = m->n_binds;
  return CB_OK;
}

int cb_matches_ensure_host(cb_matches* m) {
  if (m->host_valid) return CB_OK;
  std::vector<int32_t> tmp;
  CB_CUDA_TRY(m->d_group_ptr.download(m->group_ptr));
  CB_CUDA_TRY(m->d_pat.download(tmp));
  m->pat.assign(tmp.begin(), tmp.begin() + m->n_matches);
  CB_CUDA_TRY(m->d_root.download(tmp));
  m->root.assign(tmp.begin(), tmp.begin() + m->n_matches);
  CB_CUDA_TRY(m->d_backend.download(tmp));
  m->backend.assign(tmp.begin(), tmp.begin() + m->n_matches);
  CB_CUDA_TRY(m->d_mem_ptr.download(m->mem_ptr));
  CB_CUDA_TRY(m->d_bind_ptr.download(m->bind_ptr));
  CB_CUDA_TRY(m->d_members.download(tmp));
  m->members.assign(tmp.begin(), tmp.begin() + m->n_members);
  CB_CUDA_TRY(m->d_binds.download(tmp));
  m->binds.assign(tmp.begin(), tmp.begin() + m->n_binds);
  m->host_valid = true;
  return CB_OK;
}

extern "C" int cb_matches_download(cb_matches* m, int32_t* group_ptr, int32_t* pat, int32_t* root,
                                   int32_t* mem_ptr, int32_t* members, int32_t* bind_ptr,
                                   int32_t* binds) {
  CB_ARG_CHECK(m, "cb_matches_download: null matches");
  int rc = cb_matches_ensure_host(m);
  if (rc != CB_OK) return rc;
  auto cp = [](int32_t* dst, const std::vector<int32_t>& src, size_t count) {
    if (dst && count) std::copy(src.begin(), src.begin() + count, dst);
  };
  cp(group_ptr, m->group_ptr, (size_t)m->n_groups + 1);
  cp(pat, m->pat, (size_t)m->n_matches);
  cp(root, m->root, (size_t)m->n_matches);
  cp(mem_ptr, m->mem_ptr, (size_t)m->n_matches + 1);
  cp(members, m->members, (size_t)m->n_members);
  cp(bind_ptr, m->bind_ptr, (size_t)m->n_matches + 1);
  cp(binds, m->binds, (size_t)m->n_binds);
  return CB_OK;
}

extern "C" void cb_matches_destroy(cb_matches* m) { delete m; }
