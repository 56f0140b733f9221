// Internal structures shared by the translation units of libcollage_b200.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/collage_b200.h"
#include "fixed192.cuh"

// ------------------------------------------------------------- error state
void cb_set_error(const std::string& msg);

// Streaming multiprocessors of the current device (148 on B200), cached.
int cb_sm_count();

#define CB_CUDA_TRY(expr)                                                  \
  do {                                                                     \
    cudaError_t _e = (expr);                                               \
    if (_e != cudaSuccess) {                                               \
      cb_set_error(std::string("CUDA error: ") + cudaGetErrorString(_e) +  \
                   " at " __FILE__ ":" + std::to_string(__LINE__));        \
      return CB_ERR_CUDA;                                                  \
    }                                                                      \
  } while (0)

#define CB_ARG_CHECK(cond, msg)   \
  do {                            \
    if (!(cond)) {                \
      cb_set_error(msg);          \
      return CB_ERR_ARG;          \
    }                             \
  } while (0)

// Device buffer that frees itself.
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  cudaError_t alloc(size_t count) {
    release();
    n = count;
    if (count == 0) return cudaSuccess;
    return cudaMalloc((void**)&p, count * sizeof(T));
  }
  cudaError_t upload(const T* h, size_t count) {
    cudaError_t e = alloc(count);
    if (e != cudaSuccess || count == 0) return e;
    return cudaMemcpy(p, h, count * sizeof(T), cudaMemcpyHostToDevice);
  }
  cudaError_t upload(const std::vector<T>& v) { return upload(v.data(), v.size()); }
  cudaError_t download(std::vector<T>& v) const {
    v.resize(n);
    if (n == 0) return cudaSuccess;
    return cudaMemcpy(v.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost);
  }
};

int cb_require_device();  // CB_OK or CB_ERR_CUDA with a message

// Attribute / literal tags (graph attrs and pattern literals share them).
enum : int8_t { TAG_INT = 0, TAG_FLOAT = 1, TAG_STR = 2, TAG_BOOL = 3, TAG_OTHER = 4 };
enum : int8_t { CON_EQ = 0, CON_ONEOF = 1, CON_RANGE = 2 };

// ------------------------------------------------------------------ graph
struct cb_graph {
  int32_t n = 0;
  // host CSR
  std::vector<int32_t> kind, in_ptr, in_src, out_ptr, out_dst;
  std::vector<uint8_t> is_output;
  std::vector<double> volume;
  std::vector<int32_t> attr_ptr, attr_key;
  std::vector<int8_t> attr_tag;
  std::vector<int64_t> attr_ival;
  std::vector<double> attr_fval;
  // analysis (valid when analysed)
  bool analysed = false;
  int32_t cycle_node = -1;
  std::vector<int32_t> topo, depth, ipdom, pd_tin, pd_tout;
  std::vector<int32_t> level_ptr, level_nodes;  // pop order: (depth, index)
  std::vector<int32_t> pch_ptr, pch;            // post-dominator tree children
  // device mirror
  bool on_device = false;
  DBuf<int32_t> d_kind, d_in_ptr, d_in_src, d_out_ptr, d_out_dst;
  DBuf<uint8_t> d_is_output;
  DBuf<double> d_volume;
  DBuf<int32_t> d_attr_ptr, d_attr_key;
  DBuf<int8_t> d_attr_tag;
  DBuf<int64_t> d_attr_ival;
  DBuf<double> d_attr_fval;
  DBuf<int32_t> d_ipdom, d_pch_ptr, d_pch, d_level_nodes, d_depth;
};

int cb_graph_ensure_analysis(cb_graph* g);
int cb_graph_ensure_device(cb_graph* g);

// --------------------------------------------------------------- patterns
struct cb_patterns {
  int32_t n_pat = 0, n_kinds = 0, n_pos = 0, max_pos = 0;
  std::vector<int32_t> pat_pos_ptr, pos_kind, pos_nargs, pos_parent, pos_argidx,
      pos_sid, pos_con_ptr, con_key, con_val_ptr, pat_backend, kind_pat_ptr,
      kind_pat;
  std::vector<int8_t> con_op, val_tag;
  std::vector<int64_t> val_ival, con_lo, con_hi;
  std::vector<double> val_fval;
  bool on_device = false;
  DBuf<int32_t> d_pat_pos_ptr, d_pos_kind, d_pos_nargs, d_pos_parent,
      d_pos_argidx, d_pos_sid, d_pos_con_ptr, d_con_key, d_con_val_ptr,
      d_pat_backend, d_kind_pat_ptr, d_kind_pat;
  DBuf<int8_t> d_con_op, d_val_tag;
  DBuf<int64_t> d_val_ival, d_con_lo, d_con_hi;
  DBuf<double> d_val_fval;
};

// ---------------------------------------------------------------- matches
struct cb_matches {
  int64_t n_groups = 0, n_matches = 0, n_members = 0, n_binds = 0;
  bool by_root = false;  // groups are node indices (match_all)
  // device
  DBuf<int32_t> d_group_ptr, d_pat, d_root, d_mem_ptr, d_members, d_bind_ptr,
      d_binds, d_backend;
  DBuf<double> d_cost;
  bool costs_set = false;
  // host mirror (filled lazily)
  bool host_valid = false;
  std::vector<int32_t> group_ptr, pat, root, mem_ptr, members, bind_ptr, binds,
      backend;
  std::vector<double> cost;
};

int cb_matches_ensure_host(cb_matches* m);

// ------------------------------------------------------------ level plan
// Consecutive pop-order levels are batched: runs of narrow levels go to one
// single-CTA launch that synchronises with __syncthreads, wide levels get a
// grid of their own.
struct LevelSegment {
  int32_t lvl_begin, lvl_end;  // [begin, end) level indices
  bool narrow;
};
std::vector<LevelSegment> cb_plan_levels(const cb_graph* g, int32_t narrow_max);

// True when `func` on the current device has not yet been given a dynamic
// shared-memory limit of at least `bytes` (and records it): the attribute
// is per device, so a process driving several GPUs sets it on each.
// Thread-safe.
bool cb_smem_claim(const void* func, size_t bytes);

