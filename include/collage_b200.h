/*
 * collage_b200.h -- C ABI of the B200-native placement-search hot path.
 *
 * The reference (tensorplace, pure Python) has no foreign-function boundary;
 * the entry points below are the calls its hot path would bind if it had
 * one.  Each block names the reference function it replaces:
 *
 *   cb_graph_*        tensorplace/graph.py:71-345   ComputationGraph structure
 *                     (topo order :156-175, depths :177-182, post-dominators :224-255)
 *   cb_match_*        tensorplace/matching.py:53-115 match_at / match_all and
 *                     tensorplace/registry.py:135-145 candidates_at
 *   cb_matches_price  tensorplace/cost.py:121-138, :248-263 SimProfile.kernel_cost
 *                     via SimMeasurer.measure_kernel
 *   cb_dp_solve       tensorplace/dp.py:71-179        optimize (Algorithm 1)
 *   cb_es_plan_* /
 *   cb_fitness_*      tensorplace/evolution.py:65-119 decode + fitness, i.e.
 *                     tensorplace/cost.py:320-373 placement_cost_graphlevel
 *   cb_es_breed       tensorplace/evolution.py:205-223 selection / crossover /
 *                     mutation (device variant, counter-based RNG)
 *   cb_es_generation  tensorplace/evolution.py:233-249 one generation (breed +
 *                     evaluate), optionally as one fused kernel
 *   cb_argmin*        tensorplace/evolution.py:226-231, :245-247 best tracking
 *   cb_es_plan_units / _kernel / _set_path / _set_pool: diagnostics and tuning
 *                     knobs of this implementation (no reference counterpart)
 *
 * Conventions: plain pointers and sizes only; arrays marked "host" live in
 * host memory, "device" arrays are CUDA device pointers; `stream` is a
 * cudaStream_t passed as void* (NULL = legacy default stream).  Every call
 * returns CB_OK or an error code; cb_last_error() describes the last failure
 * of the calling thread.  There is no CPU execution path for the search:
 * calls that need a GPU fail with CB_ERR_CUDA when none is present.
 */
#ifndef COLLAGE_B200_H
#define COLLAGE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  CB_OK = 0,
  CB_ERR_CUDA = 1,     /* CUDA runtime failure or no usable device */
  CB_ERR_ARG = 2,      /* malformed arguments */
  CB_ERR_PROFILE = 3,  /* a match cannot be priced (see err array) */
  CB_ERR_INEXACT = 4,  /* a cost falls outside the exact fixed-point range */
  CB_ERR_CYCLE = 5,    /* graph is not a DAG */
  CB_ERR_LIMIT = 6,    /* a compiled-in capacity was exceeded */
  CB_ERR_STATE = 7     /* call out of order (e.g. costs not set) */
};

const char* cb_last_error(void);
int cb_abi_version(void);
/* 1 when a CUDA device is visible and usable, 0 otherwise (never fails). */
int cb_device_available(void);

/* Exactly rounded sum of n doubles (math.fsum semantics) -- exposed so the
 * host can check the accumulator; *exact=0 if an input left the range. */
int cb_fx_sum(const double* xs, int64_t n, double* out, int32_t* exact);

/* ------------------------------------------------------------------ graph */
typedef struct cb_graph cb_graph;

/* Nodes are indexed 0..n-1 in ascending node-id order.  in_src[j] is the
 * producing node index of input slot j or -1 for a graph-input reference.
 * Attributes: per node a CSR slice (attr_ptr) of (key id, tag, ival, fval)
 * with tag 0=int 1=float 2=string(id in ival) 3=bool(0/1 in ival) 4=other.
 * volume[i] = float(prod(output_shape)).  All arrays are host arrays and are
 * copied. */
int cb_graph_create(int32_t n, const int32_t* kind, const int32_t* in_ptr,
                    const int32_t* in_src, const uint8_t* is_output,
                    const double* volume, const int32_t* attr_ptr,
                    const int32_t* attr_key, const int8_t* attr_tag,
                    const int64_t* attr_ival, const double* attr_fval,
                    cb_graph** out);
void cb_graph_destroy(cb_graph* g);

/* Structural analysis (host only, no GPU needed).  topo: deterministic
 * topological order (ties by smallest index); depth: longest path from any
 * graph input; ipdom: immediate post-dominator w.r.t. a virtual sink joining
 * all outputs, -1 when only the sink post-dominates; pd_tin/pd_tout: Euler
 * interval of the post-dominator tree (d post-dominates v iff
 * tin[d] <= tin[v] && tout[v] <= tout[d]).  On a cycle returns CB_ERR_CYCLE
 * and stores the smallest stuck node index in *cycle_node. */
int cb_graph_analysis(cb_graph* g, int32_t* topo, int32_t* depth,
                      int32_t* ipdom, int32_t* pd_tin, int32_t* pd_tout,
                      int32_t* cycle_node);

/* --------------------------------------------------------------- patterns */
typedef struct cb_patterns cb_patterns;

/* Pattern trees flattened in pre-order, one record per op position
 * (wildcards carry no position; they only count towards nargs).
 *   pos_kind    op-kind id            pos_nargs  0 = any arity, else exact
 *   pos_parent  parent position (-1 for the root)
 *   pos_argidx  argument slot in the parent
 *   pos_sid     structural id of the sub-pattern rooted here (two positions
 *               may bind one node only if their sids are equal)
 * Constraints per position (pos_con_ptr): key id, op (0 Equals, 1 OneOf,
 * 2 IntRange), literal slice (con_val_ptr into val_tag/val_ival/val_fval;
 * tags as for graph attributes) and con_lo/con_hi for ranges.
 * kind_pat_ptr/kind_pat: for every op kind the patterns rooted at it in
 * registration order (the registry's root index). */
int cb_patterns_create(int32_t n_pat, int32_t n_kinds,
                       const int32_t* pat_pos_ptr, const int32_t* pos_kind,
                       const int32_t* pos_nargs, const int32_t* pos_parent,
                       const int32_t* pos_argidx, const int32_t* pos_sid,
                       const int32_t* pos_con_ptr, const int32_t* con_key,
                       const int8_t* con_op, const int32_t* con_val_ptr,
                       const int8_t* val_tag, const int64_t* val_ival,
                       const double* val_fval, const int64_t* con_lo,
                       const int64_t* con_hi, const int32_t* pat_backend,
                       const int32_t* kind_pat_ptr, const int32_t* kind_pat,
                       cb_patterns** out);
void cb_patterns_destroy(cb_patterns* p);

/* ---------------------------------------------------------------- matches */
typedef struct cb_matches cb_matches;

/* Every (anchor node, candidate pattern) pair, i.e. candidates_at for all
 * nodes.  Matches are grouped by root (group = root index), in registration
 * order inside a group. */
int cb_match_all(cb_graph* g, cb_patterns* p, cb_matches** out);
/* Explicit (root, pattern) pairs; group = pair index, 0 or 1 match each. */
int cb_match_pairs(cb_graph* g, cb_patterns* p, int32_t n_pairs,
                   const int32_t* roots, const int32_t* pats,
                   cb_matches** out);
int cb_matches_counts(const cb_matches* m, int64_t* n_groups,
                      int64_t* n_matches, int64_t* n_members,
                      int64_t* n_binds);
/* Host outputs: group_ptr[n_groups+1]; per match pat, root, mem_ptr
 * (n_matches+1) into members (sorted node indices) and bind_ptr into binds
 * (bound node per op position, pre-order). */
int cb_matches_download(cb_matches* m, int32_t* group_ptr, int32_t* pat,
                        int32_t* root, int32_t* mem_ptr, int32_t* members,
                        int32_t* bind_ptr, int32_t* binds);
void cb_matches_destroy(cb_matches* m);

/* Device pricing (SimProfile): per backend b, op kind k:
 *   coeff[b*n_kinds+k], overhead[..], has_entry[..]; has_profile[b];
 *   pw[b*pw_stride+e] = fusion_discount ** e   (computed by the host with
 *   the reference's own float pow so results are bit-identical).
 * costs_out (host, n_matches) receives every kernel cost; err_out (host,
 * n_matches) 0 ok / 1 backend without profile / 2 op without entry. */
int cb_matches_price(cb_matches* m, cb_graph* g, int32_t n_backends,
                     int32_t n_kinds, const double* coeff,
                     const double* overhead, const uint8_t* has_entry,
                     const uint8_t* has_profile, int32_t pw_stride,
                     const double* pw, double* costs_out, int8_t* err_out);
/* Host-priced costs (any Measurer), one per match. */
int cb_matches_set_costs(cb_matches* m, const double* costs);

/* --------------------------------------------------------------------- DP */
typedef struct {
  double cost_ms;           /* fsum of kernel costs + eps per kernel */
  int32_t feasible;         /* 0: no full cover exists */
  int32_t n_kernels;
  int32_t n_levels;
  int32_t n_launches;
  int64_t candidates;       /* matches examined (= relaxations) */
  int64_t ties;             /* exact-cost ties resolved by the key order */
  int64_t walk_steps;       /* nodes visited by tie walks */
  int32_t window_safe;      /* 1: no other cover rounds to the same cost */
  int32_t first_zero_candidate; /* first node in pop order without a
                                   candidate, -1 if none */
  double device_ms;         /* GPU time of the solve */
} cb_dp_result;

/* Exact op-level placement (Algorithm 1 semantics, canonical tie-break).
 * kernel_match (host, capacity n_nodes) receives the chosen match of every
 * kernel in pop order of its root. */
int cb_dp_solve(cb_graph* g, cb_matches* m, double epsilon,
                int32_t* kernel_match, cb_dp_result* res);
/* cb_dp_solve with every launch, copy and event on `stream` (cudaStream_t
 * as void*, NULL = legacy default stream); returns after the stream work. */
int cb_dp_solve_stream(cb_graph* g, cb_matches* m, double epsilon, int32_t* kernel_match,
                       cb_dp_result* res, void* stream);

/* Graph-level cost of one arbitrary placement (host code of the native
 * runtime; populations go through cb_fitness_*).  Kernels are given as node
 * index lists (kernel_ptr/kernel_nodes), a backend id and a cost each. */
int cb_placement_cost_graphlevel(cb_graph* g, int32_t n_kernels,
                                 const int32_t* kernel_ptr,
                                 const int32_t* kernel_nodes,
                                 const int32_t* kernel_backend,
                                 const double* kernel_cost, int32_t n_backends,
                                 const uint8_t* backend_is_graph,
                                 const double* region_alpha,
                                 const double* region_floor, double epsilon,
                                 double* out);

/* --------------------------------------------------------- evolutionary */
typedef struct cb_es_plan cb_es_plan;

/* kernel_match: the placement's kernels in canonical order (sorted node
 * tuples).  backend_is_graph/region_alpha/region_floor per backend id. */
int cb_es_plan_create(cb_graph* g, cb_matches* m, int32_t n_kernels,
                      const int32_t* kernel_match, int32_t n_backends,
                      const uint8_t* backend_is_graph,
                      const double* region_alpha, const double* region_floor,
                      int32_t target_backend, double epsilon,
                      cb_es_plan** out);
typedef struct {
  int32_t genome_bits;   /* eligible kernels (genome length) */
  int32_t words;         /* uint64 words per genome */
  int32_t units;         /* dynamic units (feasible eligible + fixed) */
  int32_t fixed_units;   /* contracted fixed target-backend components */
  int32_t edges;         /* dynamic adjacency edges */
  int32_t infeasible_bits;
  int32_t smem_path;     /* union-find path: 1 warp/genome in shared memory */
  int32_t frontier_slots;/* thread/genome frontier program width (0 = none) */
  double seed_cost;      /* graph-level cost of the all-zero genome */
  int32_t window_shift;  /* 128-bit window: values carried as v >> shift (-1 = none) */
  int32_t packed_labels; /* 1: frontier fits the packed-label kernels (<= 16 slots),
                            2: also the packed anchor kernel (<= 8 slots) */
  int32_t fsm_transitions; /* transitions of the finite-state program (0 = none) */
  int32_t fsm_entry_bytes; /* transition layout: 8 (also the mixed 8 / 16 layout) or 16 (+ shared delta table), or 32 */
} cb_es_plan_info;
int cb_es_plan_query(const cb_es_plan* p, cb_es_plan_info* info);
/* Evaluation path: -1 automatic (the finite-state walk when its table is
 * <= 32 MB, else the frontier program when available), 0 the union-find
 * kernels, 1 the frontier program (packed-label form when it has <= 16
 * slots), 2 the frontier program in its shared-memory-label form, 3 the
 * warp-per-genome walk, 4 the anchor walk, 5 the packed-label walk, 6 the
 * packed anchor walk, 7 the finite-state walk.  For tests and profiling; all
 * paths return identical results. */
int cb_es_plan_set_path(cb_es_plan* p, int32_t path);
/* Merged-component pool entries per genome of the anchor walk held in
 * shared memory (1..24, default min(frontier slots, 8)); entries beyond
 * live in the thread's local memory (at most F are ever held).  A tuning /
 * testing knob: results are identical for every value. */
int cb_es_plan_set_pool(cb_es_plan* p, int32_t entries);
/* Name of the fitness kernel the current path setting dispatches to
 * (static string; for reports and profiles). */
const char* cb_es_plan_kernel(const cb_es_plan* p);
/* The dynamic unit graph (diagnostics and tests; any pointer may be NULL):
 * unit_bit[units] genome bit of each unit (-1 = fixed unit), unit_cnt[units]
 * kernels each unit contributes to a region, edges[2*edges] unit pairs
 * (a < b), frontier_needed = slots the frontier program needs (may exceed
 * the kernels' cap, in which case frontier_slots is 0). */
int cb_es_plan_units(const cb_es_plan* p, int32_t* unit_bit, int32_t* unit_cnt,
                     int32_t* edges, int32_t* frontier_needed);
/* slot_kernel (host, genome_bits): canonical kernel index of each bit;
 * rep_kind (host, genome_bits): 0 infeasible, 1 same-set pattern,
 * 2 decomposed into singletons; rep_match_ptr/rep_match: replacement
 * matches per bit. */
int cb_es_plan_slots(const cb_es_plan* p, int32_t* slot_kernel,
                     int8_t* rep_kind, int32_t* rep_match_ptr,
                     int32_t* rep_match);
void cb_es_plan_destroy(cb_es_plan* p);

/* Fitness of n genomes (row stride `words` uint64, bit i of a genome is
 * bit i%64 of word i/64).  Infeasible genomes get +inf. */
int cb_fitness_device(cb_es_plan* p, const uint64_t* d_pop, int64_t n,
                      double* d_fit, void* stream);
/* Same through host buffers: H2D copy, evaluation, D2H copy. */
int cb_fitness_host(cb_es_plan* p, const uint64_t* h_pop, int64_t n,
                    double* h_fit);

/* Device breeding: children[e..n) from parents by tournament selection
 * (size `tournament`, strict-less wins), two-point crossover and per-bit
 * mutation at `mutation_rate` (geometric skipping), Philox4x32-10 keyed by
 * (seed, generation, stream_id, child).  Rows [0, n_keep) are copied from
 * `keep` (elites).  */
int cb_es_breed(cb_es_plan* p, const uint64_t* d_parents,
                const double* d_parent_fit, int64_t n_parents,
                uint64_t* d_children, int64_t n_children,
                const uint64_t* d_keep, int64_t n_keep, uint64_t seed,
                uint64_t generation, uint64_t stream_id, int32_t tournament,
                double mutation_rate, void* stream);
/* One ES generation (tensorplace/evolution.py:233-249: breed the next
 * population, evaluate it): breed n_children rows into d_children (same operators
 * and draws as cb_es_breed) and write their fitness to d_child_fit (as
 * cb_fitness_device).  Runs as a single fused kernel when the plan's walk
 * allows it (<= 8 frontier slots, 128-bit window, <= 4 words per genome),
 * else as the two launches; results are identical. */
int cb_es_generation(cb_es_plan* p, const uint64_t* d_parents,
                     const double* d_parent_fit, int64_t n_parents,
                     uint64_t* d_children, double* d_child_fit,
                     int64_t n_children, const uint64_t* d_keep, int64_t n_keep,
                     uint64_t seed, uint64_t generation, uint64_t stream_id,
                     int32_t tournament, double mutation_rate, void* stream);
/* cb_argmin plus, when d_pop is given, the best row copied to d_elite
 * (words uint64) and the best value to *d_history_slot (if not NULL):
 * the best-so-far / history bookkeeping of tensorplace/evolution.py:244-248. */
int cb_argmin_elite(const double* d_fit, int64_t n, const uint64_t* d_pop,
                    int32_t words, int64_t* d_idx, double* d_val,
                    uint64_t* d_elite, double* d_history_slot, void* stream);

/* Sharded search exchange (tensorplace/evolution.py:244-248 best tracking,
 * across ranks).  cb_elite_record: argmin of the rank's fitness and its row
 * as one record d_record[0 .. words] = [fitness bits, row].  After an
 * all-gather of the records ([world][1 + words]), cb_elite_pick writes the
 * lowest-fitness row (first rank on ties) to d_elite, its fitness to
 * *d_elite_val and, if given, to *d_history_slot. */
int cb_elite_record(const double* d_fit, int64_t n, const uint64_t* d_pop, int32_t words,
                    int64_t* d_idx, double* d_val, uint64_t* d_record, void* stream);
int cb_elite_pick(const uint64_t* d_records, int32_t world, int32_t words, uint64_t* d_elite,
                  double* d_elite_val, double* d_history_slot, void* stream);
/* 1 when cb_es_generation runs fused for this plan (and path setting). */
int cb_es_generation_fused(const cb_es_plan* p);
/* Index of the smallest fitness (first on ties) -> d_idx[0]; value ->
 * d_val[0] (tensorplace/evolution.py:226-231, :245-247 best tracking). */
int cb_argmin(const double* d_fit, int64_t n, int64_t* d_idx, double* d_val,
              void* stream);

#ifdef __cplusplus
}
#endif
#endif /* COLLAGE_B200_H */
