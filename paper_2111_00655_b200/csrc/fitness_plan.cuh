// Fitness plan: the host-built, genome-independent part of graph-level pricing.
#pragma once
#include <map>
#include <memory>
#include <mutex>

#include "cb_internal.cuh"

// One record per dynamic unit of the frontier program (thread-per-genome
// evaluation): the unit's costs, its genome bit, the frontier slot it
// occupies while it still has unvisited neighbours, and the slots of its
// earlier neighbours / of the units whose last neighbour it is.
struct __align__(16) UnitRec {
  fx192 rep;    // exact sum of its replacement kernels (region member value)
  fx192 off;    // its own kernel cost + eps (removed when offloaded)
  fx192 term1;  // round(rep) * r(cnt) + eps: its term as a region of one
  int32_t bit;  // genome bit, -1 for always-on fixed units
  int32_t cnt;  // kernels it contributes to a region
  int32_t back_off, end_off;
  uint8_t slot, nback, nend, pad;
  int32_t bit2;  // copy of `bit`
  // packed step header of the packed-label kernel (one 16-byte load):
  // x = bit, y = slot | nback << 8 | nend << 16, z = back slots (4 bits
  // each, <= 8), w = end slots (4 bits each, <= 8)
  uint4 hot;
};

struct cb_es_plan {
  int32_t k = 0;       // genome bits
  int32_t words = 0;   // uint64 words per genome
  int32_t M = 0;       // dynamic units
  int32_t n_virtual = 0;
  int32_t E = 0;
  int32_t infeasible_bits = 0;
  fx192 base_const;    // static regions + every eligible kernel's cost + eps
  fx192 eps;
  double seed_cost = 0.0;
  bool smem_path = true;
  // host copies
  std::vector<int32_t> slot_kernel, rep_match_ptr, rep_match;
  std::vector<int8_t> rep_kind;
  std::vector<int32_t> unit_slot;  // slot of unit u, -1 for virtual units
  std::vector<fx192> unit_rep, unit_off;
  std::vector<int32_t> unit_cnt;
  std::vector<int2> edges;
  std::vector<uint64_t> infeas_mask;
  std::vector<double> rt;  // r(n) of the target backend, n = 0..max
  // device copies
  DBuf<int32_t> d_unit_slot, d_unit_cnt;
  DBuf<fx192> d_unit_rep, d_unit_off;
  DBuf<int2> d_edges;
  DBuf<uint64_t> d_infeas;
  DBuf<double> d_rt;
  DBuf<unsigned long long> d_flags;
  DBuf<uint8_t> d_scratch;
  size_t scratch_per_group = 0;
  int32_t scratch_groups = 0;
  // staging for the host-buffer entry point
  DBuf<uint64_t> d_pop_stage;
  DBuf<double> d_fit_stage;
  // frontier program (0 slots = not built / too wide)
  int32_t F = 0;
  int32_t F_needed = 0;  // width of the program before the FRONTIER_MAX cap
  std::vector<UnitRec> prog;
  std::vector<uint8_t> prog_slots;
  std::vector<int32_t> prog_back_pos;  // position of each back-list entry's unit (-1 for end entries)
  DBuf<UnitRec> d_prog;
  DBuf<uint8_t> d_prog_slots;
  // sparse walk (fitness_wide.cu): last neighbour position of each program
  // position, program position of each genome bit (-1 infeasible), program
  // positions of the fixed units followed by the sentinel M
  std::vector<int32_t> prog_last, pos_of_bit, fixed_pos;
  DBuf<int32_t> d_prog_last, d_pos_of_bit, d_fixed_pos;
  // anchor kernel (fitness_anchor.cu): 128-bit window (values carried as
  // X = v >> anchor_shift), per-position step headers and 128-bit constants,
  // merged-component pool entries per genome, and the list of genomes that
  // overflowed it
  bool anchor_ok = false;
  int32_t anchor_shift = 0;
  int32_t anchor_span = 0;  // highest bit of the partial-sum bound minus anchor_shift
  DBuf<uint64_t> d_acold;   // [M][6]: rep, off, term1 as 128-bit X (packed-label walks)
  DBuf<int32_t> d_acnt;     // [M]
  bool anchor_wide_ok = false;  // packed-sum anchor walk usable (span and counts fit)
  DBuf<uint64_t> d_arec;        // [M][10]: 80-byte step records (header, term1 - off, slot-table entry)
  DBuf<uint8_t> d_alists;       // long back lists
  DBuf<int32_t> d_an_infeas_word;  // genome words holding infeasible bits, and their masks
  DBuf<uint64_t> d_an_infeas_mask;
  int32_t pool_entries = 16;  // anchor walk: merged-sum pool entries per lane in shared memory
  cudaStream_t host_stream = nullptr;  // single-chunk cb_fitness_host calls
  ~cb_es_plan() {
    if (host_stream) cudaStreamDestroy(host_stream);
  }
  // finite-state walk (fitness_fsm.cu, <= 8 slots): per-step headers and
  // the transition table
  bool fsm_ok = false;
  bool fsm_auto = false;  // chosen by the automatic path (table <= 1 MB)
  DBuf<uint32_t> d_fsm_hdr, d_fsm_table;
  int32_t fsm_layout = 0;  // transitions: 1 = 8 bytes, 2 = 16 bytes (+ shared delta table), 0 = 32 bytes
  DBuf<uint32_t> d_fsm_ctable, d_fsm_dtab;
  int32_t fsm_deltas = 0;
  bool fsm_d64 = false;  // shared delta table as sign-extended 8-byte entries (fitness_fsm.cu)
  int32_t fsm_states_max = 0;
  int64_t fsm_entries = 0;
  // tournament order keys of the parent population (es.cu)
  DBuf<uint16_t> d_keys;                // 16-bit tournament order keys (es_ops.cuh)
  DBuf<unsigned long long> d_fminmax;  // finite fitness [min, max] bit patterns for the keys
  // packed anchor walk (fitness_packed128.cu, <= 8 slots): 16-byte step headers
  bool pa_ok = false;
  DBuf<uint32_t> d_pahdr;
  bool packed_ok = true;     // every unit's back / end lists fit the packed header
  int32_t force_path = -1;  // -1 auto, 0 union-find, 1 frontier, 2 frontier (smem labels),
                            // 3 sparse warp-per-genome walk, 4 anchor walk (thread per genome),
                            // 5 packed-label walk in the 128-bit window, 6 packed anchor walk,
                            // 7 finite-state walk
};

// fitness_wide.cu: warp-per-genome sparse walk of the frontier program (F <= 128)
int launch_fitness_wide(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit,
                        cudaStream_t stream);
// fitness_anchor.cu: 128-bit window analysis + step headers (plan time);
// thread-per-genome lockstep anchor walk (F <= 64)
int build_anchor_plan(cb_es_plan* p);
// fitness_packed128.cu: packed-label walk (<= 16 slots) in the 128-bit window
int launch_fitness_packed128(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit,
                             cudaStream_t stream);
int launch_fitness_packed_anchor(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit,
                                 cudaStream_t stream);
// fitness_fsm.cu: frontier states enumerated at plan time, walk by table
int build_fsm_plan(cb_es_plan* p);
int launch_fitness_fsm(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit, cudaStream_t stream);
// fused breed + packed anchor fitness (one kernel per generation, <= 4 words)
struct BreedArgs;
bool fused_generation_ok(const cb_es_plan* p);
int launch_fused_generation(cb_es_plan* p, const BreedArgs& br, uint64_t* d_children, int64_t n,
                            double* d_fit, cudaStream_t stream);
int launch_fitness_anchor(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit,
                          cudaStream_t stream);
