// Device-side evolutionary operators for population-scale search.
//
// Operator semantics follow tensorplace/evolution.py:205-223 and :412-428:
// tournament selection (first draw, then tournament-1 challengers that win
// only when strictly fitter), two-point crossover child = a[:i] + b[i:j] +
// a[j:] with i <= j drawn from [0, k], per-bit mutation.  Randomness is
// Philox4x32-10 keyed by (seed) and countered by (child, generation, stream,
// draw) so every child is reproducible independently of launch geometry.
// Mutation draws geometric gaps between flipped bits, which is the same
// Bernoulli(rate) process per bit at O(#flips) cost.
//
// One warp per child: lane 0 draws, every lane assembles whole uint64 words
// of the child from the two parents with segment masks (coalesced rows).
#include <map>
#include <cub/cub.cuh>

#include "fitness_plan.cuh"

#include "es_ops.cuh"

#define BREED_WARPS 8
#define MAX_FLIPS 32

__global__ void __launch_bounds__(BREED_WARPS * 32)
breed_kernel(int32_t k, int32_t words, const uint64_t* __restrict__ parents,
             const double* __restrict__ fit, int64_t n_parents, uint64_t* __restrict__ children,
             int64_t n_children, const uint64_t* __restrict__ keep, int64_t n_keep, uint64_t seed,
             uint32_t generation, uint32_t stream_id, int32_t tournament, double rate,
             double log1m_rate) {
  __shared__ int64_t s_flip[BREED_WARPS][MAX_FLIPS];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t stride = (int64_t)gridDim.x * BREED_WARPS;
  for (int64_t child = (int64_t)blockIdx.x * BREED_WARPS + warp; child < n_children; child += stride) {
    uint64_t* out = children + child * words;
    if (child < n_keep) {
      for (int32_t w = lane; w < words; w += 32) out[w] = keep[child * words + w];
      continue;
    }
    int64_t pa = 0, pb = 0, ci = 0, cj = 0;
    int nflip = 0;
    bool dense = false;
    if (lane == 0) {
      Philox rng(seed, (uint32_t)child, (uint32_t)(child >> 32) ^ (generation * 0x9E3779B9u),
                 stream_id);
      for (int t = 0; t < 2; ++t) {
        int64_t best = rng.below((uint32_t)n_parents);
        for (int j = 1; j < tournament; ++j) {
          int64_t i = rng.below((uint32_t)n_parents);
          if (fit[i] < fit[best]) best = i;
        }
        if (t == 0) pa = best;
        else pb = best;
      }
      if (k >= 2) {
        int64_t x = rng.below((uint32_t)(k + 1)), y = rng.below((uint32_t)(k + 1));
        ci = x < y ? x : y;
        cj = x < y ? y : x;
      }
      // mutation positions by geometric gaps
      if (rate >= 1.0 || rate * (double)k > 8.0) {
        dense = true;
      } else if (rate > 0.0) {
        int64_t pos = -1;
        while (true) {
          double u = rng.unit();
          double gap = floor(log(u) / log1m_rate);
          if (!(gap < (double)k)) break;
          pos += 1 + (int64_t)gap;
          if (pos >= k) break;
          if (nflip == MAX_FLIPS) {
            dense = true;  // too many: fall back to per-bit draws below
            break;
          }
          s_flip[warp][nflip++] = pos;
        }
      }
    }
    pa = __shfl_sync(0xffffffffu, pa, 0);
    pb = __shfl_sync(0xffffffffu, pb, 0);
    ci = __shfl_sync(0xffffffffu, ci, 0);
    cj = __shfl_sync(0xffffffffu, cj, 0);
    nflip = __shfl_sync(0xffffffffu, nflip, 0);
    dense = __shfl_sync(0xffffffffu, dense, 0);
    __syncwarp();
    const uint64_t* A = parents + pa * words;
    const uint64_t* B = parents + pb * words;
    for (int32_t w = lane; w < words; w += 32) {
      uint64_t mb = seg_mask(ci, cj, w);
      uint64_t v = (A[w] & ~mb) | (B[w] & mb);
      if (dense) {
        Philox r2(seed ^ 0xA5A5A5A5A5A5A5A5ull, (uint32_t)child, (uint32_t)w,
                  generation ^ (stream_id << 16));
        uint64_t flips = 0;
        for (int b = 0; b < 64; ++b) {
          int64_t bit = (int64_t)w * 64 + b;
          if (bit >= k) break;
          double u = ((double)(r2.next() >> 8) + 0.5) * (1.0 / 16777216.0);
          if (u < rate) flips |= 1ull << b;
        }
        v ^= flips;
      } else {
        for (int f = 0; f < nflip; ++f) {
          int64_t pos = s_flip[warp][f];
          if ((pos >> 6) == w) v ^= 1ull << (pos & 63);
        }
      }
      if ((int64_t)(w + 1) * 64 > k) v &= (k % 64) ? ((1ull << (k % 64)) - 1ull) : ~0ull;
      out[w] = v;
    }
    __syncwarp();
  }
}

// Narrow genomes (W <= 8 words): one thread per child, the child row in
// registers.  Same draws and semantics as breed_kernel.
template <int W>
__global__ void __launch_bounds__(256)
breed_thread_kernel(int32_t k, const uint64_t* __restrict__ parents, const double* __restrict__ fit,
                    const cb_key_t* __restrict__ keys, int64_t n_parents, uint64_t* __restrict__ children, int64_t n_children,
                    const uint64_t* __restrict__ keep, int64_t n_keep, uint64_t seed,
                    uint32_t generation, uint32_t stream_id, int32_t tournament, double rate,
                    double log1m_rate) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t child = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; child < n_children;
       child += stride) {
    uint64_t v[W];
    make_child<W>(v, k, parents, fit, keys, n_parents, child, keep, n_keep, seed, generation, stream_id,
                  tournament, rate, log1m_rate);
#pragma unroll
    for (int w = 0; w < W; ++w) __stcs(children + child * W + w, v[w]);
  }
}


// Tournament order keys: the high word of each fitness (non-negative doubles
// and +inf order like their bit patterns), half the bytes of the fitness
// array so that a large population's keys stay in L2 for the random gathers.
// Finite [min, max] of the (non-negative) fitness as ordered bit patterns:
// mm[0] = ~min, mm[1] = max (both preset to 0, one memset).
__global__ void fitness_minmax_kernel(const double* __restrict__ fit, int64_t n, unsigned long long* mm) {
  unsigned long long lo = ~0ull, hi = 0ull;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double f = __ldcs(fit + i);
    if (isfinite(f)) {
      const unsigned long long u = (unsigned long long)__double_as_longlong(f);
      lo = u < lo ? u : lo;
      hi = u > hi ? u : hi;
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, lo, d), h2 = __shfl_xor_sync(0xffffffffu, hi, d);
    lo = l2 < lo ? l2 : lo;
    hi = h2 > hi ? h2 : hi;
  }
  if ((threadIdx.x & 31) == 0) {
    if (lo != ~0ull) atomicMax(mm, ~lo);
    if (hi != 0ull) atomicMax(mm + 1, hi);
  }
}

// 16-bit order keys (es_ops.cuh): floor((f - min) * 65534 / (max - min)),
// 65535 for infinite fitness.  Fitness streams through evict-first so the
// keys the tournaments gather next stay in L2.
__global__ void fitness_keys_kernel(const double* __restrict__ fit, int64_t n, const unsigned long long* mm,
                                    cb_key_t* __restrict__ keys) {
  const unsigned long long ulo = ~mm[0], uhi = mm[1];
  const double lo = __longlong_as_double((long long)ulo), hi = __longlong_as_double((long long)uhi);
  const double scale = (ulo < uhi && hi > lo) ? 65534.0 / (hi - lo) : 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double f = __ldcs(fit + i);
    keys[i] = isfinite(f) ? (cb_key_t)fmin(65534.0, floor((f - lo) * scale)) : (cb_key_t)65535;
  }
}

// Order keys of the parents into p->d_keys (two small passes over the fitness).
static int launch_keys(cb_es_plan* p, const double* d_fit, int64_t n, cudaStream_t s) {
  if (p->d_keys.n < (size_t)n) CB_CUDA_TRY(p->d_keys.alloc((size_t)n));
  if (p->d_fminmax.n < 2) CB_CUDA_TRY(p->d_fminmax.alloc(2));
  CB_CUDA_TRY(cudaMemsetAsync(p->d_fminmax.p, 0, 2 * sizeof(unsigned long long), s));
  const int64_t kb = std::min<int64_t>((n + 255) / 256, (int64_t)cb_sm_count() * 16);
  fitness_minmax_kernel<<<(unsigned)kb, 256, 0, s>>>(d_fit, n, p->d_fminmax.p);
  fitness_keys_kernel<<<(unsigned)kb, 256, 0, s>>>(d_fit, n, p->d_fminmax.p, p->d_keys.p);
  CB_CUDA_TRY(cudaGetLastError());
  return CB_OK;
}

template <int W>
static void launch_breed_thread(int32_t k, const uint64_t* parents, const double* fit,
                                const cb_key_t* keys, int64_t n_parents, uint64_t* children, int64_t n_children,
                                const uint64_t* keep, int64_t n_keep, uint64_t seed, uint32_t gen,
                                uint32_t sid, int32_t tournament, double rate, double log1m,
                                cudaStream_t s) {
  int64_t blocks = (n_children + 255) / 256;
  if (blocks > (int64_t)cb_sm_count() * 8) blocks = (int64_t)cb_sm_count() * 8;
  breed_thread_kernel<W><<<(unsigned)blocks, 256, 0, s>>>(k, parents, fit, keys, n_parents, children,
                                                           n_children, keep, n_keep, seed, gen,
                                                           sid, tournament, rate, log1m);
}

extern "C" int cb_es_breed(cb_es_plan* p, const uint64_t* d_parents, const double* d_parent_fit,
                           int64_t n_parents, uint64_t* d_children, int64_t n_children,
                           const uint64_t* d_keep, int64_t n_keep, uint64_t seed,
                           uint64_t generation, uint64_t stream_id, int32_t tournament,
                           double mutation_rate, void* stream) {
  CB_ARG_CHECK(p && d_parents && d_parent_fit && d_children && n_parents > 0 && tournament >= 1,
               "cb_es_breed: bad arguments");
  CB_ARG_CHECK(n_parents < (int64_t)0xffffffffll, "cb_es_breed: too many parents");
  CB_ARG_CHECK(n_keep == 0 || d_keep, "cb_es_breed: keep rows missing");
  cb_es_plan_info info;
  cb_es_plan_query(p, &info);
  if (n_children <= 0) return CB_OK;
  double log1m = (mutation_rate > 0.0 && mutation_rate < 1.0) ? log1p(-mutation_rate) : -1.0;
  cudaStream_t s = (cudaStream_t)stream;
  const uint32_t gen = (uint32_t)generation, sid = (uint32_t)stream_id;
  const cb_key_t* keys = nullptr;
  if (info.words <= 8) {
    const int rc = launch_keys(p, d_parent_fit, n_parents, s);
    if (rc != CB_OK) return rc;
    keys = p->d_keys.p;
  }
  switch (info.words) {
#define CB_BREED_CASE(Wn)                                                                   \
  case Wn:                                                                                  \
    launch_breed_thread<Wn>(info.genome_bits, d_parents, d_parent_fit, keys, n_parents, d_children, \
                            n_children, d_keep, n_keep, seed, gen, sid, tournament,          \
                            mutation_rate, log1m, s);                                        \
    CB_CUDA_TRY(cudaGetLastError());                                                         \
    return CB_OK;
    CB_BREED_CASE(1)
    CB_BREED_CASE(2)
    CB_BREED_CASE(3)
    CB_BREED_CASE(4)
    CB_BREED_CASE(5)
    CB_BREED_CASE(6)
    CB_BREED_CASE(7)
    CB_BREED_CASE(8)
#undef CB_BREED_CASE
    default:
      break;
  }
  int64_t blocks = (n_children + BREED_WARPS - 1) / BREED_WARPS;
  if (blocks > (int64_t)cb_sm_count() * 16) blocks = (int64_t)cb_sm_count() * 16;
  breed_kernel<<<(unsigned)blocks, BREED_WARPS * 32, 0, (cudaStream_t)stream>>>(
      info.genome_bits, info.words, d_parents, d_parent_fit, n_parents, d_children, n_children,
      d_keep, n_keep, seed, (uint32_t)generation, (uint32_t)stream_id, tournament, mutation_rate,
      log1m);
  CB_CUDA_TRY(cudaGetLastError());
  return CB_OK;
}

// One generation: breed n_children rows from the parents and price them.
// Fused into one kernel (fitness_pa_breed_kernel) when the plan runs the
// packed anchor walk and genomes have <= 4 words; otherwise the breed launch
// followed by the plan's fitness kernel.  Same children and fitness either way.
extern "C" int cb_es_generation(cb_es_plan* p, const uint64_t* d_parents, const double* d_parent_fit,
                                int64_t n_parents, uint64_t* d_children, double* d_child_fit,
                                int64_t n_children, const uint64_t* d_keep, int64_t n_keep, uint64_t seed,
                                uint64_t generation, uint64_t stream_id, int32_t tournament,
                                double mutation_rate, void* stream) {
  CB_ARG_CHECK(p && d_parents && d_parent_fit && d_children && d_child_fit && n_parents > 0 &&
                   tournament >= 1,
               "cb_es_generation: bad arguments");
  CB_ARG_CHECK(n_parents < (int64_t)0xffffffffll, "cb_es_generation: too many parents");
  CB_ARG_CHECK(n_keep == 0 || d_keep, "cb_es_generation: keep rows missing");
  if (n_children <= 0) return CB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (!fused_generation_ok(p)) {
    int rc = cb_es_breed(p, d_parents, d_parent_fit, n_parents, d_children, n_children, d_keep, n_keep,
                         seed, generation, stream_id, tournament, mutation_rate, stream);
    if (rc != CB_OK) return rc;
    return cb_fitness_device(p, d_children, n_children, d_child_fit, stream);
  }
  const int rc = launch_keys(p, d_parent_fit, n_parents, s);
  if (rc != CB_OK) return rc;
  BreedArgs br;
  br.k = p->k;
  br.parents = d_parents;
  br.fit = d_parent_fit;
  br.keys = p->d_keys.p;
  br.n_parents = n_parents;
  br.keep = d_keep;
  br.n_keep = n_keep;
  br.seed = seed;
  br.generation = (uint32_t)generation;
  br.stream_id = (uint32_t)stream_id;
  br.tournament = tournament;
  br.rate = mutation_rate;
  br.log1m_rate = (mutation_rate > 0.0 && mutation_rate < 1.0) ? log1p(-mutation_rate) : -1.0;
  return launch_fused_generation(p, br, d_children, n_children, d_child_fit, s);
}

extern "C" int cb_es_generation_fused(const cb_es_plan* p) { return p && fused_generation_ok(p) ? 1 : 0; }

// index of the smallest fitness (first on ties) -> *d_idx, value -> *d_val
static int argmin_to(const double* d_fit, int64_t n, int64_t* d_idx, double* d_val, cudaStream_t s) {
  // CUB scratch per (host thread, device): a process may drive several GPUs
  static thread_local std::map<int, std::pair<void*, size_t>> scratch;
  int dev = 0;
  cudaGetDevice(&dev);
  void*& tmp = scratch[dev].first;
  size_t& tmp_bytes = scratch[dev].second;
  size_t bytes = 0;
  CB_CUDA_TRY(cub::DeviceReduce::ArgMin(nullptr, bytes, d_fit, d_val, d_idx, n, s));
  if (bytes > tmp_bytes) {
    if (tmp) cudaFree(tmp);
    CB_CUDA_TRY(cudaMalloc(&tmp, bytes));
    tmp_bytes = bytes;
  }
  CB_CUDA_TRY(cub::DeviceReduce::ArgMin(tmp, bytes, d_fit, d_val, d_idx, n, s));
  return CB_OK;
}

// best row -> elite, best value -> history slot (one launch instead of three
// host-side copies)
__global__ void copy_elite(const int64_t* idx, const double* val, const uint64_t* __restrict__ pop,
                           int32_t words, uint64_t* elite, double* hist) {
  const int64_t i = *idx;
  if (threadIdx.x == 0 && hist) *hist = *val;
  for (int32_t w = threadIdx.x; w < words; w += blockDim.x) elite[w] = pop[i * words + w];
}

extern "C" int cb_argmin_elite(const double* d_fit, int64_t n, const uint64_t* d_pop, int32_t words,
                               int64_t* d_idx, double* d_val, uint64_t* d_elite, double* d_history_slot,
                               void* stream) {
  CB_ARG_CHECK(d_fit && d_idx && d_val && n > 0 && (!d_pop || (d_elite && words > 0)),
               "cb_argmin_elite: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  int rc = argmin_to(d_fit, n, d_idx, d_val, s);
  if (rc != CB_OK) return rc;
  if (d_pop || d_history_slot) {
    copy_elite<<<1, 32, 0, s>>>(d_idx, d_val, d_pop, d_pop ? words : 0, d_elite, d_history_slot);
    CB_CUDA_TRY(cudaGetLastError());
  }
  return CB_OK;
}

extern "C" int cb_argmin(const double* d_fit, int64_t n, int64_t* d_idx, double* d_val,
                         void* stream) {
  CB_ARG_CHECK(d_fit && d_idx && d_val && n > 0, "cb_argmin: bad arguments");
  return argmin_to(d_fit, n, d_idx, d_val, (cudaStream_t)stream);
}

// ---------------------------------------------------------------- elite exchange
// The sharded search's only exchange step: every rank contributes one record
// [best fitness bits, best row] (one all-gather), and every rank picks the
// lowest fitness (first rank on ties) on the device.

__global__ void elite_record_kernel(const int64_t* idx, const double* val, const uint64_t* __restrict__ pop,
                                    int32_t words, uint64_t* rec) {
  const int64_t i = *idx;
  if (threadIdx.x == 0) rec[0] = (uint64_t)__double_as_longlong(*val);
  for (int32_t w = threadIdx.x; w < words; w += blockDim.x) rec[1 + w] = pop[i * words + w];
}

__global__ void elite_pick_kernel(const uint64_t* __restrict__ recs, int32_t world, int32_t words,
                                  uint64_t* elite, double* elite_val, double* hist) {
  __shared__ int best;
  if (threadIdx.x == 0) {
    int b = 0;
    double bv = __longlong_as_double((long long)recs[0]);
    for (int r = 1; r < world; ++r) {
      const double v = __longlong_as_double((long long)recs[(int64_t)r * (1 + words)]);
      if (v < bv) {
        b = r;
        bv = v;
      }
    }
    best = b;
    *elite_val = bv;
    if (hist) *hist = bv;
  }
  __syncthreads();
  const uint64_t* row = recs + (int64_t)best * (1 + words) + 1;
  for (int32_t w = threadIdx.x; w < words; w += blockDim.x) elite[w] = row[w];
}

extern "C" int cb_elite_record(const double* d_fit, int64_t n, const uint64_t* d_pop, int32_t words,
                               int64_t* d_idx, double* d_val, uint64_t* d_record, void* stream) {
  CB_ARG_CHECK(d_fit && d_pop && d_idx && d_val && d_record && n > 0 && words > 0,
               "cb_elite_record: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  int rc = argmin_to(d_fit, n, d_idx, d_val, s);
  if (rc != CB_OK) return rc;
  elite_record_kernel<<<1, 128, 0, s>>>(d_idx, d_val, d_pop, words, d_record);
  CB_CUDA_TRY(cudaGetLastError());
  return CB_OK;
}

extern "C" int cb_elite_pick(const uint64_t* d_records, int32_t world, int32_t words, uint64_t* d_elite,
                             double* d_elite_val, double* d_history_slot, void* stream) {
  CB_ARG_CHECK(d_records && world > 0 && words > 0 && d_elite && d_elite_val, "cb_elite_pick: bad arguments");
  elite_pick_kernel<<<1, 128, 0, (cudaStream_t)stream>>>(d_records, world, words, d_elite, d_elite_val,
                                                         d_history_slot);
  CB_CUDA_TRY(cudaGetLastError());
  return CB_OK;
}
