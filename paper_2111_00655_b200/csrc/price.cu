// Kernel cost of every match under the simulated profiles.
//
// tensorplace/cost.py:121-138: node cost = coeff[op] * volume + overhead[op]
// (two separately rounded IEEE operations -- no FMA contraction), kernel cost
// = fsum(node costs) * fusion_discount ** (n - 1).  The power table is
// computed by the host with Python's own float pow so the product is
// bit-identical; fsum is the exact fixed-point sum rounded once.
#include "cb_internal.cuh"

__global__ void price_kernel(int64_t n_matches, const int32_t* __restrict__ mem_ptr,
                             const int32_t* __restrict__ members,
                             const int32_t* __restrict__ backend, const int32_t* __restrict__ kind,
                             const double* __restrict__ volume, int32_t n_kinds,
                             const double* __restrict__ coeff, const double* __restrict__ overhead,
                             const uint8_t* __restrict__ has_entry,
                             const uint8_t* __restrict__ has_profile, int32_t pw_stride,
                             const double* __restrict__ pw, double* __restrict__ cost,
                             int8_t* __restrict__ err) {
  int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n_matches) return;
  const int32_t b = backend[m];
  const int32_t i0 = mem_ptr[m], i1 = mem_ptr[m + 1];
  if (!has_profile[b]) {
    err[m] = 1;
    cost[m] = 0.0;
    return;
  }
  fx192 acc = fx_zero();
  bool exact = true;
  for (int32_t i = i0; i < i1; ++i) {
    const int32_t v = members[i];
    const int64_t t = (int64_t)b * n_kinds + kind[v];
    if (!has_entry[t]) {
      err[m] = 2;
      cost[m] = 0.0;
      return;
    }
    const double c = __dadd_rn(__dmul_rn(coeff[t], volume[v]), overhead[t]);
    fx192 x;
    exact &= fx_from_double(c, x);
    fx_add(acc, x);
  }
  const int32_t e = i1 - i0 - 1;
  const double base = fx_to_double(acc);
  cost[m] = (e < pw_stride) ? __dmul_rn(base, pw[(int64_t)b * pw_stride + e]) : 0.0;
  err[m] = (e < pw_stride) ? (exact ? 0 : 3) : 4;
}

extern "C" int cb_matches_price(cb_matches* m, cb_graph* g, int32_t n_backends, int32_t n_kinds,
                                const double* coeff, const double* overhead,
                                const uint8_t* has_entry, const uint8_t* has_profile,
                                int32_t pw_stride, const double* pw, double* costs_out,
                                int8_t* err_out) {
  CB_ARG_CHECK(m && g && coeff && overhead && has_entry && has_profile && pw && pw_stride > 0,
               "cb_matches_price: bad arguments");
  int rc = cb_graph_ensure_device(g);
  if (rc != CB_OK) return rc;
  const size_t tab = (size_t)n_backends * n_kinds;
  DBuf<double> d_coeff, d_over, d_pw;
  DBuf<uint8_t> d_has, d_prof;
  DBuf<int8_t> d_err;
  CB_CUDA_TRY(d_coeff.upload(coeff, tab));
  CB_CUDA_TRY(d_over.upload(overhead, tab));
  CB_CUDA_TRY(d_has.upload(has_entry, tab));
  CB_CUDA_TRY(d_prof.upload(has_profile, (size_t)n_backends));
  CB_CUDA_TRY(d_pw.upload(pw, (size_t)n_backends * pw_stride));
  CB_CUDA_TRY(d_err.alloc((size_t)m->n_matches + 1));
  if (m->n_matches > 0) {
    const int threads = 256;
    const int64_t blocks = (m->n_matches + threads - 1) / threads;
    price_kernel<<<(unsigned)blocks, threads>>>(m->n_matches, m->d_mem_ptr.p, m->d_members.p,
                                                m->d_backend.p, g->d_kind.p, g->d_volume.p,
                                                n_kinds, d_coeff.p, d_over.p, d_has.p, d_prof.p,
                                                pw_stride, d_pw.p, m->d_cost.p, d_err.p);
    CB_CUDA_TRY(cudaGetLastError());
  }
  CB_CUDA_TRY(cudaDeviceSynchronize());
  std::vector<int8_t> herr;
  std::vector<double> hcost;
  CB_CUDA_TRY(d_err.download(herr));
  CB_CUDA_TRY(m->d_cost.download(hcost));
  m->cost.assign(hcost.begin(), hcost.begin() + m->n_matches);
  if (costs_out) std::copy(m->cost.begin(), m->cost.end(), costs_out);
  bool any = false, inexact = false;
  for (int64_t i = 0; i < m->n_matches; ++i) {
    if (err_out) err_out[i] = herr[i];
    if (herr[i] == 1 || herr[i] == 2) any = true;
    if (herr[i] == 3 || herr[i] == 4) inexact = true;
  }
  m->costs_set = !any && !inexact;
  if (any) {
    cb_set_error("some matches cannot be priced (missing profile or op entry)");
    return CB_ERR_PROFILE;
  }
  if (inexact) {
    cb_set_error("a node cost falls outside the exact accumulator range [2^-75, 2^64)");
    return CB_ERR_INEXACT;
  }
  return CB_OK;
}

extern "C" int cb_matches_set_costs(cb_matches* m, const double* costs) {
  CB_ARG_CHECK(m && (costs || m->n_matches == 0), "cb_matches_set_costs: bad arguments");
  for (int64_t i = 0; i < m->n_matches; ++i) {
    fx192 t;
    if (!fx_from_double(costs[i], t)) {
      cb_set_error("kernel cost " + std::to_string(costs[i]) +
                   " is negative, non-finite or outside the exact accumulator range");
      return CB_ERR_INEXACT;
    }
  }
  CB_CUDA_TRY(m->d_cost.upload(costs, (size_t)m->n_matches));
  m->cost.assign(costs, costs + m->n_matches);
  m->costs_set = true;
  return CB_OK;
}
