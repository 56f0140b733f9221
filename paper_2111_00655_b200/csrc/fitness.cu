// Graph-level fitness of offload genomes, batched over a population.
//
// Reference semantics (tensorplace/evolution.py:65-119 and
// tensorplace/cost.py:320-373): bit i of a genome moves the i-th eligible
// kernel (canonical placement order, not on a graph inference library) to
// the target graph backend -- as one same-node-set match of that backend
// when registered, else decomposed into its singleton matches, else the
// genome is infeasible (+inf).  The decoded placement is priced by grouping
// graph-backend kernels of the same backend that touch through a data edge
// into regions; every region costs round(fsum(member costs)) * r(n) + eps
// with r(n) = max(floor, 1 - alpha * (n - 1)), every other kernel its cost +
// eps, and the total is the fsum of all terms.
//
// Plan (host, once per DP placement): everything that does not depend on the
// genome is folded into constants -- regions of other graph backends, the
// kernels' own costs -- and the genome-dependent part is reduced to a small
// "dynamic unit" graph: one unit per feasible eligible kernel plus one unit
// per connected component of fixed target-backend kernels (always on).
//
// Evaluation (device).  The plan orders the units into a "frontier
// program" (each unit holds a slot from its position to its last
// neighbour's) and launch_fitness picks the kernel by the program's width F:
//   F <= 8   fitness_fsm_kernel         (fitness_fsm.cu) tabulated state machine,
//            while its transition table stays <= 32 MB (all model configs)
//   F <= 8   fitness_pa_kernel          (fitness_packed128.cu) packed anchor labels
//   F <= 16  fitness_packed128_kernel / fitness_frontier2_kernel (this file)
//   F <= 64  fitness_anchor_kernel      (fitness_anchor.cu) union-find anchors
//   F <= 128 fitness_wide_kernel        (fitness_wide.cu) warp per genome
//   wider    fitness_smem_kernel / fitness_global_kernel (this file): warp or
//            CTA per genome, lock-free union-find over the dynamic edges
//            (shared-memory CAS, smaller root wins), exact region sums with
//            multi-limb atomics, a shuffle reduction of the 192-bit total.
// All of them return bit-identical fitness (values in the plan's 128-bit
// window where it exists, else 192-bit fixed point, rounded once).
#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <queue>

#include "cb_internal.cuh"
#include "fitness_plan.cuh"

#define FRONTIER_MAX 32   // slot cap of the thread-per-genome kernels
#define WIDE_MAX 128      // slot cap of the program (warp-per-genome sparse kernel)

static bool fx_term(double base, double r, const fx192& eps, fx192& out);

// Order the dynamic units (eligible ones in genome order, each fixed unit
// just before its first eligible neighbour), give every unit a frontier
// slot for the span between its position and its last neighbour's, and
// record the back / end slot lists.  F = number of slots = the largest
// number of units simultaneously waiting for a later neighbour.
static void build_frontier_program(cb_es_plan* P, int32_t n_elig_units) {
  const int32_t M = P->M;
  // unit adjacency as CSR (neighbours in edge order, as per-unit lists would hold them)
  std::vector<int32_t> nptr(M + 1, 0), nadj(2 * P->edges.size());
  for (const int2& e : P->edges) {
    ++nptr[e.x + 1];
    ++nptr[e.y + 1];
  }
  for (int32_t v = 0; v < M; ++v) nptr[v + 1] += nptr[v];
  {
    std::vector<int32_t> fill(nptr.begin(), nptr.end() - 1);
    for (const int2& e : P->edges) {
      nadj[fill[e.x]++] = e.y;
      nadj[fill[e.y]++] = e.x;
    }
  }
  auto nbr_begin = [&](int32_t v) { return nadj.begin() + nptr[v]; };
  auto nbr_end = [&](int32_t v) { return nadj.begin() + nptr[v + 1]; };
  std::vector<int32_t> key(M, M);
  for (int32_t v = n_elig_units; v < M; ++v)
    for (auto it = nbr_begin(v); it != nbr_end(v); ++it)
      if (*it < n_elig_units) key[v] = std::min(key[v], *it);
  std::vector<std::vector<int32_t>> before(n_elig_units + 1);
  for (int32_t v = n_elig_units; v < M; ++v) before[std::min(key[v], n_elig_units)].push_back(v);
  std::vector<int32_t> order;
  order.reserve(M);
  for (int32_t e = 0; e <= n_elig_units; ++e) {
    for (int32_t v : before[e]) order.push_back(v);
    if (e < n_elig_units) order.push_back(e);
  }
  std::vector<int32_t> pos(M);
  for (int32_t p = 0; p < M; ++p) pos[order[p]] = p;
  std::vector<int32_t> last(M);
  std::vector<int32_t> eptr(M + 1, 0), eat(M);  // ends_at as CSR (positions in increasing order)
  for (int32_t p = 0; p < M; ++p) {
    int32_t u = order[p], l = p;
    for (auto it = nbr_begin(u); it != nbr_end(u); ++it) l = std::max(l, pos[*it]);
    last[p] = l;
    ++eptr[l + 1];
  }
  for (int32_t p = 0; p < M; ++p) eptr[p + 1] += eptr[p];
  {
    std::vector<int32_t> fill(eptr.begin(), eptr.end() - 1);
    for (int32_t p = 0; p < M; ++p) eat[fill[last[p]]++] = p;
  }
  std::vector<int32_t> slot(M, -1);
  // free slots as a min-heap: every unit takes the smallest free slot
  std::priority_queue<int32_t, std::vector<int32_t>, std::greater<int32_t>> free_slots;
  int32_t used = 0;
  for (int32_t p = 0; p < M; ++p) {
    int32_t s;
    if (free_slots.empty()) {
      s = used++;
    } else {
      s = free_slots.top();
      free_slots.pop();
    }
    slot[p] = s;
    for (int32_t j = eptr[p]; j < eptr[p + 1]; ++j) free_slots.push(slot[eat[j]]);
  }
  P->F_needed = used;
  if (used > WIDE_MAX) {
    P->F = 0;
    return;
  }
  P->F = used;
  // merged-sum pool entries per lane in shared memory (anchor walk; the
  // rest in local memory): 8 measured best on the random 100k DAG (4 / 12
  // within 6 %, 16 slower: fewer resident blocks)
  P->pool_entries = std::min(used, 8);
  // sparse walk: program position of every genome bit, fixed-unit positions
  P->prog_last.assign(last.begin(), last.end());
  P->pos_of_bit.assign((size_t)std::max(P->k, 1), -1);
  P->fixed_pos.clear();
  for (int32_t p = 0; p < M; ++p) {
    const int32_t b = P->unit_slot[order[p]];
    if (b >= 0)
      P->pos_of_bit[b] = p;
    else
      P->fixed_pos.push_back(p);
  }
  P->fixed_pos.push_back(M);  // sentinel
  P->prog.resize(M);
  P->prog_slots.clear();
  P->prog_back_pos.clear();
  for (int32_t p = 0; p < M; ++p) {
    const int32_t u = order[p];
    UnitRec r;
    std::memset(&r, 0, sizeof(r));
    r.rep = P->unit_rep[u];
    r.off = P->unit_off[u];
    fx_term(fx_to_double(r.rep), P->rt[P->unit_cnt[u]], P->eps, r.term1);
    r.bit = P->unit_slot[u];
    r.bit2 = r.bit;
    r.cnt = P->unit_cnt[u];
    r.slot = (uint8_t)slot[p];
    r.back_off = (int32_t)P->prog_slots.size();
    for (auto it = nbr_begin(u); it != nbr_end(u); ++it)
      if (pos[*it] < p) {
        P->prog_slots.push_back((uint8_t)slot[pos[*it]]);
        P->prog_back_pos.push_back(pos[*it]);
      }
    r.nback = (uint8_t)(P->prog_slots.size() - r.back_off);
    r.end_off = (int32_t)P->prog_slots.size();
    for (int32_t j = eptr[p]; j < eptr[p + 1]; ++j) {
      P->prog_slots.push_back((uint8_t)slot[eat[j]]);
      P->prog_back_pos.push_back(-1);
    }
    r.nend = (uint8_t)(P->prog_slots.size() - r.end_off);
    r.hot.x = (uint32_t)r.bit;
    r.hot.y = (uint32_t)r.slot | ((uint32_t)r.nback << 8) | ((uint32_t)r.nend << 16);
    r.hot.z = r.hot.w = 0u;
    if (r.nback > 8 || r.nend > 8 || used > 16) P->packed_ok = false;
    for (int j = 0; j < r.nback && j < 8; ++j)
      r.hot.z |= (uint32_t)(P->prog_slots[r.back_off + j] & 0xF) << (4 * j);
    for (int j = 0; j < r.nend && j < 8; ++j)
      r.hot.w |= (uint32_t)(P->prog_slots[r.end_off + j] & 0xF) << (4 * j);
    P->prog[p] = r;
  }
  if (P->prog_slots.empty()) P->prog_slots.push_back(0);
}

static double region_r(double alpha, double floor_, int64_t n) {
  // max(floor, 1.0 - alpha * (n - 1)) with two separately rounded operations
  volatile double prod = alpha * (double)(n - 1);
  volatile double t = 1.0 - prod;
  return t > floor_ ? t : floor_;
}

namespace {
struct DSU {
  std::vector<int32_t> p;
  explicit DSU(int32_t n) : p(n) { std::iota(p.begin(), p.end(), 0); }
  int32_t find(int32_t x) {
    while (p[x] != x) {
      p[x] = p[p[x]];
      x = p[x];
    }
    return x;
  }
  void unite(int32_t a, int32_t b) {
    a = find(a);
    b = find(b);
    if (a != b) p[std::max(a, b)] = std::min(a, b);
  }
};
}  // namespace

static bool fx_term(double base, double r, const fx192& eps, fx192& out) {
  // exact value of (base * r) + eps, base*r rounded once as in Python
  volatile double prod = base * r;
  bool ok = fx_from_double(prod, out);
  fx_add(out, eps);
  return ok;
}

extern "C" int cb_placement_cost_graphlevel(cb_graph* g, int32_t n_kernels, const int32_t* kernel_ptr,
                                            const int32_t* kernel_nodes, const int32_t* kernel_backend,
                                            const double* kernel_cost, int32_t n_backends,
                                            const uint8_t* backend_is_graph, const double* region_alpha,
                                            const double* region_floor, double epsilon, double* out) {
  CB_ARG_CHECK(g && out && n_kernels >= 0 && (n_kernels == 0 || (kernel_ptr && kernel_nodes &&
               kernel_backend && kernel_cost)) && backend_is_graph && region_alpha && region_floor,
               "cb_placement_cost_graphlevel: bad arguments");
  const int32_t n = g->n;
  fx192 eps;
  if (!fx_from_double(epsilon, eps)) {
    cb_set_error("epsilon outside the exact range");
    return CB_ERR_INEXACT;
  }
  std::vector<int32_t> kernel_of(n, -1);
  for (int32_t k = 0; k < n_kernels; ++k) {
    CB_ARG_CHECK(kernel_backend[k] >= 0 && kernel_backend[k] < n_backends, "backend out of range");
    for (int32_t i = kernel_ptr[k]; i < kernel_ptr[k + 1]; ++i) {
      int32_t v = kernel_nodes[i];
      CB_ARG_CHECK(v >= 0 && v < n && kernel_of[v] < 0, "kernels must partition the graph");
      kernel_of[v] = k;
    }
  }
  for (int32_t v = 0; v < n; ++v) CB_ARG_CHECK(kernel_of[v] >= 0, "kernels must cover the graph");
  DSU dsu(n_kernels);
  for (int32_t v = 0; v < n; ++v)
    for (int32_t j = g->in_ptr[v]; j < g->in_ptr[v + 1]; ++j) {
      int32_t p = g->in_src[j];
      if (p < 0) continue;
      int32_t a = kernel_of[p], b = kernel_of[v];
      if (a != b && kernel_backend[a] == kernel_backend[b] && backend_is_graph[kernel_backend[a]])
        dsu.unite(a, b);
    }
  fx192 tot = fx_zero();
  bool exact = true;
  std::vector<fx192> sum(n_kernels, fx_zero());
  std::vector<int32_t> cnt(n_kernels, 0);
  for (int32_t k = 0; k < n_kernels; ++k) {
    fx192 t;
    exact &= fx_from_double(kernel_cost[k], t);
    if (!backend_is_graph[kernel_backend[k]]) {
      fx_add(tot, t);
      fx_add(tot, eps);
    } else {
      int32_t r = dsu.find(k);
      fx_add(sum[r], t);
      cnt[r] += 1;
    }
  }
  for (int32_t k = 0; k < n_kernels; ++k) {
    if (!backend_is_graph[kernel_backend[k]] || dsu.find(k) != k) continue;
    double r = region_r(region_alpha[kernel_backend[k]], region_floor[kernel_backend[k]], cnt[k]);
    fx192 t;
    exact &= fx_term(fx_to_double(sum[k]), r, eps, t);
    fx_add(tot, t);
  }
  if (!exact) {
    cb_set_error("a cost falls outside the exact accumulator range");
    return CB_ERR_INEXACT;
  }
  *out = fx_to_double(tot);
  return CB_OK;
}

extern "C" int cb_es_plan_create(cb_graph* g, cb_matches* m, int32_t n_kernels,
                                 const int32_t* kernel_match, int32_t n_backends,
                                 const uint8_t* backend_is_graph, const double* region_alpha,
                                 const double* region_floor, int32_t target_backend,
                                 double epsilon, cb_es_plan** out) {
  CB_ARG_CHECK(g && m && out && kernel_match && backend_is_graph && region_alpha && region_floor,
               "cb_es_plan_create: null argument");
  CB_ARG_CHECK(m->by_root && m->n_groups == g->n, "cb_es_plan_create: matches must come from cb_match_all");
  CB_ARG_CHECK(target_backend >= 0 && target_backend < n_backends, "cb_es_plan_create: bad target");
  if (!m->costs_set) {
    cb_set_error("cb_es_plan_create: kernel costs have not been set");
    return CB_ERR_STATE;
  }
  int rc = cb_require_device();
  if (rc != CB_OK) return rc;
  rc = cb_matches_ensure_host(m);
  if (rc != CB_OK) return rc;
  const int32_t n = g->n;
  // CB_PLAN_TIMING: per-phase host times on stderr
  const bool timing = getenv("CB_PLAN_TIMING") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto tick = [&](const char* what) {
    if (!timing) return;
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "plan %-18s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  tick("host copies");
  cb_es_plan* P = new cb_es_plan();
  auto bad = [&](const std::string& msg, int code) {
    delete P;
    cb_set_error(msg);
    return code;
  };
  if (!fx_from_double(epsilon, P->eps)) return bad("epsilon outside the exact range", CB_ERR_INEXACT);
  // kernel of every node
  std::vector<int32_t> kernel_of(n, -1);
  for (int32_t kk = 0; kk < n_kernels; ++kk) {
    int32_t mi = kernel_match[kk];
    if (mi < 0 || mi >= m->n_matches) return bad("kernel references an unknown match", CB_ERR_ARG);
    for (int32_t i = m->mem_ptr[mi]; i < m->mem_ptr[mi + 1]; ++i) {
      int32_t v = m->members[i];
      if (kernel_of[v] >= 0) return bad("placement kernels overlap", CB_ERR_ARG);
      kernel_of[v] = kk;
    }
  }
  for (int32_t v = 0; v < n; ++v)
    if (kernel_of[v] < 0) return bad("placement does not cover every node", CB_ERR_ARG);
  std::vector<int32_t> kb(n_kernels);
  std::vector<double> kc(n_kernels);
  for (int32_t kk = 0; kk < n_kernels; ++kk) {
    kb[kk] = m->backend[kernel_match[kk]];
    kc[kk] = m->cost[kernel_match[kk]];
    if (kb[kk] < 0 || kb[kk] >= n_backends) return bad("backend id out of range", CB_ERR_ARG);
  }
  // kernel adjacency through data edges
  std::vector<int2> kadj;
  for (int32_t v = 0; v < n; ++v)
    for (int32_t j = g->in_ptr[v]; j < g->in_ptr[v + 1]; ++j) {
      int32_t p = g->in_src[j];
      if (p < 0) continue;
      int32_t a = kernel_of[p], b = kernel_of[v];
      if (a != b) kadj.push_back(make_int2(std::min(a, b), std::max(a, b)));
    }
  std::sort(kadj.begin(), kadj.end(), [](int2 x, int2 y) { return x.x != y.x ? x.x < y.x : x.y < y.y; });
  kadj.erase(std::unique(kadj.begin(), kadj.end(), [](int2 x, int2 y) { return x.x == y.x && x.y == y.y; }),
             kadj.end());

  tick("kernel adjacency");
  // eligible slots and their replacements
  auto same_set = [&](int32_t a, int32_t b) {
    int32_t na = m->mem_ptr[a + 1] - m->mem_ptr[a];
    if (na != m->mem_ptr[b + 1] - m->mem_ptr[b]) return false;
    return std::equal(m->members.begin() + m->mem_ptr[a], m->members.begin() + m->mem_ptr[a + 1],
                      m->members.begin() + m->mem_ptr[b]);
  };
  std::vector<int32_t> slot_of_kernel(n_kernels, -1);
  std::vector<fx192> slot_rep;
  std::vector<int32_t> slot_cnt;
  P->rep_match_ptr.push_back(0);
  for (int32_t kk = 0; kk < n_kernels; ++kk) {
    if (backend_is_graph[kb[kk]]) continue;
    int32_t s = (int32_t)P->slot_kernel.size();
    slot_of_kernel[kk] = s;
    P->slot_kernel.push_back(kk);
    const int32_t km = kernel_match[kk];
    const int32_t r = m->root[km];
    int8_t kind = 0;
    fx192 rep = fx_zero();
    int32_t cnt = 0;
    for (int32_t c = m->group_ptr[r]; c < m->group_ptr[r + 1]; ++c)
      if (m->backend[c] == target_backend && same_set(c, km)) {
        kind = 1;
        P->rep_match.push_back(c);
        if (!fx_from_double(m->cost[c], rep)) return bad("cost outside exact range", CB_ERR_INEXACT);
        cnt = 1;
        break;
      }
    if (!kind) {
      kind = 2;
      size_t mark = P->rep_match.size();
      for (int32_t i = m->mem_ptr[km]; i < m->mem_ptr[km + 1]; ++i) {
        const int32_t u = m->members[i];
        int32_t found = -1;
        for (int32_t c = m->group_ptr[u]; c < m->group_ptr[u + 1]; ++c)
          if (m->backend[c] == target_backend && m->mem_ptr[c + 1] - m->mem_ptr[c] == 1) {
            found = c;
            break;
          }
        if (found < 0) {
          kind = 0;
          break;
        }
        P->rep_match.push_back(found);
        fx192 t;
        if (!fx_from_double(m->cost[found], t)) return bad("cost outside exact range", CB_ERR_INEXACT);
        fx_add(rep, t);
        ++cnt;
      }
      if (!kind) {
        P->rep_match.resize(mark);
        rep = fx_zero();
        cnt = 0;
      }
    }
    P->rep_kind.push_back(kind);
    P->rep_match_ptr.push_back((int32_t)P->rep_match.size());
    slot_rep.push_back(rep);
    slot_cnt.push_back(cnt);
  }
  P->k = (int32_t)P->slot_kernel.size();
  P->words = (P->k + 63) / 64;
  if (P->words == 0) P->words = 1;

  // fixed graph kernels: target-backend components become virtual units,
  // other graph backends form static regions
  DSU dsu(n_kernels);
  for (const int2& e : kadj) {
    bool ga = backend_is_graph[kb[e.x]], gb = backend_is_graph[kb[e.y]];
    if (ga && gb && kb[e.x] == kb[e.y]) dsu.unite(e.x, e.y);
  }
  fx192 cst = fx_zero();
  bool exact = true;
  std::vector<fx192> comp_sum(n_kernels, fx_zero());
  std::vector<int32_t> comp_cnt(n_kernels, 0);
  for (int32_t kk = 0; kk < n_kernels; ++kk) {
    if (!backend_is_graph[kb[kk]]) {
      fx192 t;
      exact &= fx_from_double(kc[kk], t);
      fx_add(cst, t);
      fx_add(cst, P->eps);
      continue;
    }
    int32_t r = dsu.find(kk);
    fx192 t;
    exact &= fx_from_double(kc[kk], t);
    fx_add(comp_sum[r], t);
    comp_cnt[r] += 1;
  }
  std::vector<int32_t> virtual_of(n_kernels, -1);
  std::vector<fx192> v_rep;
  std::vector<int32_t> v_cnt;
  for (int32_t kk = 0; kk < n_kernels; ++kk) {
    if (!backend_is_graph[kb[kk]] || dsu.find(kk) != kk) continue;
    if (kb[kk] == target_backend) {
      virtual_of[kk] = (int32_t)v_rep.size();
      v_rep.push_back(comp_sum[kk]);
      v_cnt.push_back(comp_cnt[kk]);
    } else {
      double base = fx_to_double(comp_sum[kk]);
      double r = region_r(region_alpha[kb[kk]], region_floor[kb[kk]], comp_cnt[kk]);
      fx192 t;
      exact &= fx_term(base, r, P->eps, t);
      fx_add(cst, t);
    }
  }
  if (!exact) return bad("a cost falls outside the exact accumulator range", CB_ERR_INEXACT);
  P->base_const = cst;

  // dynamic units: feasible eligible slots, then virtual units
  std::vector<int32_t> unit_of_slot(P->k, -1);
  P->infeas_mask.assign(P->words, 0ull);
  for (int32_t s = 0; s < P->k; ++s) {
    fx192 off;
    fx_from_double(kc[P->slot_kernel[s]], off);
    fx_add(off, P->eps);
    if (P->rep_kind[s] == 0) {
      P->infeas_mask[s >> 6] |= 1ull << (s & 63);
      P->infeasible_bits++;
      continue;
    }
    unit_of_slot[s] = (int32_t)P->unit_slot.size();
    P->unit_slot.push_back(s);
    P->unit_rep.push_back(slot_rep[s]);
    P->unit_cnt.push_back(slot_cnt[s]);
    P->unit_off.push_back(off);
  }
  const int32_t n_elig_units = (int32_t)P->unit_slot.size();
  for (size_t i = 0; i < v_rep.size(); ++i) {
    P->unit_slot.push_back(-1);
    P->unit_rep.push_back(v_rep[i]);
    P->unit_cnt.push_back(v_cnt[i]);
    P->unit_off.push_back(fx_zero());
  }
  P->n_virtual = (int32_t)v_rep.size();
  P->M = (int32_t)P->unit_slot.size();
  auto unit_of_kernel = [&](int32_t kk) -> int32_t {
    if (!backend_is_graph[kb[kk]]) {
      int32_t s = slot_of_kernel[kk];
      return unit_of_slot[s];
    }
    if (kb[kk] != target_backend) return -1;
    return n_elig_units + virtual_of[dsu.find(kk)];
  };
  for (const int2& e : kadj) {
    int32_t a = unit_of_kernel(e.x), b = unit_of_kernel(e.y);
    if (a < 0 || b < 0 || a == b) continue;
    P->edges.push_back(make_int2(std::min(a, b), std::max(a, b)));
  }
  std::sort(P->edges.begin(), P->edges.end(), [](int2 x, int2 y) { return x.x != y.x ? x.x < y.x : x.y < y.y; });
  P->edges.erase(std::unique(P->edges.begin(), P->edges.end(),
                             [](int2 x, int2 y) { return x.x == y.x && x.y == y.y; }),
                 P->edges.end());
  P->E = (int32_t)P->edges.size();
  int64_t max_cnt = 0;
  for (int32_t c : P->unit_cnt) max_cnt += c;
  P->rt.resize((size_t)max_cnt + 2);
  for (int64_t c = 0; c < (int64_t)P->rt.size(); ++c)
    P->rt[c] = region_r(region_alpha[target_backend], region_floor[target_backend], c);
  tick("units and edges");
  build_frontier_program(P, n_elig_units);
  tick("frontier program");
  // seed (all-zero genome) cost
  {
    fx192 tot = P->base_const;
    for (int32_t i = 0; i < P->n_virtual; ++i) {
      int32_t u = n_elig_units + i;
      fx192 t;
      fx_term(fx_to_double(P->unit_rep[u]), P->rt[P->unit_cnt[u]], P->eps, t);
      fx_add(tot, t);
    }
    P->seed_cost = fx_to_double(tot);
  }
  // device upload
  auto fail_cuda = [&](cudaError_t e) {
    delete P;
    cb_set_error(std::string("CUDA error in plan upload: ") + cudaGetErrorString(e));
    return CB_ERR_CUDA;
  };
  cudaError_t e;
  if ((e = P->d_unit_slot.upload(P->unit_slot)) != cudaSuccess) return fail_cuda(e);
  if ((e = P->d_unit_cnt.upload(P->unit_cnt)) != cudaSuccess) return fail_cuda(e);
  if ((e = P->d_unit_rep.upload(P->unit_rep)) != cudaSuccess) return fail_cuda(e);
  if ((e = P->d_unit_off.upload(P->unit_off)) != cudaSuccess) return fail_cuda(e);
  if ((e = P->d_edges.upload(P->edges)) != cudaSuccess) return fail_cuda(e);
  if ((e = P->d_infeas.upload(P->infeas_mask)) != cudaSuccess) return fail_cuda(e);
  if ((e = P->d_rt.upload(P->rt)) != cudaSuccess) return fail_cuda(e);
  if (P->F > 0) {
    if ((e = P->d_prog.upload(P->prog)) != cudaSuccess) return fail_cuda(e);
    if ((e = P->d_prog_slots.upload(P->prog_slots)) != cudaSuccess) return fail_cuda(e);
    if ((e = P->d_prog_last.upload(P->prog_last)) != cudaSuccess) return fail_cuda(e);
    if ((e = P->d_pos_of_bit.upload(P->pos_of_bit)) != cudaSuccess) return fail_cuda(e);
    if ((e = P->d_fixed_pos.upload(P->fixed_pos)) != cudaSuccess) return fail_cuda(e);
  }
  tick("uploads");
  if ((rc = build_anchor_plan(P)) != CB_OK || (rc = build_fsm_plan(P)) != CB_OK) {
    delete P;
    return rc;
  }
  if ((e = P->d_flags.alloc(2)) != cudaSuccess) return fail_cuda(e);
  cudaMemset(P->d_flags.p, 0, 2 * sizeof(unsigned long long));
  const size_t per_warp = (size_t)P->words * 8 + (size_t)P->M * (sizeof(fx192) + 8);
  P->smem_path = per_warp * 4 <= 200 * 1024;
  tick("anchor + fsm plans");
  *out = P;
  return CB_OK;
}

extern "C" int cb_es_plan_query(const cb_es_plan* p, cb_es_plan_info* info) {
  CB_ARG_CHECK(p && info, "cb_es_plan_query: null argument");
  info->genome_bits = p->k;
  info->words = p->words;
  info->units = p->M;
  info->fixed_units = p->n_virtual;
  info->edges = p->E;
  info->infeasible_bits = p->infeasible_bits;
  info->smem_path = p->smem_path ? 1 : 0;
  info->frontier_slots = p->F;
  info->seed_cost = p->seed_cost;
  info->window_shift = p->anchor_ok ? p->anchor_shift : -1;
  info->packed_labels = p->F > 0 && p->packed_ok ? (p->pa_ok && p->anchor_ok ? 2 : 1) : 0;
  info->fsm_transitions = p->fsm_ok ? (int32_t)std::min<int64_t>(p->fsm_entries, INT32_MAX) : 0;
  info->fsm_entry_bytes = p->fsm_ok ? (p->fsm_layout == 1 || p->fsm_layout == 3 ? 8 : p->fsm_layout == 2 ? 16 : 32) : 0;
  return CB_OK;
}

extern "C" int cb_es_plan_units(const cb_es_plan* p, int32_t* unit_bit, int32_t* unit_cnt,
                                int32_t* edges, int32_t* frontier_needed) {
  CB_ARG_CHECK(p, "cb_es_plan_units: null plan");
  if (unit_bit) std::copy(p->unit_slot.begin(), p->unit_slot.end(), unit_bit);
  if (unit_cnt) std::copy(p->unit_cnt.begin(), p->unit_cnt.end(), unit_cnt);
  if (edges)
    for (size_t i = 0; i < p->edges.size(); ++i) {
      edges[2 * i] = p->edges[i].x;
      edges[2 * i + 1] = p->edges[i].y;
    }
  if (frontier_needed) *frontier_needed = p->F_needed;
  return CB_OK;
}

extern "C" const char* cb_es_plan_kernel(const cb_es_plan* p) {
  // the kernel launch_fitness dispatches to (mirrors its decision order)
  if (!p) return "";
  const bool frontier = p->F > 0 && p->force_path != 0;
  if (frontier && p->force_path == 3) return "fitness_wide_kernel";
  if (frontier && p->fsm_ok && (p->force_path == 7 || (p->force_path == -1 && p->fsm_auto))) {
    static thread_local char fbuf[48];
    // fitness_fsm_kernel<F, W, L>: L = transition layout (1: 8 bytes, 2: 16, 3: mixed, 0: 32),
    // + 4 with the 8-byte shared delta table
    std::snprintf(fbuf, sizeof(fbuf), "fitness_fsm_kernel<%d, %d, %d>", p->F <= 4 ? 4 : p->F <= 6 ? 6 : 8,
                  p->words <= 4 ? p->words : 0,
                  p->fsm_layout + (p->fsm_d64 && p->fsm_layout != 0 ? 4 : 0));
    return fbuf;
  }
  if (frontier && p->pa_ok && p->anchor_ok && (p->force_path == 6 || p->force_path == -1)) {
    // fitness_pa_kernel<F, W>: W = genome words held in registers (0 = loaded on demand)
    static thread_local char buf[48];
    std::snprintf(buf, sizeof(buf), "fitness_pa_kernel<%d, %d>", p->F <= 4 ? 4 : p->F <= 6 ? 6 : 8,
                  p->words <= 4 ? p->words : 0);
    return buf;
  }
  if (frontier && p->packed_ok && p->anchor_ok && (p->force_path == 5 || p->force_path == -1)) {
    static const char* pk[] = {"fitness_packed128_kernel<uint32_t, 4>", "fitness_packed128_kernel<uint32_t, 6>",
                               "fitness_packed128_kernel<uint32_t, 8>", "fitness_packed128_kernel<uint64_t, 12>",
                               "fitness_packed128_kernel<uint64_t, 16>"};
    return pk[p->F <= 4 ? 0 : p->F <= 6 ? 1 : p->F <= 8 ? 2 : p->F <= 12 ? 3 : 4];
  }
  if (frontier && (p->force_path == 4 || (p->force_path == -1 && !p->packed_ok)))
    return p->anchor_ok && p->anchor_wide_ok ? "fitness_anchor_kernel" : "fitness_wide_kernel";
  if (frontier) {
    if (p->force_path != 2 && p->packed_ok) return "fitness_frontier2_kernel";
    return "fitness_frontier_kernel";
  }
  return p->smem_path ? "fitness_smem_kernel" : "fitness_global_kernel";
}

extern "C" int cb_es_plan_set_pool(cb_es_plan* p, int32_t entries) {
  CB_ARG_CHECK(p && entries >= 1 && entries <= 24, "cb_es_plan_set_pool: entries must be in [1, 24]");
  p->pool_entries = entries;
  return CB_OK;
}

extern "C" int cb_es_plan_set_path(cb_es_plan* p, int32_t path) {
  CB_ARG_CHECK(p && path >= -1 && path <= 7, "cb_es_plan_set_path: bad arguments");
  CB_ARG_CHECK(path != 7 || p->fsm_ok, "cb_es_plan_set_path: no finite-state program for this plan");
  CB_ARG_CHECK(path != 6 || (p->pa_ok && p->anchor_ok),
               "cb_es_plan_set_path: no packed anchor program (> 8 slots or values outside a 128-bit window)");
  CB_ARG_CHECK(path != 5 || (p->packed_ok && p->anchor_ok),
               "cb_es_plan_set_path: no packed 128-bit program (> 16 slots or values outside a 128-bit window)");
  CB_ARG_CHECK(path != 4 || p->anchor_ok,
               "cb_es_plan_set_path: no anchor program (> 64 slots or values outside a 128-bit window)");
  CB_ARG_CHECK(path < 1 || p->F > 0, "cb_es_plan_set_path: no frontier program for this plan");
  CB_ARG_CHECK(path < 1 || path > 2 || p->F <= FRONTIER_MAX,
               "cb_es_plan_set_path: the thread-per-genome kernels need <= 32 frontier slots");
  p->force_path = path;
  return CB_OK;
}

extern "C" int cb_es_plan_slots(const cb_es_plan* p, int32_t* slot_kernel, int8_t* rep_kind,
                                int32_t* rep_match_ptr, int32_t* rep_match) {
  CB_ARG_CHECK(p, "cb_es_plan_slots: null plan");
  if (slot_kernel) std::copy(p->slot_kernel.begin(), p->slot_kernel.end(), slot_kernel);
  if (rep_kind) std::copy(p->rep_kind.begin(), p->rep_kind.end(), rep_kind);
  if (rep_match_ptr) std::copy(p->rep_match_ptr.begin(), p->rep_match_ptr.end(), rep_match_ptr);
  if (rep_match) std::copy(p->rep_match.begin(), p->rep_match.end(), rep_match);
  return CB_OK;
}

extern "C" void cb_es_plan_destroy(cb_es_plan* p) { delete p; }

// ----------------------------------------------------------------- device
struct FitArgs {
  int32_t k, words, M, E;
  fx192 base_const, eps;
  const int32_t* unit_slot;
  const int32_t* unit_cnt;
  const fx192* unit_rep;
  const fx192* unit_off;
  const int2* edges;
  const uint64_t* infeas;
  const double* rt;
  unsigned long long* flags;
};

__device__ __forceinline__ int32_t uf_find(volatile int32_t* parent, int32_t x) {
  while (true) {
    int32_t p = parent[x];
    if (p == x) return x;
    int32_t gp = parent[p];
    if (gp != p) parent[x] = gp;  // path halving (only ever points to an ancestor)
    x = p;
  }
}

__device__ __forceinline__ void uf_union(int32_t* parent, int32_t a, int32_t b) {
  volatile int32_t* vp = parent;
  while (true) {
    a = uf_find(vp, a);
    b = uf_find(vp, b);
    if (a == b) return;
    int32_t hi = a > b ? a : b, lo = a > b ? b : a;
    if (atomicCAS(parent + hi, hi, lo) == hi) return;
  }
}

__device__ __forceinline__ void atomic_add_fx(fx192* dst, const fx192& v) {
  unsigned long long* w = reinterpret_cast<unsigned long long*>(dst->w);
  unsigned long long o0 = atomicAdd(w + 0, (unsigned long long)v.w[0]);
  unsigned long long c0 = (o0 + v.w[0]) < o0;
  unsigned long long a1 = v.w[1] + c0;
  unsigned long long c1 = a1 < c0;  // v.w[1] == max and c0
  unsigned long long o1 = atomicAdd(w + 1, a1);
  c1 += (o1 + a1) < o1;
  atomicAdd(w + 2, (unsigned long long)(v.w[2] + c1));
}

__device__ __forceinline__ fx192 shfl_xor_fx(const fx192& v, int m) {
  fx192 r;
  r.w[0] = __shfl_xor_sync(0xffffffffu, v.w[0], m);
  r.w[1] = __shfl_xor_sync(0xffffffffu, v.w[1], m);
  r.w[2] = __shfl_xor_sync(0xffffffffu, v.w[2], m);
  return r;
}

// One group (warp or CTA) evaluates one genome.  `parent`, `acc`, `cnt`
// point at this group's scratch (shared or global memory).
template <int GROUP>
__device__ void eval_genome(const FitArgs& a, const uint64_t* __restrict__ genome,
                            int32_t* parent, fx192* acc, int32_t* cnt, double* out,
                            fx192* red_scratch, int* red_flag) {
  const int t = threadIdx.x % GROUP;
  auto gsync = [&]() {
    if (GROUP == 32) __syncwarp();
    else __syncthreads();
  };
  // infeasibility
  int bad = 0;
  for (int32_t w = t; w < a.words; w += GROUP) bad |= (genome[w] & a.infeas[w]) != 0ull;
  bool any_bad;
  if (GROUP == 32) {
    any_bad = __any_sync(0xffffffffu, bad);
  } else {
    if (t == 0) *red_flag = 0;
    __syncthreads();
    if (bad) *red_flag = 1;
    __syncthreads();
    any_bad = *red_flag != 0;
    __syncthreads();
  }
  if (any_bad) {
    if (t == 0) *out = __longlong_as_double(0x7ff0000000000000ll);
    return;
  }
  // switch units on
  for (int32_t u = t; u < a.M; u += GROUP) {
    const int32_t s = a.unit_slot[u];
    const bool on = s < 0 || ((genome[s >> 6] >> (s & 63)) & 1ull);
    parent[u] = on ? u : -1;
    acc[u] = fx_zero();
    cnt[u] = 0;
  }
  gsync();
  // hook regions
  for (int32_t e = t; e < a.E; e += GROUP) {
    const int2 ed = a.edges[e];
    if (((volatile int32_t*)parent)[ed.x] >= 0 && ((volatile int32_t*)parent)[ed.y] >= 0)
      uf_union(parent, ed.x, ed.y);
  }
  gsync();
  // accumulate region sums; subtract the op-kernel terms of offloaded units
  fx192 part = fx_zero();
  for (int32_t u = t; u < a.M; u += GROUP) {
    if (((volatile int32_t*)parent)[u] < 0) continue;
    const int32_t r = uf_find((volatile int32_t*)parent, u);
    atomic_add_fx(acc + r, a.unit_rep[u]);
    atomicAdd(cnt + r, a.unit_cnt[u]);
    fx_sub(part, a.unit_off[u]);
  }
  gsync();
  bool inexact = false;
  for (int32_t u = t; u < a.M; u += GROUP) {
    if (((volatile int32_t*)parent)[u] != u) continue;
    const fx192 sum = acc[u];
    const double base = fx_to_double(sum);
    const double prod = __dmul_rn(base, a.rt[cnt[u]]);
    fx192 term;
    inexact |= !fx_from_double(prod, term);
    fx_add(term, a.eps);
    fx_add(part, term);
  }
  if (inexact) atomicAdd(a.flags + 0, 1ull);
  // reduce `part` over the group
  for (int off = 16; off > 0; off >>= 1) {
    fx192 o = shfl_xor_fx(part, off);
    fx_add(part, o);
  }
  if (GROUP == 32) {
    if (t == 0) {
      fx_add(part, a.base_const);
      *out = fx_to_double(part);
    }
  } else {
    const int warp = t >> 5;
    if ((t & 31) == 0) red_scratch[warp] = part;
    __syncthreads();
    if (t == 0) {
      fx192 tot = a.base_const;
      for (int w = 0; w < GROUP / 32; ++w) fx_add(tot, red_scratch[w]);
      *out = fx_to_double(tot);
    }
    __syncthreads();
  }
}

#define FIT_WARPS 4

__global__ void __launch_bounds__(FIT_WARPS * 32)
fitness_smem_kernel(FitArgs a, const uint64_t* __restrict__ pop, int64_t n, double* __restrict__ fit) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  const size_t per_warp = (size_t)a.M * (sizeof(fx192) + 8);
  unsigned char* base = smem + per_warp * warp;
  fx192* acc = reinterpret_cast<fx192*>(base);
  int32_t* parent = reinterpret_cast<int32_t*>(base + (size_t)a.M * sizeof(fx192));
  int32_t* cnt = parent + a.M;
  const int64_t stride = (int64_t)gridDim.x * FIT_WARPS;
  for (int64_t i = (int64_t)blockIdx.x * FIT_WARPS + warp; i < n; i += stride)
    eval_genome<32>(a, pop + i * a.words, parent, acc, cnt, fit + i, nullptr, nullptr);
}

#define FIT_CTA 256

__global__ void __launch_bounds__(FIT_CTA)
fitness_global_kernel(FitArgs a, const uint64_t* __restrict__ pop, int64_t n, double* __restrict__ fit,
                      unsigned char* scratch, size_t per_group) {
  __shared__ fx192 red[FIT_CTA / 32];
  __shared__ int flag;
  unsigned char* base = scratch + per_group * blockIdx.x;
  fx192* acc = reinterpret_cast<fx192*>(base);
  int32_t* parent = reinterpret_cast<int32_t*>(base + (size_t)a.M * sizeof(fx192));
  int32_t* cnt = parent + a.M;
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x)
    eval_genome<FIT_CTA>(a, pop + i * a.words, parent, acc, cnt, fit + i, red, &flag);
}

// ------------------------------------------------- frontier program kernel
// One thread per genome.  Units are visited in program order; an on unit
// opens a component in its slot and merges the components of its on earlier
// neighbours; when a slot's unit has seen its last neighbour the slot is
// released, and a component whose last member leaves is emitted as a
// region.  Component data (exact sum, kernel count, single-unit id) lives
// at its label slot, which is always an occupied slot.  Slot state is kept
// in shared memory, [field][slot][thread], so lanes never conflict.
#define FR_THREADS 128

template <int F>
struct FrontierSmem {
  uint64_t sum0[F][FR_THREADS];
  uint64_t sum1[F][FR_THREADS];
  uint64_t sum2[F][FR_THREADS];
  int32_t cnt[F][FR_THREADS];
  int32_t single[F][FR_THREADS];
  uint8_t label[F][FR_THREADS];
  uint8_t active[F][FR_THREADS];
};

template <int F>
__device__ __forceinline__ void fr_emit(FrontierSmem<F>& s, int L, int t, const UnitRec* __restrict__ prog,
                                        const double* __restrict__ rt, const fx192& eps, fx192& total,
                                        bool& inexact) {
  const int32_t one = s.single[L][t];
  if (one >= 0) {
    fx192 v;
    v.w[0] = __ldg(&prog[one].term1.w[0]);
    v.w[1] = __ldg(&prog[one].term1.w[1]);
    v.w[2] = __ldg(&prog[one].term1.w[2]);
    fx_add(total, v);
    return;
  }
  fx192 sum;
  sum.w[0] = s.sum0[L][t];
  sum.w[1] = s.sum1[L][t];
  sum.w[2] = s.sum2[L][t];
  const double prod = __dmul_rn(fx_to_double(sum), __ldg(rt + s.cnt[L][t]));
  fx192 term;
  inexact |= !fx_from_double(prod, term);
  fx_add(total, term);
  fx_add(total, eps);
}

template <int F>
__global__ void __launch_bounds__(FR_THREADS)
fitness_frontier_kernel(int32_t M, int32_t words, fx192 base_const, fx192 eps,
                        const UnitRec* __restrict__ prog, const uint8_t* __restrict__ slots,
                        const uint64_t* __restrict__ infeas, const double* __restrict__ rt,
                        const uint64_t* __restrict__ pop, int64_t n, double* __restrict__ fit,
                        unsigned long long* flags) {
  extern __shared__ __align__(16) unsigned char fr_smem[];
  FrontierSmem<F>& s = *reinterpret_cast<FrontierSmem<F>*>(fr_smem);
  const int t = threadIdx.x;
  bool inexact = false;
  // Lanes of a warp walk the program in lockstep: the genome loop is warp
  // uniform, infeasible / out-of-range lanes run with every unit off, and
  // multi-unit region terms (the expensive rounding) are deferred through a
  // one-entry queue that the warp drains together when any lane collides.
  const int64_t stride = (int64_t)gridDim.x * FR_THREADS;
  for (int64_t base = (int64_t)blockIdx.x * FR_THREADS + (t & ~31); base < n; base += stride) {
    const int64_t i = base + (t & 31);
    const bool in_range = i < n;
    const uint64_t* gen = pop + (in_range ? i : 0) * words;
    bool dead = !in_range;
    if (in_range)
      for (int32_t w = 0; w < words; ++w) dead |= (__ldg(gen + w) & __ldg(infeas + w)) != 0ull;
#pragma unroll
    for (int q = 0; q < F; ++q) s.active[q][t] = 0;
    fx192 total = base_const;
    fx192 pend = fx_zero();
    int32_t pend_cnt = 0;
    bool pend_valid = false;
    int32_t cached_word = -1;
    uint64_t word = 0;
    for (int32_t p = 0; p < M; ++p) {
      const UnitRec* r = prog + p;
      const int32_t bit = __ldg(&r->bit);
      bool on = !dead;
      if (bit >= 0) {
        const int32_t wi = bit >> 6;
        if (wi != cached_word) {
          word = dead ? 0ull : __ldg(gen + wi);
          cached_word = wi;
        }
        on = (word >> (bit & 63)) & 1ull;
      }
      const uint4 meta = __ldg(reinterpret_cast<const uint4*>(&r->back_off));
      // meta.x = back_off, meta.y = end_off, meta.z = slot|nback|nend|pad
      const int S = meta.z & 0xff;
      const int nback = (meta.z >> 8) & 0xff;
      const int nend = (meta.z >> 16) & 0xff;
      if (on) {
        if (bit >= 0) {
          fx192 off;
          off.w[0] = __ldg(&r->off.w[0]);
          off.w[1] = __ldg(&r->off.w[1]);
          off.w[2] = __ldg(&r->off.w[2]);
          fx_sub(total, off);
        }
        s.sum0[S][t] = __ldg(&r->rep.w[0]);
        s.sum1[S][t] = __ldg(&r->rep.w[1]);
        s.sum2[S][t] = __ldg(&r->rep.w[2]);
        s.cnt[S][t] = __ldg(&r->cnt);
        s.single[S][t] = p;
        s.label[S][t] = (uint8_t)S;
        s.active[S][t] = 1;
        for (int j = 0; j < nback; ++j) {
          const int b = __ldg(slots + meta.x + j);
          if (!s.active[b][t]) continue;
          const int A = s.label[S][t], B = s.label[b][t];
          if (A == B) continue;
          fx192 x, y;
          x.w[0] = s.sum0[A][t]; x.w[1] = s.sum1[A][t]; x.w[2] = s.sum2[A][t];
          y.w[0] = s.sum0[B][t]; y.w[1] = s.sum1[B][t]; y.w[2] = s.sum2[B][t];
          fx_add(x, y);
          s.sum0[A][t] = x.w[0]; s.sum1[A][t] = x.w[1]; s.sum2[A][t] = x.w[2];
          s.cnt[A][t] += s.cnt[B][t];
          s.single[A][t] = -1;
#pragma unroll
          for (int q = 0; q < F; ++q)
            if (s.active[q][t] && s.label[q][t] == B) s.label[q][t] = (uint8_t)A;
        }
      }
      for (int j = 0; j < nend; ++j) {
        const int e = __ldg(slots + meta.y + j);
        int emit_slot = -1;  // slot holding a multi-unit region to price now
        if (s.active[e][t]) {
          const int L = s.label[e][t];
          s.active[e][t] = 0;
          int other = -1;
#pragma unroll
          for (int q = 0; q < F; ++q)
            if (other < 0 && s.active[q][t] && s.label[q][t] == L) other = q;
          if (other < 0) {
            const int32_t one = s.single[L][t];
            if (one >= 0) {  // region of one unit: precomputed term
              fx192 v;
              v.w[0] = __ldg(&prog[one].term1.w[0]);
              v.w[1] = __ldg(&prog[one].term1.w[1]);
              v.w[2] = __ldg(&prog[one].term1.w[2]);
              fx_add(total, v);
            } else {
              const fx192 cur = {{s.sum0[L][t], s.sum1[L][t], s.sum2[L][t]}};
              const int32_t ccnt = s.cnt[L][t];
              if (!pend_valid) {
                pend = cur;
                pend_cnt = ccnt;
                pend_valid = true;
              } else {  // queue full: keep the new region, price the old one now
                s.sum0[L][t] = pend.w[0];  // slot L is free until the next unit
                s.sum1[L][t] = pend.w[1];
                s.sum2[L][t] = pend.w[2];
                s.cnt[L][t] = pend_cnt;
                pend = cur;
                pend_cnt = ccnt;
                emit_slot = L;
              }
            }
          } else if (L == e) {  // move the component to a slot that stays
            s.sum0[other][t] = s.sum0[e][t];
            s.sum1[other][t] = s.sum1[e][t];
            s.sum2[other][t] = s.sum2[e][t];
            s.cnt[other][t] = s.cnt[e][t];
            s.single[other][t] = s.single[e][t];
#pragma unroll
            for (int q = 0; q < F; ++q)
              if (s.active[q][t] && s.label[q][t] == e) s.label[q][t] = (uint8_t)other;
          }
        }
        if (__any_sync(0xffffffffu, emit_slot >= 0)) {
          if (emit_slot >= 0) {
            const int L = emit_slot;
            fx192 sum = {{s.sum0[L][t], s.sum1[L][t], s.sum2[L][t]}};
            const double prod = __dmul_rn(fx_to_double(sum), __ldg(rt + s.cnt[L][t]));
            fx192 term;
            inexact |= !fx_from_double(prod, term);
            fx_add(total, term);
            fx_add(total, eps);
          }
        }
      }
    }
    if (__any_sync(0xffffffffu, pend_valid)) {
      if (pend_valid) {
        const double prod = __dmul_rn(fx_to_double(pend), __ldg(rt + pend_cnt));
        fx192 term;
        inexact |= !fx_from_double(prod, term);
        fx_add(total, term);
        fx_add(total, eps);
      }
    }
    if (in_range) fit[i] = dead ? __longlong_as_double(0x7ff0000000000000ll) : fx_to_double(total);
  }
  if (inexact) atomicAdd(flags, 1ull);
}

// ------------------------------------- frontier program, packed-label form
// Same walk for programs with at most 16 slots, but the component labels of
// all slots live in one register (4 bits per slot) together with a nibble
// mask of the occupied slots, so relabelling, "does the component have
// another member" and slot (de)activation are a handful of branch-free ALU
// operations (SWAR zero-nibble tests) instead of loops over shared memory.
// Only the exact sums and the (count, single-unit) words sit in shared
// memory, indexed by slot.  Every step is predicated so the 32 genomes of a
// warp stay converged.
template <typename LT>
struct Nib;
template <>
struct Nib<uint32_t> {
  static constexpr uint32_t ONE = 0x11111111u, LOW3 = 0x77777777u;
};
template <>
struct Nib<uint64_t> {
  static constexpr uint64_t ONE = 0x1111111111111111ull, LOW3 = 0x7777777777777777ull;
};

template <typename LT>
__device__ __forceinline__ LT nib_eq(LT x, uint32_t v) {
  // nibble mask (0xF) of the nibbles of x equal to v
  const LT y = x ^ ((LT)v * Nib<LT>::ONE);
  const LT z = ~(((y & Nib<LT>::LOW3) + Nib<LT>::LOW3) | y | Nib<LT>::LOW3);
  return (z >> 3) * (LT)0xF;
}

template <typename LT>
__device__ __forceinline__ int nib_first(LT m) {
  if (sizeof(LT) == 8) return __ffsll((long long)m) - 1 >> 2;
  return __ffs((int)m) - 1 >> 2;
}

#define FR_QCAP 64

// Price queue entry `idx` (exact region sum, kernel count, owner lane) and
// add its term to the owner's accumulator (shared-memory multi-limb atomics:
// an owner can have several entries in one batch).
__device__ __forceinline__ void fr_price_entry(const uint64_t* qs0, const uint64_t* qs1,
                                               const uint64_t* qs2, const uint64_t* qm, int idx,
                                               const double* __restrict__ rt, const fx192& eps,
                                               uint64_t* tacc0, uint64_t* tacc1, uint64_t* tacc2,
                                               bool& inexact) {
  const fx192 sum = {{qs0[idx], qs1[idx], qs2[idx]}};
  const uint64_t m = qm[idx];
  const double prod = __dmul_rn(fx_to_double(sum), __ldg(rt + (uint32_t)m));
  fx192 term;
  inexact |= !fx_from_double(prod, term);
  fx_add(term, eps);
  const int owner = (int)(m >> 32);
  unsigned long long* w0 = reinterpret_cast<unsigned long long*>(tacc0 + owner);
  unsigned long long* w1 = reinterpret_cast<unsigned long long*>(tacc1 + owner);
  unsigned long long* w2 = reinterpret_cast<unsigned long long*>(tacc2 + owner);
  const unsigned long long o0 = atomicAdd(w0, (unsigned long long)term.w[0]);
  unsigned long long c = (o0 + term.w[0]) < o0;
  const unsigned long long a1 = term.w[1] + c;
  unsigned long long c1 = a1 < c;
  const unsigned long long o1 = atomicAdd(w1, a1);
  c1 += (o1 + a1) < o1;
  atomicAdd(w2, (unsigned long long)(term.w[2] + c1));
}

template <typename LT, int F>
__global__ void __launch_bounds__(FR_THREADS)
fitness_frontier2_kernel(int32_t M, int32_t words, fx192 base_const, fx192 eps,
                         const UnitRec* __restrict__ prog, const uint8_t* __restrict__ slots,
                         const uint64_t* __restrict__ infeas, const double* __restrict__ rt,
                         const uint64_t* __restrict__ pop, int64_t n, double* __restrict__ fit,
                         unsigned long long* flags) {
  extern __shared__ __align__(16) unsigned char fr_smem[];
  uint64_t (*s0)[FR_THREADS] = reinterpret_cast<uint64_t (*)[FR_THREADS]>(fr_smem);
  uint64_t (*s1)[FR_THREADS] = s0 + F;
  uint64_t (*s2)[FR_THREADS] = s1 + F;
  uint64_t (*cs)[FR_THREADS] = s2 + F;  // low 32: kernel count, high 32: single unit or -1
  const int t = threadIdx.x;
  const int lane = t & 31, warp = t >> 5;
  // per-warp queue of closed regions + per-lane term accumulators
  uint64_t* qbase = reinterpret_cast<uint64_t*>(cs + F) + (size_t)warp * 4 * FR_QCAP;
  uint64_t* qs0 = qbase;
  uint64_t* qs1 = qbase + FR_QCAP;
  uint64_t* qs2 = qbase + 2 * FR_QCAP;
  uint64_t* qm = qbase + 3 * FR_QCAP;  // low 32: kernel count, high 32: owner lane
  uint64_t* tbase = reinterpret_cast<uint64_t*>(cs + F) + (size_t)(FR_THREADS / 32) * 4 * FR_QCAP +
                    (size_t)warp * 96;
  uint64_t* tacc0 = tbase;
  uint64_t* tacc1 = tbase + 32;
  uint64_t* tacc2 = tbase + 64;
  tacc0[lane] = tacc1[lane] = tacc2[lane] = 0ull;
  __syncwarp();
  int qn = 0;
  bool inexact = false;
  const int64_t stride = (int64_t)gridDim.x * FR_THREADS;
  for (int64_t base = (int64_t)blockIdx.x * FR_THREADS + (t & ~31); base < n; base += stride) {
    const int64_t i = base + (t & 31);
    const bool in_range = i < n;
    const uint64_t* gen = pop + (in_range ? i : 0) * words;
    bool dead = !in_range;
    if (in_range)
      for (int32_t w = 0; w < words; ++w) dead |= (__ldg(gen + w) & __ldg(infeas + w)) != 0ull;
    LT lab = 0;  // nibble s: label of slot s
    LT act = 0;  // 0xF in nibble s while slot s is occupied
    fx192 total = base_const;
    int32_t cached_word = -1;
    uint64_t word = 0;
    for (int32_t p = 0; p < M; ++p) {
      const UnitRec* r = prog + p;
      const uint4 hot = __ldg(&r->hot);  // bit, slot|nback|nend, back nibbles, end nibbles
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
        if (bit >= 0) {
          const fx192 off = {{__ldg(&r->off.w[0]), __ldg(&r->off.w[1]), __ldg(&r->off.w[2])}};
          fx_sub(total, off);
        }
        s0[S][t] = __ldg(&r->rep.w[0]);
        s1[S][t] = __ldg(&r->rep.w[1]);
        s2[S][t] = __ldg(&r->rep.w[2]);
        cs[S][t] = ((uint64_t)(uint32_t)p << 32) | (uint32_t)__ldg(&r->cnt);
        act |= nibS;
        lab = (lab & ~nibS) | ((LT)S << (4 * S));
      }
      for (int j = 0; j < nback; ++j) {
        const int b = (hot.z >> (4 * j)) & 0xF;
        const uint32_t B = (uint32_t)(lab >> (4 * b)) & 0xF;
        const bool merge = on && ((act >> (4 * b)) & 1) && B != (uint32_t)S;
        if (merge) {
          fx192 x = {{s0[S][t], s1[S][t], s2[S][t]}};
          const fx192 y = {{s0[B][t], s1[B][t], s2[B][t]}};
          fx_add(x, y);
          s0[S][t] = x.w[0];
          s1[S][t] = x.w[1];
          s2[S][t] = x.w[2];
          const uint32_t c = (uint32_t)cs[S][t] + (uint32_t)cs[B][t];
          cs[S][t] = 0xffffffff00000000ull | c;
          const LT m = nib_eq<LT>(lab, B) & act;
          lab = (lab & ~m) | (((LT)S * Nib<LT>::ONE) & m);
        }
      }
      for (int j = 0; j < nend; ++j) {
        const int e = (hot.w >> (4 * j)) & 0xF;
        const LT nibE = (LT)0xF << (4 * e);
        int emit_slot = -1;
        if (act & nibE) {
          const uint32_t X = (uint32_t)(lab >> (4 * e)) & 0xF;
          act &= ~nibE;
          const LT others = nib_eq<LT>(lab, X) & act;
          if (others == 0) {  // last member leaves: the region is complete
            const uint64_t cw = cs[e][t];
            const int32_t one = (int32_t)(cw >> 32);
            if (one >= 0) {
              const UnitRec* tp = prog + one;
              const fx192 v = {{__ldg(&tp->term1.w[0]), __ldg(&tp->term1.w[1]),
                                __ldg(&tp->term1.w[2])}};
              fx_add(total, v);
            } else {
              emit_slot = e;  // multi-unit region: queued for warp-wide pricing
            }
          } else if (X == (uint32_t)e) {  // data moves to a member that stays
            const int tgt = nib_first<LT>(others);
            s0[tgt][t] = s0[e][t];
            s1[tgt][t] = s1[e][t];
            s2[tgt][t] = s2[e][t];
            cs[tgt][t] = cs[e][t];
            lab = (lab & ~others) | (((LT)tgt * Nib<LT>::ONE) & others);
          }
        }
        // Closed multi-unit regions of all lanes go to the warp's queue; once
        // 32 are waiting, every lane prices one (full-warp utilisation) and
        // adds the term to its owner's accumulator.
        const unsigned closing = __ballot_sync(0xffffffffu, emit_slot >= 0);
        if (closing) {
          if (emit_slot >= 0) {
            const int at = qn + __popc(closing & ((1u << lane) - 1u));
            qs0[at] = s0[emit_slot][t];
            qs1[at] = s1[emit_slot][t];
            qs2[at] = s2[emit_slot][t];
            qm[at] = ((uint64_t)lane << 32) | (uint32_t)cs[emit_slot][t];
          }
          qn += __popc(closing);
          if (qn >= 32) {
            __syncwarp();
            fr_price_entry(qs0, qs1, qs2, qm, lane, rt, eps, tacc0, tacc1, tacc2, inexact);
            __syncwarp();
            if (lane < qn - 32) {
              qs0[lane] = qs0[32 + lane];
              qs1[lane] = qs1[32 + lane];
              qs2[lane] = qs2[32 + lane];
              qm[lane] = qm[32 + lane];
            }
            __syncwarp();
            qn -= 32;
          }
        }
      }
    }
    __syncwarp();
    if (lane < qn) fr_price_entry(qs0, qs1, qs2, qm, lane, rt, eps, tacc0, tacc1, tacc2, inexact);
    qn = 0;
    __syncwarp();
    {
      const fx192 acc = {{tacc0[lane], tacc1[lane], tacc2[lane]}};
      fx_add(total, acc);
      tacc0[lane] = tacc1[lane] = tacc2[lane] = 0ull;
    }
    __syncwarp();
    if (in_range) fit[i] = dead ? __longlong_as_double(0x7ff0000000000000ll) : fx_to_double(total);
  }
  if (inexact) atomicAdd(flags, 1ull);
}

template <typename LT, int F>
static int launch_frontier2_t(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit,
                              cudaStream_t stream);

static FitArgs make_args(cb_es_plan* p) {
  FitArgs a;
  a.k = p->k;
  a.words = p->words;
  a.M = p->M;
  a.E = p->E;
  a.base_const = p->base_const;
  a.eps = p->eps;
  a.unit_slot = p->d_unit_slot.p;
  a.unit_cnt = p->d_unit_cnt.p;
  a.unit_rep = p->d_unit_rep.p;
  a.unit_off = p->d_unit_off.p;
  a.edges = p->d_edges.p;
  a.infeas = p->d_infeas.p;
  a.rt = p->d_rt.p;
  a.flags = p->d_flags.p;
  return a;
}

int cb_sm_count() {
  static int cached = 0;
  if (!cached) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    if (cached <= 0) cached = 148;
  }
  return cached;
}

template <int F>
static int launch_frontier_t(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit,
                             cudaStream_t stream) {
  const size_t smem = sizeof(FrontierSmem<F>);
  if (cb_smem_claim((const void*)fitness_frontier_kernel<F>, smem))
    CB_CUDA_TRY(cudaFuncSetAttribute(fitness_frontier_kernel<F>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  CB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fitness_frontier_kernel<F>,
                                                            FR_THREADS, smem));
  if (per_sm < 1) per_sm = 1;
  const int64_t want = (n + FR_THREADS - 1) / FR_THREADS;
  const int64_t grid = std::min<int64_t>(want, (int64_t)per_sm * cb_sm_count());
  fitness_frontier_kernel<F><<<(unsigned)grid, FR_THREADS, smem, stream>>>(
      p->M, p->words, p->base_const, p->eps, p->d_prog.p, p->d_prog_slots.p, p->d_infeas.p,
      p->d_rt.p, d_pop, n, d_fit, p->d_flags.p);
  CB_CUDA_TRY(cudaGetLastError());
  return CB_OK;
}

template <typename LT, int F>
static int launch_frontier2_t(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit,
                              cudaStream_t stream) {
  const size_t smem = ((size_t)4 * F * FR_THREADS + (size_t)(FR_THREADS / 32) * (4 * FR_QCAP + 96)) *
                      sizeof(uint64_t);
  if (cb_smem_claim((const void*)fitness_frontier2_kernel<LT, F>, smem))
    CB_CUDA_TRY(cudaFuncSetAttribute(fitness_frontier2_kernel<LT, F>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  CB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fitness_frontier2_kernel<LT, F>,
                                                            FR_THREADS, smem));
  if (per_sm < 1) per_sm = 1;
  const int64_t want = (n + FR_THREADS - 1) / FR_THREADS;
  const int64_t grid = std::min<int64_t>(want, (int64_t)per_sm * cb_sm_count());
  fitness_frontier2_kernel<LT, F><<<(unsigned)grid, FR_THREADS, smem, stream>>>(
      p->M, p->words, p->base_const, p->eps, p->d_prog.p, p->d_prog_slots.p, p->d_infeas.p,
      p->d_rt.p, d_pop, n, d_fit, p->d_flags.p);
  CB_CUDA_TRY(cudaGetLastError());
  return CB_OK;
}

static int launch_fitness(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit,
                          cudaStream_t stream) {
  if (n <= 0) return CB_OK;
  const bool frontier = p->F > 0 && p->force_path != 0;
  if (frontier && p->force_path == 3) return launch_fitness_wide(p, d_pop, n, d_fit, stream);
  if (frontier && p->fsm_ok && (p->force_path == 7 || (p->force_path == -1 && p->fsm_auto)))
    return launch_fitness_fsm(p, d_pop, n, d_fit, stream);
  if (frontier && p->pa_ok && p->anchor_ok && (p->force_path == 6 || p->force_path == -1))
    return launch_fitness_packed_anchor(p, d_pop, n, d_fit, stream);
  if (frontier && p->packed_ok && p->anchor_ok && (p->force_path == 5 || p->force_path == -1))
    return launch_fitness_packed128(p, d_pop, n, d_fit, stream);
  if (frontier && (p->force_path == 4 || (p->force_path == -1 && !p->packed_ok)))
    return p->anchor_ok ? launch_fitness_anchor(p, d_pop, n, d_fit, stream)
                        : launch_fitness_wide(p, d_pop, n, d_fit, stream);
  if (frontier) {
    if (p->force_path != 2 && p->packed_ok) {
      // smallest slot count that fits: less shared memory, more resident warps
      if (p->F <= 4) return launch_frontier2_t<uint32_t, 4>(p, d_pop, n, d_fit, stream);
      if (p->F <= 6) return launch_frontier2_t<uint32_t, 6>(p, d_pop, n, d_fit, stream);
      if (p->F <= 8) return launch_frontier2_t<uint32_t, 8>(p, d_pop, n, d_fit, stream);
      if (p->F <= 12) return launch_frontier2_t<uint64_t, 12>(p, d_pop, n, d_fit, stream);
      if (p->F <= 16) return launch_frontier2_t<uint64_t, 16>(p, d_pop, n, d_fit, stream);
    }
    if (p->F <= 8) return launch_frontier_t<8>(p, d_pop, n, d_fit, stream);
    if (p->F <= 16) return launch_frontier_t<16>(p, d_pop, n, d_fit, stream);
    return launch_frontier_t<32>(p, d_pop, n, d_fit, stream);
  }
  FitArgs a = make_args(p);
  if (p->smem_path) {
    const size_t smem = (size_t)FIT_WARPS * p->M * (sizeof(fx192) + 8);
    if (smem > 48 * 1024 && cb_smem_claim((const void*)fitness_smem_kernel, smem))
      CB_CUDA_TRY(cudaFuncSetAttribute(fitness_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)std::max<size_t>(smem, 48 * 1024)));
    int per_sm = 0;
    CB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fitness_smem_kernel,
                                                              FIT_WARPS * 32, smem));
    if (per_sm < 1) per_sm = 1;
    int64_t want = (n + FIT_WARPS - 1) / FIT_WARPS;
    int64_t grid = std::min<int64_t>(want, (int64_t)per_sm * cb_sm_count());
    fitness_smem_kernel<<<(unsigned)grid, FIT_WARPS * 32, smem, stream>>>(a, d_pop, n, d_fit);
  } else {
    const size_t per_group = ((size_t)p->M * (sizeof(fx192) + 8) + 255) & ~(size_t)255;
    int64_t grid = std::min<int64_t>(n, (int64_t)4 * cb_sm_count());
    if (p->scratch_per_group != per_group || p->scratch_groups < grid) {
      CB_CUDA_TRY(p->d_scratch.alloc(per_group * grid));
      p->scratch_per_group = per_group;
      p->scratch_groups = (int32_t)grid;
    }
    fitness_global_kernel<<<(unsigned)grid, FIT_CTA, 0, stream>>>(a, d_pop, n, d_fit, p->d_scratch.p,
                                                                   per_group);
  }
  CB_CUDA_TRY(cudaGetLastError());
  return CB_OK;
}

extern "C" int cb_fitness_device(cb_es_plan* p, const uint64_t* d_pop, int64_t n, double* d_fit,
                                 void* stream) {
  CB_ARG_CHECK(p && (n == 0 || (d_pop && d_fit)), "cb_fitness_device: bad arguments");
  return launch_fitness(p, d_pop, n, d_fit, (cudaStream_t)stream);
}

extern "C" int cb_fitness_host(cb_es_plan* p, const uint64_t* h_pop, int64_t n, double* h_fit) {
  CB_ARG_CHECK(p && (n == 0 || (h_pop && h_fit)), "cb_fitness_host: bad arguments");
  if (n == 0) return CB_OK;
  const size_t words = (size_t)n * p->words;
  if (p->d_pop_stage.n < words) CB_CUDA_TRY(p->d_pop_stage.alloc(words));
  if (p->d_fit_stage.n < (size_t)n) CB_CUDA_TRY(p->d_fit_stage.alloc((size_t)n));
  // Chunked pipeline: the H2D copy of chunk i+1 and the D2H copy of chunk
  // i-1 overlap the fitness kernel of chunk i (copies are asynchronous when
  // the host buffers are pinned), and consecutive chunks' kernels alternate
  // between two streams so one fills the SMs the other's tail leaves idle.
  // A chunk holds at least 512 genomes per SM (half a wave of the walks)
  // and at most an eighth of the batch.
  int64_t per_sm = 512;  // A/B (tools/e2e_ab.py): 512 > 256, 1024, 2048 on the 100k DAG
  if (const char* e = getenv("CB_HOST_CHUNK_PER_SM")) per_sm = std::max(1, atoi(e));
  const int64_t chunk = std::max<int64_t>((int64_t)cb_sm_count() * per_sm, (n + 7) / 8);
  if (n <= chunk) {
    // one chunk (small batches, e.g. one `evolve` generation): copy in, price,
    // copy out on the plan's own stream -- no per-call stream / event setup
    if (!p->host_stream) CB_CUDA_TRY(cudaStreamCreateWithFlags(&p->host_stream, cudaStreamNonBlocking));
    cudaStream_t s1 = p->host_stream;
    CB_CUDA_TRY(cudaMemcpyAsync(p->d_pop_stage.p, h_pop, words * sizeof(uint64_t), cudaMemcpyHostToDevice, s1));
    int rc1 = launch_fitness(p, p->d_pop_stage.p, n, p->d_fit_stage.p, s1);
    if (rc1 != CB_OK) return rc1;
    CB_CUDA_TRY(cudaMemcpyAsync(h_fit, p->d_fit_stage.p, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, s1));
    CB_CUDA_TRY(cudaStreamSynchronize(s1));
    unsigned long long flags1[2] = {0, 0};
    CB_CUDA_TRY(cudaMemcpy(flags1, p->d_flags.p, sizeof(flags1), cudaMemcpyDeviceToHost));
    if (flags1[0]) {
      cb_set_error("a region cost fell outside the exact accumulator range");
      return CB_ERR_INEXACT;
    }
    return CB_OK;
  }
  cudaStream_t s_in, s_run2[2], s_out;
  CB_CUDA_TRY(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking));
  CB_CUDA_TRY(cudaStreamCreateWithFlags(&s_run2[0], cudaStreamNonBlocking));
  CB_CUDA_TRY(cudaStreamCreateWithFlags(&s_run2[1], cudaStreamNonBlocking));
  CB_CUDA_TRY(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking));
  int64_t ci = 0;
  std::vector<cudaEvent_t> copied, priced;
  int rc = CB_OK;
  for (int64_t lo = 0; lo < n && rc == CB_OK; lo += chunk) {
    const int64_t cnt = std::min<int64_t>(chunk, n - lo);
    cudaEvent_t e_in, e_run;
    cudaEventCreateWithFlags(&e_in, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&e_run, cudaEventDisableTiming);
    copied.push_back(e_in);
    priced.push_back(e_run);
    uint64_t* dpop = p->d_pop_stage.p + (size_t)lo * p->words;
    double* dfit = p->d_fit_stage.p + lo;
    if (cudaMemcpyAsync(dpop, h_pop + (size_t)lo * p->words, (size_t)cnt * p->words * sizeof(uint64_t),
                        cudaMemcpyHostToDevice, s_in) != cudaSuccess) {
      rc = CB_ERR_CUDA;
      break;
    }
    cudaEventRecord(e_in, s_in);
    // the global union-find kernel shares one scratch area: keep it on one stream
    const bool shared_scratch = !(p->F > 0 && p->force_path != 0) && !p->smem_path;
    cudaStream_t s_run = s_run2[shared_scratch ? 0 : (ci++ & 1)];
    cudaStreamWaitEvent(s_run, e_in, 0);
    rc = launch_fitness(p, dpop, cnt, dfit, s_run);
    cudaEventRecord(e_run, s_run);
    cudaStreamWaitEvent(s_out, e_run, 0);
    if (cudaMemcpyAsync(h_fit + lo, dfit, (size_t)cnt * sizeof(double), cudaMemcpyDeviceToHost,
                        s_out) != cudaSuccess)
      rc = CB_ERR_CUDA;
  }
  cudaError_t se = cudaStreamSynchronize(s_out);
  cudaStreamSynchronize(s_run2[0]);
  cudaStreamSynchronize(s_run2[1]);
  cudaStreamSynchronize(s_in);
  for (cudaEvent_t e : copied) cudaEventDestroy(e);
  for (cudaEvent_t e : priced) cudaEventDestroy(e);
  cudaStreamDestroy(s_in);
  cudaStreamDestroy(s_run2[0]);
  cudaStreamDestroy(s_run2[1]);
  cudaStreamDestroy(s_out);
  if (rc == CB_ERR_CUDA || se != cudaSuccess) {
    cb_set_error(std::string("cb_fitness_host: ") + cudaGetErrorString(cudaGetLastError()));
    return CB_ERR_CUDA;
  }
  if (rc != CB_OK) return rc;
  unsigned long long flags[2] = {0, 0};
  CB_CUDA_TRY(cudaMemcpy(flags, p->d_flags.p, sizeof(flags), cudaMemcpyDeviceToHost));
  if (flags[0]) {
    cb_set_error("a region cost fell outside the exact accumulator range");
    return CB_ERR_INEXACT;
  }
  return CB_OK;
}
