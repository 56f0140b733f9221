/*
 * oracle.c -- CPU restatement of the reference placement-search hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker: tests/, smoke() and
 * bench.py's cpu_baseline / --impl reference legs may call it; the product
 * (paper_2111_00655_b200) never does.  It restates the reference algorithms
 * literally, without the device reformulations:
 *
 *   or_match_at      tensorplace/matching.py:53-103 (recursive walk with a
 *                    per-node bound-subtree map, then the single-exit check)
 *   or_kernel_cost   tensorplace/cost.py:121-138 (node cost, fsum, discount)
 *   or_dp            tensorplace/dp.py:71-179 (Algorithm 1: frontier queue in
 *                    (depth, id) order, one state per covered node set,
 *                    every stored state relaxed for every candidate, ties on
 *                    the sorted (registration index, node tuple) key)
 *   or_fitness       tensorplace/evolution.py:65-119, :346-371 (decode) and
 *                    tensorplace/cost.py:320-373 (graph-level cost)
 *
 * fsum is restated as an exact Kulisch accumulator over the whole double
 * range followed by one round-to-nearest-even, which is what math.fsum
 * returns.  Pinned against reference outputs in tests/golden/.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ exact sum */
#define KL 36 /* 64-bit limbs; bit 0 weighs 2^-1152 */
typedef struct {
  uint64_t w[KL];
  int bad;
} ksum;

static void ks_zero(ksum* k) { memset(k, 0, sizeof(*k)); }

static void ks_add(ksum* k, double d) {
  uint64_t bits;
  memcpy(&bits, &d, 8);
  if ((bits << 1) == 0) return;
  if (bits >> 63 || ((bits >> 52) & 0x7ff) == 0x7ff) {
    k->bad = 1;
    return;
  }
  int ex = (int)((bits >> 52) & 0x7ff);
  uint64_t m = bits & ((1ull << 52) - 1);
  int e;
  if (ex == 0) e = -1074;
  else {
    m |= 1ull << 52;
    e = ex - 1075;
  }
  int pos = e + 1152;
  int limb = pos >> 6, off = pos & 63;
  uint64_t lo = m << off, hi = off ? (m >> (64 - off)) : 0;
  uint64_t s = k->w[limb] + lo;
  uint64_t c = s < lo;
  k->w[limb] = s;
  int i = limb + 1;
  uint64_t add = hi + c; /* hi < 2^53 so no overflow */
  while (add && i < KL) {
    uint64_t t = k->w[i] + add;
    add = t < add;
    k->w[i] = t;
    ++i;
  }
}

static void ks_merge(ksum* a, const ksum* b) {
  uint64_t c = 0;
  for (int i = 0; i < KL; ++i) {
    uint64_t t = a->w[i] + c;
    uint64_t c1 = t < c;
    uint64_t s = t + b->w[i];
    c = c1 + (s < t);
    a->w[i] = s;
  }
  a->bad |= b->bad;
}

static int ks_bit(const ksum* k, int i) { return (int)((k->w[i >> 6] >> (i & 63)) & 1ull); }

static double ks_round(const ksum* k) {
  int top = -1;
  for (int i = KL - 1; i >= 0 && top < 0; --i)
    if (k->w[i]) top = i * 64 + 63 - __builtin_clzll(k->w[i]);
  if (top < 0) return 0.0;
  /* value = sum bit_i 2^(i-1152); take 53 bits from `top` down */
  int low = top - 52;
  if (low < 0) low = 0; /* subnormal territory: never reached for costs */
  /* bits [low, top] (at most 53) from the two limbs they span */
  int lb = low >> 6, lo = low & 63;
  unsigned __int128 win = (unsigned __int128)k->w[lb];
  if (lb + 1 < KL) win |= (unsigned __int128)k->w[lb + 1] << 64;
  uint64_t m = (uint64_t)(win >> lo) & ((top - low == 63) ? ~0ull : ((1ull << (top - low + 1)) - 1ull));
  if (low > 0) {
    int rb = ks_bit(k, low - 1);
    /* sticky: any bit below low - 1, limb by limb */
    int sticky = 0, b = low - 2;
    if (b >= 0) {
      int limb = b >> 6, off = b & 63;
      uint64_t mask = off == 63 ? ~0ull : ((1ull << (off + 1)) - 1ull);
      sticky = (k->w[limb] & mask) != 0;
      for (int i = limb - 1; i >= 0 && !sticky; --i) sticky = k->w[i] != 0;
    }
    if (rb && (sticky || (m & 1))) m += 1;
  }
  return ldexp((double)m, low - 1152);
}

/* ---------------------------------------------------------------- graph */
typedef struct {
  int n;
  const int32_t *kind, *in_ptr, *in_src;
  const uint8_t* is_output;
  const double* volume;
  const int32_t *attr_ptr, *attr_key;
  const int8_t* attr_tag;
  const int64_t* attr_ival;
  const double* attr_fval;
  int32_t *out_ptr, *out_dst; /* distinct consumers */
  int32_t* depth;
  int32_t* pop; /* nodes in (depth, index) order */
} og_t;

typedef struct {
  int n_pat;
  const int32_t *pos_ptr, *kind, *nargs, *parent, *argidx, *sid, *con_ptr, *con_key;
  const int8_t* con_op;
  const int32_t* con_val_ptr;
  const int8_t* val_tag;
  const int64_t* val_ival;
  const double* val_fval;
  const int64_t *con_lo, *con_hi;
  const int32_t* backend;
} op_t;

static int cmp_pop(const void* a, const void* b, void* ctx);

static og_t* g_sort_ctx;
static int cmp_pop_q(const void* a, const void* b) {
  int x = *(const int*)a, y = *(const int*)b;
  if (g_sort_ctx->depth[x] != g_sort_ctx->depth[y]) return g_sort_ctx->depth[x] - g_sort_ctx->depth[y];
  return x - y;
}

/* topological order (Kahn, smallest index first) -> depths and pop order;
 * restates graph.py:156-182 */
static int og_prepare(og_t* g) {
  int n = g->n;
  int* cnt = calloc(n + 1, sizeof(int));
  g->out_ptr = calloc(n + 1, sizeof(int32_t));
  /* collect distinct consumers */
  int nnz = g->in_ptr[n];
  int32_t* tmp_dst = malloc(sizeof(int32_t) * (nnz + 1));
  int32_t* fill = calloc(n + 1, sizeof(int32_t));
  for (int v = 0; v < n; ++v)
    for (int j = g->in_ptr[v]; j < g->in_ptr[v + 1]; ++j)
      if (g->in_src[j] >= 0) cnt[g->in_src[j] + 1]++;
  for (int v = 0; v < n; ++v) cnt[v + 1] += cnt[v];
  for (int v = 0; v < n; ++v)
    for (int j = g->in_ptr[v]; j < g->in_ptr[v + 1]; ++j) {
      int s = g->in_src[j];
      if (s < 0) continue;
      int at = cnt[s] + fill[s];
      int dup = 0;
      for (int q = cnt[s]; q < at; ++q) dup |= tmp_dst[q] == v;
      if (!dup) tmp_dst[cnt[s] + fill[s]++] = v;
    }
  g->out_dst = malloc(sizeof(int32_t) * (nnz + 1));
  int k = 0;
  for (int v = 0; v < n; ++v) {
    g->out_ptr[v] = k;
    for (int q = 0; q < fill[v]; ++q) g->out_dst[k++] = tmp_dst[cnt[v] + q];
  }
  g->out_ptr[n] = k;
  free(tmp_dst);
  free(fill);
  free(cnt);
  /* Kahn with a binary heap over indices */
  int* pend = calloc(n, sizeof(int));
  for (int v = 0; v < n; ++v) {
    for (int j = g->in_ptr[v]; j < g->in_ptr[v + 1]; ++j) {
      int s = g->in_src[j], dup = 0;
      if (s < 0) continue;
      for (int q = g->in_ptr[v]; q < j; ++q) dup |= g->in_src[q] == s;
      if (!dup) pend[v]++;
    }
  }
  int* heap = malloc(sizeof(int) * (n + 1));
  int hn = 0;
#define HPUSH(x)                                                          \
  do {                                                                    \
    int _i = hn++;                                                        \
    heap[_i] = (x);                                                       \
    while (_i && heap[(_i - 1) / 2] > heap[_i]) {                         \
      int _t = heap[_i]; heap[_i] = heap[(_i - 1) / 2]; heap[(_i - 1) / 2] = _t; \
      _i = (_i - 1) / 2;                                                  \
    }                                                                     \
  } while (0)
  for (int v = 0; v < n; ++v)
    if (!pend[v]) HPUSH(v);
  g->depth = calloc(n, sizeof(int32_t));
  int done = 0;
  while (hn) {
    int v = heap[0];
    heap[0] = heap[--hn];
    int i = 0;
    for (;;) {
      int l = 2 * i + 1, r = l + 1, m = i;
      if (l < hn && heap[l] < heap[m]) m = l;
      if (r < hn && heap[r] < heap[m]) m = r;
      if (m == i) break;
      int t = heap[i]; heap[i] = heap[m]; heap[m] = t;
      i = m;
    }
    int d = -1;
    for (int j = g->in_ptr[v]; j < g->in_ptr[v + 1]; ++j)
      if (g->in_src[j] >= 0 && g->depth[g->in_src[j]] > d) d = g->depth[g->in_src[j]];
    g->depth[v] = d + 1;
    ++done;
    for (int j = g->out_ptr[v]; j < g->out_ptr[v + 1]; ++j)
      if (--pend[g->out_dst[j]] == 0) HPUSH(g->out_dst[j]);
  }
#undef HPUSH
  free(heap);
  free(pend);
  if (done != n) return -1;
  g->pop = malloc(sizeof(int32_t) * (n + 1));
  for (int v = 0; v < n; ++v) g->pop[v] = v;
  g_sort_ctx = g;
  qsort(g->pop, n, sizeof(int32_t), cmp_pop_q);
  return 0;
}

static void og_free(og_t* g) {
  free(g->out_ptr);
  free(g->out_dst);
  free(g->depth);
  free(g->pop);
}

/* -------------------------------------------------------------- matcher */
static int int_like(int8_t t) { return t == 0 || t == 3; }

static int py_eq(int8_t ta, int64_t ia, double fa, int8_t tb, int64_t ib, double fb) {
  if (ta == 2 || tb == 2) return ta == tb && ia == ib;
  if (ta == 4 || tb == 4) return 0;
  if (int_like(ta) && int_like(tb)) return ia == ib;
  if (ta == 1 && tb == 1) return fa == fb;
  double f = int_like(ta) ? fb : fa;
  int64_t i = int_like(ta) ? ia : ib;
  if (f != f || f != floor(f) || f < -9223372036854775808.0 || f >= 9223372036854775808.0) return 0;
  return (int64_t)f == i;
}

static int cons_ok(const og_t* g, const op_t* p, int P, int node) {
  for (int c = p->con_ptr[P]; c < p->con_ptr[P + 1]; ++c) {
    int slot = -1;
    for (int j = g->attr_ptr[node]; j < g->attr_ptr[node + 1]; ++j)
      if (g->attr_key[j] == p->con_key[c]) slot = j;
    if (slot < 0) return 0;
    if (p->con_op[c] == 2) {
      if (g->attr_tag[slot] != 0) return 0;
      if (g->attr_ival[slot] < p->con_lo[c] || g->attr_ival[slot] > p->con_hi[c]) return 0;
      continue;
    }
    int any = 0;
    for (int v = p->con_val_ptr[c]; v < p->con_val_ptr[c + 1]; ++v)
      any |= py_eq(g->attr_tag[slot], g->attr_ival[slot], g->attr_fval[slot], p->val_tag[v],
                   p->val_ival[v], p->val_fval[v]);
    if (!any) return 0;
  }
  return 1;
}

typedef struct {
  int* bind;   /* local position -> node */
  int* sidmap; /* node -> structural id bound there, -1 */
  int* touched;
  int ntouched;
} walk_t;

static int walk(const og_t* g, const op_t* p, int base, int local, int node, walk_t* w) {
  int P = base + local;
  if (g->kind[node] != p->kind[P]) return 0;
  if (!cons_ok(g, p, P, node)) return 0;
  int arity = g->in_ptr[node + 1] - g->in_ptr[node];
  if (p->nargs[P] && p->nargs[P] != arity) return 0;
  int prior = w->sidmap[node];
  if (prior >= 0 && prior != p->sid[P]) return 0;
  if (prior < 0) w->touched[w->ntouched++] = node;
  w->sidmap[node] = p->sid[P];
  w->bind[local] = node;
  return 1;
}

/* Children are visited in argument order: the compiled tables list every
 * position in pre-order, so scanning forward for `parent == local` yields
 * them in order. */
static int walk_all(const og_t* g, const op_t* p, int pat, int local, int node, walk_t* w) {
  int base = p->pos_ptr[pat], npos = p->pos_ptr[pat + 1] - base;
  if (!walk(g, p, base, local, node, w)) return 0;
  for (int q = local + 1; q < npos; ++q) {
    if (p->parent[base + q] != local) continue;
    int producer = g->in_src[g->in_ptr[node] + p->argidx[base + q]];
    if (producer < 0) return 0;
    if (!walk_all(g, p, pat, q, producer, w)) return 0;
  }
  return 1;
}

static int cmp_int(const void* a, const void* b) {
  int x = *(const int*)a, y = *(const int*)b;
  return (x > y) - (x < y);
}

/* match_at: returns 1 and fills members (sorted) / bind; restates
 * matching.py:53-103 */
static int match_at_impl(const og_t* g, const op_t* p, int root, int pat, walk_t* w,
                         int* members, int* nmem) {
  w->ntouched = 0;
  int ok = walk_all(g, p, pat, 0, root, w);
  for (int i = 0; i < w->ntouched; ++i) w->sidmap[w->touched[i]] = -1;
  if (!ok) return 0;
  int base = p->pos_ptr[pat], npos = p->pos_ptr[pat + 1] - base;
  int k = 0;
  for (int i = 0; i < npos; ++i) {
    int v = w->bind[i], dup = 0;
    for (int j = 0; j < k; ++j) dup |= members[j] == v;
    if (!dup) members[k++] = v;
  }
  qsort(members, k, sizeof(int), cmp_int);
  *nmem = k;
  for (int i = 0; i < k; ++i) {
    int u = members[i];
    if (u == root) continue;
    if (g->is_output[u]) return 0;
    for (int j = g->out_ptr[u]; j < g->out_ptr[u + 1]; ++j) {
      int c = g->out_dst[j];
      if (!bsearch(&c, members, k, sizeof(int), cmp_int)) return 0;
    }
  }
  return 1;
}

/* Table of all candidate matches: for every node, the patterns rooted at
 * its kind in registration order (registry.py:135-145). */
typedef struct {
  int n_match;
  int32_t *group_ptr, *pat, *root, *mem_ptr, *members, *bind_ptr, *binds;
} mt_t;

static void mt_free(mt_t* m) {
  free(m->group_ptr); free(m->pat); free(m->root); free(m->mem_ptr);
  free(m->members); free(m->bind_ptr); free(m->binds);
}

static int build_matches(const og_t* g, const op_t* p, const int32_t* kind_pat_ptr,
                         const int32_t* kind_pat, int n_kinds, mt_t* mt) {
  int n = g->n, maxpos = 1;
  for (int i = 0; i < p->n_pat; ++i)
    if (p->pos_ptr[i + 1] - p->pos_ptr[i] > maxpos) maxpos = p->pos_ptr[i + 1] - p->pos_ptr[i];
  walk_t w;
  w.bind = malloc(sizeof(int) * maxpos);
  w.touched = malloc(sizeof(int) * (maxpos + 1));
  w.sidmap = malloc(sizeof(int) * (n + 1));
  for (int v = 0; v < n; ++v) w.sidmap[v] = -1;
  int cap = 1024, mcap = 4096, bcap = 4096;
  memset(mt, 0, sizeof(*mt));
  mt->group_ptr = calloc(n + 1, sizeof(int32_t));
  mt->pat = malloc(sizeof(int32_t) * cap);
  mt->root = malloc(sizeof(int32_t) * cap);
  mt->mem_ptr = malloc(sizeof(int32_t) * (cap + 1));
  mt->bind_ptr = malloc(sizeof(int32_t) * (cap + 1));
  mt->members = malloc(sizeof(int32_t) * mcap);
  mt->binds = malloc(sizeof(int32_t) * bcap);
  int* mem = malloc(sizeof(int) * maxpos);
  int cnt = 0, nm = 0, nb = 0;
  mt->mem_ptr[0] = 0;
  mt->bind_ptr[0] = 0;
  for (int v = 0; v < n; ++v) {
    mt->group_ptr[v] = cnt;
    int k = g->kind[v];
    if (k < 0 || k >= n_kinds) continue;
    for (int j = kind_pat_ptr[k]; j < kind_pat_ptr[k + 1]; ++j) {
      int pat = kind_pat[j], nmem;
      if (!match_at_impl(g, p, v, pat, &w, mem, &nmem)) continue;
      int npos = p->pos_ptr[pat + 1] - p->pos_ptr[pat];
      if (cnt + 1 >= cap) {
        cap *= 2;
        mt->pat = realloc(mt->pat, sizeof(int32_t) * cap);
        mt->root = realloc(mt->root, sizeof(int32_t) * cap);
        mt->mem_ptr = realloc(mt->mem_ptr, sizeof(int32_t) * (cap + 1));
        mt->bind_ptr = realloc(mt->bind_ptr, sizeof(int32_t) * (cap + 1));
      }
      while (nm + nmem >= mcap) { mcap *= 2; mt->members = realloc(mt->members, sizeof(int32_t) * mcap); }
      while (nb + npos >= bcap) { bcap *= 2; mt->binds = realloc(mt->binds, sizeof(int32_t) * bcap); }
      mt->pat[cnt] = pat;
      mt->root[cnt] = v;
      for (int i = 0; i < nmem; ++i) mt->members[nm++] = mem[i];
      for (int i = 0; i < npos; ++i) mt->binds[nb++] = w.bind[i];
      ++cnt;
      mt->mem_ptr[cnt] = nm;
      mt->bind_ptr[cnt] = nb;
    }
  }
  mt->group_ptr[n] = cnt;
  mt->n_match = cnt;
  free(mem);
  free(w.bind);
  free(w.touched);
  free(w.sidmap);
  return 0;
}

/* ----------------------------------------------------------- kernel cost */
/* cost.py:121-138; err: 1 no profile, 2 op without entry */
static double kernel_cost(const og_t* g, const mt_t* mt, int m, int backend, int n_kinds,
                          const double* coeff, const double* overhead, const uint8_t* has,
                          const uint8_t* has_prof, int pw_stride, const double* pw, int* err) {
  *err = 0;
  if (!has_prof[backend]) { *err = 1; return 0.0; }
  ksum ks;
  ks_zero(&ks);
  int nn = mt->mem_ptr[m + 1] - mt->mem_ptr[m];
  for (int i = mt->mem_ptr[m]; i < mt->mem_ptr[m + 1]; ++i) {
    int v = mt->members[i];
    long t = (long)backend * n_kinds + g->kind[v];
    if (!has[t]) { *err = 2; return 0.0; }
    volatile double prod = coeff[t] * g->volume[v];
    volatile double c = prod + overhead[t];
    ks_add(&ks, c);
  }
  volatile double base = ks_round(&ks);
  return base * pw[(long)backend * pw_stride + (nn - 1)];
}

/* -------------------------------------------------------------- state DP */
typedef struct {
  int W;            /* uint64 words per cover */
  int n_states, cap;
  uint64_t* cover;  /* n_states * W */
  ksum* sum;        /* exact sum of the state's terms */
  double* cost;
  int32_t* klen;
  int32_t** key;    /* match ids sorted by element order */
  /* open addressing */
  int hcap;
  int32_t* htab;
} states_t;

static uint64_t hash_cover(const uint64_t* c, int W) {
  uint64_t h = 1469598103934665603ull;
  for (int i = 0; i < W; ++i) {
    h ^= c[i];
    h *= 1099511628211ull;
    h ^= h >> 29;
  }
  return h;
}

static int st_find(states_t* s, const uint64_t* c) {
  uint64_t h = hash_cover(c, s->W) & (uint64_t)(s->hcap - 1);
  while (s->htab[h] >= 0) {
    if (!memcmp(s->cover + (size_t)s->htab[h] * s->W, c, sizeof(uint64_t) * s->W)) return s->htab[h];
    h = (h + 1) & (uint64_t)(s->hcap - 1);
  }
  return -1;
}

static void st_rehash(states_t* s) {
  free(s->htab);
  s->htab = malloc(sizeof(int32_t) * s->hcap);
  for (int i = 0; i < s->hcap; ++i) s->htab[i] = -1;
  for (int i = 0; i < s->n_states; ++i) {
    uint64_t h = hash_cover(s->cover + (size_t)i * s->W, s->W) & (uint64_t)(s->hcap - 1);
    while (s->htab[h] >= 0) h = (h + 1) & (uint64_t)(s->hcap - 1);
    s->htab[h] = i;
  }
}

static int st_add(states_t* s, const uint64_t* c) {
  if (s->n_states + 1 >= s->cap) {
    s->cap *= 2;
    s->cover = realloc(s->cover, sizeof(uint64_t) * (size_t)s->cap * s->W);
    s->sum = realloc(s->sum, sizeof(ksum) * (size_t)s->cap);
    s->cost = realloc(s->cost, sizeof(double) * (size_t)s->cap);
    s->klen = realloc(s->klen, sizeof(int32_t) * (size_t)s->cap);
    s->key = realloc(s->key, sizeof(int32_t*) * (size_t)s->cap);
  }
  int id = s->n_states++;
  memcpy(s->cover + (size_t)id * s->W, c, sizeof(uint64_t) * s->W);
  s->key[id] = NULL;
  s->klen[id] = 0;
  if (2 * s->n_states > s->hcap) {
    s->hcap *= 2;
    st_rehash(s);
  } else {
    uint64_t h = hash_cover(c, s->W) & (uint64_t)(s->hcap - 1);
    while (s->htab[h] >= 0) h = (h + 1) & (uint64_t)(s->hcap - 1);
    s->htab[h] = id;
  }
  return id;
}

/* element order: (registration index, sorted node tuple) -- placement.py:40-41 */
static int elem_cmp(const mt_t* mt, int a, int b) {
  if (mt->pat[a] != mt->pat[b]) return mt->pat[a] < mt->pat[b] ? -1 : 1;
  int i = mt->mem_ptr[a], ie = mt->mem_ptr[a + 1], j = mt->mem_ptr[b], je = mt->mem_ptr[b + 1];
  for (; i < ie && j < je; ++i, ++j)
    if (mt->members[i] != mt->members[j]) return mt->members[i] < mt->members[j] ? -1 : 1;
  return (ie - i) - (je - j);
}

static int key_cmp(const mt_t* mt, const int32_t* a, int na, const int32_t* b, int nb) {
  for (int i = 0; i < na && i < nb; ++i) {
    int c = elem_cmp(mt, a[i], b[i]);
    if (c) return c;
  }
  return na - nb;
}

/* Returns 0 ok, 1 uncoverable, 2 state cap exceeded.  kernels_out receives
 * the chosen match ids (any order), *n_kernels their count. */
int or_dp(int n, const int32_t* kind, const int32_t* in_ptr, const int32_t* in_src,
          const uint8_t* is_output, int n_match, const int32_t* group_ptr,
          const int32_t* pat, const int32_t* mem_ptr, const int32_t* members,
          const double* cost, double eps, int max_states, int32_t* kernels_out,
          int32_t* n_kernels, double* cost_out, int64_t* relaxations, int32_t* states_peak,
          int32_t* first_zero) {
  og_t g;
  memset(&g, 0, sizeof(g));
  g.n = n; g.kind = kind; g.in_ptr = in_ptr; g.in_src = in_src; g.is_output = is_output;
  if (og_prepare(&g) != 0) { og_free(&g); return 3; }
  mt_t mt;
  memset(&mt, 0, sizeof(mt));
  mt.n_match = n_match;
  mt.group_ptr = (int32_t*)group_ptr; mt.pat = (int32_t*)pat; mt.mem_ptr = (int32_t*)mem_ptr;
  mt.members = (int32_t*)members;
  int W = (n + 63) / 64;
  if (W == 0) W = 1;
  /* per candidate: node bitset and external predecessors bitset */
  uint64_t* mset = calloc((size_t)n_match * W + 1, sizeof(uint64_t));
  uint64_t* mext = calloc((size_t)n_match * W + 1, sizeof(uint64_t));
  for (int m = 0; m < n_match; ++m) {
    uint64_t* s = mset + (size_t)m * W;
    for (int i = mem_ptr[m]; i < mem_ptr[m + 1]; ++i) s[members[i] >> 6] |= 1ull << (members[i] & 63);
    uint64_t* e = mext + (size_t)m * W;
    for (int i = mem_ptr[m]; i < mem_ptr[m + 1]; ++i) {
      int v = members[i];
      for (int j = in_ptr[v]; j < in_ptr[v + 1]; ++j) {
        int p = in_src[j];
        if (p >= 0 && !((s[p >> 6] >> (p & 63)) & 1)) e[p >> 6] |= 1ull << (p & 63);
      }
    }
  }
  states_t st;
  memset(&st, 0, sizeof(st));
  st.W = W; st.cap = 1024; st.hcap = 2048;
  st.cover = calloc((size_t)st.cap * W, sizeof(uint64_t));
  st.sum = malloc(sizeof(ksum) * st.cap);
  st.cost = malloc(sizeof(double) * st.cap);
  st.klen = malloc(sizeof(int32_t) * st.cap);
  st.key = malloc(sizeof(int32_t*) * st.cap);
  st.htab = malloc(sizeof(int32_t) * st.hcap);
  for (int i = 0; i < st.hcap; ++i) st.htab[i] = -1;
  uint64_t* zero = calloc(W, sizeof(uint64_t));
  int s0 = st_add(&st, zero);
  ks_zero(&st.sum[s0]);
  st.cost[s0] = 0.0;
  uint64_t* nc = malloc(sizeof(uint64_t) * W);
  int32_t* nkey = malloc(sizeof(int32_t) * (n + 1));
  int rc = 0;
  int64_t relax = 0;
  *first_zero = -1;
  for (int t = 0; t < n && rc == 0; ++t) {
    int v = g.pop[t];
    if (group_ptr[v] == group_ptr[v + 1] && *first_zero < 0) *first_zero = v;
    for (int m = group_ptr[v]; m < group_ptr[v + 1] && rc == 0; ++m) {
      const uint64_t* ms = mset + (size_t)m * W;
      const uint64_t* me = mext + (size_t)m * W;
      int snap = st.n_states;
      for (int s = 0; s < snap; ++s) {
        const uint64_t* cv = st.cover + (size_t)s * W;
        int ok = 1;
        for (int i = 0; i < W && ok; ++i) ok = !(cv[i] & ms[i]) && !(me[i] & ~cv[i]);
        if (!ok) continue;
        ++relax;
        ksum nsum = st.sum[s];
        ks_add(&nsum, cost[m]);
        ks_add(&nsum, eps);
        double ncost = ks_round(&nsum);
        for (int i = 0; i < W; ++i) nc[i] = cv[i] | ms[i];
        int cur = st_find(&st, nc);
        if (cur >= 0 && ncost > st.cost[cur]) continue;
        /* key: insert m into the sorted key of s */
        int len = st.klen[s], k2 = 0, placed = 0;
        for (int i = 0; i < len; ++i) {
          if (!placed && elem_cmp(&mt, m, st.key[s][i]) < 0) { nkey[k2++] = m; placed = 1; }
          nkey[k2++] = st.key[s][i];
        }
        if (!placed) nkey[k2++] = m;
        if (cur < 0 || ncost < st.cost[cur] ||
            key_cmp(&mt, nkey, k2, st.key[cur], st.klen[cur]) < 0) {
          if (cur < 0) {
            cur = st_add(&st, nc);
            cv = st.cover + (size_t)s * W; /* realloc may have moved it */
          }
          st.sum[cur] = nsum;
          st.cost[cur] = ncost;
          free(st.key[cur]);
          st.key[cur] = malloc(sizeof(int32_t) * (k2 + 1));
          memcpy(st.key[cur], nkey, sizeof(int32_t) * k2);
          st.klen[cur] = k2;
        }
      }
      if (max_states > 0 && st.n_states > max_states) rc = 2;
    }
  }
  *relaxations = relax;
  *states_peak = st.n_states;
  if (rc == 0) {
    uint64_t* full = calloc(W, sizeof(uint64_t));
    for (int v = 0; v < n; ++v) full[v >> 6] |= 1ull << (v & 63);
    int f = st_find(&st, full);
    if (f < 0) rc = 1;
    else {
      *n_kernels = st.klen[f];
      memcpy(kernels_out, st.key[f], sizeof(int32_t) * st.klen[f]);
      *cost_out = st.cost[f];
    }
    free(full);
  }
  for (int i = 0; i < st.n_states; ++i) free(st.key[i]);
  free(st.key); free(st.klen); free(st.cost); free(st.sum); free(st.cover); free(st.htab);
  free(zero); free(nc); free(nkey); free(mset); free(mext);
  og_free(&g);
  return rc;
}

/* --------------------------------------------------------------- public */
/* Match every node against its root-kind candidates; results are returned
 * through malloc'ed arrays the caller frees with or_free. */
int or_match_all(int n, const int32_t* kind, const int32_t* in_ptr, const int32_t* in_src,
                 const uint8_t* is_output, const int32_t* attr_ptr, const int32_t* attr_key,
                 const int8_t* attr_tag, const int64_t* attr_ival, const double* attr_fval,
                 int n_pat, const int32_t* pos_ptr, const int32_t* pkind, const int32_t* nargs,
                 const int32_t* parent, const int32_t* argidx, const int32_t* sid,
                 const int32_t* con_ptr, const int32_t* con_key, const int8_t* con_op,
                 const int32_t* con_val_ptr, const int8_t* val_tag, const int64_t* val_ival,
                 const double* val_fval, const int64_t* con_lo, const int64_t* con_hi,
                 int n_kinds, const int32_t* kind_pat_ptr, const int32_t* kind_pat,
                 int32_t** group_ptr, int32_t** pat, int32_t** mem_ptr, int32_t** members,
                 int32_t** bind_ptr, int32_t** binds, int32_t* n_match) {
  og_t g;
  memset(&g, 0, sizeof(g));
  g.n = n; g.kind = kind; g.in_ptr = in_ptr; g.in_src = in_src; g.is_output = is_output;
  g.attr_ptr = attr_ptr; g.attr_key = attr_key; g.attr_tag = attr_tag; g.attr_ival = attr_ival;
  g.attr_fval = attr_fval;
  if (og_prepare(&g) != 0) { og_free(&g); return 3; }
  op_t p = {n_pat, pos_ptr, pkind, nargs, parent, argidx, sid, con_ptr, con_key, con_op,
            con_val_ptr, val_tag, val_ival, val_fval, con_lo, con_hi, NULL};
  mt_t mt;
  build_matches(&g, &p, kind_pat_ptr, kind_pat, n_kinds, &mt);
  *group_ptr = mt.group_ptr; *pat = mt.pat; *mem_ptr = mt.mem_ptr; *members = mt.members;
  *bind_ptr = mt.bind_ptr; *binds = mt.binds; *n_match = mt.n_match;
  free(mt.root);
  og_free(&g);
  return 0;
}

void or_free(void* p) { free(p); }

/* Kernel cost of every match (cost.py:121-138).  err_out per match. */
int or_price(int n_match, const int32_t* root_kind_unused, const int32_t* mem_ptr,
             const int32_t* members, const int32_t* backend, const int32_t* kind,
             const double* volume, int n_kinds, const double* coeff, const double* overhead,
             const uint8_t* has, const uint8_t* has_prof, int pw_stride, const double* pw,
             double* cost_out, int8_t* err_out) {
  (void)root_kind_unused;
  og_t g;
  memset(&g, 0, sizeof(g));
  g.kind = kind; g.volume = volume;
  mt_t mt;
  memset(&mt, 0, sizeof(mt));
  mt.mem_ptr = (int32_t*)mem_ptr; mt.members = (int32_t*)members;
  for (int m = 0; m < n_match; ++m) {
    int err;
    cost_out[m] = kernel_cost(&g, &mt, m, backend[m], n_kinds, coeff, overhead, has, has_prof,
                              pw_stride, pw, &err);
    err_out[m] = (int8_t)err;
  }
  return 0;
}

/* ------------------------------------------------------------ fitness */
static int uf_find(int* p, int x) {
  while (p[x] != x) { p[x] = p[p[x]]; x = p[x]; }
  return x;
}

/* Graph-level cost of n_genomes genomes (row stride `words` uint64).
 * kernels: the DP placement's matches in canonical order. */
int or_fitness(int n, const int32_t* in_ptr, const int32_t* in_src, const int32_t* group_ptr,
               const int32_t* mem_ptr, const int32_t* members, const int32_t* mbackend,
               const double* mcost, int n_kernels, const int32_t* kernel_match,
               int n_backends, const uint8_t* is_graph, const double* alpha,
               const double* floor_, int target, double eps, const uint64_t* genomes,
               int64_t n_genomes, int words, int threads, double* out) {
  /* eligible slots and their replacements (evolution.py:77-97) */
  int* slot_kernel = malloc(sizeof(int) * (n_kernels + 1));
  int k = 0;
  for (int i = 0; i < n_kernels; ++i)
    if (!is_graph[mbackend[kernel_match[i]]]) slot_kernel[k++] = i;
  int* rep_ptr = malloc(sizeof(int) * (k + 1));
  int* rep = malloc(sizeof(int) * (n + 1));
  int* rep_ok = malloc(sizeof(int) * (k + 1));
  int nr = 0;
  for (int s = 0; s < k; ++s) {
    int km = kernel_match[slot_kernel[s]];
    int nn = mem_ptr[km + 1] - mem_ptr[km];
    int r = -1;
    /* the kernel's root is its member without consumers inside -> the match root
       is recovered from the group that contains km */
    int lo = 0, hi = n; /* last v with group_ptr[v] <= km */
    while (hi - lo > 1) {
      int mid = (lo + hi) / 2;
      if (group_ptr[mid] <= km) lo = mid;
      else hi = mid;
    }
    while (lo + 1 < n && group_ptr[lo + 1] <= km) ++lo;
    int root = lo;
    rep_ptr[s] = nr;
    rep_ok[s] = 0;
    for (int c = group_ptr[root]; c < group_ptr[root + 1]; ++c) {
      if (mbackend[c] != target || mem_ptr[c + 1] - mem_ptr[c] != nn) continue;
      if (!memcmp(members + mem_ptr[c], members + mem_ptr[km], sizeof(int32_t) * nn)) { r = c; break; }
    }
    if (r >= 0) {
      rep[nr++] = r;
      rep_ok[s] = 1;
      continue;
    }
    int all = 1;
    for (int i = mem_ptr[km]; i < mem_ptr[km + 1] && all; ++i) {
      int u = members[i], f = -1;
      for (int c = group_ptr[u]; c < group_ptr[u + 1]; ++c)
        if (mbackend[c] == target && mem_ptr[c + 1] - mem_ptr[c] == 1) { f = c; break; }
      if (f < 0) all = 0;
      else rep[nr++] = f;
    }
    if (!all) nr = rep_ptr[s];
    rep_ok[s] = all ? 2 : 0;
  }
  rep_ptr[k] = nr;
  int maxk = n_kernels + n + 1;
  /* per-thread scratch, allocated once: the decoded kernel list, the kernel
     of every node, union-find parents and the region buckets */
#pragma omp parallel num_threads(threads)
  {
    int* dk = malloc(sizeof(int) * maxk);
    int* kernel_of = malloc(sizeof(int) * (n + 1));
    int* par = malloc(sizeof(int) * (maxk + 1));
    int* rid = malloc(sizeof(int) * (maxk + 1));
    int* rcnt = malloc(sizeof(int) * (maxk + 2));
    int* rmem = malloc(sizeof(int) * (maxk + 1));
    int* rb = malloc(sizeof(int) * (maxk + 1));
#pragma omp for schedule(dynamic, 4)
    for (int64_t gi = 0; gi < n_genomes; ++gi) {
      const uint64_t* bits = genomes + gi * words;
      int infeasible = 0;
      for (int s = 0; s < k && !infeasible; ++s)
        if (((bits[s >> 6] >> (s & 63)) & 1) && !rep_ok[s]) infeasible = 1;
      if (infeasible) { out[gi] = INFINITY; continue; }
      /* decoded placement as a list of matches (evolution.py decode) */
      int nd = 0, s = 0;
      for (int i = 0; i < n_kernels; ++i) {
        int flip = 0;
        if (s < k && slot_kernel[s] == i) {
          flip = (bits[s >> 6] >> (s & 63)) & 1;
          if (flip) for (int j = rep_ptr[s]; j < rep_ptr[s + 1]; ++j) dk[nd++] = rep[j];
          ++s;
        }
        if (!flip) dk[nd++] = kernel_match[i];
      }
      for (int i = 0; i < nd; ++i)
        for (int j = mem_ptr[dk[i]]; j < mem_ptr[dk[i] + 1]; ++j) kernel_of[members[j]] = i;
      /* union-find over same-backend graph kernels that touch (cost.py:339-357) */
      for (int i = 0; i < nd; ++i) par[i] = i;
      for (int v = 0; v < n; ++v) {
        int ki = kernel_of[v], b = mbackend[dk[ki]];
        if (!is_graph[b]) continue;
        for (int j = in_ptr[v]; j < in_ptr[v + 1]; ++j) {
          int p = in_src[j];
          if (p < 0) continue;
          int pk = kernel_of[p];
          if (pk != ki && mbackend[dk[pk]] == b) {
            int ra = uf_find(par, pk), rb2 = uf_find(par, ki);
            if (ra != rb2) { if (ra < rb2) par[rb2] = ra; else par[ra] = rb2; }
          }
        }
      }
      /* terms: every other kernel's cost + eps; every region's
         round(fsum(members)) * r(n) + eps (cost.py:359-373) */
      ksum total, rs;
      ks_zero(&total);
      int nr = 0;
      for (int i = 0; i < nd; ++i) rid[i] = -1;
      for (int i = 0; i < nd; ++i) {
        int b = mbackend[dk[i]];
        if (!is_graph[b]) { ks_add(&total, mcost[dk[i]]); ks_add(&total, eps); continue; }
        int r = uf_find(par, i);
        if (rid[r] < 0) { rid[r] = nr; rcnt[nr] = 0; rb[nr] = b; ++nr; }
        rcnt[rid[r]]++;
      }
      /* bucket the members of every region (counting sort by region) */
      int acc = 0;
      for (int r = 0; r < nr; ++r) { int c = rcnt[r]; rcnt[r] = acc; acc += c; }
      rcnt[nr] = acc;
      for (int i = 0; i < nd; ++i) {
        if (!is_graph[mbackend[dk[i]]]) continue;
        rmem[rcnt[rid[uf_find(par, i)]]++] = i;
      }
      for (int r = nr; r > 0; --r) rcnt[r] = rcnt[r - 1];
      rcnt[0] = 0;
      for (int r = 0; r < nr; ++r) {
        ks_zero(&rs);
        for (int q = rcnt[r]; q < rcnt[r + 1]; ++q) ks_add(&rs, mcost[dk[rmem[q]]]);
        int b = rb[r], cnt = rcnt[r + 1] - rcnt[r];
        volatile double prod = alpha[b] * (double)(cnt - 1);
        volatile double t = 1.0 - prod;
        double rr = t > floor_[b] ? t : floor_[b];
        volatile double term = ks_round(&rs) * rr;
        ks_add(&total, term);
        ks_add(&total, eps);
      }
      out[gi] = ks_round(&total);
    }
    free(dk); free(kernel_of); free(par); free(rid); free(rcnt); free(rmem); free(rb);
  }
  free(slot_kernel); free(rep_ptr); free(rep); free(rep_ok);
  return k;
}

/* ------------------------------------------------- independent exact DP */
/*
 * or_dp_subtree -- a second, independent solver for the reference optimum,
 * for graphs whose covered-set state space is out of reach (NasNet-A,
 * 10-step NasRNN, the 100k-node random DAG).
 *
 * What it computes is the reference's result (tensorplace/dp.py:71-179):
 * the partition of the graph into registered matches with the smallest
 * fsum of (kernel cost + epsilon), ties broken by the canonical key
 * (placement.py:78-82: sorted (registration index, node tuple) pairs).
 * The covered-set DP reaches exactly these partitions (dp.py:10-14), and a
 * match may only expose its root (matching.py:104-110), so every non-root
 * member of a kernel is post-dominated by the kernel's root.  Hence the
 * kernels of any partition nest along the post-dominator tree and
 *
 *   OPT(r) = min over matches m rooted at r of
 *            cost(m) + eps + sum of OPT(x) for x not in m with ipdom(x) in m
 *
 * with the answer the sum of OPT(x) over the tree's roots.  Written apart
 * from the device solver on purpose:
 *   - post-dominator SETS are built literally as graph.py:224-237 does
 *     (intersection of the successors' sets, plus the node), as sorted
 *     arrays of topological indices; ipdom is the set's member with the
 *     smallest topological index (graph.py:239-251);
 *   - sums are exact Kulisch accumulators (ksum), not 192-bit fixed point;
 *   - ties are settled by materialising both candidate kernel lists,
 *     sorting them and comparing them as the reference compares keys
 *     (key_cmp above), not by a symmetric-difference walk.
 * It also reports the smallest positive exact regret of any (node,
 * candidate) decision, from which the caller decides whether rounded
 * comparisons (the reference compares rounded state costs) could pick a
 * different partition: every pair of same-cover states differs by a sum of
 * such regrets.
 *
 * Returns 0 ok, 1 uncoverable, 3 cycle, 4 memory cap for the literal
 * post-dominator sets exceeded.
 */
static int ks_cmp(const ksum* a, const ksum* b) {
  for (int i = KL - 1; i >= 0; --i)
    if (a->w[i] != b->w[i]) return a->w[i] < b->w[i] ? -1 : 1;
  return 0;
}

/* a - b for a >= b */
static void ks_sub(ksum* out, const ksum* a, const ksum* b) {
  uint64_t br = 0;
  for (int i = 0; i < KL; ++i) {
    uint64_t x = a->w[i], y = b->w[i];
    uint64_t d = x - y - br;
    br = (x < y) || (x == y && br) || (x - y < br);
    out->w[i] = d;
  }
  out->bad = a->bad | b->bad;
}

static int elem_cmp_q(const void* a, const void* b, void* ctx) {
  return elem_cmp((const mt_t*)ctx, *(const int32_t*)a, *(const int32_t*)b);
}

static const mt_t* g_mt_ctx;
static int elem_cmp_qs(const void* a, const void* b) {
  return elem_cmp(g_mt_ctx, *(const int32_t*)a, *(const int32_t*)b);
}

typedef struct {
  int n;
  const int32_t *mem_ptr, *members;
  const int32_t *ch_ptr, *ch; /* post-dominator children */
  const int32_t* choice;
  int32_t* mark; /* stamp per node */
  int32_t* stack;
} sol_ctx;

/* kernels of the subtree solution of option (m at r), appended to out */
static int collect(sol_ctx* c, int m, int32_t* out, int nout, int* stamp) {
  /* members of m, then for each member its pdom children outside m */
  int sp = 0;
  ++*stamp;
  int st = *stamp;
  out[nout++] = m;
  for (int i = c->mem_ptr[m]; i < c->mem_ptr[m + 1]; ++i) c->mark[c->members[i]] = st;
  for (int i = c->mem_ptr[m]; i < c->mem_ptr[m + 1]; ++i) {
    int y = c->members[i];
    for (int j = c->ch_ptr[y]; j < c->ch_ptr[y + 1]; ++j)
      if (c->mark[c->ch[j]] != st) c->stack[sp++] = c->ch[j];
  }
  while (sp) {
    int x = c->stack[--sp];
    int mx = c->choice[x];
    out[nout++] = mx;
    /* children of mx's members outside mx: members of mx are exactly the
       nodes whose chain reaches x inside mx */
    ++*stamp;
    int s2 = *stamp;
    for (int i = c->mem_ptr[mx]; i < c->mem_ptr[mx + 1]; ++i) c->mark[c->members[i]] = s2;
    for (int i = c->mem_ptr[mx]; i < c->mem_ptr[mx + 1]; ++i) {
      int y = c->members[i];
      for (int j = c->ch_ptr[y]; j < c->ch_ptr[y + 1]; ++j)
        if (c->mark[c->ch[j]] != s2) c->stack[sp++] = c->ch[j];
    }
  }
  return nout;
}

int or_dp_subtree(int n, const int32_t* kind, const int32_t* in_ptr, const int32_t* in_src,
                  const uint8_t* is_output, int n_match, const int32_t* group_ptr,
                  const int32_t* pat, const int32_t* mem_ptr, const int32_t* members,
                  const double* cost, double eps, int64_t max_set_entries,
                  int32_t* kernels_out, int32_t* n_kernels, double* cost_out,
                  double* min_regret_out, int32_t* ipdom_out, int64_t* ties_out) {
  og_t g;
  memset(&g, 0, sizeof(g));
  g.n = n; g.kind = kind; g.in_ptr = in_ptr; g.in_src = in_src; g.is_output = is_output;
  if (og_prepare(&g) != 0) { og_free(&g); return 3; }
  /* topological order: Kahn, smallest index first (graph.py:156-176) */
  int32_t* topo = malloc(sizeof(int32_t) * (n + 1));
  int32_t* tix = malloc(sizeof(int32_t) * (n + 1));
  {
    int* pend = calloc(n + 1, sizeof(int));
    for (int v = 0; v < n; ++v)
      for (int j = g.out_ptr[v]; j < g.out_ptr[v + 1]; ++j) pend[g.out_dst[j]]++;
    /* min-heap of ready indices */
    int* heap = malloc(sizeof(int) * (n + 1));
    int hn = 0, done = 0;
    for (int v = 0; v < n; ++v)
      if (!pend[v]) {
        int i = hn++;
        heap[i] = v;
        while (i && heap[(i - 1) / 2] > heap[i]) { int t = heap[i]; heap[i] = heap[(i - 1) / 2]; heap[(i - 1) / 2] = t; i = (i - 1) / 2; }
      }
    while (hn) {
      int v = heap[0];
      heap[0] = heap[--hn];
      for (int i = 0;;) {
        int l = 2 * i + 1, r = l + 1, m = i;
        if (l < hn && heap[l] < heap[m]) m = l;
        if (r < hn && heap[r] < heap[m]) m = r;
        if (m == i) break;
        int t = heap[i]; heap[i] = heap[m]; heap[m] = t;
        i = m;
      }
      tix[v] = done;
      topo[done++] = v;
      for (int j = g.out_ptr[v]; j < g.out_ptr[v + 1]; ++j)
        if (--pend[g.out_dst[j]] == 0) {
          int i = hn++;
          heap[i] = g.out_dst[j];
          while (i && heap[(i - 1) / 2] > heap[i]) { int t = heap[i]; heap[i] = heap[(i - 1) / 2]; heap[(i - 1) / 2] = t; i = (i - 1) / 2; }
        }
    }
    free(heap);
    free(pend);
  }
  /* literal post-dominator sets (graph.py:224-237), without the virtual
     sink (it post-dominates every node): sorted topological indices */
  int32_t** pset = calloc(n + 1, sizeof(int32_t*));
  int32_t* plen = calloc(n + 1, sizeof(int32_t));
  int64_t entries = 0;
  int rc = 0;
  int32_t* tmp = malloc(sizeof(int32_t) * (n + 1));
  int32_t* tmp2 = malloc(sizeof(int32_t) * (n + 1));
  for (int t = n - 1; t >= 0 && rc == 0; --t) {
    int v = topo[t];
    int nc = 0;
    if (!is_output[v]) {
      int first = 1;
      for (int j = g.out_ptr[v]; j < g.out_ptr[v + 1]; ++j) {
        int s = g.out_dst[j];
        if (first) {
          memcpy(tmp, pset[s], sizeof(int32_t) * plen[s]);
          nc = plen[s];
          first = 0;
        } else {
          int a = 0, b = 0, k = 0;
          while (a < nc && b < plen[s]) {
            if (tmp[a] < pset[s][b]) ++a;
            else if (tmp[a] > pset[s][b]) ++b;
            else { tmp2[k++] = tmp[a]; ++a; ++b; }
          }
          memcpy(tmp, tmp2, sizeof(int32_t) * k);
          nc = k;
        }
      }
    } /* an output's successors include the sink, whose set is {sink} */
    pset[v] = malloc(sizeof(int32_t) * (nc + 1));
    pset[v][0] = t;
    memcpy(pset[v] + 1, tmp, sizeof(int32_t) * nc);
    plen[v] = nc + 1;
    entries += nc + 1;
    if (max_set_entries > 0 && entries > max_set_entries) rc = 4;
  }
  free(tmp2);
  int32_t* ipdom = malloc(sizeof(int32_t) * (n + 1));
  if (rc == 0)
    for (int v = 0; v < n; ++v) {
      /* strict post-dominators: the set without v itself; the nearest one has
         the smallest topological index (graph.py:239-251) */
      int best = -1;
      for (int i = 0; i < plen[v]; ++i)
        if (pset[v][i] != tix[v] && (best < 0 || pset[v][i] < best)) best = pset[v][i];
      ipdom[v] = best < 0 ? -1 : topo[best];
      if (ipdom_out) ipdom_out[v] = ipdom[v];
    }
  for (int v = 0; v < n; ++v) free(pset[v]);
  free(pset);
  free(plen);
  if (rc) {
    free(tmp); free(ipdom); free(topo); free(tix); og_free(&g);
    return rc;
  }
  /* children lists of the post-dominator tree */
  int32_t* ch_ptr = calloc(n + 2, sizeof(int32_t));
  int32_t* ch = malloc(sizeof(int32_t) * (n + 1));
  for (int v = 0; v < n; ++v) ch_ptr[(ipdom[v] < 0 ? n : ipdom[v]) + 1]++;
  for (int v = 0; v <= n; ++v) ch_ptr[v + 1] += ch_ptr[v];
  {
    int32_t* fill = calloc(n + 1, sizeof(int32_t));
    for (int v = 0; v < n; ++v) {
      int p = ipdom[v] < 0 ? n : ipdom[v];
      ch[ch_ptr[p] + fill[p]++] = v;
    }
    free(fill);
  }
  ksum* opt = malloc(sizeof(ksum) * (size_t)(n + 1));
  uint8_t* feas = calloc(n + 1, 1);
  int32_t* choice = malloc(sizeof(int32_t) * (n + 1));
  int32_t* mark = calloc(n + 1, sizeof(int32_t));
  int stamp = 0;
  int32_t* stack = malloc(sizeof(int32_t) * (n + 1));
  int32_t* la = malloc(sizeof(int32_t) * (n + 1));
  int32_t* lb = malloc(sizeof(int32_t) * (n + 1));
  sol_ctx sc = {n, mem_ptr, members, ch_ptr, ch, choice, mark, stack};
  ksum minreg;
  int have_reg = 0;
  int64_t ties = 0;
  memset(&minreg, 0, sizeof(minreg));
  g_mt_ctx = NULL;
  mt_t mt;
  memset(&mt, 0, sizeof(mt));
  mt.pat = (int32_t*)pat; mt.mem_ptr = (int32_t*)mem_ptr; mt.members = (int32_t*)members;
  g_mt_ctx = &mt;
  ksum* vals = malloc(sizeof(ksum) * 64);
  int vcap = 64;
  for (int t = 0; t < n; ++t) {
    int r = topo[t];
    int c0 = group_ptr[r], c1 = group_ptr[r + 1];
    if (c1 - c0 > vcap) { vcap = c1 - c0; vals = realloc(vals, sizeof(ksum) * vcap); }
    uint8_t* ok = calloc(c1 - c0 + 1, 1);
    int best = -1;
    for (int m = c0; m < c1; ++m) {
      ksum* s = &vals[m - c0];
      ks_zero(s);
      ks_add(s, cost[m]);
      ks_add(s, eps);
      ++stamp;
      for (int i = mem_ptr[m]; i < mem_ptr[m + 1]; ++i) mark[members[i]] = stamp;
      int good = 1;
      /* every member other than r must hang below r inside m (true for any
         valid match); checked, not assumed */
      for (int i = mem_ptr[m]; i < mem_ptr[m + 1] && good; ++i) {
        int y = members[i];
        if (y != r && (ipdom[y] < 0 || mark[ipdom[y]] != stamp)) good = 0;
      }
      for (int i = mem_ptr[m]; i < mem_ptr[m + 1] && good; ++i) {
        int y = members[i];
        for (int j = ch_ptr[y]; j < ch_ptr[y + 1] && good; ++j) {
          int x = ch[j];
          if (mark[x] == stamp) continue;
          if (!feas[x]) good = 0;
          else ks_merge(s, &opt[x]);
        }
      }
      ok[m - c0] = (uint8_t)good;
      if (!good) continue;
      if (best < 0) { best = m; continue; }
      int c = ks_cmp(s, &vals[best - c0]);
      if (c < 0) best = m;
      else if (c == 0) {
        ++ties;
        int na = collect(&sc, m, la, 0, &stamp);
        /* collect() for `best` needs choice[] of the children only */
        int nb = collect(&sc, best, lb, 0, &stamp);
        qsort(la, na, sizeof(int32_t), elem_cmp_qs);
        qsort(lb, nb, sizeof(int32_t), elem_cmp_qs);
        if (key_cmp(&mt, la, na, lb, nb) < 0) best = m;
      }
    }
    if (best >= 0) {
      feas[r] = 1;
      choice[r] = best;
      opt[r] = vals[best - c0];
      for (int m = c0; m < c1; ++m) {
        if (!ok[m - c0] || m == best) continue;
        int c = ks_cmp(&vals[m - c0], &opt[r]);
        if (c <= 0) continue;
        ksum d;
        ks_sub(&d, &vals[m - c0], &opt[r]);
        if (!have_reg || ks_cmp(&d, &minreg) < 0) { minreg = d; have_reg = 1; }
      }
    } else {
      feas[r] = 0;
      choice[r] = -1;
    }
    free(ok);
  }
  /* the answer: the tree roots' subtree solutions */
  ksum total;
  ks_zero(&total);
  int feasible = 1, nk = 0;
  for (int j = ch_ptr[n]; j < ch_ptr[n + 1]; ++j) {
    int x = ch[j];
    if (!feas[x]) { feasible = 0; break; }
    ks_merge(&total, &opt[x]);
    /* kernels of x's solution */
    int start = nk;
    nk = collect(&sc, choice[x], kernels_out, nk, &stamp);
    (void)start;
  }
  if (!feasible) rc = 1;
  else {
    *n_kernels = nk;
    *cost_out = ks_round(&total);
    *min_regret_out = have_reg ? ks_round(&minreg) : INFINITY;
    if (have_reg && ks_round(&minreg) == 0.0) *min_regret_out = 5e-324; /* below any double */
  }
  if (ties_out) *ties_out = ties;
  free(vals); free(la); free(lb); free(stack); free(mark); free(choice); free(feas); free(opt);
  free(ch); free(ch_ptr); free(tmp); free(ipdom); free(topo); free(tix);
  og_free(&g);
  return rc;
}
