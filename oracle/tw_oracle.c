/* TEST INFRASTRUCTURE ONLY — CPU oracle (plain-C restatement) of the
 * reference core `timewalk` (/root/reference/proj/core). See tw_oracle.h.
 * Scalar, single-threaded, written for clarity; sized for the parity cases
 * (≤ a few million edges). Compiled with -ffp-contract=off so every fp64
 * expression rounds exactly like the reference's x86-64 build (no FMA).
 */
#define _GNU_SOURCE
#include "tw_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define TIME_UNSET INT64_MIN   /* types.hpp:23 kTimeUnset */
#define TIME_INFINITE INT64_MAX /* types.hpp:25 kTimeInfinite */

void two_free(void* p) { free(p); }

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ---------------------------------------------------------------- rng ---- */

/* rng.hpp:8-13 splitmix64 finalizer */
uint64_t two_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* Philox4x32-10, counter/key layout of oracle/philox_shadow/timewalk/rng.hpp */
static uint64_t philox_bits(uint64_t seed, uint64_t walk, uint64_t hop, uint64_t ordinal) {
  uint32_t c0 = (uint32_t)walk, c1 = (uint32_t)hop, c2 = (uint32_t)ordinal;
  uint32_t c3 = (uint32_t)(walk >> 32) ^ (uint32_t)(hop >> 32) ^ (uint32_t)(ordinal >> 32);
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return ((uint64_t)c1 << 32) | c0;
}

/* rng.hpp:25 (state = mix64(seed ^ 0x6a09e667f3bcc909)), :27-33 (bits) */
uint64_t two_rng_bits(int kind, uint64_t seed, uint64_t walk, uint64_t hop, uint64_t ordinal) {
  if (kind == TWO_RNG_PHILOX) return philox_bits(seed, walk, hop, ordinal);
  const uint64_t state = two_mix64(seed ^ 0x6a09e667f3bcc909ULL);
  uint64_t h = two_mix64(state ^ walk);
  h = two_mix64(h ^ hop);
  return two_mix64(h ^ ordinal);
}

/* rng.hpp:36-39 */
double two_rng_uniform(int kind, uint64_t seed, uint64_t walk, uint64_t hop, uint64_t ordinal) {
  return (double)(two_rng_bits(kind, seed, walk, hop, ordinal) >> 11) * 0x1.0p-53;
}

/* ---------------------------------------------------------- generators --- */

/* synthetic.cpp:17-20 draw_mod */
static uint64_t draw_mod(uint64_t seed, uint64_t stream, uint64_t i, uint64_t bound) {
  return two_rng_bits(TWO_RNG_SPLITMIX, seed, stream, i, 0) % bound;
}

typedef struct {
  two_edge* e;
  uint64_t n, cap;
} edge_vec;

static void ev_push(edge_vec* v, int64_t s, int64_t d, int64_t t) {
  if (v->n == v->cap) {
    v->cap = v->cap ? 2 * v->cap : 1024;
    v->e = (two_edge*)realloc(v->e, v->cap * sizeof(two_edge));
  }
  v->e[v->n].src = s;
  v->e[v->n].dst = d;
  v->e[v->n].t = t;
  v->n++;
}

/* synthetic.cpp:24-36 */
uint64_t two_gen_uniform(uint64_t nodes, uint64_t edges, int64_t t_max, uint64_t seed, two_edge** out) {
  two_edge* e = (two_edge*)malloc((edges ? edges : 1) * sizeof(two_edge));
  for (uint64_t i = 0; i < edges; ++i) {
    e[i].src = (int64_t)draw_mod(seed, 1, i, nodes);
    e[i].dst = (int64_t)draw_mod(seed, 2, i, nodes);
    e[i].t = (int64_t)draw_mod(seed, 3, i, (uint64_t)t_max + 1);
  }
  *out = e;
  return edges;
}

/* synthetic.cpp:38-99 */
uint64_t two_gen_hub_skewed(uint64_t bg_nodes, uint64_t bg_edges, uint64_t seed, two_edge** out) {
  edge_vec v = {0};
  int64_t next_id = (int64_t)bg_nodes;
#define FRESH() (next_id++)
  /* plant_funnel :50-56, plant_out_ladder :60-67 */
#define FUNNEL(width, t0, hubvar)                                       \
  do {                                                                  \
    hubvar = FRESH();                                                   \
    for (uint64_t i_ = 0; i_ < (uint64_t)(width); ++i_)                 \
      ev_push(&v, FRESH(), hubvar, (int64_t)(t0) + (int64_t)i_);        \
  } while (0)
#define LADDER(hub, groups, t0, sink_count)                             \
  do {                                                                  \
    int64_t* sinks_ = (int64_t*)malloc((sink_count) * sizeof(int64_t)); \
    for (uint64_t s_ = 0; s_ < (uint64_t)(sink_count); ++s_) sinks_[s_] = FRESH(); \
    for (uint64_t g_ = 0; g_ < (uint64_t)(groups); ++g_)                \
      ev_push(&v, hub, sinks_[g_ % (sink_count)], (int64_t)(t0) + (int64_t)g_); \
    free(sinks_);                                                       \
  } while (0)
  int64_t mega, bd, bc, wd, wc;
  FUNNEL(2600, 1000, mega);
  LADDER(mega, 5000, 10000, 200);
  FUNNEL(40, 1000, bd);
  LADDER(bd, 4500, 10000, 50);
  FUNNEL(40, 1000, bc);
  LADDER(bc, 150, 10000, 50);
  FUNNEL(3, 1000, wd);
  LADDER(wd, 700, 10000, 20);
  FUNNEL(3, 1000, wc);
  LADDER(wc, 60, 10000, 20);
  {
    const int64_t spreader = FRESH();
    LADDER(spreader, 40, 500, 40);
  }
  for (uint64_t i = 0; i < bg_edges; ++i) {
    const double u = (double)(two_rng_bits(TWO_RNG_SPLITMIX, seed, 2, i, 1) >> 11) * 0x1.0p-53;
    int64_t dst = (int64_t)((double)bg_nodes * u * u * u);
    if (dst > (int64_t)bg_nodes - 1) dst = (int64_t)bg_nodes - 1;
    ev_push(&v, (int64_t)draw_mod(seed, 1, i, bg_nodes), dst, (int64_t)draw_mod(seed, 3, i, 20000));
  }
#undef FRESH
#undef FUNNEL
#undef LADDER
  *out = v.e;
  return v.n;
}

/* synthetic.cpp:101-124 */
uint64_t two_gen_mega_hub(uint32_t feeders, uint64_t seed, two_edge** out) {
  edge_vec v = {0};
  const int64_t hub = 0;
  int64_t next_id = 1;
  for (uint32_t i = 0; i < feeders; ++i) ev_push(&v, next_id++, hub, 100 + (int64_t)i);
  int64_t sinks[16];
  for (int s = 0; s < 16; ++s) sinks[s] = next_id++;
  const int64_t t0 = 100 + (int64_t)feeders + 100;
  for (uint32_t g = 0; g < 64; ++g) ev_push(&v, hub, sinks[g % 16], t0 + (int64_t)g);
  const int64_t bg = next_id;
  for (uint64_t i = 0; i < 1000; ++i) {
    ev_push(&v, bg + (int64_t)draw_mod(seed, 1, i, 100), bg + (int64_t)draw_mod(seed, 2, i, 100),
            (int64_t)draw_mod(seed, 3, i, 5000));
  }
  *out = v.e;
  return v.n;
}

/* synthetic.cpp:126-141 */
uint64_t two_gen_time_ladder(uint64_t edges, uint32_t rungs, uint64_t seed, two_edge** out) {
  uint64_t node_count = edges / rungs;
  if (node_count < 2) node_count = 2;
  two_edge* e = (two_edge*)malloc(node_count * rungs * sizeof(two_edge));
  uint64_t i = 0;
  for (uint64_t v = 0; v < node_count; ++v) {
    for (uint32_t r = 0; r < rungs; ++r, ++i) {
      e[i].src = (int64_t)v;
      e[i].dst = (int64_t)draw_mod(seed, 2, i, node_count);
      e[i].t = (int64_t)r;
    }
  }
  *out = e;
  return node_count * rungs;
}

/* SURVEY §8(d) C5 law; background draws as synthetic.cpp:92-96 */
void two_gen_stream(uint64_t nodes, uint64_t first, uint64_t count, uint64_t seed, two_edge* out) {
  for (uint64_t k = 0; k < count; ++k) {
    const uint64_t i = first + k;
    const double u = (double)(two_rng_bits(TWO_RNG_SPLITMIX, seed, 2, i, 1) >> 11) * 0x1.0p-53;
    int64_t dst = (int64_t)((double)nodes * u * u * u);
    if (dst > (int64_t)nodes - 1) dst = (int64_t)nodes - 1;
    out[k].src = (int64_t)draw_mod(seed, 1, i, nodes);
    out[k].dst = dst;
    out[k].t = (int64_t)(i / 4);
  }
}

/* ------------------------------------------------------------ samplers --- */

/* samplers.cpp:10-13 require_picker_args */
static int picker_args_ok(double u, uint64_t n) { return n != 0 && (u >= 0.0) && u < 1.0; }

/* samplers.cpp:17-21 */
static uint64_t pick_uniform(double u, uint64_t n) {
  const uint64_t i = (uint64_t)(u * (double)n);
  return i >= n ? n - 1 : i;
}

/* samplers.cpp:23-40 */
static double cum_linear(int64_t k) { return 0.5 * (double)k * (double)(k + 1); }
static uint64_t pick_linear(double u, uint64_t n) {
  const double nn = (double)n;
  const double total = 0.5 * nn * (nn + 1.0);
  const double r = u * total;
  const double x = 0.5 * (-1.0 + sqrt(1.0 + 4.0 * u * nn * (nn + 1.0)));
  int64_t i = (int64_t)x;
  if (i < 0) i = 0;
  if (i >= (int64_t)n) i = (int64_t)n - 1;
  while (i > 0 && cum_linear(i) > r) --i;
  while (i + 1 < (int64_t)n && cum_linear(i + 1) <= r) ++i;
  return (uint64_t)i;
}

/* samplers.cpp:42-55, kExponentialExactLimit = 700 (samplers.hpp:52) */
static uint64_t pick_exponential(double u, uint64_t n) {
  if (n == 1) return 0;
  double x;
  if (n <= 700) {
    x = log1p(u * expm1((double)n));
  } else {
    x = (double)n + log(u);
  }
  if (!(x > 0.0)) return 0;
  const uint64_t i = (uint64_t)x;
  return i >= n ? n - 1 : i;
}

int two_pick_index(int kind, double u, uint64_t n, uint64_t* out) {
  if (!picker_args_ok(u, n)) return TWO_EINVAL;
  switch (kind) {
    case TWO_UNIFORM: *out = pick_uniform(u, n); return TWO_OK;
    case TWO_LINEAR: *out = pick_linear(u, n); return TWO_OK;
    case TWO_EXPINDEX: *out = pick_exponential(u, n); return TWO_OK;
    default: return TWO_EINVAL;
  }
}

/* lower_bound over [first, last) of doubles: first k with a[k] >= r */
static uint64_t lower_bound_d(const double* a, uint64_t first, uint64_t last, double r) {
  uint64_t lo = first, hi = last;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (a[mid] < r) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

/* samplers.cpp:74-80 */
uint64_t two_pick_weighted(double u, const double* prefix, uint64_t n) {
  const double r = u * prefix[n - 1];
  uint64_t k = lower_bound_d(prefix, 0, n, r);
  if (k == n) --k;
  return k;
}

/* samplers.cpp:82-90 */
uint64_t two_pick_weighted_range(double u, const double* prefix, uint64_t begin, uint64_t end, double base) {
  const double r = base + u * (prefix[end - 1] - base);
  uint64_t k = lower_bound_d(prefix, begin, end, r);
  if (k == end) --k;
  return k - begin;
}

/* samplers.cpp:92-103 */
uint64_t two_oracle_pick(double u, const double* weights, uint64_t n) {
  double total = 0.0;
  for (uint64_t i = 0; i < n; ++i) total += weights[i];
  const double r = u * total;
  double cum = 0.0;
  for (uint64_t k = 0; k < n; ++k) {
    cum += weights[k];
    if (r < cum) return k;
  }
  return n - 1;
}

/* ---------------------------------------------------------- edge store --- */

typedef struct {
  int64_t t, src, dst;
  uint64_t idx;
} sort_rec;

/* (time, source, target) then input ordinal: the three stable LSD passes of
 * edge_store.cpp:42-55 yield exactly this order. */
static int cmp_rec(const void* a, const void* b) {
  const sort_rec* x = (const sort_rec*)a;
  const sort_rec* y = (const sort_rec*)b;
  if (x->t != y->t) return x->t < y->t ? -1 : 1;
  if ((uint64_t)x->src != (uint64_t)y->src) return (uint64_t)x->src < (uint64_t)y->src ? -1 : 1;
  if ((uint64_t)x->dst != (uint64_t)y->dst) return (uint64_t)x->dst < (uint64_t)y->dst ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx ? 1 : 0);
}

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* edge_store.hpp:133-140 */
uint32_t two_ref_neighbor(const two_store* s, uint64_t pos, uint32_t owner) {
  const uint32_t e = s->ref_edge[pos];
  switch (s->mode) {
    case TWO_FORWARD: return s->dst[e];
    case TWO_BACKWARD: return s->src[e];
    default: return s->src[e] == owner ? s->dst[e] : s->src[e];
  }
}

/* edge_store.cpp:120-124 owner_of */
static uint32_t owner_of(const two_store* s, uint64_t i, int side) {
  if (s->mode == TWO_BACKWARD) return s->dst[i];
  if (s->mode == TWO_UNDIRECTED && side == 1) return s->dst[i];
  return s->src[i];
}

void two_store_free(two_store* s) {
  if (!s) return;
  free(s->src); free(s->dst); free(s->t); free(s->ext);
  free(s->ts_off); free(s->ts_time); free(s->ts_w);
  free(s->n_off); free(s->n_tsidx); free(s->mk_time); free(s->mk_start);
  free(s->ref_edge); free(s->wprefix); free(s->adj_off); free(s->adj);
  free(s);
}

#define XALLOC(n, T) ((T*)calloc((n) ? (n) : 1, sizeof(T)))

/* edge_store.cpp:27-254 EdgeStore::build */
two_store* two_build(const two_edge* edges, uint64_t m, int mode, int* status) {
  /* :32-38 validation */
  if (m >= UINT32_MAX / 2) { *status = TWO_EINVAL; return NULL; }
  for (uint64_t i = 0; i < m; ++i) {
    if (edges[i].t < 0 || edges[i].src < 0 || edges[i].dst < 0) { *status = TWO_EINVAL; return NULL; }
  }
  two_store* s = XALLOC(1, two_store);
  s->mode = mode;
  s->m = m;

  /* :42-55 canonical order */
  sort_rec* rec = XALLOC(m, sort_rec);
  for (uint64_t i = 0; i < m; ++i) {
    rec[i].t = edges[i].t; rec[i].src = edges[i].src; rec[i].dst = edges[i].dst; rec[i].idx = i;
  }
  qsort(rec, m, sizeof(sort_rec), cmp_rec);

  /* :57-89 densify: internal id = rank of external id among endpoints */
  uint64_t* ep = XALLOC(2 * m, uint64_t);
  for (uint64_t i = 0; i < m; ++i) { ep[2 * i] = (uint64_t)rec[i].src; ep[2 * i + 1] = (uint64_t)rec[i].dst; }
  qsort(ep, 2 * m, sizeof(uint64_t), cmp_u64);
  uint64_t V = 0;
  for (uint64_t k = 0; k < 2 * m; ++k) if (k == 0 || ep[k] != ep[k - 1]) ep[V++] = ep[k];
  s->V = V;
  s->ext = XALLOC(V, int64_t);
  for (uint64_t v = 0; v < V; ++v) s->ext[v] = (int64_t)ep[v];
  free(ep);
  s->src = XALLOC(m, uint32_t);
  s->dst = XALLOC(m, uint32_t);
  s->t = XALLOC(m, int64_t);
  for (uint64_t i = 0; i < m; ++i) {
    uint32_t a = 0, b = 0;
    two_find_node(s, rec[i].src, &a);
    two_find_node(s, rec[i].dst, &b);
    s->src[i] = a; s->dst[i] = b; s->t[i] = rec[i].t;
  }
  free(rec);

  /* :91-98 timestamp groups */
  uint64_t Z = 0;
  for (uint64_t i = 0; i < m; ++i) if (i == 0 || s->t[i] != s->t[i - 1]) ++Z;
  s->Z = Z;
  s->ts_off = XALLOC(Z + 1, uint64_t);
  s->ts_time = XALLOC(Z, int64_t);
  s->ts_w = XALLOC(Z, double);
  for (uint64_t i = 0, g = 0; i < m; ++i) {
    if (i == 0 || s->t[i] != s->t[i - 1]) { s->ts_off[g] = i; s->ts_time[g] = s->t[i]; ++g; }
  }
  s->ts_off[Z] = m;
  /* :100-110 group weights anchored at the newest group */
  if (Z > 0) {
    const int64_t anchor = s->ts_time[Z - 1];
    double acc = 0.0;
    for (uint64_t g = 0; g < Z; ++g) {
      acc += exp((double)(s->ts_time[g] - anchor));
      s->ts_w[g] = acc;
    }
  }

  /* :112-214 node view */
  const int sides = mode == TWO_UNDIRECTED ? 2 : 1;
  const uint64_t P = mode == TWO_UNDIRECTED ? 2 * m : m;
  s->P = P;
  uint64_t* region = XALLOC(V, uint64_t);
  uint64_t* groups = XALLOC(V, uint64_t);
  int64_t* anchor = XALLOC(V, int64_t);
  int64_t* last = XALLOC(V, int64_t);
  for (uint64_t v = 0; v < V; ++v) last[v] = -1;
  for (uint64_t i = 0; i < m; ++i) { /* pass 1 :135-162 */
    for (int sd = 0; sd < sides; ++sd) {
      const uint32_t v = owner_of(s, i, sd);
      ++region[v];
      if (last[v] != s->t[i]) { ++groups[v]; last[v] = s->t[i]; }
      anchor[v] = s->t[i];
    }
  }
  s->n_off = XALLOC(V + 1, uint64_t);
  s->n_tsidx = XALLOC(V + 1, uint64_t);
  uint64_t ea = 0, ga = 0;
  for (uint64_t v = 0; v < V; ++v) { /* :164-174 */
    s->n_off[v] = ea; s->n_tsidx[v] = ga; ea += region[v]; ga += groups[v];
  }
  s->n_off[V] = ea;
  s->n_tsidx[V] = ga;
  s->Q = ga;
  s->ref_edge = XALLOC(P, uint32_t);
  s->mk_time = XALLOC(ga, int64_t);
  s->mk_start = XALLOC(ga, uint32_t);
  s->wprefix = XALLOC(P, double);
  uint64_t* ecur = XALLOC(V, uint64_t);
  uint64_t* gcur = XALLOC(V, uint64_t);
  double* wacc = XALLOC(V, double);
  for (uint64_t v = 0; v < V; ++v) { ecur[v] = s->n_off[v]; gcur[v] = s->n_tsidx[v]; last[v] = -1; }
  for (uint64_t i = 0; i < m; ++i) { /* pass 2 :176-214 */
    const int64_t t = s->t[i];
    for (int sd = 0; sd < sides; ++sd) {
      const uint32_t v = owner_of(s, i, sd);
      const uint64_t pos = ecur[v]++;
      s->ref_edge[pos] = (uint32_t)i;
      if (last[v] != t) {
        s->mk_time[gcur[v]] = t;
        s->mk_start[gcur[v]] = (uint32_t)pos;
        ++gcur[v];
        last[v] = t;
      }
      wacc[v] += exp((double)(t - anchor[v]));
      s->wprefix[pos] = wacc[v];
    }
  }
  free(region); free(groups); free(anchor); free(last); free(ecur); free(gcur); free(wacc);

  /* :216-250 sorted unique traversal neighbours */
  s->adj_off = XALLOC(V + 1, uint64_t);
  s->adj = XALLOC(P, uint32_t);
  uint64_t A = 0;
  for (uint64_t v = 0; v < V; ++v) {
    const uint64_t lo = s->n_off[v], hi = s->n_off[v + 1];
    uint32_t* seg = s->adj + A;
    for (uint64_t pos = lo; pos < hi; ++pos) seg[pos - lo] = two_ref_neighbor(s, pos, (uint32_t)v);
    qsort(seg, hi - lo, sizeof(uint32_t), cmp_u32);
    uint64_t u = 0;
    for (uint64_t k = 0; k < hi - lo; ++k) if (k == 0 || seg[k] != seg[k - 1]) seg[u++] = seg[k];
    s->adj_off[v] = A;
    A += u;
  }
  s->adj_off[V] = A;
  s->A = A;
  *status = TWO_OK;
  return s;
}

/* edge_store.cpp:264-268 (hash map in the reference; binary search here —
 * ext is ascending because ids are ranks) */
int two_find_node(const two_store* s, int64_t external, uint32_t* out) {
  uint64_t lo = 0, hi = s->V;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if ((uint64_t)s->ext[mid] < (uint64_t)external) lo = mid + 1;
    else hi = mid;
  }
  if (lo < s->V && s->ext[lo] == external) { *out = (uint32_t)lo; return 1; }
  return 0;
}

/* upper_bound on mark times: first g with t < time[g] */
static uint64_t ub_time(const int64_t* mt, uint64_t n, int64_t t) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (t < mt[mid]) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}
/* lower_bound on mark times: first g with time[g] >= t */
static uint64_t lb_time(const int64_t* mt, uint64_t n, int64_t t) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (mt[mid] < t) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

static int supports(const two_store* s, int dir) {
  if (s->mode == TWO_UNDIRECTED) return 1;
  return (s->mode == TWO_FORWARD) == (dir == 0);
}

/* walk_engine.cpp:18-34 causal_slice == edge_store.cpp:277-302 */
static void causal_slice(const two_store* s, uint32_t v, int64_t t, int dir, uint64_t* c, uint64_t* e,
                         uint64_t* gcount) {
  const uint64_t lo = s->n_off[v], hi = s->n_off[v + 1];
  const int64_t* mt = s->mk_time + s->n_tsidx[v];
  const uint32_t* ms = s->mk_start + s->n_tsidx[v];
  const uint64_t G = s->n_tsidx[v + 1] - s->n_tsidx[v];
  if (dir == 0) {
    const uint64_t g = ub_time(mt, G, t);
    *c = g == G ? hi : ms[g];
    *e = hi;
    if (gcount) *gcount = G - g;
  } else {
    const uint64_t g = lb_time(mt, G, t);
    *c = lo;
    *e = g == G ? hi : ms[g];
    if (gcount) *gcount = g;
  }
}

int two_temporal_neighborhood(const two_store* s, int64_t v, int64_t t, int dir, uint64_t* out3) {
  uint32_t iv;
  out3[0] = out3[1] = out3[2] = 0;
  if (!two_find_node(s, v, &iv)) return TWO_OK; /* :272-273 unknown -> empty */
  if (!supports(s, dir)) return TWO_EINVAL;      /* :279-281 */
  const uint64_t lo = s->n_off[iv], hi = s->n_off[iv + 1];
  if (lo == hi) { out3[0] = out3[1] = lo; return TWO_OK; }
  causal_slice(s, iv, t, dir, &out3[0], &out3[1], &out3[2]);
  return TWO_OK;
}

/* edge_store.cpp:310-314 */
int two_adjacent(const two_store* s, uint32_t a, uint32_t b) {
  uint64_t lo = s->adj_off[a], hi = s->adj_off[a + 1];
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (s->adj[mid] < b) lo = mid + 1;
    else hi = mid;
  }
  return lo < s->adj_off[a + 1] && s->adj[lo] == b;
}

/* edge_store.cpp:316-323 */
int two_adjacent_after(const two_store* s, uint32_t a, uint32_t b, int64_t t, int dir) {
  uint64_t c, e;
  causal_slice(s, a, t, dir, &c, &e, NULL);
  for (uint64_t pos = c; pos < e; ++pos) if (two_ref_neighbor(s, pos, a) == b) return 1;
  return 0;
}

/* edge_store.cpp:325-332 */
uint64_t two_export_suffix(const two_store* s, int64_t cutoff, two_edge** out) {
  uint64_t lo = 0, hi = s->m;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (s->t[mid] < cutoff) lo = mid + 1;
    else hi = mid;
  }
  const uint64_t n = s->m - lo;
  two_edge* e = (two_edge*)malloc((n ? n : 1) * sizeof(two_edge));
  for (uint64_t i = lo; i < s->m; ++i) {
    e[i - lo].src = s->ext[s->src[i]];
    e[i - lo].dst = s->ext[s->dst[i]];
    e[i - lo].t = s->t[i];
  }
  *out = e;
  return n;
}

/* -------------------------------------------------------------- window --- */

static two_store* empty_store(int mode) {
  int st;
  return two_build(NULL, 0, mode, &st);
}

/* window_manager.cpp:9-12 */
two_window* two_window_create(int64_t duration, int mode, int* status) {
  if (duration <= 0) { *status = TWO_EINVAL; return NULL; }
  two_window* w = XALLOC(1, two_window);
  w->duration = duration;
  w->mode = mode;
  w->store = empty_store(mode);
  w->t_high = TIME_UNSET;
  *status = TWO_OK;
  return w;
}

void two_window_free(two_window* w) {
  if (!w) return;
  two_store_free(w->store);
  free(w);
}

/* window_manager.hpp:51-53 */
static int64_t cutoff_for(const two_window* w, int64_t high) {
  return high > w->duration ? high - w->duration : 0;
}

/* window_manager.cpp:14-62 */
int two_window_ingest(two_window* w, const two_edge* batch, uint64_t n, two_batch_stats* out) {
  const double started = now_s();
  two_batch_stats st;
  memset(&st, 0, sizeof st);
  st.ingested = n;
  if (n == 0) { /* :21-28 */
    st.retained = w->store->m;
    w->stats = st;
    w->batch_count++;
    if (out) *out = st;
    return TWO_OK;
  }
  int64_t batch_high = TIME_UNSET;
  for (uint64_t i = 0; i < n; ++i) if (batch[i].t > batch_high) batch_high = batch[i].t;
  const int64_t new_high = w->t_high > batch_high ? w->t_high : batch_high;
  const int64_t cutoff = cutoff_for(w, new_high);
  two_edge* merged = NULL;
  const uint64_t surv = two_export_suffix(w->store, cutoff, &merged);
  st.evicted = w->store->m - surv;
  merged = (two_edge*)realloc(merged, (surv + n) * sizeof(two_edge));
  uint64_t k = surv;
  for (uint64_t i = 0; i < n; ++i) {
    if (batch[i].t >= cutoff) merged[k++] = batch[i];
    else st.dropped_late++;
  }
  int status;
  two_store* rebuilt = two_build(merged, k, w->mode, &status);
  free(merged);
  if (!rebuilt) return status;
  st.retained = rebuilt->m;
  st.rebuild_duration = now_s() - started;
  two_store_free(w->store);
  w->store = rebuilt;
  w->t_high = new_high;
  w->stats = st;
  w->batch_count++;
  if (out) *out = st;
  return TWO_OK;
}

/* window_manager.cpp:64-69 */
int two_window_bounds(const two_window* w, int64_t* lo, int64_t* hi) {
  if (w->batch_count == 0 || w->t_high == TIME_UNSET) return TWO_ELOGIC;
  *lo = cutoff_for(w, w->t_high);
  *hi = w->t_high;
  return TWO_OK;
}

/* --------------------------------------------------------------- walks --- */

/* walk_engine.cpp:189-196 */
static int thresholds_ok(const two_thresholds* t) {
  if (t->w_warp < 1 || t->w_warp > t->block_dim || t->block_dim > t->w_max) return 0;
  if (t->g_warp_cap > t->g_block_cap) return 0;
  return 1;
}

/* walk_engine.cpp:198-206 */
static int config_ok(const two_walk_config* c) {
  if (c->walk_length < 1) return 0;
  if (c->start_mode == 0 && c->walks_per_node == 0) return 0;
  if (c->node2vec && (c->p <= 0.0 || c->q <= 0.0)) return 0;
  return 1;
}

typedef struct {
  uint32_t* cur;
  int64_t* time;
  uint32_t* prev;
  uint8_t* has_prev;
  uint8_t* alive;
  uint32_t* length;
} walk_states;

/* walk_engine.cpp:39-44: time of the group containing pos */
static int64_t time_at_position(const two_store* s, uint32_t v, uint64_t pos) {
  const int64_t* mt = s->mk_time + s->n_tsidx[v];
  const uint32_t* ms = s->mk_start + s->n_tsidx[v];
  const uint64_t G = s->n_tsidx[v + 1] - s->n_tsidx[v];
  uint64_t lo = 0, hi = G;
  while (lo < hi) { /* first g with pos < start[g] */
    const uint64_t mid = lo + (hi - lo) / 2;
    if (pos < ms[mid]) hi = mid;
    else lo = mid + 1;
  }
  return mt[lo - 1];
}

/* walk_engine.cpp:49-63 */
static uint64_t draw_weighted_local(const two_store* s, double u, uint64_t c, uint64_t e) {
  const int64_t anchor = s->t[s->ref_edge[e - 1]];
  double total = 0.0;
  for (uint64_t pos = c; pos < e; ++pos) total += exp((double)(s->t[s->ref_edge[pos]] - anchor));
  const double r = u * total;
  double cum = 0.0;
  for (uint64_t pos = c; pos < e; ++pos) {
    cum += exp((double)(s->t[s->ref_edge[pos]] - anchor));
    if (r < cum) return pos - c;
  }
  return e - 1 - c;
}

/* walk_engine.cpp:65-84 */
static uint64_t draw_index(const two_store* s, int bias, double u, uint64_t lo, uint64_t c, uint64_t e) {
  const uint64_t n = e - c;
  switch (bias) {
    case TWO_UNIFORM: return pick_uniform(u, n);
    case TWO_LINEAR: return pick_linear(u, n);
    case TWO_EXPINDEX: return pick_exponential(u, n);
    default: {
      const double* prefix = s->wprefix;
      const double base = c > lo ? prefix[c - 1] : 0.0;
      const double mass = prefix[e - 1] - base;
      if (!(mass > 0.0) || !isfinite(mass)) return draw_weighted_local(s, u, c, e);
      return two_pick_weighted_range(u, prefix, c, e, base);
    }
  }
}

/* samplers.hpp:74-86 node2vec_accept */
static int node2vec_accept(const two_store* s, const two_walk_config* c, uint32_t prev, uint32_t cand,
                           int64_t t, double u_accept) {
  double beta;
  if (cand == prev) {
    beta = 1.0 / c->p;
  } else if (c->temporal_adjacency ? two_adjacent_after(s, prev, cand, t, c->direction)
                                   : two_adjacent(s, prev, cand)) {
    beta = 1.0;
  } else {
    beta = 1.0 / c->q;
  }
  double bmax = 1.0 / c->p; /* samplers.hpp:27-29 beta_max */
  if (1.0 > bmax) bmax = 1.0;
  if (1.0 / c->q > bmax) bmax = 1.0 / c->q;
  return u_accept < beta / bmax;
}

/* walk_engine.cpp:88-145 hop_walk */
static int hop_walk(const two_store* s, const two_walk_config* c, uint32_t w, walk_states* st, two_walkset* ws) {
  const uint32_t v = st->cur[w];
  const int64_t t = st->time[w];
  const uint64_t lo = s->n_off[v];
  uint64_t cc, e;
  causal_slice(s, v, t, c->direction, &cc, &e, NULL);
  if (cc == e) { st->alive[w] = 0; return 0; }
  const uint64_t hop = st->length[w];
  uint64_t idx;
  if (c->node2vec && st->has_prev[w]) {
    const uint32_t prev = st->prev[w];
    idx = 0;
    for (int r = 0; r < 64; ++r) { /* kNode2VecMaxRetries samplers.hpp:89 */
      const double u = two_rng_uniform(c->rng, c->seed, w, hop, 2 * (uint64_t)r);
      idx = draw_index(s, c->bias, u, lo, cc, e);
      const uint32_t cand = two_ref_neighbor(s, cc + idx, v);
      const double ua = two_rng_uniform(c->rng, c->seed, w, hop, 2 * (uint64_t)r + 1);
      if (node2vec_accept(s, c, prev, cand, t, ua)) break;
    }
  } else {
    const double u = two_rng_uniform(c->rng, c->seed, w, hop, 0);
    idx = draw_index(s, c->bias, u, lo, cc, e);
  }
  const uint64_t pos = cc + idx;
  const uint32_t next = two_ref_neighbor(s, pos, v);
  const int64_t next_time = time_at_position(s, v, pos);
  const uint32_t slot = st->length[w];
  ws->nodes[(uint64_t)w * ws->stride + slot] = s->ext[next];
  ws->times[(uint64_t)w * ws->stride + slot] = next_time;
  st->length[w] = slot + 1;
  if (c->node2vec) { st->prev[w] = v; st->has_prev[w] = 1; }
  st->cur[w] = next;
  st->time[w] = next_time;
  if (st->length[w] >= ws->stride) st->alive[w] = 0;
  return 1;
}

/* walk_engine.cpp:147-155 */
static void seed_walk(walk_states* st, two_walkset* ws, uint64_t w, int64_t ext, uint32_t v, int64_t sentinel) {
  ws->nodes[w * ws->stride] = ext;
  ws->times[w * ws->stride] = sentinel;
  st->cur[w] = v;
  st->time[w] = sentinel;
  st->length[w] = 1;
  st->alive[w] = ws->stride > 1;
}

/* walk_engine.cpp:284-299 */
uint64_t two_sample_start_edge(const two_store* s, int bias, double u1, double u2) {
  const uint64_t Z = s->Z;
  uint64_t g;
  switch (bias) {
    case TWO_UNIFORM: g = pick_uniform(u1, Z); break;
    case TWO_LINEAR: g = pick_linear(u1, Z); break;
    case TWO_EXPINDEX: g = pick_exponential(u1, Z); break;
    default: g = two_pick_weighted(u1, s->ts_w, Z); break;
  }
  const uint64_t lo = s->ts_off[g], hi = s->ts_off[g + 1];
  uint64_t off = (uint64_t)(u2 * (double)(hi - lo));
  if (off >= hi - lo) off = hi - lo - 1;
  return lo + off;
}

void two_walkset_free(two_walkset* w) {
  if (!w) return;
  free(w->nodes); free(w->times); free(w->lengths);
  w->nodes = NULL; w->times = NULL; w->lengths = NULL;
}

typedef struct {
  uint32_t node, walk;
} node_walk;

static int cmp_node_walk(const void* a, const void* b) {
  const node_walk* x = (const node_walk*)a;
  const node_walk* y = (const node_walk*)b;
  if (x->node != y->node) return x->node < y->node ? -1 : 1;
  return 0; /* ties keep order: sorted by a stable merge below */
}

/* stable sort of (node, walk) pairs by node: insertion into buckets */
static void stable_sort_by_node(node_walk* a, uint64_t n, uint64_t V) {
  uint64_t* cnt = XALLOC(V + 1, uint64_t);
  for (uint64_t i = 0; i < n; ++i) cnt[a[i].node + 1]++;
  for (uint64_t v = 0; v < V; ++v) cnt[v + 1] += cnt[v];
  node_walk* tmp = XALLOC(n, node_walk);
  for (uint64_t i = 0; i < n; ++i) tmp[cnt[a[i].node]++] = a[i];
  memcpy(a, tmp, n * sizeof(node_walk));
  free(tmp);
  free(cnt);
  (void)cmp_node_walk;
}

/* walk_engine.cpp:362-429 generate_walks (+ init_walks :208-282,
 * schedule_step :301-345 for the step/tier statistics). */
int two_generate(const two_store* s, const two_walk_config* c, const two_thresholds* th, int variant,
                 two_walkset* out, two_walk_stats* stats) {
  const double started = now_s();
  two_thresholds dflt = {4, 256, 8192, 512, 4096};
  if (!th) th = &dflt;
  memset(out, 0, sizeof *out);
  if (!config_ok(c) || !thresholds_ok(th)) return TWO_EINVAL;
  if (!supports(s, c->direction)) return TWO_EINVAL;
  const int64_t sentinel = c->direction == 0 ? TIME_UNSET : TIME_INFINITE; /* types.hpp:47-49 */

  uint64_t count = 0;
  uint32_t* start_nodes = NULL;
  uint64_t n_start = 0;
  if (c->start_mode == 0) {
    start_nodes = XALLOC(s->V, uint32_t);
    for (uint64_t v = 0; v < s->V; ++v) if (s->n_off[v] != s->n_off[v + 1]) start_nodes[n_start++] = (uint32_t)v;
    count = n_start * (uint64_t)c->walks_per_node;
    out->stride = c->walk_length;
  } else {
    if (s->m == 0) return TWO_EINVAL;
    count = c->total_walks;
    out->stride = c->walk_length > 2 ? c->walk_length : 2;
  }
  if (count >= UINT32_MAX) { free(start_nodes); return TWO_EINVAL; }
  out->walk_count = count;
  out->nodes = XALLOC(count * out->stride, int64_t);
  out->times = XALLOC(count * out->stride, int64_t);
  out->lengths = XALLOC(count, uint32_t);
  walk_states st;
  st.cur = XALLOC(count, uint32_t);
  st.time = XALLOC(count, int64_t);
  st.prev = XALLOC(count, uint32_t);
  st.has_prev = XALLOC(count, uint8_t);
  st.alive = XALLOC(count, uint8_t);
  st.length = XALLOC(count, uint32_t);
  if (c->start_mode == 0) {
    uint64_t w = 0;
    for (uint64_t i = 0; i < n_start; ++i)
      for (uint32_t j = 0; j < c->walks_per_node; ++j, ++w)
        seed_walk(&st, out, w, s->ext[start_nodes[i]], start_nodes[i], sentinel);
  } else {
    const int forward = c->direction == 0;
    for (uint64_t w = 0; w < count; ++w) {
      const double u1 = two_rng_uniform(c->rng, c->seed, w, 0, 0);
      const double u2 = two_rng_uniform(c->rng, c->seed, w, 0, 1);
      const uint64_t eidx = two_sample_start_edge(s, c->start_bias, u1, u2);
      const uint32_t from = forward ? s->src[eidx] : s->dst[eidx];
      const uint32_t to = forward ? s->dst[eidx] : s->src[eidx];
      seed_walk(&st, out, w, s->ext[from], from, sentinel);
      out->nodes[w * out->stride + 1] = s->ext[to];
      out->times[w * out->stride + 1] = s->t[eidx];
      st.length[w] = 2;
      st.cur[w] = to;
      st.time[w] = s->t[eidx];
      if (c->node2vec) { st.prev[w] = from; st.has_prev[w] = 1; }
      st.alive[w] = out->stride > 2;
    }
  }
  free(start_nodes);

  two_walk_stats ws;
  memset(&ws, 0, sizeof ws);
  if (variant == 2) { /* FullWalk :380-392 */
    uint32_t max_hops = 0;
    for (uint64_t w = 0; w < count; ++w) {
      const uint32_t init_len = st.length[w];
      while (st.alive[w]) hop_walk(s, c, (uint32_t)w, &st, out);
      if (st.length[w] - init_len > max_hops) max_hops = st.length[w] - init_len;
    }
    ws.steps = max_hops;
  } else { /* Coop / CoopDirect :393-418 */
    node_walk* plan = XALLOC(count, node_walk);
    uint32_t* cand = XALLOC(count, uint32_t);
    uint64_t n_cand = count;
    for (uint64_t i = 0; i < count; ++i) cand[i] = (uint32_t)i;
    for (;;) {
      uint64_t n = 0;
      for (uint64_t i = 0; i < n_cand; ++i) { /* partition_flagged primitives.cpp:140-148 */
        if (st.alive[cand[i]]) { plan[n].walk = cand[i]; plan[n].node = st.cur[cand[i]]; ++n; }
      }
      if (n == 0) break;
      ++ws.steps;
      stable_sort_by_node(plan, n, s->V);
      for (uint64_t i = 0; i < n;) { /* run_length_encode + tiering :313-343 */
        uint64_t j = i + 1;
        while (j < n && plan[j].node == plan[i].node) ++j;
        const uint64_t W = j - i;
        const uint64_t G = s->n_tsidx[plan[i].node + 1] - s->n_tsidx[plan[i].node];
        if (W < th->w_warp) ws.solo++;
        else if (W <= th->block_dim) { if (G <= th->g_warp_cap) ws.warp_cached++; else ws.warp_direct++; }
        else if (W <= th->w_max) { if (G <= th->g_block_cap) ws.block_cached++; else ws.block_direct++; }
        else ws.multi_block += (W + th->w_max - 1) / th->w_max; /* count_tier :157-161 */
        i = j;
      }
      for (uint64_t i = 0; i < n; ++i) hop_walk(s, c, plan[i].walk, &st, out);
      for (uint64_t i = 0; i < n; ++i) cand[i] = plan[i].walk;
      n_cand = n;
    }
    free(plan);
    free(cand);
  }
  for (uint64_t w = 0; w < count; ++w) { /* :420-426 */
    out->lengths[w] = st.length[w];
    if (st.length[w] >= 2) { ws.walks++; ws.hops += st.length[w] - 1; }
  }
  free(st.cur); free(st.time); free(st.prev); free(st.has_prev); free(st.alive); free(st.length);
  ws.wall_seconds = now_s() - started;
  if (stats) *stats = ws;
  return TWO_OK;
}

/* -------------------------------------------------------------- replay --- */

void two_replay_free(two_replay_result* r) {
  if (!r) return;
  if (r->walks) for (uint64_t b = 0; b < r->batches; ++b) two_walkset_free(&r->walks[b]);
  free(r->ingest); free(r->walk); free(r->walks);
  memset(r, 0, sizeof *r);
}

/* replay.cpp:16-53 (validation :7-14) */
int two_replay(const two_edge* edges, uint64_t n, const two_replay_config* c, two_replay_result* out) {
  memset(out, 0, sizeof *out);
  if (c->batch_duration <= 0 || c->window_duration < c->batch_duration) return TWO_EINVAL;
  if (!config_ok(&c->walk) || !thresholds_ok(&c->thresholds)) return TWO_EINVAL;
  if (n == 0) return TWO_OK;
  int status;
  two_window* win = two_window_create(c->window_duration, c->mode, &status);
  if (!win) return status;
  uint64_t cap = 16;
  out->ingest = XALLOC(cap, two_batch_stats);
  out->walk = XALLOC(cap, two_walk_stats);
  out->walks = XALLOC(cap, two_walkset);
  const int64_t origin = edges[0].t;
  int64_t boundary = origin + c->batch_duration;
  uint64_t begin = 0;
  status = TWO_OK;
  for (uint64_t i = 0; i <= n && status == TWO_OK; ++i) {
    const int at_end = i == n;
    if (at_end || edges[i].t >= boundary) {
      if (i > begin) { /* flush :28-40 */
        if (out->batches == cap) {
          cap *= 2;
          out->ingest = (two_batch_stats*)realloc(out->ingest, cap * sizeof(two_batch_stats));
          out->walk = (two_walk_stats*)realloc(out->walk, cap * sizeof(two_walk_stats));
          out->walks = (two_walkset*)realloc(out->walks, cap * sizeof(two_walkset));
        }
        const uint64_t b = out->batches;
        memset(&out->walk[b], 0, sizeof(two_walk_stats));
        memset(&out->walks[b], 0, sizeof(two_walkset));
        status = two_window_ingest(win, edges + begin, i - begin, &out->ingest[b]);
        if (status == TWO_OK && c->generate && win->store->m > 0) {
          status = two_generate(win->store, &c->walk, &c->thresholds, c->variant, &out->walks[b], &out->walk[b]);
          if (!c->keep_walks) two_walkset_free(&out->walks[b]);
        }
        out->batches++;
        begin = i;
      }
      if (!at_end) { /* :46-47 jump the boundary past any gap */
        const int64_t spans = (edges[i].t - origin) / c->batch_duration + 1;
        boundary = origin + spans * c->batch_duration;
      }
    }
  }
  two_window_free(win);
  return status;
}
