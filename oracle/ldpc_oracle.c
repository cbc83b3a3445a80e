/*
 * ldpc_oracle.c -- CPU ORACLE (test infrastructure only; see ldpc_oracle.h).
 *
 * fp64 restatement of arxiv/paper_1202_1060 proj/include/ldpc/*.hpp in plain
 * C. The operation order of every floating-point expression follows the
 * reference so that results are bit-identical to the reference compiled with
 * the same compiler flags and libm (pinned in tests/test_oracle.py against
 * oracle/_ref, the unmodified reference headers).
 */
#include "ldpc_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

const char *orc_last_error(void) { return g_err; }

static int fail(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return -1;
}

/* ======================================================================
 * rng.hpp
 * ==================================================================== */

/* rng.hpp:10-15 */
uint64_t orc_splitmix64(uint64_t *state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/* rng.hpp:19-25 */
uint64_t orc_mix_seed(uint64_t seed, uint64_t stream) {
  uint64_t s = seed;
  uint64_t z = orc_splitmix64(&s);
  s ^= 0xd1342543de82ef95ull * (stream + 1);
  z ^= orc_splitmix64(&s);
  return z;
}

/* rng.hpp:31-34 */
void orc_rng_seed(orc_rng *r, uint64_t seed) {
  uint64_t s = seed;
  for (int i = 0; i < 4; ++i) r->s[i] = orc_splitmix64(&s);
  r->spare = 0.0;
  r->has_spare = 0;
}

static inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* rng.hpp:36-46 (xoshiro256++) */
uint64_t orc_rng_u64(orc_rng *r) {
  uint64_t *s = r->s;
  const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}

/* rng.hpp:49: uniform on (0, 1] */
double orc_rng_unit(orc_rng *r) { return (double)((orc_rng_u64(r) >> 11) + 1) * 0x1.0p-53; }

/* rng.hpp:52-64: Box-Muller, cos first, sin cached */
double orc_rng_gauss(orc_rng *r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  const double u1 = orc_rng_unit(r);
  const double u2 = orc_rng_unit(r);
  const double radius = sqrt(-2.0 * log(u1));
  const double angle = 6.283185307179586476925286766559 * u2;
  r->spare = radius * sin(angle);
  r->has_spare = 1;
  return radius * cos(angle);
}

/* rng.hpp:67-73 */
uint64_t orc_rng_below(orc_rng *r, uint64_t n) {
  const uint64_t threshold = (0 - n) % n;
  for (;;) {
    const uint64_t x = orc_rng_u64(r);
    if (x >= threshold) return x % n;
  }
}

/* rng.hpp:75-82 (Fisher-Yates from the back) */
void orc_rng_shuffle(orc_rng *r, int32_t *a, int64_t n) {
  for (uint64_t i = (uint64_t)n; i > 1; --i) {
    const uint64_t j = orc_rng_below(r, i);
    int32_t t = a[i - 1];
    a[i - 1] = a[j];
    a[j] = t;
  }
}

/* ======================================================================
 * channel.hpp
 * ==================================================================== */

/* channel.hpp:21-24 */
double orc_sigma2_from_ebn0(double ebn0_db, double rate) {
  if (!(rate > 0.0) || rate > 1.0) {
    fail("code rate must be in (0, 1]");
    return NAN;
  }
  return 1.0 / (2.0 * rate * pow(10.0, ebn0_db / 10.0));
}

/* channel.hpp:38-46 */
int orc_transmit_all_zero(double sigma2, uint64_t seed, int n, uint64_t frame_id, double *llr) {
  if (n < 1) return fail("frame length must be >= 1");
  orc_rng rng;
  orc_rng_seed(&rng, orc_mix_seed(seed, frame_id));
  const double sigma = sqrt(sigma2);
  const double scale = 2.0 / sigma2;
  for (int i = 0; i < n; ++i) llr[i] = scale * (1.0 + sigma * orc_rng_gauss(&rng));
  return 0;
}

/* ======================================================================
 * tanner.hpp
 * ==================================================================== */

struct orc_graph {
  int n, m, E;
  int32_t *row_off; /* check_edge_offset, tanner.hpp:27 */
  int32_t *cols;    /* check_adj flattened (CN-major edge order) */
  int32_t *var_off;
  int32_t *var_cns;   /* var_adj, ascending CN ids */
  int32_t *var_edges; /* var_edge_ids */
};

/* build_from_check_lists, tanner.hpp:79-114 */
orc_graph *orc_graph_create(int n, int m, const int32_t *row_off, const int32_t *cols) {
  if (n < 1 || m < 1) {
    fail("graph must have at least one VN and one CN");
    return NULL;
  }
  if (row_off[0] != 0) {
    fail("row offsets must start at 0");
    return NULL;
  }
  const int E = row_off[m];
  char *seen = calloc((size_t)n, 1);
  for (int r = 0; r < m; ++r) {
    const int deg = row_off[r + 1] - row_off[r];
    if (deg < 2) {
      free(seen);
      fail("check node %d has degree < 2", r);
      return NULL;
    }
    for (int e = row_off[r]; e < row_off[r + 1]; ++e) {
      const int v = cols[e];
      if (v < 0 || v >= n) {
        free(seen);
        fail("VN index out of range in check node %d", r);
        return NULL;
      }
      if (seen[v]) {
        free(seen);
        fail("duplicate VN in check node %d", r);
        return NULL;
      }
      seen[v] = 1;
    }
    for (int e = row_off[r]; e < row_off[r + 1]; ++e) seen[cols[e]] = 0;
  }
  free(seen);

  orc_graph *g = calloc(1, sizeof *g);
  g->n = n;
  g->m = m;
  g->E = E;
  g->row_off = malloc(sizeof(int32_t) * (size_t)(m + 1));
  g->cols = malloc(sizeof(int32_t) * (size_t)(E > 0 ? E : 1));
  memcpy(g->row_off, row_off, sizeof(int32_t) * (size_t)(m + 1));
  memcpy(g->cols, cols, sizeof(int32_t) * (size_t)E);
  g->var_off = calloc((size_t)n + 1, sizeof(int32_t));
  g->var_cns = malloc(sizeof(int32_t) * (size_t)(E > 0 ? E : 1));
  g->var_edges = malloc(sizeof(int32_t) * (size_t)(E > 0 ? E : 1));
  for (int e = 0; e < E; ++e) g->var_off[cols[e] + 1]++;
  for (int v = 0; v < n; ++v) {
    if (g->var_off[v + 1] == 0) {
      orc_graph_destroy(g);
      fail("isolated VN %d", v);
      return NULL;
    }
    g->var_off[v + 1] += g->var_off[v];
  }
  int32_t *fill = malloc(sizeof(int32_t) * (size_t)n);
  for (int v = 0; v < n; ++v) fill[v] = g->var_off[v];
  /* tanner.hpp:103-109: CNs visited in ascending order -> var_adj ascending */
  for (int r = 0; r < m; ++r)
    for (int e = row_off[r]; e < row_off[r + 1]; ++e) {
      const int v = cols[e];
      g->var_cns[fill[v]] = r;
      g->var_edges[fill[v]] = e;
      fill[v]++;
    }
  free(fill);
  return g;
}

void orc_graph_destroy(orc_graph *g) {
  if (!g) return;
  free(g->row_off);
  free(g->cols);
  free(g->var_off);
  free(g->var_cns);
  free(g->var_edges);
  free(g);
}

int orc_graph_n_edges(const orc_graph *g) { return g->E; }

void orc_graph_var_view(const orc_graph *g, int32_t *var_off, int32_t *var_cns, int32_t *var_edges) {
  if (var_off) memcpy(var_off, g->var_off, sizeof(int32_t) * (size_t)(g->n + 1));
  if (var_cns) memcpy(var_cns, g->var_cns, sizeof(int32_t) * (size_t)g->E);
  if (var_edges) memcpy(var_edges, g->var_edges, sizeof(int32_t) * (size_t)g->E);
}

/* random_regular_graph, tanner.hpp:356-393 */
int orc_random_regular(int n, int dv, int dc, uint64_t seed, int32_t *cols_out) {
  if (n < 1 || dv < 1 || dc < 2) return fail("need n_vars >= 1, d_v >= 1, d_c >= 2");
  const long long sockets = (long long)n * dv;
  if (sockets % dc != 0) return fail("socket count %lld is not divisible by d_c", sockets);
  const int m = (int)(sockets / dc);
  orc_rng rng;
  orc_rng_seed(&rng, seed);
  int32_t *perm = malloc(sizeof(int32_t) * (size_t)sockets);
  for (long long i = 0; i < sockets; ++i) perm[i] = (int32_t)i;
  char *seen = calloc((size_t)n, 1);
  for (int attempt = 0; attempt < 20000; ++attempt) {
    orc_rng_shuffle(&rng, perm, sockets);
    int simple = 1;
    for (int r = 0; r < m && simple; ++r) {
      for (int k = 0; k < dc; ++k) {
        const int vn = perm[r * dc + k] / dv;
        if (seen[vn]) {
          simple = 0;
          break;
        }
        seen[vn] = 1;
      }
      for (int k = 0; k < dc; ++k) seen[perm[r * dc + k] / dv] = 0;
    }
    if (!simple) continue;
    for (long long i = 0; i < sockets; ++i) cols_out[i] = perm[i] / dv;
    free(perm);
    free(seen);
    return m;
  }
  free(perm);
  free(seen);
  return fail("could not draw a duplicate-free regular graph after 20000 attempts");
}

/* ======================================================================
 * schedule.hpp
 * ==================================================================== */

static int contains(const int32_t *a, int n, int32_t x) {
  for (int i = 0; i < n; ++i)
    if (a[i] == x) return 1;
  return 0;
}

/* detail::generate_groups, schedule.hpp:54-115 */
int orc_generate_groups(int M, int G, double overlap, uint64_t rng_seed, int32_t *grp_off, int32_t *grp_cns,
                        int max_slots) {
  orc_rng rng;
  orc_rng_seed(&rng, rng_seed);
  int32_t *pool = malloc(sizeof(int32_t) * (size_t)M);
  for (int i = 0; i < M; ++i) pool[i] = i;
  orc_rng_shuffle(&rng, pool, M);
  int rc = 0;
  grp_off[0] = 0;
  if (overlap == 0.0) { /* schedule.hpp:60-70 */
    const int base = M / G, extra = M % G;
    int next = 0;
    for (int g = 0; g < G; ++g) {
      const int size = base + (g < extra ? 1 : 0);
      if (next + size > max_slots) {
        rc = fail("slot buffer too small");
        goto out;
      }
      memcpy(grp_cns + next, pool + next, sizeof(int32_t) * (size_t)size);
      next += size;
      grp_off[g + 1] = next;
    }
    rc = next;
    goto out;
  }
  {
    const double denom = G - (G - 1) * overlap; /* schedule.hpp:72-77 */
    const int nominal = (int)ceil(M / denom);
    const int k = (int)llround(nominal * overlap);
    if (G > 1 && 2 * k > nominal) {
      rc = fail("infeasible (G, r): overlap %d exceeds the fresh half of N_G=%d", k, nominal);
      goto out;
    }
    int next = 0, w = 0;
    int32_t *cand = malloc(sizeof(int32_t) * (size_t)(M > 0 ? M : 1));
    /* group 0: take_fresh(nominal), schedule.hpp:87-89 */
    {
      int got = nominal < M - next ? nominal : M - next;
      if (w + got > max_slots) {
        free(cand);
        rc = fail("slot buffer too small");
        goto out;
      }
      memcpy(grp_cns + w, pool + next, sizeof(int32_t) * (size_t)got);
      next += got;
      w += got;
      grp_off[1] = w;
      const int want = nominal < M ? nominal : M;
      if (got < want) {
        free(cand);
        rc = fail("infeasible (G, r): first group cannot be filled");
        goto out;
      }
    }
    for (int g = 1; g < G; ++g) { /* schedule.hpp:90-112 */
      const int32_t *prev = grp_cns + grp_off[g - 1];
      const int nprev = grp_off[g] - grp_off[g - 1];
      int nc = 0;
      if (g == 1) {
        memcpy(cand, prev, sizeof(int32_t) * (size_t)nprev);
        nc = nprev;
      } else {
        const int32_t *pp = grp_cns + grp_off[g - 2];
        const int npp = grp_off[g - 1] - grp_off[g - 2];
        for (int i = 0; i < nprev; ++i)
          if (!contains(pp, npp, prev[i])) cand[nc++] = prev[i];
      }
      orc_rng_shuffle(&rng, cand, nc);
      const int k_take = k < nc ? k : nc;
      int fresh_want = nominal - k_take;
      if (g == G - 1) fresh_want = M - next;
      const int got = fresh_want < M - next ? fresh_want : M - next;
      if (w + k_take + got > max_slots) {
        free(cand);
        rc = fail("slot buffer too small");
        goto out;
      }
      memcpy(grp_cns + w, cand, sizeof(int32_t) * (size_t)k_take);
      w += k_take;
      if (g < G - 1 && got < fresh_want) {
        free(cand);
        rc = fail("infeasible (G, r): fresh pool exhausted at group %d", g + 1);
        goto out;
      }
      memcpy(grp_cns + w, pool + next, sizeof(int32_t) * (size_t)got);
      next += got;
      w += got;
      grp_off[g + 1] = w;
      if (grp_off[g + 1] == grp_off[g]) {
        free(cand);
        rc = fail("infeasible (G, r): empty group %d", g + 1);
        goto out;
      }
    }
    free(cand);
    if (next != M) {
      rc = fail("infeasible (G, r): groups do not cover all CNs");
      goto out;
    }
    rc = w;
  }
out:
  free(pool);
  return rc;
}

/* iteration_budget, schedule.hpp:206-210 */
int orc_iteration_budget(int n_checks, int i_max, int kind, int n_groups, int group_size, double overlap) {
  if (kind != ORC_NONDISJOINT || overlap == 0.0) return i_max;
  const double extra = (n_groups - 1) * (double)group_size * overlap;
  return (int)floor((double)n_checks * i_max / (n_checks + extra));
}

/* ======================================================================
 * decoder.hpp
 * ==================================================================== */

#define ORC_LLR_CLAMP 30.0 /* decoder.hpp:18 */

static inline double clamp_d(double x, double lo, double hi) { return x < lo ? lo : (hi < x ? hi : x); }
static inline double clamp_llr(double x) { return clamp_d(x, -ORC_LLR_CLAMP, ORC_LLR_CLAMP); } /* :20 */

/* check_update, decoder.hpp:59-87 (tanh rule, per-edge division, exclusion
 * products when the full product is exactly zero) */
void orc_check_update(int degree, const double *v2c, double *c2v) {
  double terms_small[64];
  double *terms = degree <= 64 ? terms_small : malloc(sizeof(double) * (size_t)degree);
  double product = 1.0;
  for (int k = 0; k < degree; ++k) {
    terms[k] = tanh(0.5 * v2c[k]);
    product *= terms[k];
  }
  const double cap = 1.0 - 1e-15;
  if (product == 0.0) {
    for (int k = 0; k < degree; ++k) {
      double excl = 1.0;
      for (int j = 0; j < degree; ++j)
        if (j != k) excl *= terms[j];
      excl = clamp_d(excl, -cap, cap);
      c2v[k] = clamp_llr(2.0 * atanh(excl));
    }
  } else {
    for (int k = 0; k < degree; ++k) {
      double excl = clamp_d(product / terms[k], -cap, cap);
      c2v[k] = clamp_llr(2.0 * atanh(excl));
    }
  }
  if (terms != terms_small) free(terms);
}

typedef struct {
  double *ch;  /* channel_llr (clamped) */
  double *v2c; /* per edge */
  double *c2v; /* per edge */
  double *total;
  uint8_t *hard;
  int32_t *touched;
  char *mark;
  int32_t *regroup_off, *regroup_cns; /* per-iteration regroup buffers */
} dstate;

static void state_alloc(dstate *st, const orc_graph *g, int n_groups) {
  st->ch = malloc(sizeof(double) * (size_t)g->n);
  st->v2c = malloc(sizeof(double) * (size_t)g->E);
  st->c2v = malloc(sizeof(double) * (size_t)g->E);
  st->total = malloc(sizeof(double) * (size_t)g->n);
  st->hard = malloc((size_t)g->n);
  st->touched = malloc(sizeof(int32_t) * (size_t)g->n);
  st->mark = calloc((size_t)g->n, 1);
  st->regroup_off = malloc(sizeof(int32_t) * (size_t)(n_groups + 1));
  st->regroup_cns = malloc(sizeof(int32_t) * (size_t)(2 * g->m + 1));
}

static void state_free(dstate *st) {
  free(st->ch);
  free(st->v2c);
  free(st->c2v);
  free(st->total);
  free(st->hard);
  free(st->touched);
  free(st->mark);
  free(st->regroup_off);
  free(st->regroup_cns);
}

/* init_state, decoder.hpp:39-52 */
static void init_state(dstate *st, const orc_graph *g, const double *llr) {
  for (int v = 0; v < g->n; ++v) st->ch[v] = clamp_llr(llr[v]);
  for (int e = 0; e < g->E; ++e) st->c2v[e] = 0.0;
  for (int v = 0; v < g->n; ++v)
    for (int j = g->var_off[v]; j < g->var_off[v + 1]; ++j) st->v2c[g->var_edges[j]] = st->ch[v];
  for (int v = 0; v < g->n; ++v) {
    st->total[v] = 0.0;
    st->hard[v] = 0;
  }
}

/* var_update, decoder.hpp:91-105 (exclusion sum in adjacency order) */
static double var_update(const dstate *st, const orc_graph *g, int v, int exclude_m) {
  double sum = st->ch[v];
  for (int j = g->var_off[v]; j < g->var_off[v + 1]; ++j) {
    if (g->var_cns[j] == exclude_m) continue;
    sum += st->c2v[g->var_edges[j]];
  }
  return sum;
}

static int cmp_i32(const void *a, const void *b) {
  const int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

/* run_subiteration, decoder.hpp:112-127 */
static void run_subiteration(dstate *st, const orc_graph *g, const int32_t *grp, int gsize) {
  for (int i = 0; i < gsize; ++i) {
    const int m = grp[i];
    const int off = g->row_off[m];
    orc_check_update(g->row_off[m + 1] - off, st->v2c + off, st->c2v + off);
  }
  int nt = 0; /* sorted unique touched VNs */
  for (int i = 0; i < gsize; ++i) {
    const int m = grp[i];
    for (int e = g->row_off[m]; e < g->row_off[m + 1]; ++e) {
      const int v = g->cols[e];
      if (!st->mark[v]) {
        st->mark[v] = 1;
        st->touched[nt++] = v;
      }
    }
  }
  qsort(st->touched, (size_t)nt, sizeof(int32_t), cmp_i32);
  for (int t = 0; t < nt; ++t) {
    const int v = st->touched[t];
    st->mark[v] = 0;
    for (int j = g->var_off[v]; j < g->var_off[v + 1]; ++j)
      st->v2c[g->var_edges[j]] = clamp_llr(var_update(st, g, v, g->var_cns[j]));
  }
}

/* syndrome_weight, decoder.hpp:129-137 */
static int syndrome_weight(const orc_graph *g, const uint8_t *bits) {
  int weight = 0;
  for (int m = 0; m < g->m; ++m) {
    int parity = 0;
    for (int e = g->row_off[m]; e < g->row_off[m + 1]; ++e) parity ^= bits[g->cols[e]];
    weight += parity;
  }
  return weight;
}

/* decode, decoder.hpp:143-181 (early_stop=1); early_stop=0 is the
 * fixed-iteration composition used by acceptance.cpp:142-146 */
static int decode_impl(dstate *st, const orc_graph *g, const orc_schedule *s, uint64_t frame_id, const double *llr,
                       int max_iters, int early_stop, uint8_t *bits, int32_t *iterations, uint8_t *converged,
                       double *posterior, int32_t *trace, int64_t *cn_updates) {
  if (max_iters < 1) return fail("max_iters must be >= 1");
  init_state(st, g, llr);
  const int32_t *goff = s->grp_off, *gcns = s->grp_cns;
  int G = s->n_groups;
  uint64_t seed = s->seed;
  if (s->per_frame && s->kind != ORC_FLOODING) {
    /* run_frame (sim.hpp:113-117): sched.seed = mix_seed(schedule_seed,
     * frame_id); groups = schedule_groups_for(sched, M, 1) */
    seed = orc_mix_seed(s->seed, frame_id);
    const double ov = s->kind == ORC_NONDISJOINT ? s->overlap : 0.0;
    if (orc_generate_groups(g->m, s->n_groups, ov, orc_mix_seed(seed, 1), st->regroup_off, st->regroup_cns,
                            2 * g->m + 1) < 0)
      return -1;
    goff = st->regroup_off;
    gcns = st->regroup_cns;
  }
  int64_t cnu = 0;
  int conv = 0, iters = 0;
  if (trace)
    for (int i = 0; i < max_iters; ++i) trace[i] = -1;
  for (int iter = 1; iter <= max_iters; ++iter) {
    if (iter > 1 && s->regroup && s->kind != ORC_FLOODING) { /* decoder.hpp:153-156 */
      const double ov = s->kind == ORC_NONDISJOINT ? s->overlap : 0.0;
      if (orc_generate_groups(g->m, s->n_groups, ov, orc_mix_seed(seed, (uint64_t)iter), st->regroup_off,
                              st->regroup_cns, 2 * g->m + 1) < 0)
        return -1;
      goff = st->regroup_off;
      gcns = st->regroup_cns;
      G = s->n_groups;
    }
    for (int k = 0; k < G; ++k) {
      run_subiteration(st, g, gcns + goff[k], goff[k + 1] - goff[k]);
      cnu += goff[k + 1] - goff[k];
    }
    for (int v = 0; v < g->n; ++v) { /* decoder.hpp:162-167 */
      double total = st->ch[v];
      for (int j = g->var_off[v]; j < g->var_off[v + 1]; ++j) total += st->c2v[g->var_edges[j]];
      st->total[v] = total;
      st->hard[v] = total >= 0.0 ? 0 : 1;
    }
    const int weight = syndrome_weight(g, st->hard);
    if (trace) trace[iter - 1] = weight;
    iters = iter;
    conv = weight == 0;
    if (conv && early_stop) break;
  }
  if (!early_stop) iters = max_iters;
  if (bits) memcpy(bits, st->hard, (size_t)g->n);
  if (iterations) *iterations = iters;
  if (converged) *converged = (uint8_t)conv;
  if (posterior) memcpy(posterior, st->total, sizeof(double) * (size_t)g->n);
  if (cn_updates) *cn_updates = cnu;
  return 0;
}

static int check_schedule(const orc_graph *g, const orc_schedule *s) {
  if (s->n_groups < 1) return fail("schedule needs at least one group");
  if (s->per_frame) return 0; /* groups are generated per frame */
  for (int k = 0; k < s->n_groups; ++k)
    for (int i = s->grp_off[k]; i < s->grp_off[k + 1]; ++i)
      if (s->grp_cns[i] < 0 || s->grp_cns[i] >= g->m) return fail("group CN index out of range");
  return 0;
}

int orc_decode(const orc_graph *g, const orc_schedule *s, const double *llr, int max_iters, int early_stop,
               uint8_t *bits, int32_t *iterations, uint8_t *converged, double *posterior, int32_t *trace,
               int64_t *cn_updates) {
  if (check_schedule(g, s)) return -1;
  dstate st;
  state_alloc(&st, g, s->n_groups);
  const int rc = decode_impl(&st, g, s, 0, llr, max_iters, early_stop, bits, iterations, converged, posterior,
                             trace, cn_updates);
  state_free(&st);
  return rc;
}

int orc_run_subiterations(const orc_graph *g, const orc_schedule *s, const double *llr, int n_subiters,
                          double *c2v_out, double *v2c_out) {
  if (check_schedule(g, s)) return -1;
  dstate st;
  state_alloc(&st, g, s->n_groups);
  init_state(&st, g, llr);
  for (int t = 0; t < n_subiters; ++t) {
    const int k = t % s->n_groups;
    run_subiteration(&st, g, s->grp_cns + s->grp_off[k], s->grp_off[k + 1] - s->grp_off[k]);
  }
  if (c2v_out) memcpy(c2v_out, st.c2v, sizeof(double) * (size_t)g->E);
  if (v2c_out) memcpy(v2c_out, st.v2c, sizeof(double) * (size_t)g->E);
  state_free(&st);
  return 0;
}

/* ---- frame-parallel workers (sim.hpp:136-150) -------------------------- */

typedef struct {
  const orc_graph *g;
  const orc_schedule *s;
  const float *llr;
  int64_t frames;
  int max_iters, early_stop;
  uint8_t *bits;
  int32_t *iterations;
  uint8_t *converged;
  float *posterior;
  int32_t *trace;
  int64_t next; /* atomic work counter */
  int rc;
} batch_job;

static void *batch_worker(void *arg) {
  batch_job *J = arg;
  const orc_graph *g = J->g;
  dstate st;
  state_alloc(&st, g, J->s->n_groups);
  double *llr = malloc(sizeof(double) * (size_t)g->n);
  double *post = malloc(sizeof(double) * (size_t)g->n);
  for (;;) {
    const int64_t f = __atomic_fetch_add(&J->next, 1, __ATOMIC_RELAXED);
    if (f >= J->frames) break;
    for (int v = 0; v < g->n; ++v) llr[v] = (double)J->llr[f * g->n + v];
    int32_t it = 0;
    uint8_t cv = 0;
    if (decode_impl(&st, g, J->s, (uint64_t)f, llr, J->max_iters, J->early_stop, J->bits ? J->bits + f * g->n : NULL,
                    &it, &cv,
                    J->posterior ? post : NULL, J->trace ? J->trace + f * J->max_iters : NULL, NULL)) {
      J->rc = -1;
      break;
    }
    if (J->iterations) J->iterations[f] = it;
    if (J->converged) J->converged[f] = cv;
    if (J->posterior)
      for (int v = 0; v < g->n; ++v) J->posterior[f * g->n + v] = (float)post[v];
  }
  free(llr);
  free(post);
  state_free(&st);
  return NULL;
}

static void run_pool(void *(*fn)(void *), void *job, int threads) {
  if (threads < 1) threads = 1;
  pthread_t *tid = malloc(sizeof(pthread_t) * (size_t)threads);
  for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, fn, job);
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  free(tid);
}

int orc_decode_batch_f32(const orc_graph *g, const orc_schedule *s, const float *llr, int64_t frames, int max_iters,
                         int early_stop, int threads, uint8_t *bits, int32_t *iterations, uint8_t *converged,
                         float *posterior, int32_t *trace) {
  if (check_schedule(g, s)) return -1;
  if (max_iters < 1) return fail("max_iters must be >= 1");
  batch_job J = {g, s, llr, frames, max_iters, early_stop, bits, iterations, converged, posterior, trace, 0, 0};
  run_pool(batch_worker, &J, threads);
  return J.rc;
}

typedef struct {
  double sigma2;
  uint64_t seed;
  int n;
  uint64_t frame0;
  int64_t frames;
  float *llr;
  int64_t next;
} tx_job;

static void *tx_worker(void *arg) {
  tx_job *J = arg;
  double *buf = malloc(sizeof(double) * (size_t)J->n);
  for (;;) {
    const int64_t f = __atomic_fetch_add(&J->next, 1, __ATOMIC_RELAXED);
    if (f >= J->frames) break;
    orc_transmit_all_zero(J->sigma2, J->seed, J->n, J->frame0 + (uint64_t)f, buf);
    for (int i = 0; i < J->n; ++i) J->llr[f * J->n + i] = (float)buf[i];
  }
  free(buf);
  return NULL;
}

int orc_transmit_batch_f32(double sigma2, uint64_t seed, int n, uint64_t frame0, int64_t frames, float *llr,
                           int threads) {
  if (n < 1) return fail("frame length must be >= 1");
  tx_job J = {sigma2, seed, n, frame0, frames, llr, 0};
  run_pool(tx_worker, &J, threads);
  return 0;
}

typedef struct {
  const orc_graph *g;
  const orc_schedule *s;
  double sigma2;
  uint64_t seed, frame0;
  int64_t frames;
  int max_iters, early_stop, round_f32;
  int64_t next;
  int64_t counters[6];
  pthread_mutex_t mu;
  int rc;
} sim_job;

/* run_frame + aggregation, sim.hpp:111-124 and :162-181 */
static void *sim_worker(void *arg) {
  sim_job *J = arg;
  const orc_graph *g = J->g;
  dstate st;
  state_alloc(&st, g, J->s->n_groups);
  double *llr = malloc(sizeof(double) * (size_t)g->n);
  uint8_t *bits = malloc((size_t)g->n);
  int64_t c[6] = {0, 0, 0, 0, 0, 0};
  for (;;) {
    const int64_t f = __atomic_fetch_add(&J->next, 1, __ATOMIC_RELAXED);
    if (f >= J->frames) break;
    orc_transmit_all_zero(J->sigma2, J->seed, g->n, J->frame0 + (uint64_t)f, llr);
    if (J->round_f32)
      for (int v = 0; v < g->n; ++v) llr[v] = (double)(float)llr[v];
    int32_t it = 0;
    uint8_t cv = 0;
    if (decode_impl(&st, g, J->s, J->frame0 + (uint64_t)f, llr, J->max_iters, J->early_stop, bits, &it, &cv, NULL,
                    NULL, NULL)) {
      J->rc = -1;
      break;
    }
    int be = 0;
    for (int v = 0; v < g->n; ++v) be += bits[v];
    c[0] += 1;
    c[1] += be;
    c[2] += be > 0;
    c[3] += cv;
    c[4] += it;
    c[5] += cv ? it : 0;
  }
  pthread_mutex_lock(&J->mu);
  for (int i = 0; i < 6; ++i) J->counters[i] += c[i];
  pthread_mutex_unlock(&J->mu);
  free(llr);
  free(bits);
  state_free(&st);
  return NULL;
}

int orc_simulate(const orc_graph *g, const orc_schedule *s, double sigma2, uint64_t channel_seed,
                 uint64_t frame_begin, int64_t frame_count, int max_iters, int early_stop, int round_f32, int threads,
                 int64_t *counters) {
  if (check_schedule(g, s)) return -1;
  if (max_iters < 1) return fail("max_iters must be >= 1");
  sim_job J;
  memset(&J, 0, sizeof J);
  J.g = g;
  J.s = s;
  J.sigma2 = sigma2;
  J.seed = channel_seed;
  J.frame0 = frame_begin;
  J.frames = frame_count;
  J.max_iters = max_iters;
  J.early_stop = early_stop;
  J.round_f32 = round_f32;
  pthread_mutex_init(&J.mu, NULL);
  run_pool(sim_worker, &J, threads);
  pthread_mutex_destroy(&J.mu);
  for (int i = 0; i < 6; ++i) counters[i] = J.counters[i];
  return J.rc;
}
