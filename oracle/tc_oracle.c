/*
 * tc_oracle.c -- plain-C restatement of the reference pruned color-coding DP.
 *
 * TEST INFRASTRUCTURE ONLY (see tc_oracle.h).  Follows, function by function,
 * /root/reference/proj/include/treecount/{rng,graph,synthgen,color_index,
 * templates,count_table,la_kernels,engines,estimator}.hpp; each function
 * names the file:line it restates.  Build with -O2 -ffp-contract=off so the
 * fp64 arithmetic matches the reference's own -O3 (no -march) build bit for
 * bit (SURVEY finding 10).
 */
#include "tc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* rng.hpp:13-37 -- std::mt19937_64 ([rand.predef]) and Rng::below/unit      */
/* ------------------------------------------------------------------------ */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL
#define MT_A 0xB5026F5AA96619E9ULL

void orc_mt_seed(orc_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = MT_N;
}

static void mt_twist(orc_mt64* g) {
  uint64_t* x = g->mt;
  int k;
  for (k = 0; k < MT_N - MT_M; ++k) {
    uint64_t y = (x[k] & MT_UPPER) | (x[k + 1] & MT_LOWER);
    x[k] = x[k + MT_M] ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
  }
  for (; k < MT_N - 1; ++k) {
    uint64_t y = (x[k] & MT_UPPER) | (x[k + 1] & MT_LOWER);
    x[k] = x[k + (MT_M - MT_N)] ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
  }
  uint64_t y = (x[MT_N - 1] & MT_UPPER) | (x[0] & MT_LOWER);
  x[MT_N - 1] = x[MT_M - 1] ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
  g->idx = 0;
}

uint64_t orc_mt_next(orc_mt64* g) {
  if (g->idx >= MT_N) mt_twist(g);
  uint64_t z = g->mt[g->idx++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= (z >> 43);
  return z;
}

/* rng.hpp:21-27 */
static uint32_t rng_below(orc_mt64* g, uint32_t bound, uint64_t limit_override) {
  const uint64_t limit = limit_override ? limit_override : (UINT64_MAX / bound) * (uint64_t)bound;
  uint64_t x = orc_mt_next(g);
  while (x >= limit) x = orc_mt_next(g);
  return (uint32_t)(x % bound);
}

/* rng.hpp:30 */
static double rng_unit(orc_mt64* g) { return (double)(orc_mt_next(g) >> 11) * 0x1.0p-53; }

/* count_table.hpp:90-99 */
void orc_random_coloring(int32_t n, int k, uint64_t seed, uint64_t limit_override, uint8_t* out) {
  orc_mt64* g = (orc_mt64*)malloc(sizeof(orc_mt64));
  orc_mt_seed(g, seed);
  for (int32_t i = 0; i < n; ++i)
    out[i] = (uint8_t)(k == 1 ? 0 : rng_below(g, (uint32_t)k, limit_override));
  free(g);
}

/* ------------------------------------------------------------------------ */
/* graph.hpp:46-95 -- from_edges + build_csc                                 */
/* ------------------------------------------------------------------------ */
static void radix_sort_u64(uint64_t* a, int64_t m) {
  uint64_t* tmp = (uint64_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(uint64_t));
  int64_t* cnt = (int64_t*)malloc(65536 * sizeof(int64_t));
  for (int pass = 0; pass < 4; ++pass) {
    const int sh = 16 * pass;
    memset(cnt, 0, 65536 * sizeof(int64_t));
    for (int64_t i = 0; i < m; ++i) cnt[(a[i] >> sh) & 0xFFFF]++;
    int64_t s = 0;
    for (int d = 0; d < 65536; ++d) { int64_t c = cnt[d]; cnt[d] = s; s += c; }
    for (int64_t i = 0; i < m; ++i) tmp[cnt[(a[i] >> sh) & 0xFFFF]++] = a[i];
    uint64_t* t = a; a = tmp; tmp = t;
  }
  /* 4 passes: result is back in the caller's buffer */
  free(tmp == a ? NULL : tmp);
  free(cnt);
}

int orc_csr_from_edges(const int32_t* edges, int64_t m, int32_t n_hint, int32_t* n_out,
                       int64_t** row_ptr_out, int32_t** col_out, int64_t* nnz_out) {
  int32_t n = n_hint;
  if (n < 0) {
    int32_t mx = -1;
    for (int64_t e = 0; e < 2 * m; ++e) if (edges[e] > mx) mx = edges[e];
    n = mx + 1;
  }
  for (int64_t e = 0; e < 2 * m; ++e)
    if (edges[e] < 0 || edges[e] >= n) return -1;          /* graph.hpp:73-76 */
  uint64_t* key = (uint64_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(uint64_t));
  int64_t mm = 0;
  for (int64_t e = 0; e < m; ++e) {
    uint32_t u = (uint32_t)edges[2 * e], v = (uint32_t)edges[2 * e + 1];
    if (u > v) { uint32_t t = u; u = v; v = t; }              /* graph.hpp:77-79 */
    if (u == v) continue;                                     /* graph.hpp:80 */
    key[mm++] = ((uint64_t)u << 32) | v;
  }
  radix_sort_u64(key, mm);                                    /* graph.hpp:81 */
  int64_t w = 0;
  for (int64_t i = 0; i < mm; ++i)                            /* graph.hpp:82 */
    if (w == 0 || key[i] != key[w - 1]) key[w++] = key[i];
  int64_t* rp = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t i = 0; i < w; ++i) { rp[(key[i] >> 32) + 1]++; rp[(key[i] & 0xFFFFFFFFu) + 1]++; }
  for (int32_t v = 0; v < n; ++v) rp[v + 1] += rp[v];
  int32_t* col = (int32_t*)malloc((size_t)(rp[n] > 0 ? rp[n] : 1) * sizeof(int32_t));
  int64_t* fill = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  memcpy(fill, rp, (size_t)n * sizeof(int64_t));
  /* lower neighbours first (ascending u), then higher (ascending v): each
   * row comes out sorted, as the per-row std::sort in graph.hpp:92 does */
  for (int64_t i = 0; i < w; ++i) { uint32_t u = key[i] >> 32, v = key[i] & 0xFFFFFFFFu; col[fill[v]++] = (int32_t)u; }
  for (int64_t i = 0; i < w; ++i) { uint32_t u = key[i] >> 32, v = key[i] & 0xFFFFFFFFu; col[fill[u]++] = (int32_t)v; }
  free(fill);
  free(key);
  *n_out = n;
  *row_ptr_out = rp;
  *col_out = col;
  *nnz_out = rp[n];
  return 0;
}

/* synthgen.hpp:40-74 */
int orc_generate_rmat(int scale, int64_t nedges, double a, double b, double c, double d,
                      uint64_t seed, int32_t* n_out, int64_t** row_ptr, int32_t** col,
                      int64_t* nnz) {
  if (scale < 1 || scale > 26 || nedges < 1 || fabs(a + b + c + d - 1.0) > 1e-9) return -1;
  const int32_t n = (int32_t)(1LL << scale);
  orc_mt64* g = (orc_mt64*)malloc(sizeof(orc_mt64));
  orc_mt_seed(g, seed);
  int32_t* e = (int32_t*)malloc((size_t)nedges * 2 * sizeof(int32_t));
  const double ab = a + b, abc = ab + c;
  for (int64_t i = 0; i < nedges; ++i) {
    int32_t row = 0, cl = 0;
    for (int level = 0; level < scale; ++level) {
      const double u = rng_unit(g);
      row <<= 1; cl <<= 1;
      if (u < a) {
      } else if (u < ab) { cl |= 1; }
      else if (u < abc) { row |= 1; }
      else { row |= 1; cl |= 1; }
    }
    e[2 * i] = row; e[2 * i + 1] = cl;
  }
  free(g);
  int rc = orc_csr_from_edges(e, nedges, n, n_out, row_ptr, col, nnz);
  free(e);
  return rc;
}

void orc_free(void* p) { free(p); }

/* ------------------------------------------------------------------------ */
/* color_index.hpp:20-82 -- combinadic                                       */
/* ------------------------------------------------------------------------ */
int64_t orc_binom(int a, int b) {
  if (b < 0 || a < 0 || b > a) return 0;
  int64_t r = 1;
  for (int i = 1; i <= b; ++i) r = r * (a - b + i) / i;
  return r;
}

/* color_index.hpp:44-56: sum over 1-based positions of C(c_pos, pos) */
int64_t orc_index_of(const int* colors, int h) {
  int64_t idx = 0;
  for (int pos = 1; pos <= h; ++pos) idx += orc_binom(colors[pos - 1], pos);
  return idx;
}

/* color_index.hpp:60-72: greedy unrank, largest position first */
void orc_set_of(int k, int64_t index, int h, int* colors) {
  int c = k - 1;
  for (int pos = h; pos >= 1; --pos) {
    while (orc_binom(c, pos) > index) --c;
    colors[pos - 1] = c;
    index -= orc_binom(c, pos);
    --c;
  }
}

/* color_index.hpp:103-180 */
typedef struct { int32_t is, ia; } orc_pair;
static int cmp_pair(const void* x, const void* y) {
  const orc_pair* a = (const orc_pair*)x; const orc_pair* b = (const orc_pair*)y;
  if (a->is != b->is) return a->is < b->is ? -1 : 1;
  return a->ia < b->ia ? -1 : (a->ia > b->ia);
}

int orc_split_table(int k, int parent_size, int active_size, int32_t* active_index,
                    int32_t* passive_index, int32_t* grouped_parent, int32_t* grouped_active) {
  const int passive_size = parent_size - active_size;
  if (active_size < 1 || passive_size < 1 || parent_size > k) return -1;
  const int64_t parent_cols = orc_binom(k, parent_size);
  const int64_t passive_cols = orc_binom(k, passive_size);
  const int pairs = (int)orc_binom(parent_size, active_size);
  const int partners = (int)orc_binom(k - passive_size, active_size);
  orc_pair* groups = (orc_pair*)malloc((size_t)(passive_cols * partners) * sizeof(orc_pair));
  int* gcount = (int*)calloc((size_t)passive_cols, sizeof(int));
  int parent[ORC_MAXK], act[ORC_MAXK], pas[ORC_MAXK], choose[ORC_MAXK];
  for (int64_t is = 0; is < parent_cols; ++is) {
    orc_set_of(k, is, parent_size, parent);
    for (int i = 0; i < active_size; ++i) choose[i] = i;      /* lexicographic positions */
    int pair = 0;
    for (;;) {
      int ai = 0, pi = 0;
      for (int pos = 0, ci = 0; pos < parent_size; ++pos) {
        if (ci < active_size && choose[ci] == pos) { act[ai++] = parent[pos]; ++ci; }
        else pas[pi++] = parent[pos];
      }
      const int32_t ia = (int32_t)orc_index_of(act, active_size);
      const int32_t ip = (int32_t)orc_index_of(pas, passive_size);
      const int64_t slot = is * pairs + pair;
      if (active_index) active_index[slot] = ia;
      if (passive_index) passive_index[slot] = ip;
      orc_pair pr = {(int32_t)is, ia};
      groups[(int64_t)ip * partners + gcount[ip]++] = pr;
      ++pair;
      int move = active_size - 1;
      while (move >= 0 && choose[move] == parent_size - active_size + move) --move;
      if (move < 0) break;
      ++choose[move];
      for (int j = move + 1; j < active_size; ++j) choose[j] = choose[j - 1] + 1;
    }
  }
  for (int64_t ip = 0; ip < passive_cols; ++ip) {
    if (gcount[ip] != partners) { free(groups); free(gcount); return -2; }
    qsort(groups + ip * partners, (size_t)partners, sizeof(orc_pair), cmp_pair);
    for (int q = 0; q < partners; ++q) {
      if (grouped_parent) grouped_parent[ip * partners + q] = groups[ip * partners + q].is;
      if (grouped_active) grouped_active[ip * partners + q] = groups[ip * partners + q].ia;
    }
  }
  free(groups);
  free(gcount);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* templates.hpp:37-90,174-259 -- validation and the partition plan          */
/* ------------------------------------------------------------------------ */
typedef struct { int k; int deg[ORC_MAXK]; int nb[ORC_MAXK][ORC_MAXK]; } orc_tadj;

static int tadj_build(int k, const int32_t* edges, orc_tadj* t) {
  if (k < 1 || k > ORC_MAXK) return -1;
  t->k = k;
  memset(t->deg, 0, sizeof(t->deg));
  for (int e = 0; e < k - 1; ++e) {
    int u = edges[2 * e], v = edges[2 * e + 1];
    if (u < 0 || v < 0 || u >= k || v >= k || u == v) return -1;
    t->nb[u][t->deg[u]++] = v;
    t->nb[v][t->deg[v]++] = u;
  }
  for (int v = 0; v < k; ++v)  /* sorted neighbours (templates.hpp:28-31) */
    for (int i = 1; i < t->deg[v]; ++i)
      for (int j = i; j > 0 && t->nb[v][j - 1] > t->nb[v][j]; --j) {
        int s = t->nb[v][j]; t->nb[v][j] = t->nb[v][j - 1]; t->nb[v][j - 1] = s;
      }
  /* connectivity (templates.hpp:46-64) */
  uint32_t seen = 1u; int stack[ORC_MAXK], sp = 0; stack[sp++] = 0; int count = 1;
  while (sp) {
    int v = stack[--sp];
    for (int i = 0; i < t->deg[v]; ++i) {
      int w = t->nb[v][i];
      if (!(seen >> w & 1u)) { seen |= 1u << w; ++count; stack[sp++] = w; }
    }
  }
  return count == k ? 0 : -1;
}

/* templates.hpp:225-240: DFS from `from` inside `mask`, skipping from->blocked */
static uint32_t reachable(const orc_tadj* t, uint32_t mask, int from, int blocked) {
  uint32_t out = 1u << from; int stack[ORC_MAXK], sp = 0; stack[sp++] = from;
  while (sp) {
    int v = stack[--sp];
    for (int i = 0; i < t->deg[v]; ++i) {
      int w = t->nb[v][i];
      if (v == from && w == blocked) continue;
      if (!(mask >> w & 1u) || (out >> w & 1u)) continue;
      out |= 1u << w; stack[sp++] = w;
    }
  }
  return out;
}

static int popcount32(uint32_t x) { int c = 0; while (x) { x &= x - 1; ++c; } return c; }

static int plan_build(const orc_tadj* t, orc_plan* p, int* order_len, uint32_t mask, int root) {
  const int id = p->num_nodes++;
  p->size[id] = popcount32(mask);
  p->node_root[id] = root;
  p->active_child[id] = p->passive_child[id] = p->parent[id] = -1;
  if (p->size[id] > 1) {
    int tau = -1;                                  /* templates.hpp:189-197 */
    for (int i = 0; i < t->deg[root]; ++i)
      if (mask >> t->nb[root][i] & 1u) { tau = t->nb[root][i]; break; }
    uint32_t act = reachable(t, mask, root, tau);
    uint32_t pas = mask & ~act;
    int a = plan_build(t, p, order_len, act, root);
    int q = plan_build(t, p, order_len, pas, tau);
    p->active_child[id] = a; p->passive_child[id] = q;
    p->parent[a] = id; p->parent[q] = id;
  }
  p->dp_order[(*order_len)++] = id;
  return id;
}

int orc_partition(int k, const int32_t* edges, int root, orc_plan* plan) {
  orc_tadj t;
  if (tadj_build(k, edges, &t) != 0) return -1;
  if (root < 0) {                                  /* templates.hpp:67-74 */
    root = 0;
    for (int v = 1; v < k; ++v) if (t.deg[v] > t.deg[root]) root = v;
  }
  if (root >= k) return -1;
  memset(plan, 0, sizeof(*plan));
  plan->k = k; plan->root = root;
  int len = 0;
  plan_build(&t, plan, &len, k == 32 ? 0xFFFFFFFFu : ((1u << k) - 1u), root);
  return 0;
}

/* count_table.hpp:113-133 */
int64_t orc_estimate_bytes(const orc_plan* plan, int64_t n) {
  char live[ORC_MAXNODES] = {0};
  int64_t peak = 0;
  for (int s = 0; s < plan->num_nodes; ++s) {
    int id = plan->dp_order[s];
    live[id] = 1;
    int64_t cols = 0;
    for (int j = 0; j < plan->num_nodes; ++j) if (live[j]) cols += orc_binom(plan->k, plan->size[j]);
    if (cols > peak) peak = cols;
    if (plan->size[id] > 1) { live[plan->active_child[id]] = 0; live[plan->passive_child[id]] = 0; }
  }
  return 8 * n * peak;
}

/* ------------------------------------------------------------------------ */
/* templates.hpp:265-339 -- |Aut(T)| via AHU canonical strings               */
/* ------------------------------------------------------------------------ */
typedef struct { char* canon; uint64_t aut; } orc_ahu;
static int cmp_ahu(const void* x, const void* y) {
  return strcmp(((const orc_ahu*)x)->canon, ((const orc_ahu*)y)->canon);
}

static orc_ahu ahu_rooted(const orc_tadj* t, int v, int parent) {   /* :270-294 */
  orc_ahu ch[ORC_MAXK]; int nc = 0; size_t len = 2;
  for (int i = 0; i < t->deg[v]; ++i) {
    int w = t->nb[v][i];
    if (w == parent) continue;
    ch[nc] = ahu_rooted(t, w, v);
    len += strlen(ch[nc].canon); ++nc;
  }
  qsort(ch, (size_t)nc, sizeof(orc_ahu), cmp_ahu);
  orc_ahu r; r.aut = 1; r.canon = (char*)malloc(len + 1);
  char* o = r.canon; *o++ = '(';
  int i = 0;
  while (i < nc) {
    int j = i;
    while (j < nc && strcmp(ch[j].canon, ch[i].canon) == 0) ++j;
    for (int run = 2; run <= j - i; ++run) r.aut *= (uint64_t)run;
    for (int c = i; c < j; ++c) { size_t l = strlen(ch[c].canon); memcpy(o, ch[c].canon, l); o += l; r.aut *= ch[c].aut; }
    i = j;
  }
  *o++ = ')'; *o = 0;
  for (int c = 0; c < nc; ++c) free(ch[c].canon);
  return r;
}

uint64_t orc_automorphisms(int k, const int32_t* edges) {
  orc_tadj t;
  if (tadj_build(k, edges, &t) != 0) return 0;
  if (k == 1) return 1;
  /* tree centers (templates.hpp:297-320) */
  int degree[ORC_MAXK], frontier[ORC_MAXK] = {0}, nf = 0, remaining = k;
  for (int v = 0; v < k; ++v) { degree[v] = t.deg[v]; if (degree[v] == 1) frontier[nf++] = v; }
  while (remaining > 2) {
    int next[ORC_MAXK], nn = 0;
    remaining -= nf;
    for (int f = 0; f < nf; ++f) {
      int v = frontier[f]; degree[v] = 0;
      for (int i = 0; i < t.deg[v]; ++i) if (--degree[t.nb[v][i]] == 1) next[nn++] = t.nb[v][i];
    }
    memcpy(frontier, next, sizeof(int) * (size_t)nn); nf = nn;
  }
  if (nf == 2 && frontier[1] < frontier[0]) { int s = frontier[0]; frontier[0] = frontier[1]; frontier[1] = s; }
  if (nf == 1) { orc_ahu r = ahu_rooted(&t, frontier[0], -1); free(r.canon); return r.aut; }
  orc_ahu a = ahu_rooted(&t, frontier[0], frontier[1]);
  orc_ahu b = ahu_rooted(&t, frontier[1], frontier[0]);
  uint64_t aut = a.aut * b.aut;
  if (strcmp(a.canon, b.canon) == 0) aut *= 2;
  free(a.canon); free(b.canon);
  return aut;
}

/* ------------------------------------------------------------------------ */
/* engines.hpp:106-152,224-268 + la_kernels.hpp:50-114 -- the vectorized DP  */
/* ------------------------------------------------------------------------ */
double orc_run_iteration(int32_t n, const int64_t* row_ptr, const int32_t* col,
                         const orc_plan* plan, const uint8_t* colors, double* per_vertex,
                         double** node_tables) {
  const int k = plan->k;
  double* tab[ORC_MAXNODES] = {0};
  double* staged = (double*)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
  for (int s = 0; s < plan->num_nodes; ++s) {
    const int id = plan->dp_order[s];
    const int64_t cs = orc_binom(k, plan->size[id]);
    if (plan->size[id] == 1) {                       /* count_table.hpp:102-107 */
      tab[id] = (double*)calloc((size_t)n * (size_t)k, sizeof(double));
      for (int32_t i = 0; i < n; ++i) tab[id][(size_t)colors[i] * (size_t)n + (size_t)i] = 1.0;
      continue;
    }
    const int a = plan->active_child[id], p = plan->passive_child[id];
    const int sa = plan->size[a], sp = plan->size[p];
    const int64_t cp = orc_binom(k, sp);
    const int partners = (int)orc_binom(k - sp, sa);
    int32_t* gp = (int32_t*)malloc((size_t)(cp * partners) * sizeof(int32_t));
    int32_t* ga = (int32_t*)malloc((size_t)(cp * partners) * sizeof(int32_t));
    orc_split_table(k, plan->size[id], sa, NULL, NULL, gp, ga);
    if (node_tables) {
      for (int c = 0; c < 2; ++c) {
        int child = c ? p : a;
        if (plan->size[child] > 1 && !node_tables[child]) {
          size_t bytes = (size_t)n * (size_t)orc_binom(k, plan->size[child]) * sizeof(double);
          node_tables[child] = (double*)malloc(bytes);
          memcpy(node_tables[child], tab[child], bytes);
        }
      }
    }
    double* out = (double*)calloc((size_t)n * (size_t)cs, sizeof(double));
    /* SpMM phase, in place (engines.hpp:226-246, la_kernels.hpp:83-102):
     * per-entry order is ascending neighbour id, independent of batch Z */
    double* P = tab[p];
    for (int64_t c = 0; c < cp; ++c) {
      double* colp = P + (size_t)c * (size_t)n;
      memcpy(staged, colp, (size_t)n * sizeof(double));
      for (int32_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) acc += staged[col[e]];
        colp[i] = acc;
      }
    }
    /* eMA phase, grouped by passive column (engines.hpp:252-268) */
    double* A = tab[a];
    for (int64_t ip = 0; ip < cp; ++ip) {
      const double* colp = P + (size_t)ip * (size_t)n;
      for (int q = 0; q < partners; ++q) {
        double* o = out + (size_t)gp[ip * partners + q] * (size_t)n;
        const double* av = A + (size_t)ga[ip * partners + q] * (size_t)n;
        for (int32_t i = 0; i < n; ++i) o[i] += av[i] * colp[i];
      }
    }
    free(gp); free(ga);
    free(tab[a]); free(tab[p]); tab[a] = tab[p] = NULL;   /* engines.hpp:149-151 */
    tab[id] = out;
  }
  const int full = plan->dp_order[plan->num_nodes - 1];
  double total = 0.0;                                       /* engines.hpp:125-129 */
  for (int32_t i = 0; i < n; ++i) total += tab[full][i];
  if (per_vertex) memcpy(per_vertex, tab[full], (size_t)n * sizeof(double));
  if (node_tables && !node_tables[full]) {
    size_t bytes = (size_t)n * (size_t)orc_binom(k, plan->size[full]) * sizeof(double);
    node_tables[full] = (double*)malloc(bytes);
    memcpy(node_tables[full], tab[full], bytes);
  }
  free(tab[full]);
  free(staged);
  return total;
}

/* ------------------------------------------------------------------------ */
/* estimator.hpp:29-33,49-93                                                 */
/* ------------------------------------------------------------------------ */
double orc_colorful_probability(int k) {
  double p = 1.0;
  for (int i = 1; i <= k; ++i) p *= (double)i / (double)k;
  return p;
}

void orc_estimate(int32_t n, const int64_t* row_ptr, const int32_t* col, int k,
                  const int32_t* edges, int root, int iterations, uint64_t seed,
                  double* rooted_totals, double* estimate, double* stderr_of_mean,
                  uint64_t* aut_out) {
  orc_plan plan;
  orc_partition(k, edges, root, &plan);
  const uint64_t aut = orc_automorphisms(k, edges);
  uint8_t* colors = (uint8_t*)malloc((size_t)(n > 0 ? n : 1));
  for (int i = 0; i < iterations; ++i) {
    orc_random_coloring(n, k, seed + (uint64_t)i, 0, colors);
    rooted_totals[i] = orc_run_iteration(n, row_ptr, col, &plan, colors, NULL, NULL);
  }
  free(colors);
  double mean = 0.0;
  for (int i = 0; i < iterations; ++i) mean += rooted_totals[i];
  mean /= (double)iterations;
  double var = 0.0;
  for (int i = 0; i < iterations; ++i) var += (rooted_totals[i] - mean) * (rooted_totals[i] - mean);
  const double scale = 1.0 / ((double)aut * orc_colorful_probability(k));
  *estimate = mean * scale;
  *stderr_of_mean = iterations > 1
      ? sqrt(var / ((double)iterations * (double)(iterations - 1))) * scale : 0.0;
  *aut_out = aut;
}
