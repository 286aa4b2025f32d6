/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the all-points
 * minimax path distance (APPD) of arxiv 2407.07058.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or helper with the CUDA product path
 * (paper_2407_07058_b200/csrc); neither side includes or links the other.
 *
 * Citations: "P:Lnn" = PAPER.md line nn, "S:Lnn" = SPEC.md line nn.
 *
 * What is here (each function cites the passage it follows):
 *   oracle_r1_dist2 / oracle_r1_weight  points -> weight, the pinned R1 formula
 *   oracle_metric_weight (+ _metric API)  NEXT-3: Manhattan / Chebyshev weights
 *                                       (reading Q6: Euclidean, fixed
 *                                       order fmaf chain, fp32)
 *   oracle_dist_f64                     fp64 Euclidean distance (R1 checker)
 *   oracle_prim_*                       Prim's O(n^2) array-scan MST
 *   oracle_appd_*                       Algorithm 4, calculate and copy:
 *                                       Prim -> sort descending -> remove the
 *                                       edges one by one, traverse tree1 and
 *                                       tree2, copy the weight
 *   oracle_appd_points_rows             the same, keeping only writes whose
 *                                       row lies in a window (R5)
 *   oracle_floyd                        minimax Floyd-Warshall variant
 *                                          -- checker
 *   oracle_brute                        Eq. 1-2 by enumerating every simple
 *                                       path, n <= 9    -- checker
 *   oracle_mst_path                     max edge on the MST path -- checker
 *
 *   oracle_appd_weights_f64 / oracle_prim_weights_f64
 *                                       NEXT-3: the same on fp64 weights
 * Precision: the paper does not fix one; BASELINE.json fixes fp32 weights.
 * Every APPD value is a copied weight (only comparisons are made), so the
 * oracle works on the fp32 weights directly.  -0.0 is read as +0.0 (DESIGN.md
 * reading Q5).  Every function here is pinned by tests/test_oracle_*.py; no
 * function is "parity unpinned".
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-math-errno -mfma -shared -fPIC
 * (no -ffast-math: fmaf must be the single correctly rounded fused op).
 */
#define _POSIX_C_SOURCE 199309L
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define ORACLE_OK 0
#define ORACLE_ERR_ARG 1
#define ORACLE_ERR_NOMEM 6

typedef struct {
  int64_t writes;     /* off-diagonal pair writes (each writes M[a][b] and M[b][a]) */
  int64_t traversed;  /* vertices visited by the tree1/tree2 traversals */
  double t_mst;       /* seconds in Prim (incl. R1 weights in points mode) */
  double t_sort;      /* seconds sorting MST edges */
  double t_copy;      /* seconds in remove / traverse / copy */
} oracle_stats;

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

/* -0.0 -> +0.0; every other value unchanged (reading Q5). */
static float canon(float w) { return w == 0.0f ? 0.0f : w; }

/* ---------------------------------------------------------------------------
 * R1: weight of the complete-graph edge between two points ("A dataset
 * X can be straightforwardly converted to a complete graph"; S:L52-55 fixes
 * Euclidean).  Pinned order: acc = +0; for k = 0..d-1: t = fl(x_i[k] - x_j[k]);
 * acc = fmaf(t, t, acc).  The weight is sqrtf(acc).
 * ------------------------------------------------------------------------- */
float oracle_r1_dist2(const float* xi, const float* xj, int64_t d) {
  float acc = 0.0f;
  for (int64_t k = 0; k < d; k++) {
    float t = xi[k] - xj[k];
    acc = fmaf(t, t, acc);
  }
  return acc;
}

float oracle_r1_weight(const float* xi, const float* xj, int64_t d) {
  return sqrtf(oracle_r1_dist2(xi, xj, d));
}

/* ---------------------------------------------------------------------------
 * NEXT-3 ("other point metrics"): pluggable point metrics.
 * metric 0: R1 above (Euclidean); 1: Manhattan, acc = +0; for k in order:
 * acc = fl(acc + |fl(x_i[k] - x_j[k])|); 2: Chebyshev, acc = max over k of
 * |fl(x_i[k] - x_j[k])|.  The weight is the distance itself (no square root).
 * ------------------------------------------------------------------------- */
float oracle_metric_weight(const float* xi, const float* xj, int64_t d, int metric) {
  if (metric == 0) return oracle_r1_weight(xi, xj, d);
  float acc = 0.0f;
  for (int64_t k = 0; k < d; k++) {
    float t = fabsf(xi[k] - xj[k]);
    if (metric == 1) acc = acc + t;
    else if (t > acc) acc = t;
  }
  return acc;
}

/* fp64 Euclidean distance, the checker R1 is held to (BASELINE north star: 1e-5 rel). */
double oracle_dist_f64(const float* xi, const float* xj, int64_t d) {
  double s = 0.0;
  for (int64_t k = 0; k < d; k++) {
    double t = (double)xi[k] - (double)xj[k];
    s += t * t;
  }
  return sqrt(s);
}

/* Row block [r0, r0+R) of the R1 weight matrix, row-major R x n. */
void oracle_points_weights(const float* X, int64_t n, int64_t d, int64_t r0, int64_t R, float* Wblk) {
  for (int64_t i = 0; i < R; i++)
    for (int64_t j = 0; j < n; j++)
      Wblk[i * n + j] = (r0 + i == j) ? 0.0f : oracle_r1_weight(X + (r0 + i) * d, X + j * d, d);
}

/* ---------------------------------------------------------------------------
 * Edge weight source: a dense matrix W or points X (R1 computed on the fly).
 * sense = +1 minimax (minimum spanning tree), -1 widest (maximum spanning tree,
 * P:L119 "constructing a maximum spanning tree and sort the edges in ascending
 * order"; S:L133 implements it as minimum-sense Prim on negated weights).
 * ------------------------------------------------------------------------- */
typedef struct {
  const float* W;
  const float* X;
  int64_t n, d;
  int metric;       /* points: 0 R1, 1 Manhattan, 2 Chebyshev */
  const double* Wd; /* NEXT-3: fp64 weight matrix ("float64"), used when W and X are NULL */
} wsrc;

/* Weights are handled as doubles: every fp32 weight converts exactly, and the method only
 * compares and copies weights, so the fp32 results are unchanged by the wider type. */
static double wget(const wsrc* s, int64_t i, int64_t j) {
  if (s->W) return canon(s->W[i * s->n + j]);
  if (s->Wd) { double w = s->Wd[i * s->n + j]; return w == 0.0 ? 0.0 : w; }
  return oracle_metric_weight(s->X + i * s->d, s->X + j * s->d, s->d, s->metric);
}

/* ---------------------------------------------------------------------------
 * R2. Prim's algorithm, O(n^2) array scan ("The complexity of
 * constructing a MST with prim's algorithm is O(n^2)").  Start vertex 0
 * (S:L133); among equal keys the smallest vertex id is chosen.  The
 * edge that attaches the vertex chosen at step s (s >= 1) gets seq = s-1.
 * For sense -1 the keys are the negated weights; the recorded weight is the
 * original one.
 * ------------------------------------------------------------------------- */
static int prim(const wsrc* s, int sense, int32_t* eu, int32_t* ev, double* ew) {
  int64_t n = s->n;
  double* key = (double*)malloc(sizeof(double) * n);
  int32_t* parent = (int32_t*)malloc(sizeof(int32_t) * n);
  unsigned char* done = (unsigned char*)calloc(n, 1);
  if (!key || !parent || !done) {
    free(key); free(parent); free(done);
    return ORACLE_ERR_NOMEM;
  }
  for (int64_t i = 0; i < n; i++) { key[i] = INFINITY; parent[i] = -1; }
  key[0] = -INFINITY;
  for (int64_t step = 0; step < n; step++) {
    int64_t v = -1;
    for (int64_t u = 0; u < n; u++)
      if (!done[u] && (v < 0 || key[u] < key[v])) v = u; /* strict <: smallest id wins ties */
    done[v] = 1;
    if (step > 0) {
      eu[step - 1] = parent[v];
      ev[step - 1] = (int32_t)v;
      ew[step - 1] = sense > 0 ? key[v] : -key[v];
    }
    for (int64_t u = 0; u < n; u++) {
      if (done[u]) continue;
      double w = wget(s, v, u);
      double k = sense > 0 ? w : -w;
      /* an edge of weight +inf (points whose squared distance overflows fp32) is still an
       * edge of the complete graph (reading Q14): the first tree vertex to
       * offer one becomes the parent */
      if (parent[u] < 0 || k < key[u]) { key[u] = k; parent[u] = (int32_t)v; }
    }
  }
  free(key); free(parent); free(done);
  return ORACLE_OK;
}

static int prim_f32(const wsrc* s, int sense, int32_t* eu, int32_t* ev, float* ew) {
  double* w = (double*)malloc(sizeof(double) * (s->n > 1 ? s->n - 1 : 1));
  if (!w) return ORACLE_ERR_NOMEM;
  int rc = prim(s, sense, eu, ev, w);
  for (int64_t e = 0; rc == ORACLE_OK && e < s->n - 1; e++) ew[e] = (float)w[e]; /* exact: copies of fp32 weights */
  free(w);
  return rc;
}

int oracle_prim_weights(const float* W, int64_t n, int sense, int32_t* eu, int32_t* ev, float* ew) {
  if (!W || n < 1) return ORACLE_ERR_ARG;
  wsrc s = {W, NULL, n, 0, 0, NULL};
  return prim_f32(&s, sense, eu, ev, ew);
}

int oracle_prim_points(const float* X, int64_t n, int64_t d, int32_t* eu, int32_t* ev, float* ew) {
  if (!X || n < 1 || d < 1) return ORACLE_ERR_ARG;
  wsrc s = {NULL, X, n, d, 0, NULL};
  return prim_f32(&s, +1, eu, ev, ew);
}

/* NEXT-3: Prim on an fp64 weight matrix. */
int oracle_prim_weights_f64(const double* W, int64_t n, int sense, int32_t* eu, int32_t* ev, double* ew) {
  if (!W || n < 1) return ORACLE_ERR_ARG;
  wsrc s = {NULL, NULL, n, 0, 0, W};
  return prim(&s, sense, eu, ev, ew);
}

/* ---------------------------------------------------------------------------
 * R3. Sort the MST edges "in descending order" for minimax, ascending
 * for widest.  Ties: ascending seq, so the order is total.
 * ------------------------------------------------------------------------- */
typedef struct {
  double w;
  int32_t seq;
} sort_item;

static int cmp_desc(const void* a, const void* b) {
  const sort_item* x = (const sort_item*)a;
  const sort_item* y = (const sort_item*)b;
  if (x->w > y->w) return -1;
  if (x->w < y->w) return 1;
  return (x->seq > y->seq) - (x->seq < y->seq);
}

static int cmp_asc(const void* a, const void* b) {
  const sort_item* x = (const sort_item*)a;
  const sort_item* y = (const sort_item*)b;
  if (x->w < y->w) return -1;
  if (x->w > y->w) return 1;
  return (x->seq > y->seq) - (x->seq < y->seq);
}

/* ---------------------------------------------------------------------------
 * R4. Remove the edges one by one in the sorted order ("remove the edges
 * from the MST one-by-one, from large to small. Only by this we can get the two
 * sub-trees, tree1 and tree2. By traversing each sub-tree, nodes of the two
 * sub-trees can be obtained"), and copy the removed edge's weight into every
 * cell tree1 x tree2 (each cell is accessed only once).  Traversal is
 * an iterative DFS over the live forest.  Only rows in [r0, r0+R) are
 * stored (R5); R = n stores everything.  M is R x n, row-major.
 * ------------------------------------------------------------------------- */
/* M (fp32) or Md (fp64) receives the output; every stored value is a copied weight */
static int algo4(const wsrc* s, int sense, int64_t r0, int64_t R, float* M, double* Md, oracle_stats* st) {
  int64_t n = s->n;
  oracle_stats local = {0, 0, 0, 0, 0};
  if (n == 1) {
    if (R == 1) { if (Md) Md[0] = 0.0; else M[0] = 0.0f; }
    if (st) *st = local;
    return ORACLE_OK;
  }
  int64_t m = n - 1;
  int32_t* eu = (int32_t*)malloc(sizeof(int32_t) * m);
  int32_t* ev = (int32_t*)malloc(sizeof(int32_t) * m);
  double* ew = (double*)malloc(sizeof(double) * m);
  sort_item* order = (sort_item*)malloc(sizeof(sort_item) * m);
  /* forest adjacency in CSR form with a live flag per edge */
  int64_t* off = (int64_t*)calloc(n + 1, sizeof(int64_t));
  int32_t* adj_v = (int32_t*)malloc(sizeof(int32_t) * 2 * m);
  int32_t* adj_e = (int32_t*)malloc(sizeof(int32_t) * 2 * m);
  unsigned char* live = (unsigned char*)malloc(m);
  int32_t* stack = (int32_t*)malloc(sizeof(int32_t) * n);
  int32_t* tree1 = (int32_t*)malloc(sizeof(int32_t) * n);
  int32_t* tree2 = (int32_t*)malloc(sizeof(int32_t) * n);
  int32_t* mark = (int32_t*)malloc(sizeof(int32_t) * n);
  int rc = ORACLE_OK;
  if (!eu || !ev || !ew || !order || !off || !adj_v || !adj_e || !live || !stack || !tree1 || !tree2 || !mark) {
    rc = ORACLE_ERR_NOMEM;
    goto out;
  }

  double t0 = now_s();
  rc = prim(s, sense, eu, ev, ew);
  if (rc) goto out;
  double t1 = now_s();
  for (int64_t e = 0; e < m; e++) { order[e].w = ew[e]; order[e].seq = (int32_t)e; }
  qsort(order, m, sizeof(sort_item), sense > 0 ? cmp_desc : cmp_asc);
  double t2 = now_s();

  for (int64_t e = 0; e < m; e++) { off[eu[e] + 1]++; off[ev[e] + 1]++; live[e] = 1; }
  for (int64_t i = 0; i < n; i++) off[i + 1] += off[i];
  {
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * n);
    if (!fill) { rc = ORACLE_ERR_NOMEM; goto out; }
    memcpy(fill, off, sizeof(int64_t) * n);
    for (int64_t e = 0; e < m; e++) {
      adj_v[fill[eu[e]]] = ev[e]; adj_e[fill[eu[e]]++] = (int32_t)e;
      adj_v[fill[ev[e]]] = eu[e]; adj_e[fill[ev[e]]++] = (int32_t)e;
    }
    free(fill);
  }
  for (int64_t i = 0; i < n; i++) mark[i] = -1;
  for (int64_t i = 0; i < R; i++) { /* diagonal: the empty path */
    if (Md) Md[i * n + (r0 + i)] = 0.0; else M[i * n + (r0 + i)] = 0.0f;
  }

  for (int64_t k = 0; k < m; k++) {
    int32_t e = order[k].seq;
    double w = ew[e];
    live[e] = 0; /* delete the edge from the forest */
    int32_t* trees[2] = {tree1, tree2};
    int64_t sizes[2] = {0, 0};
    int32_t roots[2] = {eu[e], ev[e]};
    for (int side = 0; side < 2; side++) {
      /* iterative DFS from roots[side] over live edges; mark with a fresh stamp */
      int32_t stamp = (int32_t)(2 * k + side);
      int64_t sp = 0, cnt = 0;
      stack[sp++] = roots[side];
      mark[roots[side]] = stamp;
      while (sp) {
        int32_t a = stack[--sp];
        trees[side][cnt++] = a;
        for (int64_t p = off[a]; p < off[a + 1]; p++) {
          if (!live[adj_e[p]]) continue;
          int32_t b = adj_v[p];
          if (mark[b] != stamp) { mark[b] = stamp; stack[sp++] = b; }
        }
      }
      sizes[side] = cnt;
    }
    local.traversed += sizes[0] + sizes[1];
    /* copy: M[a][b] = M[b][a] = w for a in tree1, b in tree2 */
    for (int64_t x = 0; x < sizes[0]; x++) {
      int64_t a = tree1[x];
      for (int64_t y = 0; y < sizes[1]; y++) {
        int64_t b = tree2[y];
        if (Md) {
          if (a >= r0 && a < r0 + R) Md[(a - r0) * n + b] = w;
          if (b >= r0 && b < r0 + R) Md[(b - r0) * n + a] = w;
        } else {
          if (a >= r0 && a < r0 + R) M[(a - r0) * n + b] = (float)w;
          if (b >= r0 && b < r0 + R) M[(b - r0) * n + a] = (float)w;
        }
      }
    }
    local.writes += sizes[0] * sizes[1];
  }
  double t3 = now_s();
  local.t_mst = t1 - t0;
  local.t_sort = t2 - t1;
  local.t_copy = t3 - t2;
  if (st) *st = local;
out:
  free(eu); free(ev); free(ew); free(order); free(off); free(adj_v); free(adj_e);
  free(live); free(stack); free(tree1); free(tree2); free(mark);
  return rc;
}

/* Algorithm 4 on a weight matrix.  sense +1 minimax, -1 widest. */
int oracle_appd_weights(const float* W, int64_t n, int sense, float* M, oracle_stats* st) {
  if (!W || !M || n < 1 || (sense != 1 && sense != -1)) return ORACLE_ERR_ARG;
  wsrc s = {W, NULL, n, 0, 0, NULL};
  return algo4(&s, sense, 0, n, M, NULL, st);
}

/* NEXT-3: Algorithm 4 on an fp64 weight matrix ("float64"), fp64 output.  The
 * method only compares and copies weights, so it is the same procedure in the wider type. */
int oracle_appd_weights_f64(const double* W, int64_t n, int sense, double* M, oracle_stats* st) {
  if (!W || !M || n < 1 || (sense != 1 && sense != -1)) return ORACLE_ERR_ARG;
  wsrc s = {NULL, NULL, n, 0, 0, W};
  return algo4(&s, sense, 0, n, NULL, M, st);
}

/* Algorithm 4 on points (complete graph of R1 weights). */
int oracle_appd_points(const float* X, int64_t n, int64_t d, float* M, oracle_stats* st) {
  if (!X || !M || n < 1 || d < 1) return ORACLE_ERR_ARG;
  wsrc s = {NULL, X, n, d, 0, NULL};
  return algo4(&s, +1, 0, n, M, NULL, st);
}

/* Algorithm 4 on points under a pluggable metric (NEXT-3). */
int oracle_appd_points_metric(const float* X, int64_t n, int64_t d, int metric, float* M, oracle_stats* st) {
  if (!X || !M || n < 1 || d < 1 || metric < 0 || metric > 2) return ORACLE_ERR_ARG;
  wsrc s = {NULL, X, n, d, metric, NULL};
  return algo4(&s, +1, 0, n, M, NULL, st);
}

/* Row block [r0, r0+R) of the metric weight matrix, row-major R x n. */
void oracle_points_weights_metric(const float* X, int64_t n, int64_t d, int metric, int64_t r0, int64_t R,
                                  float* Wblk) {
  for (int64_t i = 0; i < R; i++)
    for (int64_t j = 0; j < n; j++)
      Wblk[i * n + j] = (r0 + i == j) ? 0.0f : oracle_metric_weight(X + (r0 + i) * d, X + j * d, d, metric);
}

/* R5: rows [r0, r0+R) only, M is R x n. */
int oracle_appd_points_rows(const float* X, int64_t n, int64_t d, int64_t r0, int64_t R, float* M,
                            oracle_stats* st) {
  if (!X || !M || n < 1 || d < 1 || r0 < 0 || R < 1 || r0 + R > n) return ORACLE_ERR_ARG;
  wsrc s = {NULL, X, n, d, 0, NULL};
  return algo4(&s, +1, r0, R, M, NULL, st);
}

int oracle_appd_weights_rows(const float* W, int64_t n, int64_t r0, int64_t R, float* M, oracle_stats* st) {
  if (!W || !M || n < 1 || r0 < 0 || R < 1 || r0 + R > n) return ORACLE_ERR_ARG;
  wsrc s = {W, NULL, n, 0, 0, NULL};
  return algo4(&s, +1, r0, R, M, NULL, st);
}

/* ---------------------------------------------------------------------------
 * Checker: the minimax variant of Floyd-Warshall ("a modified version of
 * the Floyd-Warshall algorithm", Fig. floyd, O(n^3) P:L84):
 * k outermost, M[i][j] = min(M[i][j], max(M[i][k], M[k][j])).  With
 * sense -1 (widest) min and max swap.  The diagonal is reset to +0 afterwards
 * (reading Q3: with negative weights the relaxation drives M[i][i] below 0).
 * ------------------------------------------------------------------------- */
int oracle_floyd(const float* W, int64_t n, int sense, float* M) {
  if (!W || !M || n < 1) return ORACLE_ERR_ARG;
  for (int64_t i = 0; i < n * n; i++) M[i] = canon(W[i]);
  for (int64_t k = 0; k < n; k++)
    for (int64_t i = 0; i < n; i++)
      for (int64_t j = 0; j < n; j++) {
        float a = M[i * n + k], b = M[k * n + j];
        if (sense > 0) {
          float c = a > b ? a : b;
          if (c < M[i * n + j]) M[i * n + j] = c;
        } else {
          float c = a < b ? a : b;
          if (c > M[i * n + j]) M[i * n + j] = c;
        }
      }
  for (int64_t i = 0; i < n; i++) M[i * n + i] = 0.0f;
  return ORACLE_OK;
}

/* ---------------------------------------------------------------------------
 * Checker: Eq. 1-2 by brute force.  Phi = { max_weight(p) : p a
 * path from i to j }, M(i,j) = min(Phi).  Enumerates every simple path (a
 * non-simple path never has a smaller maximum than the simple path inside it).
 * n <= 9.  sense -1: the widest problem (maximise the minimum).
 * ------------------------------------------------------------------------- */
static void brute_dfs(const float* W, int64_t n, int sense, int64_t src, int64_t v, unsigned visited,
                      float bott, float* best) {
  for (int64_t u = 0; u < n; u++) {
    if (visited & (1u << u)) continue;
    float w = canon(W[v * n + u]);
    float b = (v == src) ? w : (sense > 0 ? (w > bott ? w : bott) : (w < bott ? w : bott));
    float* cell = &best[src * n + u];
    if (sense > 0 ? b < *cell : b > *cell) *cell = b;
    brute_dfs(W, n, sense, src, u, visited | (1u << u), b, best);
  }
}

int oracle_brute(const float* W, int64_t n, int sense, float* M) {
  if (!W || !M || n < 1 || n > 9) return ORACLE_ERR_ARG;
  for (int64_t i = 0; i < n * n; i++) M[i] = sense > 0 ? INFINITY : -INFINITY;
  for (int64_t s = 0; s < n; s++) brute_dfs(W, n, sense, s, s, 1u << s, 0.0f, M);
  for (int64_t i = 0; i < n; i++) M[i * n + i] = 0.0f;
  return ORACLE_OK;
}

/* ---------------------------------------------------------------------------
 * Checker: "the path between any two nodes in a minimum spanning tree (MST) is
 * a minimax path".  Builds the MST with Prim (minimum sense), then for
 * each source walks the tree once carrying the maximum edge seen so far.
 * ------------------------------------------------------------------------- */
int oracle_mst_path(const float* W, int64_t n, float* M) {
  if (!W || !M || n < 1) return ORACLE_ERR_ARG;
  if (n == 1) { M[0] = 0.0f; return ORACLE_OK; }
  int64_t m = n - 1;
  int32_t* eu = (int32_t*)malloc(sizeof(int32_t) * m);
  int32_t* ev = (int32_t*)malloc(sizeof(int32_t) * m);
  float* ew = (float*)malloc(sizeof(float) * m);
  int64_t* off = (int64_t*)calloc(n + 1, sizeof(int64_t));
  int32_t* adj_v = (int32_t*)malloc(sizeof(int32_t) * 2 * m);
  float* adj_w = (float*)malloc(sizeof(float) * 2 * m);
  int32_t* stack = (int32_t*)malloc(sizeof(int32_t) * n);
  int32_t* from = (int32_t*)malloc(sizeof(int32_t) * n);
  int rc = ORACLE_OK;
  if (!eu || !ev || !ew || !off || !adj_v || !adj_w || !stack || !from) { rc = ORACLE_ERR_NOMEM; goto out; }
  {
    wsrc s = {W, NULL, n, 0, 0, NULL};
    rc = prim_f32(&s, +1, eu, ev, ew);
    if (rc) goto out;
  }
  for (int64_t e = 0; e < m; e++) { off[eu[e] + 1]++; off[ev[e] + 1]++; }
  for (int64_t i = 0; i < n; i++) off[i + 1] += off[i];
  {
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * n);
    if (!fill) { rc = ORACLE_ERR_NOMEM; goto out; }
    memcpy(fill, off, sizeof(int64_t) * n);
    for (int64_t e = 0; e < m; e++) {
      adj_v[fill[eu[e]]] = ev[e]; adj_w[fill[eu[e]]++] = ew[e];
      adj_v[fill[ev[e]]] = eu[e]; adj_w[fill[ev[e]]++] = ew[e];
    }
    free(fill);
  }
  for (int64_t src = 0; src < n; src++) {
    float* row = M + src * n;
    int64_t sp = 0;
    stack[sp++] = (int32_t)src;
    from[src] = -1;
    row[src] = 0.0f;
    while (sp) {
      int32_t a = stack[--sp];
      for (int64_t p = off[a]; p < off[a + 1]; p++) {
        int32_t b = adj_v[p];
        if (b == from[a]) continue;
        from[b] = a;
        float w = adj_w[p];
        row[b] = (a == src) ? w : (row[a] > w ? row[a] : w);
        stack[sp++] = b;
      }
    }
  }
out:
  free(eu); free(ev); free(ew); free(off); free(adj_v); free(adj_w); free(stack); free(from);
  return rc;
}

/* FNV-1a 64 over bytes, used for golden row-block manifests. */
uint64_t oracle_fnv1a64(const void* p, int64_t bytes) {
  const unsigned char* c = (const unsigned char*)p;
  uint64_t h = 1469598103934665603ULL;
  for (int64_t i = 0; i < bytes; i++) { h ^= c[i]; h *= 1099511628211ULL; }
  return h;
}
