/*
 * evoke_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for the n x 73 vertex-orbit
 * matrix of EVOKE (arXiv 1911.10616).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this code.
 * It shares no code, header, table or generator with the CUDA path.
 *
 * What it computes:
 *   - P:139-142 (Sec. 1.1 "Problem Description"): for every vertex v and every
 *     orbit theta, the number of times v occurs in a copy of theta; "we ask for
 *     induced counts".
 *   - P:366-388 (Def. "auto"): orbits = classes of the automorphism relation.
 *   - P:400-404 ("Induced vs non-induced"): an induced copy is a vertex subset
 *     with all its edges and non-edges.  So DIM(v,theta) = #{ U : v in U,
 *     G[U] isomorphic to H(theta), v mapped into the orbit theta }.
 *   - P:419-422 (Def. "unlabeled-match"): non-induced DM(v,theta) = number of
 *     distinct (not-necessarily-induced) copies (U,F), F subset of E(G[U]),
 *     with (U,F) isomorphic to H and v mapped into theta.  Only the tiny-graph
 *     brute force below computes DM (used to pin the catalog to the paper's
 *     equations and to Fig. 11).
 *
 * The orbit numbering (Fig. 2) is not in the text (the figure is
 * an empty TikZ macro).  The catalog below is the reading given in DESIGN.md
 * ("R1"), pinned by tests against the paper's printed equations (Lemma
 * 4vertexorbit P:704-751, Thm B.1, Fig. 11) and the
 * textual anchors P:129-146.
 *
 * Enumeration: ESU (exclusive-subgraph extension; each connected induced
 * vertex set of size 2..5 produced exactly once, minimum vertex = root) and an
 * all-subsets brute force used to pin ESU.  Counts are accumulated in wrapping
 * uint64 (reading R20: counts are exact modulo 2^64).
 *
 * parity unpinned: none of the functions here -- see tests/test_oracle_*.py.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define NORB 73
#define NPAT 30

/* ------------------------------------------------------------------------- */
/* Pattern catalog H0..H29 (Fig. 2 reading, R1).                    */
/* Each pattern: k vertices, edge list, and the orbit id of every vertex.     */
/* ------------------------------------------------------------------------- */
typedef struct {
  int k;
  int ne;
  int e[10][2];
  int orb[5];
} pattern_t;

static const pattern_t CATALOG[NPAT] = {
  /* H0  edge                     */ {2, 1, {{0,1}}, {0,0}},
  /* H1  path P3 (1 end, 2 mid)   */ {3, 2, {{0,1},{1,2}}, {1,2,1}},
  /* H2  triangle                 */ {3, 3, {{0,1},{0,2},{1,2}}, {3,3,3}},
  /* H3  path P4 (4 end, 5 mid)   */ {4, 3, {{0,1},{1,2},{2,3}}, {4,5,5,4}},
  /* H4  claw (6 leaf, 7 centre)  */ {4, 3, {{0,1},{0,2},{0,3}}, {7,6,6,6}},
  /* H5  4-cycle                  */ {4, 4, {{0,1},{1,2},{2,3},{3,0}}, {8,8,8,8}},
  /* H6  paw: tail 9, tri deg2 10, centre 11 */
  {4, 4, {{0,1},{0,2},{1,2},{0,3}}, {11,10,10,9}},
  /* H7  diamond: off-chord 12, chord 13 */
  {4, 5, {{0,1},{0,2},{0,3},{1,2},{1,3}}, {13,13,12,12}},
  /* H8  K4                       */ {4, 6, {{0,1},{0,2},{0,3},{1,2},{1,3},{2,3}}, {14,14,14,14}},
  /* H9  path P5: 15 end, 16 next, 17 centre */
  {5, 4, {{0,1},{1,2},{2,3},{3,4}}, {15,16,17,16,15}},
  /* H10 chair: 18 long-arm end, 19 short leaves, 20 long-arm middle, 21 centre */
  {5, 4, {{0,1},{0,2},{0,3},{3,4}}, {21,19,19,20,18}},
  /* H11 star K1,4: 22 leaf, 23 centre */
  {5, 4, {{0,1},{0,2},{0,3},{0,4}}, {23,22,22,22,22}},
  /* H12 bull: 24 pendants, 25 apex, 26 pendant-bearing triangle vertices */
  {5, 5, {{0,1},{0,2},{1,2},{1,3},{2,4}}, {25,26,26,24,24}},
  /* H13 triangle + 2-path: 27 end, 28 path middle, 29 tri deg2, 30 attach */
  {5, 5, {{0,1},{0,2},{1,2},{2,3},{3,4}}, {29,29,30,28,27}},
  /* H14 cricket: 31 pendants, 32 tri deg2, 33 centre */
  {5, 5, {{0,1},{0,2},{1,2},{0,3},{0,4}}, {33,32,32,31,31}},
  /* H15 5-cycle                  */ {5, 5, {{0,1},{1,2},{2,3},{3,4},{4,0}}, {34,34,34,34,34}},
  /* H16 banner (C4 + pendant): 35 pendant, 36 opposite, 37 adjacent, 38 attach */
  {5, 5, {{0,1},{1,2},{2,3},{3,0},{0,4}}, {38,37,36,37,35}},
  /* H17 diamond + pendant on chord vertex: 39 pendant, 40 off-chord, 41 chord, 42 attach */
  {5, 6, {{0,1},{0,2},{0,3},{1,2},{1,3},{0,4}}, {42,41,40,40,39}},
  /* H18 bowtie: 43 wings, 44 centre */
  {5, 6, {{0,1},{0,2},{1,2},{0,3},{0,4},{3,4}}, {44,43,43,43,43}},
  /* H19 diamond + pendant on off-chord vertex: 45 pendant, 46 free off-chord, 47 attach, 48 chord */
  {5, 6, {{0,1},{0,2},{0,3},{1,2},{1,3},{2,4}}, {48,48,47,46,45}},
  /* H20 K2,3: 49 degree-2 side, 50 degree-3 side */
  {5, 6, {{0,2},{0,3},{0,4},{1,2},{1,3},{1,4}}, {50,50,49,49,49}},
  /* H21 house: 51 floor, 52 roof, 53 eaves */
  {5, 6, {{0,1},{1,2},{2,3},{3,0},{4,0},{4,1}}, {53,53,51,51,52}},
  /* H22 book K1,1,3: 54 pages, 55 spine */
  {5, 7, {{0,1},{0,2},{0,3},{0,4},{1,2},{1,3},{1,4}}, {55,55,54,54,54}},
  /* H23 K4 + pendant: 56 pendant, 57 free K4 vertices, 58 attach */
  {5, 7, {{0,1},{0,2},{0,3},{1,2},{1,3},{2,3},{0,4}}, {58,57,57,57,56}},
  /* H24 gem (P4 + hub): 59 path ends, 60 path middles, 61 hub */
  {5, 7, {{0,1},{1,2},{2,3},{4,0},{4,1},{4,2},{4,3}}, {59,60,60,59,61}},
  /* H25 K2,3 + edge in the 3-side: 62 degree 2, 63 non-adjacent deg 3, 64 adjacent deg 3 */
  {5, 7, {{0,2},{0,3},{0,4},{1,2},{1,3},{1,4},{2,3}}, {63,63,64,64,62}},
  /* H26 K4 + degree-2 vertex: 65 degree 2, 66 degree 3, 67 degree 4 */
  {5, 8, {{0,1},{0,2},{0,3},{1,2},{1,3},{2,3},{4,0},{4,1}}, {67,67,66,66,65}},
  /* H27 wheel W4: 68 rim, 69 hub */
  {5, 8, {{0,1},{1,2},{2,3},{3,0},{4,0},{4,1},{4,2},{4,3}}, {68,68,68,68,69}},
  /* H28 K5 minus edge (3,4): 70 degree 3, 71 degree 4 */
  {5, 9, {{0,1},{0,2},{0,3},{0,4},{1,2},{1,3},{1,4},{2,3},{2,4}}, {71,71,71,70,70}},
  /* H29 K5                       */
  {5, 10, {{0,1},{0,2},{0,3},{0,4},{1,2},{1,3},{1,4},{2,3},{2,4},{3,4}}, {72,72,72,72,72}},
};

/* bit index of position pair (i,j), i<j: pairs ordered (0,1),(0,2),(1,2),(0,3),... */
static inline int pair_bit(int i, int j) {
  if (i > j) { int t = i; i = j; j = t; }
  return j * (j - 1) / 2 + i;
}

/* Lookup tables: for k = 2..5 and every mask over the C(k,2) position pairs,
 * orbit id per position (or -1 if the mask is not a connected spanning graph). */
static signed char TABLE2[1 << 1][2];
static signed char TABLE3[1 << 3][3];
static signed char TABLE4[1 << 6][4];
static signed char TABLE5[1 << 10][5];
static int g_tables_ready = 0;

static signed char *table_row(int k, int mask) {
  switch (k) {
    case 2: return TABLE2[mask];
    case 3: return TABLE3[mask];
    case 4: return TABLE4[mask];
    default: return TABLE5[mask];
  }
}

static int mask_connected(int k, int mask) {
  int seen = 1, frontier = 1;
  while (frontier) {
    int nf = 0;
    for (int a = 0; a < k; a++) {
      if (!(frontier >> a & 1)) continue;
      for (int b = 0; b < k; b++) {
        if (a == b) continue;
        if ((mask >> pair_bit(a, b) & 1) && !(seen >> b & 1)) { seen |= 1 << b; nf |= 1 << b; }
      }
    }
    frontier = nf;
  }
  return seen == (1 << k) - 1;
}

static int popcount_i(int x) { int c = 0; while (x) { c += x & 1; x >>= 1; } return c; }

/* next permutation (lexicographic) of p[0..k-1]; returns 0 after the last */
static int next_perm(int *p, int k) {
  int i = k - 2;
  while (i >= 0 && p[i] > p[i + 1]) i--;
  if (i < 0) return 0;
  int j = k - 1;
  while (p[j] < p[i]) j--;
  int t = p[i]; p[i] = p[j]; p[j] = t;
  for (int a = i + 1, b = k - 1; a < b; a++, b--) { t = p[a]; p[a] = p[b]; p[b] = t; }
  return 1;
}

static int pattern_mask(const pattern_t *P, const int *perm) {
  /* mask obtained by placing pattern vertex a at position perm[a] */
  int m = 0;
  for (int e = 0; e < P->ne; e++) m |= 1 << pair_bit(perm[P->e[e][0]], perm[P->e[e][1]]);
  return m;
}

static void build_tables(void) {
  if (g_tables_ready) return;
  for (int k = 2; k <= 5; k++) {
    int npairs = k * (k - 1) / 2;
    for (int mask = 0; mask < (1 << npairs); mask++) {
      signed char *row = table_row(k, mask);
      for (int i = 0; i < k; i++) row[i] = -1;
      if (!mask_connected(k, mask)) continue;
      for (int p = 0; p < NPAT && row[0] < 0; p++) {
        const pattern_t *P = &CATALOG[p];
        if (P->k != k || P->ne != popcount_i(mask)) continue;
        int perm[5] = {0, 1, 2, 3, 4};
        do {
          if (pattern_mask(P, perm) == mask) {
            for (int a = 0; a < k; a++) row[perm[a]] = (signed char)P->orb[a];
            break;
          }
        } while (next_perm(perm, k));
      }
    }
  }
  g_tables_ready = 1;
}

/* ------------------------------------------------------------------------- */
/* Catalog self-description (used by tests to pin the catalog).              */
/* ------------------------------------------------------------------------- */
int oracle_num_patterns(void) { return NPAT; }

/* Writes k, ne, edges (2*ne ints), orbit per vertex (k ints). */
int oracle_pattern(int p, int *k, int *ne, int *edges, int *orb) {
  if (p < 0 || p >= NPAT) return -1;
  const pattern_t *P = &CATALOG[p];
  *k = P->k; *ne = P->ne;
  for (int e = 0; e < P->ne; e++) { edges[2 * e] = P->e[e][0]; edges[2 * e + 1] = P->e[e][1]; }
  for (int a = 0; a < P->k; a++) orb[a] = P->orb[a];
  return 0;
}

/* Automorphism classes by exhaustive permutation (Def. "auto").
 * cls[a] = smallest vertex b such that some automorphism maps a to b. */
int oracle_automorphism_classes(int p, int *cls, int *num_aut) {
  if (p < 0 || p >= NPAT) return -1;
  const pattern_t *P = &CATALOG[p];
  int k = P->k, ident[5] = {0, 1, 2, 3, 4};
  int base = pattern_mask(P, ident);
  for (int a = 0; a < k; a++) cls[a] = a;
  int perm[5] = {0, 1, 2, 3, 4}, cnt = 0;
  do {
    if (pattern_mask(P, perm) == base) {
      cnt++;
      for (int a = 0; a < k; a++) if (perm[a] < cls[a]) cls[a] = perm[a];
    }
  } while (next_perm(perm, k));
  *num_aut = cnt;
  return 0;
}

/* classify a mask over k positions: writes orbit per position, returns 0 if
 * connected spanning, -1 otherwise */
int oracle_classify(int k, int mask, int *orb) {
  build_tables();
  if (k < 2 || k > 5) return -1;
  signed char *row = table_row(k, mask);
  if (row[0] < 0) return -1;
  for (int i = 0; i < k; i++) orb[i] = row[i];
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Graph: cleaned simple undirected graph in sorted adjacency form.          */
/* ------------------------------------------------------------------------- */
typedef struct {
  int64_t n;
  int64_t *rp;   /* n+1 */
  int32_t *adj;  /* rp[n] */
} graph_t;

static int cmp_u64(const void *a, const void *b) {
  uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
  return x < y ? -1 : x > y;
}

/* Input cleaning ("removed directions ... omitted duplicates and self
 * loops"); ids are kept (row v = vertex v). Returns 0 or -1 on bad input. */
static int graph_build(graph_t *g, int64_t n, int64_t m, const int32_t *edges) {
  g->n = n; g->rp = NULL; g->adj = NULL;
  uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(2 * m + 1));
  if (!keys) return -1;
  int64_t cnt = 0;
  for (int64_t e = 0; e < m; e++) {
    int64_t a = edges[2 * e], b = edges[2 * e + 1];
    if (a < 0 || b < 0 || a >= n || b >= n) { free(keys); return -1; }
    if (a == b) continue;
    keys[cnt++] = ((uint64_t)a << 32) | (uint64_t)b;
    keys[cnt++] = ((uint64_t)b << 32) | (uint64_t)a;
  }
  qsort(keys, (size_t)cnt, sizeof(uint64_t), cmp_u64);
  int64_t u = 0;
  for (int64_t i = 0; i < cnt; i++)
    if (i == 0 || keys[i] != keys[i - 1]) keys[u++] = keys[i];
  g->rp = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  g->adj = (int32_t *)malloc(sizeof(int32_t) * (size_t)(u + 1));
  for (int64_t i = 0; i < u; i++) g->rp[(keys[i] >> 32) + 1]++;
  for (int64_t v = 0; v < n; v++) g->rp[v + 1] += g->rp[v];
  for (int64_t i = 0; i < u; i++) g->adj[i] = (int32_t)(keys[i] & 0xffffffffu);
  free(keys);
  return 0;
}

static void graph_free(graph_t *g) { free(g->rp); free(g->adj); }

static int has_edge(const graph_t *g, int a, int b) {
  int64_t lo = g->rp[a], hi = g->rp[a + 1];
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (g->adj[mid] < b) lo = mid + 1; else hi = mid;
  }
  return lo < g->rp[a + 1] && g->adj[lo] == b;
}

/* adjacency mask of the ordered vertex list S[0..k-1] */
static int subset_mask(const graph_t *g, const int *S, int k) {
  int m = 0;
  for (int j = 1; j < k; j++)
    for (int i = 0; i < j; i++)
      if (has_edge(g, S[i], S[j])) m |= 1 << pair_bit(i, j);
  return m;
}

/* credit every position of the induced subgraph S */
static void credit(const graph_t *g, const int *S, int k, uint64_t *out) {
  int mask = subset_mask(g, S, k);
  signed char *row = table_row(k, mask);
  for (int i = 0; i < k; i++) out[(int64_t)S[i] * NORB + row[i]] += 1u;
}

/* ------------------------------------------------------------------------- */
/* ESU: every connected induced subgraph on 2..5 vertices exactly once.       */
/* ------------------------------------------------------------------------- */
typedef struct {
  const graph_t *g;
  int32_t *buf[6];     /* extension set of each depth, capacity cap_ext */
  int64_t cap_ext;
  uint64_t *out;       /* n*73 accumulator, or NULL (rooted mode)  */
  uint64_t *row;       /* rooted mode: 73 accumulator for S[0]     */
  int root_filter;     /* 1: only extend with ids > root            */
  uint64_t work, cap;  /* rooted mode: number of sets, cap (0 = none) */
  int aborted;
} esu_ctx;

static int in_set(const int *S, int k, int x) {
  for (int i = 0; i < k; i++) if (S[i] == x) return 1;
  return 0;
}

static int adjacent_to_set(const graph_t *g, const int *S, int k, int x) {
  for (int i = 0; i < k; i++) if (has_edge(g, S[i], x)) return 1;
  return 0;
}

static void esu_extend(esu_ctx *c, int *S, int k, int32_t *ext, int64_t next) {
  if (c->aborted) return;
  if (k >= 2) {
    if (c->out) credit(c->g, S, k, c->out);
    else {
      int mask = subset_mask(c->g, S, k);
      c->row[table_row(k, mask)[0]] += 1u;
      c->work++;
      if (c->cap && c->work >= c->cap) { c->aborted = 1; return; }
    }
  }
  if (k == 5) return;
  const graph_t *g = c->g;
  int root = S[0];
  /* Wernicke's ESU: pick w from the extension set; the new extension set is
   * the rest of the old one plus the exclusive neighbours of w. */
  int32_t *ext2 = c->buf[k];
  while (next > 0) {
    int w = ext[--next];
    int64_t n2 = 0;
    for (int64_t i = 0; i < next; i++) ext2[n2++] = ext[i];
    S[k] = w;
    for (int64_t p = g->rp[w]; p < g->rp[w + 1]; p++) {
      int u = g->adj[p];
      if (c->root_filter && u <= root) continue;
      if (in_set(S, k + 1, u)) continue;
      if (adjacent_to_set(g, S, k, u)) continue;  /* u in N(S) => not exclusive */
      if (n2 >= c->cap_ext) { c->aborted = 2; return; }
      ext2[n2++] = u;
    }
    if (!c->out) {  /* rooted mode: the cap bounds work (sets + extension elements) */
      c->work += (uint64_t)n2;
      if (c->cap && c->work >= c->cap) { c->aborted = 1; return; }
    }
    esu_extend(c, S, k + 1, ext2, n2);
    if (c->aborted) return;
  }
}

/* per-depth extension buffers: an extension set holds at most the exclusive
 * neighbourhoods of the (<= 4) vertices added so far */
static int ctx_alloc(esu_ctx *c, const graph_t *g) {
  int64_t dmax = 0;
  for (int64_t v = 0; v < g->n; v++) if (g->rp[v + 1] - g->rp[v] > dmax) dmax = g->rp[v + 1] - g->rp[v];
  c->cap_ext = 5 * dmax + 16;
  for (int i = 0; i < 6; i++) {
    c->buf[i] = (int32_t *)malloc(sizeof(int32_t) * (size_t)c->cap_ext);
    if (!c->buf[i]) return -1;
  }
  return 0;
}
static void ctx_free(esu_ctx *c) { for (int i = 0; i < 6; i++) free(c->buf[i]); }

/* Induced orbit counts of all vertices by ESU over all roots.
 * Returns 0, -1 (bad input), -2 (extension set overflow). */
int oracle_orbits_esu(int64_t n, int64_t m, const int32_t *edges, uint64_t *out, int threads) {
  build_tables();
  graph_t g;
  if (graph_build(&g, n, m, edges)) return -1;
  memset(out, 0, sizeof(uint64_t) * (size_t)n * NORB);
  int status = 0;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
#pragma omp parallel
  {
    uint64_t *acc = (uint64_t *)calloc((size_t)n * NORB, sizeof(uint64_t));
    esu_ctx c;
    memset(&c, 0, sizeof(c));
    c.g = &g; c.out = acc; c.root_filter = 1;
    if (ctx_alloc(&c, &g)) c.aborted = 3;
#pragma omp for schedule(dynamic, 1)
    for (int64_t r = 0; r < n; r++) {
      if (c.aborted) continue;
      int S[5];
      int64_t ne = 0;
      S[0] = (int)r;
      for (int64_t p = g.rp[r]; p < g.rp[r + 1]; p++)
        if (g.adj[p] > r) c.buf[5][ne++] = g.adj[p];
      esu_extend(&c, S, 1, c.buf[5], ne);
    }
#pragma omp critical
    {
      if (c.aborted) status = -2;
      for (int64_t i = 0; i < n * NORB; i++) out[i] += acc[i];
    }
    ctx_free(&c);
    free(acc);
  }
  graph_free(&g);
  return status;
}

/* One exact row DIM(root, .) by rooted ESU (no id filter: every connected set
 * containing root exactly once).  cap = max number of sets (0 = unlimited).
 * Returns 0 on success, 1 if the cap was hit (row incomplete), <0 on error. */
int oracle_orbit_row(int64_t n, int64_t m, const int32_t *edges, int64_t root,
                     uint64_t *row, uint64_t cap) {
  build_tables();
  graph_t g;
  if (root < 0 || root >= n) return -1;
  if (graph_build(&g, n, m, edges)) return -1;
  memset(row, 0, sizeof(uint64_t) * NORB);
  esu_ctx c;
  memset(&c, 0, sizeof(c));
  c.g = &g; c.row = row; c.cap = cap;
  if (ctx_alloc(&c, &g)) { graph_free(&g); return -2; }
  int S[5];
  int64_t ne = 0;
  S[0] = (int)root;
  for (int64_t p = g.rp[root]; p < g.rp[root + 1]; p++) c.buf[5][ne++] = g.adj[p];
  esu_extend(&c, S, 1, c.buf[5], ne);
  ctx_free(&c);
  graph_free(&g);
  if (c.aborted == 2) return -2;
  return c.aborted ? 1 : 0;
}

/* Same, for many roots (one thread per root). status[i] as oracle_orbit_row. */
int oracle_orbit_rows(int64_t n, int64_t m, const int32_t *edges, int64_t nroots,
                      const int64_t *roots, uint64_t *rows, int *status, uint64_t cap,
                      int threads) {
  build_tables();
  graph_t g;
  if (graph_build(&g, n, m, edges)) return -1;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
#pragma omp parallel
  {
    esu_ctx c;
    memset(&c, 0, sizeof(c));
    int bad_alloc = ctx_alloc(&c, &g);
#pragma omp for schedule(dynamic, 1)
    for (int64_t i = 0; i < nroots; i++) {
      int64_t root = roots[i];
      uint64_t *row = rows + i * NORB;
      memset(row, 0, sizeof(uint64_t) * NORB);
      if (root < 0 || root >= n || bad_alloc) { status[i] = -1; continue; }
      c.row = row; c.cap = cap; c.work = 0; c.aborted = 0; c.g = &g;
      int S[5];
      int64_t ne = 0;
      S[0] = (int)root;
      for (int64_t p = g.rp[root]; p < g.rp[root + 1]; p++) c.buf[5][ne++] = g.adj[p];
      esu_extend(&c, S, 1, c.buf[5], ne);
      status[i] = c.aborted == 2 ? -2 : (c.aborted ? 1 : 0);
    }
    ctx_free(&c);
  }
  graph_free(&g);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* All-subsets brute force (pins ESU on tiny graphs): every k-subset, k=2..5, */
/* connectivity by the mask table, credit.                                    */
/* ------------------------------------------------------------------------- */
int oracle_orbits_bruteforce(int64_t n, int64_t m, const int32_t *edges, uint64_t *out) {
  build_tables();
  graph_t g;
  if (n > 64) return -1;
  if (graph_build(&g, n, m, edges)) return -1;
  memset(out, 0, sizeof(uint64_t) * (size_t)n * NORB);
  int S[5];
  for (int k = 2; k <= 5; k++) {
    /* lexicographic k-subsets of 0..n-1 */
    if (k > n) break;
    for (int i = 0; i < k; i++) S[i] = i;
    for (;;) {
      int mask = subset_mask(&g, S, k);
      signed char *row = table_row(k, mask);
      if (row[0] >= 0)
        for (int i = 0; i < k; i++) out[(int64_t)S[i] * NORB + row[i]] += 1u;
      int i = k - 1;
      while (i >= 0 && S[i] == n - k + i) i--;
      if (i < 0) break;
      S[i]++;
      for (int j = i + 1; j < k; j++) S[j] = S[j - 1] + 1;
    }
  }
  graph_free(&g);
  return 0;
}

/* Non-induced brute force DM(v,theta) (Def. unlabeled-match):
 * every k-subset U and every edge subset F of E(G[U]) that is connected and
 * spanning on U is one distinct copy; credit its positions. Tiny graphs only. */
int oracle_noninduced_bruteforce(int64_t n, int64_t m, const int32_t *edges, uint64_t *out) {
  build_tables();
  graph_t g;
  if (n > 40) return -1;
  if (graph_build(&g, n, m, edges)) return -1;
  memset(out, 0, sizeof(uint64_t) * (size_t)n * NORB);
  int S[5];
  for (int k = 2; k <= 5; k++) {
    if (k > n) break;
    for (int i = 0; i < k; i++) S[i] = i;
    for (;;) {
      int full = subset_mask(&g, S, k);
      /* enumerate sub-masks F of full (including full itself) */
      for (int F = full;; F = (F - 1) & full) {
        signed char *row = table_row(k, F);
        if (F && row[0] >= 0)
          for (int i = 0; i < k; i++) out[(int64_t)S[i] * NORB + row[i]] += 1u;
        if (F == 0) break;
      }
      int i = k - 1;
      while (i >= 0 && S[i] == n - k + i) i--;
      if (i < 0) break;
      S[i]++;
      for (int j = i + 1; j < k; j++) S[j] = S[j - 1] + 1;
    }
  }
  graph_free(&g);
  return 0;
}

/* Simple clique / triangle totals by plain enumeration (used for whole-matrix
 * invariants at sizes the ESU cannot reach: Sigma_v DIM3 = 3 #K3, Sigma_v DIM14 =
 * 4 #K4, Sigma_v DIM72 = 5 #K5; cliques = P:702 / P:861-864).
 * Each clique is counted once, at its first vertex in the paper's degree order
 * (vertices ordered by degree, ties by id): for every vertex a, the
 * pairwise-adjacent 2-, 3- and 4-subsets of its later neighbours N>(a), taken
 * in increasing list position.  The order only bounds |N>(a)|; any total order
 * counts every clique exactly once.
 * counts[0] = #triangles, counts[1] = #4-cliques, counts[2] = #5-cliques; only cliques
 * of at most kmax (3..5) vertices are counted (the others are left 0), so the invariants
 * reach graphs whose 5-cliques number in the 10^10s. */
static int later(const graph_t *g, int a, int b) {  /* b after a in degree order */
  int64_t da = g->rp[a + 1] - g->rp[a], db = g->rp[b + 1] - g->rp[b];
  return db > da || (db == da && b > a);
}

int oracle_clique_totals(int64_t n, int64_t m, const int32_t *edges, uint64_t *counts, int threads, int kmax) {
  graph_t g;
  if (graph_build(&g, n, m, edges)) return -1;
  /* N>(a) for every a, in increasing id order (a filtered copy of the sorted list) */
  int64_t *orp = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  int32_t *oadj = (int32_t *)malloc(sizeof(int32_t) * (size_t)(g.rp[n] / 2 + 1));
  if (!orp || !oadj) { free(orp); free(oadj); graph_free(&g); return -1; }
  for (int64_t a = 0; a < n; a++) {
    orp[a + 1] = orp[a];
    for (int64_t p = g.rp[a]; p < g.rp[a + 1]; p++)
      if (later(&g, (int)a, g.adj[p])) oadj[orp[a + 1]++] = g.adj[p];
  }
  uint64_t t3 = 0, t4 = 0, t5 = 0;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
#pragma omp parallel for schedule(dynamic, 64) reduction(+:t3, t4, t5)
  for (int64_t a = 0; a < n; a++) {
    for (int64_t pb = orp[a]; pb < orp[a + 1]; pb++) {
      int b = oadj[pb];
      for (int64_t pc = pb + 1; pc < orp[a + 1]; pc++) {
        int c = oadj[pc];
        if (!has_edge(&g, b, c)) continue;
        t3++;
        if (kmax < 4) continue;
        for (int64_t pd = pc + 1; pd < orp[a + 1]; pd++) {
          int d = oadj[pd];
          if (!has_edge(&g, b, d) || !has_edge(&g, c, d)) continue;
          t4++;
          if (kmax < 5) continue;
          for (int64_t pe = pd + 1; pe < orp[a + 1]; pe++) {
            int e = oadj[pe];
            if (has_edge(&g, b, e) && has_edge(&g, c, e) && has_edge(&g, d, e)) t5++;
          }
        }
      }
    }
  }
  counts[0] = t3; counts[1] = t4; counts[2] = t5;
  free(orp); free(oadj);
  graph_free(&g);
  return 0;
}

/* The same clique totals (cliques = P:702 / P:861-864, each counted once at its first
 * vertex in the degree order of P:432-437) with the inner membership tests done on a
 * local adjacency bitmap, for the graphs where the plain loop nest above is too slow
 * (config 3's 5-cliques, config 5's 4- and 5-cliques).  For every vertex a:
 *   L = N>(a) listed in degree order; row i of the bitmap holds bit j (j > i) iff
 *   L[i] ~ L[j].  A clique {a} + S, S a pairwise-adjacent subset of L, is found once, from
 *   its member of least position: triangles = sum_i |row i|, 4-cliques = sum over bits j of
 *   row i of |row i & row j|, 5-cliques = sum over bits l of (row i & row j) of
 *   |row i & row j & row l|.
 * Pinned against oracle_clique_totals (itself pinned against all-subsets brute force) in
 * tests/test_oracle_pins.py; kmax as there. */
static int64_t *g_ord_rank;  /* rank of each vertex in degree order (read-only in the loop) */
static int cmp_by_rank(const void *x, const void *y) {
  int64_t a = g_ord_rank[*(const int32_t *)x], b = g_ord_rank[*(const int32_t *)y];
  return (a > b) - (a < b);
}

int oracle_clique_totals_bits(int64_t n, int64_t m, const int32_t *edges, uint64_t *counts, int threads,
                              int kmax) {
  graph_t g;
  if (graph_build(&g, n, m, edges)) return -1;
  /* degree order (ties by id) as a rank: sort ids by (degree, id) */
  int64_t *key = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t *rank = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t *orp = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  int32_t *oadj = (int32_t *)malloc(sizeof(int32_t) * (size_t)(g.rp[n] / 2 + 1));
  if (!key || !rank || !orp || !oadj) { free(key); free(rank); free(orp); free(oadj); graph_free(&g); return -1; }
  for (int64_t v = 0; v < n; v++) key[v] = ((g.rp[v + 1] - g.rp[v]) << 32) | v;  /* degree < 2^31 */
  qsort(key, (size_t)n, sizeof(int64_t), cmp_u64);  /* non-negative keys: unsigned order = signed order */
  for (int64_t r = 0; r < n; r++) rank[key[r] & 0xffffffffLL] = r;
  free(key);
  /* N>(a): the later neighbours of a, listed in degree order */
  int64_t kmax_list = 0;
  for (int64_t a = 0; a < n; a++) {
    orp[a + 1] = orp[a];
    for (int64_t p = g.rp[a]; p < g.rp[a + 1]; p++)
      if (rank[g.adj[p]] > rank[a]) oadj[orp[a + 1]++] = g.adj[p];
    if (orp[a + 1] - orp[a] > kmax_list) kmax_list = orp[a + 1] - orp[a];
  }
  g_ord_rank = rank;
  for (int64_t a = 0; a < n; a++) qsort(oadj + orp[a], (size_t)(orp[a + 1] - orp[a]), sizeof(int32_t), cmp_by_rank);
  uint64_t t3 = 0, t4 = 0, t5 = 0;
  int fail = 0;
  const int64_t W = (kmax_list + 63) / 64;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
#pragma omp parallel reduction(+:t3, t4, t5) reduction(|:fail)
  {
    int32_t *pos = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));  /* position in L, or -1 */
    uint64_t *row = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(kmax_list * W + 1));
    uint64_t *c2 = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(W + 1));
    const int ok = pos && row && c2;
    if (ok) for (int64_t v = 0; v < n; v++) pos[v] = -1;
    {
#pragma omp for schedule(dynamic, 16)
      for (int64_t a = 0; a < n; a++) {
        if (!ok) { fail = 1; continue; }  /* every thread still reaches the worksharing loop */
        const int32_t *L = oadj + orp[a];
        const int64_t k = orp[a + 1] - orp[a], w = (k + 63) / 64;
        if (k < 2) continue;
        for (int64_t i = 0; i < k; i++) pos[L[i]] = (int32_t)i;
        memset(row, 0, sizeof(uint64_t) * (size_t)(k * w));
        /* L[i] ~ L[j] with j > i  <=>  L[j] in N>(L[i]) and in L */
        for (int64_t i = 0; i < k; i++)
          for (int64_t p = orp[L[i]]; p < orp[L[i] + 1]; p++) {
            int32_t j = pos[oadj[p]];
            if (j >= 0) row[i * w + j / 64] |= 1ULL << (j % 64);
          }
        for (int64_t i = 0; i < k; i++) {
          const uint64_t *ri = row + i * w;
          for (int64_t q = 0; q < w; q++) t3 += (uint64_t)__builtin_popcountll(ri[q]);
          if (kmax < 4) continue;
          for (int64_t q = 0; q < w; q++)
            for (uint64_t bits = ri[q]; bits; bits &= bits - 1) {
              int64_t j = q * 64 + __builtin_ctzll(bits);
              const uint64_t *rj = row + j * w;
              for (int64_t s = 0; s < w; s++) { c2[s] = ri[s] & rj[s]; t4 += (uint64_t)__builtin_popcountll(c2[s]); }
              if (kmax < 5) continue;
              for (int64_t s = 0; s < w; s++)
                for (uint64_t b2 = c2[s]; b2; b2 &= b2 - 1) {
                  const uint64_t *rl = row + (s * 64 + __builtin_ctzll(b2)) * w;
                  for (int64_t u = 0; u < w; u++) t5 += (uint64_t)__builtin_popcountll(c2[u] & rl[u]);
                }
            }
        }
        for (int64_t i = 0; i < k; i++) pos[L[i]] = -1;
      }
    }
    free(pos); free(row); free(c2);
  }
  counts[0] = t3; counts[1] = t4; counts[2] = t5;
  free(rank); free(orp); free(oadj);
  graph_free(&g);
  return fail ? -1 : 0;
}

/* Per-vertex clique counts: out[v*3 + 0] = #triangles, + 1 = #4-cliques, + 2 = #5-cliques
 * that contain v (cliques = P:702 / P:861-864).  A clique is an induced copy of itself and
 * all its vertices are one orbit, so these are three columns of the orbit matrix by their
 * definition: DIM(v, theta3) = DM(v, theta3) = T(v), DIM(v, theta14) = K4(v),
 * DIM(v, theta72) = K5(v) -- exact on every vertex, hubs included, at sizes the ESU cannot
 * reach (used by the GPU tests on the full configs).
 * Enumeration exactly as in oracle_clique_totals_bits (each clique found once, from its
 * first vertex a in the degree order of P:432-437 and its members of increasing position
 * in L = N>(a), membership on the local bitmap); here every clique found adds 1 to each of
 * its members instead of 1 to a total.  Members shared by all the cliques of an inner loop
 * get that loop's count in one addition; the last member is credited bit by bit.
 * Counts wrap modulo 2^64 (reading R20).  kmax as above (columns beyond kmax stay 0).
 * Pinned in tests/test_oracle_pins.py against the ESU columns 3/14/72, the all-subsets
 * brute force, K_n and the totals (sum_v = k * #K_k). */
int oracle_clique_counts_vertex(int64_t n, int64_t m, const int32_t *edges, uint64_t *out, int threads,
                                int kmax) {
  graph_t g;
  if (graph_build(&g, n, m, edges)) return -1;
  int64_t *key = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t *rank = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t *orp = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  int32_t *oadj = (int32_t *)malloc(sizeof(int32_t) * (size_t)(g.rp[n] / 2 + 1));
  if (!key || !rank || !orp || !oadj) { free(key); free(rank); free(orp); free(oadj); graph_free(&g); return -1; }
  for (int64_t v = 0; v < n; v++) key[v] = ((g.rp[v + 1] - g.rp[v]) << 32) | v;
  qsort(key, (size_t)n, sizeof(int64_t), cmp_u64);
  for (int64_t r = 0; r < n; r++) rank[key[r] & 0xffffffffLL] = r;
  free(key);
  int64_t kmax_list = 0;
  for (int64_t a = 0; a < n; a++) {
    orp[a + 1] = orp[a];
    for (int64_t p = g.rp[a]; p < g.rp[a + 1]; p++)
      if (rank[g.adj[p]] > rank[a]) oadj[orp[a + 1]++] = g.adj[p];
    if (orp[a + 1] - orp[a] > kmax_list) kmax_list = orp[a + 1] - orp[a];
  }
  g_ord_rank = rank;
  for (int64_t a = 0; a < n; a++) qsort(oadj + orp[a], (size_t)(orp[a + 1] - orp[a]), sizeof(int32_t), cmp_by_rank);
  memset(out, 0, sizeof(uint64_t) * (size_t)n * 3);
  int fail = 0;
  const int64_t W = (kmax_list + 63) / 64;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
#pragma omp parallel reduction(|:fail)
  {
    int32_t *pos = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1));
    uint64_t *row = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(kmax_list * W + 1));
    uint64_t *c2 = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(W + 1));
    uint64_t *loc = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(kmax_list * 3 + 3));  /* credits of L[i] */
    const int ok = pos && row && c2 && loc;
    if (ok) for (int64_t v = 0; v < n; v++) pos[v] = -1;
    {
#pragma omp for schedule(dynamic, 16)
      for (int64_t a = 0; a < n; a++) {
        if (!ok) { fail = 1; continue; }
        const int32_t *L = oadj + orp[a];
        const int64_t k = orp[a + 1] - orp[a], w = (k + 63) / 64;
        if (k < 2) continue;
        for (int64_t i = 0; i < k; i++) pos[L[i]] = (int32_t)i;
        memset(row, 0, sizeof(uint64_t) * (size_t)(k * w));
        memset(loc, 0, sizeof(uint64_t) * (size_t)(k * 3));
        for (int64_t i = 0; i < k; i++)
          for (int64_t p = orp[L[i]]; p < orp[L[i] + 1]; p++) {
            int32_t j = pos[oadj[p]];
            if (j >= 0) row[i * w + j / 64] |= 1ULL << (j % 64);
          }
        uint64_t a3 = 0, a4 = 0, a5 = 0;  /* cliques found at a: a is a member of each */
        for (int64_t i = 0; i < k; i++) {
          const uint64_t *ri = row + i * w;
          for (int64_t q = 0; q < w; q++)
            for (uint64_t bits = ri[q]; bits; bits &= bits - 1) {
              const int64_t j = q * 64 + __builtin_ctzll(bits);
              /* triangle {a, L[i], L[j]} */
              a3++; loc[i * 3]++; loc[j * 3]++;
              if (kmax < 4) continue;
              const uint64_t *rj = row + j * w;
              for (int64_t s = 0; s < w; s++) c2[s] = ri[s] & rj[s];
              for (int64_t s = 0; s < w; s++)
                for (uint64_t b2 = c2[s]; b2; b2 &= b2 - 1) {
                  const int64_t l = s * 64 + __builtin_ctzll(b2);
                  /* 4-clique {a, L[i], L[j], L[l]} */
                  a4++; loc[i * 3 + 1]++; loc[j * 3 + 1]++; loc[l * 3 + 1]++;
                  if (kmax < 5) continue;
                  const uint64_t *rl = row + l * w;
                  for (int64_t u = 0; u < w; u++)
                    for (uint64_t b3 = c2[u] & rl[u]; b3; b3 &= b3 - 1) {
                      const int64_t p5 = u * 64 + __builtin_ctzll(b3);
                      /* 5-clique {a, L[i], L[j], L[l], L[p5]} */
                      a5++; loc[i * 3 + 2]++; loc[j * 3 + 2]++; loc[l * 3 + 2]++; loc[p5 * 3 + 2]++;
                    }
                }
            }
        }
        for (int c = 0; c < 3; c++) {
          const uint64_t av = c == 0 ? a3 : c == 1 ? a4 : a5;
          if (av) {
#pragma omp atomic
            out[a * 3 + c] += av;
          }
        }
        for (int64_t i = 0; i < k; i++) {
          for (int c = 0; c < 3; c++)
            if (loc[i * 3 + c]) {
#pragma omp atomic
              out[(int64_t)L[i] * 3 + c] += loc[i * 3 + c];
            }
          pos[L[i]] = -1;
        }
      }
    }
    free(pos); free(row); free(c2); free(loc);
  }
  free(rank); free(orp); free(oadj);
  graph_free(&g);
  return fail ? -1 : 0;
}

/* Non-induced counts DM(u, theta_0..13) of the orbits with at most 4 vertices on EVERY
 * vertex, by Lemma "4vertexorbit" read line by line, from the plain
 * definitions of its inputs: d(u); T(u,v) = |N(u) & N(v)| for every edge (a merge
 * of the two sorted lists); T(u) = (1/2) sum_{v in N(u)} T(u,v); C4(u) = sum_{x != u}
 * C(c(u,x), 2), c(u,x) = #common neighbours = #wedges u-w-x (a 4-cycle through u is its
 * opposite vertex x and two of their common neighbours).  K4(u) (theta_14) is
 * oracle_clique_counts_vertex's column 1 and is not computed here.
 * out[u*15 + i] = DM(u, theta_i), i = 0..13 (slot 14 left 0), wrapping modulo 2^64
 * (reading R20).  with_c4 = 0 skips theta_8 (left 0): its wedge walk is O(sum d^2).
 * These are the NON-induced counts of Def. "unlabeled-match": the GPU tests
 * compare them with the non-induced mode of the product on every vertex of the
 * full configs, hub rows included.  Pinned against oracle_noninduced_bruteforce on random
 * graphs and against K_n / K_{a,b} closed forms in tests/test_oracle_pins.py. */
static uint64_t binom_u64(uint64_t x, int k) {  /* C(x, k) mod 2^64, k <= 3, via 128-bit products */
  if (x < (uint64_t)k) return 0;
  unsigned __int128 r = 1;
  for (int i = 0; i < k; i++) r *= (unsigned __int128)(x - (uint64_t)i);
  for (int i = 2; i <= k; i++) r /= (unsigned)i;  /* x < 2^40: the product is exact in 128 bits */
  return (uint64_t)r;
}

int oracle_dm4_vertex(int64_t n, int64_t m, const int32_t *edges, uint64_t *out, int threads, int with_c4) {
  graph_t g;
  if (graph_build(&g, n, m, edges)) return -1;
  const int64_t M2 = g.rp[n];
  uint32_t *te = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(M2 + 1));  /* T(u,v) per list slot */
  uint64_t *T = (uint64_t *)calloc((size_t)n + 1, sizeof(uint64_t));
  uint64_t *dm1 = (uint64_t *)calloc((size_t)n + 1, sizeof(uint64_t));
  if (!te || !T || !dm1) { free(te); free(T); free(dm1); graph_free(&g); return -1; }
  memset(out, 0, sizeof(uint64_t) * (size_t)n * 15);
  int fail = 0;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
  /* T(u,v) for every edge, both directions; T(u); DM(u, theta_1) */
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t u = 0; u < n; u++) {
    uint64_t tu = 0, s1 = 0;
    for (int64_t p = g.rp[u]; p < g.rp[u + 1]; p++) {
      const int v = g.adj[p];
      int64_t a = g.rp[u], b = g.rp[v];
      uint32_t c = 0;
      while (a < g.rp[u + 1] && b < g.rp[v + 1]) {
        if (g.adj[a] < g.adj[b]) a++;
        else if (g.adj[a] > g.adj[b]) b++;
        else { c++; a++; b++; }
      }
      te[p] = c;
      tu += c;
      s1 += (uint64_t)(g.rp[v + 1] - g.rp[v]) - 1;
    }
    T[u] = tu / 2;
    dm1[u] = s1;
  }
#pragma omp parallel reduction(|:fail)
  {
    uint32_t *cnt = with_c4 ? (uint32_t *)calloc((size_t)n + 1, sizeof(uint32_t)) : NULL;
    int32_t *touched = with_c4 ? (int32_t *)malloc(sizeof(int32_t) * (size_t)(n + 1)) : NULL;
    const int ok = !with_c4 || (cnt && touched);
#pragma omp for schedule(dynamic, 16)
    for (int64_t u = 0; u < n; u++) {
      if (!ok) { fail = 1; continue; }
      uint64_t *o = out + u * 15;
      const uint64_t d = (uint64_t)(g.rp[u + 1] - g.rp[u]);
      uint64_t s4 = 0, s6 = 0, s9 = 0, s10 = 0, s12 = 0, s13 = 0;
      for (int64_t p = g.rp[u]; p < g.rp[u + 1]; p++) {
        const int v = g.adj[p];
        const uint64_t dv = (uint64_t)(g.rp[v + 1] - g.rp[v]), tuv = te[p];
        s4 += dm1[v];
        s6 += binom_u64(dv - 1, 2);
        s9 += T[v] - tuv;
        s10 += tuv * (dv - 2);
        s13 += binom_u64(tuv, 2);
        /* triangles t = (u, v, x) with v < x: x in N(u) & N(v); add T(v,x) - 1 */
        int64_t a = g.rp[u], b = g.rp[v];
        while (a < g.rp[u + 1] && b < g.rp[v + 1]) {
          if (g.adj[a] < g.adj[b]) a++;
          else if (g.adj[a] > g.adj[b]) b++;
          else { if (g.adj[b] > v) s12 += (uint64_t)te[b] - 1; a++; b++; }  /* slot b = x in N(v) */
        }
      }
      o[0] = d;
      o[1] = dm1[u];
      o[2] = binom_u64(d, 2);
      o[3] = T[u];
      o[4] = s4 - 2 * o[2] - 2 * o[3];
      o[5] = o[1] * (d - 1) - 2 * o[3];
      o[6] = s6;
      o[7] = binom_u64(d, 3);
      o[9] = s9;
      o[10] = s10;
      o[11] = o[3] * (d - 2);
      o[12] = s12;
      o[13] = s13;
      if (with_c4) {
        int64_t nt = 0;
        for (int64_t p = g.rp[u]; p < g.rp[u + 1]; p++) {
          const int w = g.adj[p];
          for (int64_t q = g.rp[w]; q < g.rp[w + 1]; q++) {
            const int x = g.adj[q];
            if (x == u) continue;
            if (cnt[x]++ == 0) touched[nt++] = x;
          }
        }
        uint64_t c4 = 0;
        for (int64_t i = 0; i < nt; i++) { c4 += binom_u64(cnt[touched[i]], 2); cnt[touched[i]] = 0; }
        o[8] = c4;
      }
    }
    free(cnt); free(touched);
  }
  free(te); free(T); free(dm1);
  graph_free(&g);
  return fail ? -1 : 0;
}

/* Non-induced 5-cycle count of chosen vertices: out[r] = DM(roots[r], theta_34) = the number
 * of 5-cycles of G through v = roots[r] (the 5-cycle pattern has one orbit, theta_34: "each
 * vertex of the Petersen graph is in 6 five-cycles"; Def. "unlabeled-match" P:419-422),
 * straight from the definition: a 5-cycle through v is v-a-x-y-b-v with five distinct
 * vertices and the five edges present; each is met twice (once per direction), so the
 * number of such (a, x, y, b) is halved.  The walk is O(#4-paths from v) -- cheap for a hub
 * of a sparse graph, where the rooted ESU (all connected 5-sets around the hub) is not.
 * status[r] = 0 done, 1 abandoned after `cap` innermost steps (cap = 0: no cap).
 * Pinned against oracle_noninduced_bruteforce column 34 and K_n / C_5 / Petersen closed
 * forms in tests/test_oracle_pins.py. */
int oracle_c5_rows(int64_t n, int64_t m, const int32_t *edges, int64_t nroots, const int64_t *roots,
                   uint64_t *out, int *status, uint64_t cap, int threads) {
  graph_t g;
  if (graph_build(&g, n, m, edges)) return -1;
  unsigned char *nv = (unsigned char *)calloc((size_t)n + 1, 1);  /* nv[b] = 1 iff b ~ v */
  if (!nv) { graph_free(&g); return -1; }
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
  for (int64_t r = 0; r < nroots; r++) {
    const int64_t v = roots[r];
    if (v < 0 || v >= n) { free(nv); graph_free(&g); return -1; }
    for (int64_t p = g.rp[v]; p < g.rp[v + 1]; p++) nv[g.adj[p]] = 1;
    uint64_t cnt = 0, steps = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(+:cnt, steps)
    for (int64_t pa = g.rp[v]; pa < g.rp[v + 1]; pa++) {
      const int a = g.adj[pa];
      for (int64_t px = g.rp[a]; px < g.rp[a + 1]; px++) {
        const int x = g.adj[px];
        if (x == v) continue;
        if (cap && steps > cap) break;  /* this thread's share alone is past the cap */
        for (int64_t py = g.rp[x]; py < g.rp[x + 1]; py++) {
          const int y = g.adj[py];
          if (y == v || y == a) continue;
          steps += (uint64_t)(g.rp[y + 1] - g.rp[y]);
          for (int64_t pb = g.rp[y]; pb < g.rp[y + 1]; pb++) {
            const int b = g.adj[pb];
            if (b == v || b == a || b == x) continue;
            cnt += nv[b];
          }
        }
      }
    }
    for (int64_t p = g.rp[v]; p < g.rp[v + 1]; p++) nv[g.adj[p]] = 0;
    status[r] = (cap && steps > cap) ? 1 : 0;
    out[r] = status[r] ? 0 : cnt / 2;
  }
  free(nv);
  graph_free(&g);
  return 0;
}
