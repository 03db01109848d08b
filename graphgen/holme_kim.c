/* Holme-Kim power-law cluster graph generator (Holme & Kim 2002: preferential
 * attachment with triad formation).  Input generation only: no orbit-counting
 * arithmetic lives here.  Deterministic for a given seed (splitmix64 stream).
 *
 * Each new vertex s attaches m edges: the first by preferential attachment
 * (uniform pick from the degree-weighted multiset), each further one with
 * probability p as a triad-formation step (a random neighbour of the last
 * preferential target that is not yet adjacent to s), otherwise by another
 * preferential-attachment pick.  Starts from m isolated vertices.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static uint64_t sm_state;
static inline uint64_t sm_next(void) {
  uint64_t z = (sm_state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static inline double sm_unif(void) { return (double)(sm_next() >> 11) * (1.0 / 9007199254740992.0); }
static inline uint64_t sm_below(uint64_t n) { return sm_next() % n; }

typedef struct { int32_t *v; int32_t n, cap; } vec_t;
static void vpush(vec_t *a, int32_t x) {
  if (a->n == a->cap) { a->cap = a->cap ? 2 * a->cap : 8; a->v = (int32_t *)realloc(a->v, sizeof(int32_t) * a->cap); }
  a->v[a->n++] = x;
}
static int vhas(const vec_t *a, int32_t x) { for (int i = 0; i < a->n; i++) if (a->v[i] == x) return 1; return 0; }

/* writes up to (n-m)*m edges into edges[2*k]; returns the number written */
int64_t holme_kim(int64_t n, int m, double p, uint64_t seed, int32_t *edges) {
  sm_state = seed * 0x2545F4914F6CDD1Dull + 12345;
  vec_t *adj = (vec_t *)calloc((size_t)n, sizeof(vec_t));
  int64_t rep_cap = 2 * (n * (int64_t)m + m) + 16, rep_n = 0;
  int32_t *rep = (int32_t *)malloc(sizeof(int32_t) * (size_t)rep_cap);
  for (int i = 0; i < m; i++) rep[rep_n++] = i;
  int64_t ne = 0;
  int32_t *targets = (int32_t *)malloc(sizeof(int32_t) * (size_t)m);
  for (int64_t s = m; s < n; s++) {
    /* m distinct targets sampled from the repeated-nodes multiset */
    int nt = 0;
    while (nt < m) {
      int32_t x = rep[sm_below((uint64_t)rep_n)];
      int dup = 0;
      for (int i = 0; i < nt; i++) if (targets[i] == x) { dup = 1; break; }
      if (!dup) targets[nt++] = x;
    }
    int32_t target = targets[--nt];
    vpush(&adj[s], target); vpush(&adj[target], (int32_t)s);
    edges[2 * ne] = (int32_t)s; edges[2 * ne + 1] = target; ne++;
    rep[rep_n++] = target;
    int count = 1;
    while (count < m) {
      if (sm_unif() < p) {
        /* triad formation: neighbours of target not adjacent to s */
        vec_t *nb = &adj[target];
        int cand = 0;
        for (int i = 0; i < nb->n; i++) if (nb->v[i] != s && !vhas(&adj[s], nb->v[i])) cand++;
        if (cand > 0) {
          int pick = (int)sm_below((uint64_t)cand), seen = 0;
          int32_t nbr = -1;
          for (int i = 0; i < nb->n; i++) {
            if (nb->v[i] != s && !vhas(&adj[s], nb->v[i])) { if (seen == pick) { nbr = nb->v[i]; break; } seen++; }
          }
          vpush(&adj[s], nbr); vpush(&adj[nbr], (int32_t)s);
          edges[2 * ne] = (int32_t)s; edges[2 * ne + 1] = nbr; ne++;
          rep[rep_n++] = nbr;
          count++;
          continue;
        }
      }
      if (nt == 0) break;
      target = targets[--nt];
      if (!vhas(&adj[s], target)) {
        vpush(&adj[s], target); vpush(&adj[target], (int32_t)s);
        edges[2 * ne] = (int32_t)s; edges[2 * ne + 1] = target; ne++;
      }
      rep[rep_n++] = target;
      count++;
    }
    for (int i = 0; i < m; i++) rep[rep_n++] = (int32_t)s;
  }
  for (int64_t i = 0; i < n; i++) free(adj[i].v);
  free(adj); free(rep); free(targets);
  return ne;
}
