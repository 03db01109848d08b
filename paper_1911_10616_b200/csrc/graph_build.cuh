// graph_build.cuh -- step a1-a3 of SURVEY 8(a): canonicalise the input (drop
// direction, duplicates, self-loops), degeneracy order by k-core peeling (orientation
// G-> of P:432-437 with the north star's degeneracy rank), relabel vertices by rank and
// build the undirected CSR (sorted) plus the oriented edge arrays.
#pragma once
#include <cooperative_groups.h>
#include "common.cuh"
#include "sched.cuh"

namespace cg = cooperative_groups;

// ---- a1: canonical keys -----------------------------------------------------
// key = (min << 32) | max for every non-loop pair, UINT64_MAX for self-loops; sets
// *bad if an id is outside [0,n).
__global__ void k_make_keys(const int32_t* __restrict__ edges, int64_t m, int32_t n,
                            u64* __restrict__ keys, int* bad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    int32_t a = edges[2 * e], b = edges[2 * e + 1];
    if (a < 0 || b < 0 || a >= n || b >= n) { *bad = 1; keys[e] = ~0ull; continue; }
    if (a == b) { keys[e] = ~0ull; continue; }
    u32 lo = (u32)min(a, b), hi = (u32)max(a, b);
    keys[e] = ((u64)lo << 32) | hi;
  }
}

// CSR input -> keys (row v, col[k])
__global__ void k_make_keys_csr(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                int32_t n, u64* __restrict__ keys, int* bad) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    for (int64_t k = rowptr[v]; k < rowptr[v + 1]; k++) {
      int32_t b = col[k];
      if (b < 0 || b >= n) { *bad = 1; keys[k] = ~0ull; continue; }
      if (b == v) { keys[k] = ~0ull; continue; }
      u32 lo = (u32)min(v, b), hi = (u32)max(v, b);
      keys[k] = ((u64)lo << 32) | hi;
    }
  }
}

__global__ void k_check_rowptr(const int64_t* __restrict__ rowptr, int32_t n, int* bad) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    if (rowptr[v + 1] < rowptr[v]) *bad = 1;
  if (blockIdx.x == 0 && threadIdx.x == 0 && rowptr[0] != 0) *bad = 1;
}

// degrees of the cleaned graph in original ids; keys[0..m) unique, valid
__global__ void k_degrees(const u64* __restrict__ keys, int64_t m, int32_t* __restrict__ deg) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    u64 k = keys[e];
    atomicAdd(&deg[(int32_t)(k >> 32)], 1);
    atomicAdd(&deg[(int32_t)(k & 0xffffffffu)], 1);
  }
}

// unsorted adjacency (original ids) for peeling
__global__ void k_fill_adj0(const u64* __restrict__ keys, int64_t m, int64_t* __restrict__ cursor,
                            int32_t* __restrict__ adj) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    u64 k = keys[e];
    int32_t a = (int32_t)(k >> 32), b = (int32_t)(k & 0xffffffffu);
    adj[atomicAdd((unsigned long long*)&cursor[a], 1ull)] = b;
    adj[atomicAdd((unsigned long long*)&cursor[b], 1ull)] = a;
  }
}

// ---- a2: k-core peeling (cooperative, grid-synchronised rounds) ---------------
// Round r removes every alive vertex whose current degree is <= k (the current core
// level); rnd[v] = r.  When no such vertex exists the level rises to the minimum alive
// degree.  The total order (rnd, id) is a degeneracy order: every vertex has at most
// k_max = degeneracy later neighbours (reading R19).
struct PeelCtl {
  int cnt[2];
  int minv;
  int level;
  int rounds;
  int nalive;
};

#define PEEL_BT 1024           // threads per CTA
#define PEEL_SWITCH 2048       // alive vertices at or below which one CTA finishes the peel
#define PEEL_GRID 64           // CTAs of the grid-wide phase (cheaper grid barriers; rounds are small)
#define PEEL_CLUSTER 16        // CTAs of the cluster variant (non-portable cluster size)
#define PEEL_CLUSTER_MAXN (1 << 18)  // graphs up to this many vertices use the cluster variant

// Rounds of the peel are identical in both phases: the frontier L[p] (alive vertices of
// current degree <= k) gets rnd = round, their alive neighbours lose one degree each, and
// a neighbour whose degree drops to exactly k joins the next frontier.  When a frontier is
// empty the level rises to the minimum alive degree.  Phase 1 runs the rounds over the
// whole grid (grid.sync between steps) while many vertices are alive; once at most
// PEEL_SWITCH remain, they are compacted into a list and block 0 finishes alone with
// block barriers (each late round touches few vertices, so a grid-wide barrier per round
// would dominate).
// CLUSTER: the whole grid is one thread-block cluster and the barriers between rounds are
// hardware cluster barriers (cheaper than a cooperative grid barrier); used when the graph is
// small enough for one cluster.
template <bool CLUSTER>
__global__ void __launch_bounds__(PEEL_BT) k_peel(int32_t n, const int64_t* __restrict__ rp,
                                                  const int32_t* __restrict__ adj, int32_t* __restrict__ deg,
                                                  int32_t* __restrict__ rnd, int32_t* __restrict__ list0,
                                                  int32_t* __restrict__ list1, int32_t* __restrict__ alive0,
                                                  int32_t* __restrict__ alive1, PeelCtl* ctl, int peel_switch) {
  struct Sync {
    __device__ __forceinline__ void sync() const {
      if (CLUSTER) cg::this_cluster().sync();
      else cg::this_grid().sync();
    }
  } grid;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const int warp = (int)(tid >> 5), nwarps = (int)(nthreads >> 5), lane = threadIdx.x & 31;
  int32_t* lists[2] = {list0, list1};
  int k = 0, round = 0, p = 0, removed = 0;
  for (int32_t v = tid; v < n; v += nthreads) rnd[v] = -1;
  if (tid == 0) { ctl->cnt[0] = 0; ctl->cnt[1] = 0; ctl->minv = 0x7fffffff; ctl->nalive = 0; }
  grid.sync();
  // ---- phase 1: grid-wide rounds
  while (n - removed > peel_switch) {
    int cur = *(volatile int*)&ctl->cnt[p];
    if (cur == 0) {
      for (int32_t v = tid; v < n; v += nthreads)
        if (rnd[v] < 0) atomicMin(&ctl->minv, deg[v]);
      grid.sync();
      int mv = *(volatile int*)&ctl->minv;
      if (mv > k) k = mv;
      for (int32_t v = tid; v < n; v += nthreads)
        if (rnd[v] < 0 && deg[v] <= k) lists[p][atomicAdd(&ctl->cnt[p], 1)] = v;
      grid.sync();
      cur = *(volatile int*)&ctl->cnt[p];
      if (tid == 0) ctl->minv = 0x7fffffff;
    }
    int32_t* L = lists[p];
    for (int64_t i = tid; i < cur; i += nthreads) rnd[L[i]] = round;
    if (tid == 0) ctl->cnt[p ^ 1] = 0;
    grid.sync();
    for (int i = warp; i < cur; i += nwarps) {
      int32_t v = L[i];
      for (int64_t s = rp[v] + lane; s < rp[v + 1]; s += 32) {
        int32_t w = adj[s];
        if (rnd[w] < 0) {
          int old = atomicSub(&deg[w], 1);
          if (old == k + 1) lists[p ^ 1][atomicAdd(&ctl->cnt[p ^ 1], 1)] = w;
        }
      }
    }
    removed += cur;
    round++;
    grid.sync();
    p ^= 1;
  }
  if (removed >= n) {
    if (tid == 0) { ctl->level = k; ctl->rounds = round; }
    return;
  }
  // compact the alive vertices (the pending frontier L[p] stays as it is)
  for (int32_t v = tid; v < n; v += nthreads)
    if (rnd[v] < 0) alive0[atomicAdd(&ctl->nalive, 1)] = v;
  grid.sync();
  if (blockIdx.x != 0) return;
  // ---- phase 2: one CTA
  __shared__ int s_cnt[2], s_minv, s_na;
  int32_t* al[2] = {alive0, alive1};
  int ap = 0;
  int nalive = *(volatile int*)&ctl->nalive;
  if (threadIdx.x == 0) { s_cnt[p] = *(volatile int*)&ctl->cnt[p]; s_cnt[p ^ 1] = 0; s_minv = 0x7fffffff; s_na = 0; }
  __syncthreads();
  const int bw = threadIdx.x >> 5, nbw = PEEL_BT / 32;
  while (removed < n) {
    int cur = s_cnt[p];
    if (cur == 0) {
      // level up: minimum alive degree, compacting the alive list on the way
      for (int i = threadIdx.x; i < nalive; i += PEEL_BT) {
        const int32_t v = al[ap][i];
        if (rnd[v] < 0) {
          atomicMin(&s_minv, deg[v]);
          al[ap ^ 1][atomicAdd(&s_na, 1)] = v;
        }
      }
      __syncthreads();
      ap ^= 1;
      nalive = s_na;
      if (s_minv > k) k = s_minv;
      for (int i = threadIdx.x; i < nalive; i += PEEL_BT) {
        const int32_t v = al[ap][i];
        if (deg[v] <= k) lists[p][atomicAdd(&s_cnt[p], 1)] = v;
      }
      __syncthreads();
      cur = s_cnt[p];
      __syncthreads();
      if (threadIdx.x == 0) { s_minv = 0x7fffffff; s_na = 0; }
    }
    int32_t* L = lists[p];
    for (int i = threadIdx.x; i < cur; i += PEEL_BT) rnd[L[i]] = round;
    if (threadIdx.x == 0) s_cnt[p ^ 1] = 0;
    __syncthreads();
    // the adjacency lists of the frontier flattened over the whole CTA: late rounds remove
    // a few hubs with long lists, which a warp per vertex would walk alone
    __shared__ int64_t s_pre[PEEL_BT + 1];
    __shared__ int64_t s_base[PEEL_BT];
    block_flat<PEEL_BT>(cur, s_pre,
        [&](int64_t i) -> int64_t {
          const int32_t v = L[i];
          s_base[threadIdx.x] = rp[v];
          return rp[v + 1] - rp[v];
        },
        [&](int li, int64_t kk) {
          const int32_t w = adj[s_base[li] + kk];
          if (rnd[w] < 0) {
            const int old = atomicSub(&deg[w], 1);
            if (old == k + 1) lists[p ^ 1][atomicAdd(&s_cnt[p ^ 1], 1)] = w;
          }
        },
        [&](int64_t, int) {});
    (void)bw; (void)nbw;
    removed += cur;
    round++;
    __syncthreads();
    p ^= 1;
  }
  if (threadIdx.x == 0) { ctl->level = k; ctl->rounds = round; }
}

// order keys: (round << 32) | id
__global__ void k_order_keys(const int32_t* __restrict__ rnd, int32_t n, u64* __restrict__ keys) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    keys[v] = ((u64)(u32)rnd[v] << 32) | (u32)v;
}

// perm[new] = old, inv[old] = new
__global__ void k_perm(const u64* __restrict__ sorted, int32_t n, int32_t* __restrict__ perm,
                       int32_t* __restrict__ inv) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int32_t old = (int32_t)(sorted[i] & 0xffffffffu);
    perm[i] = old;
    inv[old] = i;
  }
}

// ---- a3: relabelled directed keys, both directions ---------------------------
__global__ void k_relabel_keys(const u64* __restrict__ keys, int64_t m, const int32_t* __restrict__ inv,
                               u64* __restrict__ dk) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    u64 k = keys[e];
    u32 a = (u32)inv[(int32_t)(k >> 32)], b = (u32)inv[(int32_t)(k & 0xffffffffu)];
    dk[2 * e] = ((u64)a << 32) | b;
    dk[2 * e + 1] = ((u64)b << 32) | a;
  }
}

__global__ void k_split_keys(const u64* __restrict__ dk, int64_t m2, int32_t* __restrict__ ci,
                             int32_t* __restrict__ degc) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m2;
       s += (int64_t)gridDim.x * blockDim.x) {
    u64 k = dk[s];
    ci[s] = (int32_t)(k & 0xffffffffu);
    atomicAdd(&degc[(int32_t)(k >> 32)], 1);
  }
}

// dm[u] = number of neighbours < u; dplus[u] = d(u) - dm[u]
__global__ void k_split_counts(int32_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                               int32_t* __restrict__ dm, int64_t* __restrict__ dplus, int32_t* __restrict__ deg) {
  for (int32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
    int64_t lo = lower_bound_dev<int32_t>(ci, rp[u], rp[u + 1], u);
    dm[u] = (int32_t)(lo - rp[u]);
    dplus[u] = rp[u + 1] - lo;
    deg[u] = (int32_t)(rp[u + 1] - rp[u]);
  }
}

// per-slot edge ids, oriented arrays.  src of slot s = high half of the sorted key.
__global__ void k_edge_arrays(const u64* __restrict__ dk, int64_t m2, const int64_t* __restrict__ rp,
                              const int32_t* __restrict__ ci, const int32_t* __restrict__ dm,
                              const int64_t* __restrict__ orow, int32_t* __restrict__ eid,
                              int32_t* __restrict__ ocol, int32_t* __restrict__ esrc,
                              int32_t* __restrict__ edst, int64_t* __restrict__ eslot_hi) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m2;
       s += (int64_t)gridDim.x * blockDim.x) {
    int32_t u = (int32_t)(dk[s] >> 32);
    int32_t w = ci[s];
    if (w > u) {
      int64_t e = orow[u] + (s - rp[u] - dm[u]);
      eid[s] = (int32_t)e;
      ocol[e] = w;
      esrc[e] = u;
      edst[e] = w;
    } else {
      int64_t lo = rp[w] + dm[w];
      int64_t pos = lower_bound_dev<int32_t>(ci, lo, rp[w + 1], u);
      int64_t e = orow[w] + (pos - lo);
      eid[s] = (int32_t)e;
      eslot_hi[e] = s;
    }
  }
}
