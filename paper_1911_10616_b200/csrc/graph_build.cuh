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
  int cnt[3];
  int minv;
  int level;
  int rounds;
  int rounds1;  // rounds of the grid-wide phase
  int nalive;
  unsigned long long t0, t1, t2;  // %globaltimer at start, at the phase switch, at the end
};

#define PEEL_BT 1024           // threads per CTA
#define PEEL_SWITCH 8192       // vertices left at or below which one CTA finishes the peel locally
#define PEEL_CLUSTER 16        // CTAs of the cluster variant (non-portable cluster size)
#define PEEL_CLUSTER_MAXN (1 << 18)  // graphs up to this many vertices use the cluster variant
// shared bytes per local vertex of phase 2: ldeg, lrnd (int32), lbeg (u32), lcnt, two frontier
// lists (u16)
#define PEEL_LOCAL_BYTES 20

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Round r removes the frontier L_r: alive vertices whose current degree is <= k (the current
// core level).  A vertex is stamped rnd = r when it joins L_r, so one barrier per round
// suffices: while L_r is walked, every neighbour w not yet stamped loses one degree, and the
// one decrement that takes d(w) from k+1 to k stamps w with r+1 and appends it to L_{r+1}
// (decrements of stamped vertices are skipped; their degree no longer matters).  When a
// frontier is empty the level rises to the minimum degree of the unstamped vertices, which
// are stamped as the next frontier if their degree is <= that level.  The three frontier
// counters rotate (read r, append r+1, reset r+2) so no counter is reset while it is read.
// Phase 1 runs the rounds over the whole grid while many vertices are alive.  Once at most
// peel_switch (<= PEEL_SWITCH) vertices are left (unstamped, or stamped for the pending
// round), the grid gives them local ids and copies the subgraph they induce into ladj
// (local ids, at the vertices' own CSR positions); block 0 then finishes with every per-vertex
// state in shared memory and block barriers: the late rounds touch few vertices each, so the
// grid-wide barrier and the dependent L2 round trips of a global round would dominate.  The
// result -- rnd, hence the order (rnd, id) -- is the same in both phases and for any grid
// size: the set L_{r+1} is fixed by the degrees, not by the schedule.
// CLUSTER: the whole grid is one thread-block cluster and the barriers between rounds are
// hardware cluster barriers (cheaper than a cooperative grid barrier); used when the graph is
// small enough for one cluster.
template <bool CLUSTER>
__global__ void __launch_bounds__(PEEL_BT) k_peel(int32_t n, const int64_t* __restrict__ rp,
                                                  const int32_t* __restrict__ adj, int32_t* __restrict__ deg,
                                                  int32_t* __restrict__ rnd, int32_t* __restrict__ list0,
                                                  int32_t* __restrict__ list1, int32_t* __restrict__ lidmap,
                                                  int32_t* __restrict__ loc, int32_t* __restrict__ lcnt,
                                                  uint16_t* __restrict__ ladj, PeelCtl* ctl, int peel_switch) {
  struct Sync {
    __device__ __forceinline__ void sync() const {
      if (CLUSTER) cg::this_cluster().sync();
      else cg::this_grid().sync();
    }
  } grid;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const int warp = (int)(tid >> 5), nwarps = (int)(nthreads >> 5), lane = threadIdx.x & 31;
  int k = 0, round = 0, p = 0, removed = 0;
  // (selects instead of an array indexed by p: a dynamically indexed local array lives in
  // local memory)
  auto lists = [&](int q) { return q ? list1 : list0; };
  for (int32_t v = tid; v < n; v += nthreads) { rnd[v] = -1; lidmap[v] = -1; }
  if (tid == 0) {
    ctl->cnt[0] = 0; ctl->cnt[1] = 0; ctl->cnt[2] = 0; ctl->minv = 0x7fffffff; ctl->nalive = 0;
    ctl->t0 = globaltimer();
  }
  grid.sync();
  // ---- phase 1: grid-wide rounds, one barrier each
  while (n - removed > peel_switch) {
    const int c = round % 3, c1 = (round + 1) % 3, c2 = (round + 2) % 3;
    int cur = *(volatile int*)&ctl->cnt[c];
    if (cur == 0) {
      for (int32_t v = tid; v < n; v += nthreads)
        if (rnd[v] < 0) atomicMin(&ctl->minv, deg[v]);
      grid.sync();
      const int mv = *(volatile int*)&ctl->minv;
      if (mv > k) k = mv;
      for (int32_t v = tid; v < n; v += nthreads)
        if (rnd[v] < 0 && deg[v] <= k) {
          rnd[v] = round;
          lists(p)[atomicAdd(&ctl->cnt[c], 1)] = v;
        }
      grid.sync();
      cur = *(volatile int*)&ctl->cnt[c];
      if (tid == 0) ctl->minv = 0x7fffffff;  // read again only after the next round's barrier
    }
    if (tid == 0) ctl->cnt[c2] = 0;
    const int32_t* L = lists(p);
    int32_t* Ln = lists(p ^ 1);
    // `per` frontier vertices per warp step (up to 32, as many as keep every warp busy), their
    // (vertex, neighbour) pairs flattened over the lanes: a warp per vertex left most lanes
    // idle on the large degree-8 frontiers of config 4's first rounds, while a small frontier
    // needs a warp per vertex to spread its lists
    const int per = max(1, min(32, cur / nwarps));
    for (int i0 = warp * per; i0 < cur; i0 += nwarps * per) {
      int64_t b0 = 0;
      int len = 0;
      if (lane < per && i0 + lane < cur) {
        const int32_t v = L[i0 + lane];
        b0 = rp[v];
        len = (int)(rp[v + 1] - b0);
      }
      warp_flat(len, [&](int j, int kk, bool valid) {
        const int64_t bj = __shfl_sync(FULL_MASK, b0, j);
        bool hit = false;
        int32_t w = 0;
        if (valid) {
          // no stamp test first: a stamped vertex had degree <= k when stamped and k only
          // grows, so its decrement can never return k + 1 (one dependent load less per round)
          w = adj[bj + kk];
          hit = atomicSub(&deg[w], 1) == k + 1;
          if (hit) rnd[w] = round + 1;
        }
        warp_append(hit, w, Ln, &ctl->cnt[c1]);
      });
    }
    removed += cur;
    round++;
    grid.sync();
    p ^= 1;
  }
  if (tid == 0) { ctl->rounds1 = round; ctl->t1 = globaltimer(); }
  if (removed >= n) {
    if (tid == 0) { ctl->level = k; ctl->rounds = round; ctl->t2 = ctl->t1; }
    return;
  }
  // ---- switch: local ids for the vertices left (unstamped, or stamped for the pending round)
  for (int32_t v = tid; v < n; v += nthreads) {
    const int r = rnd[v];
    if (r < 0 || r == round) {
      const int l = atomicAdd(&ctl->nalive, 1);
      loc[l] = v;
      lidmap[v] = l;
    }
  }
  grid.sync();
  const int S = *(volatile int*)&ctl->nalive;
  // the induced subgraph in local ids, ladj[rp[v] + j] for j < lcnt[l] (warp per vertex,
  // ballot compaction keeps the neighbours in CSR order)
  for (int l = warp; l < S; l += nwarps) {
    const int32_t v = loc[l];
    const int64_t b = rp[v], e = rp[v + 1];
    int cnt = 0;
    for (int64_t s0 = b; s0 < e; s0 += 32) {
      const int64_t s = s0 + lane;
      const int lw = s < e ? lidmap[adj[s]] : -1;
      const unsigned bal = __ballot_sync(FULL_MASK, lw >= 0);
      if (lw >= 0) ladj[b + cnt + __popc(bal & ((1u << lane) - 1))] = (uint16_t)lw;
      cnt += __popc(bal);
    }
    if (lane == 0) lcnt[l] = cnt;
  }
  grid.sync();
  if (blockIdx.x != 0) return;
  // ---- phase 2: block 0, per-vertex state in shared memory
  extern __shared__ int32_t peel_sh[];
  int32_t* ldeg = peel_sh;                                   // current degree
  int32_t* lrnd = ldeg + peel_switch;                        // round, -1 = unstamped
  u32* lbeg = (u32*)(lrnd + peel_switch);                    // CSR position (2m < 2^31)
  uint16_t* lc = (uint16_t*)(lbeg + peel_switch);            // local degree at the switch
  uint16_t* lq0 = lc + peel_switch;
  uint16_t* lq1 = lq0 + peel_switch;
  auto lq = [&](int q) { return q ? lq1 : lq0; };
  __shared__ int s_cnt[3], s_minv;
  if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_minv = 0x7fffffff;
  __syncthreads();
  const int c0 = round % 3;
  for (int l = threadIdx.x; l < S; l += PEEL_BT) {
    const int32_t v = loc[l];
    const int r = rnd[v];
    ldeg[l] = lcnt[l];
    lc[l] = (uint16_t)lcnt[l];
    lbeg[l] = (u32)rp[v];
    lrnd[l] = r;
    if (r >= 0) lq(p)[atomicAdd(&s_cnt[c0], 1)] = (uint16_t)l;  // the pending frontier
  }
  __syncthreads();
  const int removed0 = removed;
  while (removed - removed0 < S) {
    const int c = round % 3, c1 = (round + 1) % 3, c2 = (round + 2) % 3;
    int cur = s_cnt[c];
    if (cur == 0) {
      for (int l = threadIdx.x; l < S; l += PEEL_BT)
        if (lrnd[l] < 0) atomicMin(&s_minv, ldeg[l]);
      __syncthreads();
      if (s_minv > k) k = s_minv;
      for (int l = threadIdx.x; l < S; l += PEEL_BT)
        if (lrnd[l] < 0 && ldeg[l] <= k) {
          lrnd[l] = round;
          lq(p)[atomicAdd(&s_cnt[c], 1)] = (uint16_t)l;
        }
      __syncthreads();
      cur = s_cnt[c];
      __syncthreads();
      if (threadIdx.x == 0) s_minv = 0x7fffffff;
    }
    if (threadIdx.x == 0) s_cnt[c2] = 0;
    const uint16_t* L = lq(p);
    uint16_t* Ln = lq(p ^ 1);
    // a warp per frontier vertex, its local list over the lanes (no scan or search: one
    // barrier per round)
    const int wl = threadIdx.x >> 5, ln = threadIdx.x & 31;
    for (int f = wl; f < cur; f += PEEL_BT / 32) {
      const int l = L[f];
      const u32 b0 = lbeg[l];
      const int len = lc[l];
      for (int t = ln; t < len; t += 32) {
        const int w = ladj[b0 + (u32)t];
        const int old = atomicSub(&ldeg[w], 1);  // stamped w: old <= k (see phase 1)
        if (old == k + 1) {
          lrnd[w] = round + 1;
          Ln[atomicAdd(&s_cnt[c1], 1)] = (uint16_t)w;
        }
      }
    }
    __syncthreads();
    removed += cur;
    round++;
    p ^= 1;
  }
  for (int l = threadIdx.x; l < S; l += PEEL_BT) rnd[loc[l]] = lrnd[l];
  if (threadIdx.x == 0) { ctl->level = k; ctl->rounds = round; ctl->t2 = globaltimer(); }
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
// directed keys (x << kb) | y in new ids, kb = bits(n): 2 kb key bits instead of 32 + kb (one
// radix pass less on config 4's 32 M keys)
__global__ void k_relabel_keys(const u64* __restrict__ keys, int64_t m, const int32_t* __restrict__ inv,
                               u64* __restrict__ dk, int kb) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    u64 k = keys[e];
    u32 a = (u32)inv[(int32_t)(k >> 32)], b = (u32)inv[(int32_t)(k & 0xffffffffu)];
    dk[2 * e] = ((u64)a << kb) | b;
    dk[2 * e + 1] = ((u64)b << kb) | a;
  }
}

// (degrees from the sorted keys: the slot that ends a run of equal rows writes its length,
// found by a search back to the run's start -- no atomics on the rows' counters)
__global__ void k_split_keys(const u64* __restrict__ dk, int64_t m2, int32_t* __restrict__ ci,
                             int32_t* __restrict__ degc, int kb) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m2;
       s += (int64_t)gridDim.x * blockDim.x) {
    const u64 k = dk[s];
    ci[s] = (int32_t)(k & ((1ull << kb) - 1));
    const u64 row = k >> kb;
    if (s + 1 == m2 || (dk[s + 1] >> kb) != row) {  // last slot of its row
      // first slot of the row: gallop back from s, then bisect (O(log d) loads)
      int64_t hi = s, step = 1, lo = s - 1;
      while (lo >= 0 && (dk[lo] >> kb) == row) {
        hi = lo;
        lo = s - (step <<= 1);
      }
      lo = lo < 0 ? 0 : lo + 1;  // dk[lo - 1] (if any) belongs to an earlier row; dk[hi] to this one
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((dk[mid] >> kb) < row) lo = mid + 1; else hi = mid;
      }
      degc[(int32_t)row] = (int32_t)(s - lo + 1);
    }
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
                              int32_t* __restrict__ edst, int64_t* __restrict__ eslot_hi,
                              int32_t* __restrict__ twin, int kb) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m2;
       s += (int64_t)gridDim.x * blockDim.x) {
    int32_t u = (int32_t)(dk[s] >> kb);
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
      twin[s] = (int32_t)pos;  // (the other slot's twin: k_twin_hi, once eslot_hi is complete)
    }
  }
}
// twin of the slots of higher neighbours: the slot of u in N(w), w > u, is eslot_hi[e(u,w)]
// (a gather along u's out-part, coalesced, instead of a scattered write above)
__global__ void k_twin_hi(int32_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ dm,
                          const int64_t* __restrict__ orow, const int64_t* __restrict__ eslot_hi,
                          const int32_t* __restrict__ eid, int64_t m2, const u64* __restrict__ dk,
                          int32_t* __restrict__ twin, int kb) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m2; s += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = (int32_t)(dk[s] >> kb);
    if (s >= rp[u] + dm[u]) twin[s] = (int32_t)eslot_hi[eid[s]];
  }
}

// out8 rows (DGraph::out8): one 32-byte row per vertex holding a short out-list
__global__ void k_out8(int32_t n, const int64_t* __restrict__ orow, const int32_t* __restrict__ ocol,
                       int4* __restrict__ out8) {
  for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const int64_t b = orow[j];
    const int d = (int)(orow[j + 1] - b);
    int r[OUT8];
#pragma unroll
    for (int t = 0; t < OUT8; t++) r[t] = t < d ? ocol[b + t] : -1;
    if (d > OUT8) r[0] = OUT8_LONG;
    out8[2 * (size_t)j] = make_int4(r[0], r[1], r[2], r[3]);
    out8[2 * (size_t)j + 1] = make_int4(r[4], r[5], r[6], r[7]);
  }
}
