// pairs.cuh -- step a7 of SURVEY 8(a): the pair (wedge) pass.
//
// One CTA per source u holds, for every x at distance <= 2, the pair quantities of
// Theorem B.1 (readings R11, R14):
//   W(u,x)  = |N(u) & N(x)|                       (2-hop expansion, phase A)
//   D(u,x)  = #edges inside N(u) & N(x)            (diamond expansion, phase B)
// TT(u,x) = sum_{v in N(u)&N(x)} T(v,x) - W[u~x] (R14) enters theta51 only through
// sum_x TT(u,x)(W-1), which is summed per wedge in phase D once W is final (no table).
// Emits:  C4(u)=DM8, theta36, theta50, theta51, theta63 for u (phase C);
//   E5 = C4(u,v) = sum_{x in N(v)\u} (W(u,x)-1) per edge, and the centre credits
//   theta49(v) += C(W(u,x)-1,2), theta62(v) += D(u,x) for x>u in N(v) (phase D);
//   theta64(v) += sum over diamonds (u; v,w; x), x>u, of W(u,x)-2 (phase E):
//   DM64(v) = sum_{pairs {a,x} in N(v)} |N(v)&N(a)&N(x)| (W(a,x)-2) seen from the pair.
//
// Tables: sources whose 2-hop estimate fits use an open-addressing hash in shared memory
// (on-chip, no DRAM traffic); the others a dense packed u64 (W | D<<32) table per CTA in
// global memory, with the CTA count chosen so the tables stay L2-resident.  All wedge and
// diamond visits are flattened over the CTA by a block prefix sum + binary search
// (load-balanced, coalesced along each adjacency list).
#pragma once
#include <cub/block/block_scan.cuh>
#include "common.cuh"

struct PairOut {
  u64 *R8, *R36, *R50, *R51, *R63, *R49, *R62, *R64, *C4e;
};

__device__ __forceinline__ int64_t slot_of_lo_in_hi(const DGraph& g, int32_t e) { return g.eslot_hi[e]; }
__device__ __forceinline__ int64_t slot_of_hi_in_lo(const DGraph& g, int32_t e) {
  const int32_t a = g.esrc[e];
  return g.rp[a] + g.dm[a] + (e - g.orow[a]);
}

#define PAIR_THREADS 512
#define PAIR_CHUNK 1024          // neighbours of u per prefix-sum chunk
#define PAIR_HASH_CAP 16384      // shared hash entries (keys + W + D = 192 KB)
#define EMPTY_KEY (-1)

// ---- table abstractions ---------------------------------------------------------
struct SharedHashTable {
  int32_t* keys;
  u32* w;
  u32* d;
  u32 mask;
  __device__ __forceinline__ u32 h0(int32_t x) const { return ((u32)x * 0x9E3779B1u) & mask; }
  __device__ __forceinline__ u32 insert(int32_t x) {
    u32 h = h0(x);
    for (;;) {
      const int32_t k = keys[h];
      if (k == x) return h;
      if (k == EMPTY_KEY) {
        const int32_t old = atomicCAS(&keys[h], EMPTY_KEY, x);
        if (old == EMPTY_KEY || old == x) return h;
      }
      h = (h + 1) & mask;
    }
  }
  __device__ __forceinline__ u32 find(int32_t x) const {
    u32 h = h0(x);
    while (keys[h] != x) h = (h + 1) & mask;
    return h;
  }
  __device__ __forceinline__ void add_w(int32_t x) { atomicAdd(&w[insert(x)], 1u); }
  __device__ __forceinline__ void add_d(int32_t x) { atomicAdd(&d[find(x)], 1u); }
  __device__ __forceinline__ void get(int32_t x, u64& wv, u64& dv) const {
    const u32 h = find(x);
    wv = w[h];
    dv = d[h];
  }
  __device__ __forceinline__ u64 get_w(int32_t x) const { return w[find(x)]; }
  // W(u,x) or 0 when x is not at distance 2 (not in the table)
  __device__ __forceinline__ u64 get_w_or0(int32_t x) const {
    u32 h = h0(x);
    for (;;) {
      const int32_t k = keys[h];
      if (k == x) return w[h];
      if (k == EMPTY_KEY) return 0;
      h = (h + 1) & mask;
    }
  }
};

struct GlobalDenseTable {
  u64* t;        // [n] W | D << 32
  int32_t* L;    // touched list
  int* ntouch;   // shared counter
  __device__ __forceinline__ void add_w(int32_t x) {
    const u64 old = atomicAdd(&t[x], 1ull);
    if ((old & 0xffffffffull) == 0) L[atomicAdd(ntouch, 1)] = x;
  }
  __device__ __forceinline__ void add_d(int32_t x) { atomicAdd(&t[x], 1ull << 32); }
  __device__ __forceinline__ void get(int32_t x, u64& wv, u64& dv) const {
    const u64 v = t[x];
    wv = v & 0xffffffffull;
    dv = v >> 32;
  }
  __device__ __forceinline__ u64 get_w(int32_t x) const { return t[x] & 0xffffffffull; }
  __device__ __forceinline__ u64 get_w_or0(int32_t x) const { return t[x] & 0xffffffffull; }
};

// ---- flattened iteration over the slots of N(v), v in N(u) -------------------------
// f(v, s_uv, t) for every slot t of N(v), v = ci[s_uv], s_uv in [r0, r1).
template <typename F>
__device__ __forceinline__ void flat_wedges(const DGraph& g, int64_t r0, int64_t r1, int64_t* pre, F f) {
  typedef cub::BlockScan<int64_t, PAIR_THREADS> Scan;
  __shared__ typename Scan::TempStorage scan_tmp;
  for (int64_t c0 = r0; c0 < r1; c0 += PAIR_CHUNK) {
    const int cn = (int)min((int64_t)PAIR_CHUNK, r1 - c0);
    // each thread owns two entries of the chunk (PAIR_CHUNK = 2 * PAIR_THREADS)
    int64_t a0 = 0, a1 = 0;
    const int i0 = 2 * threadIdx.x, i1 = i0 + 1;
    if (i0 < cn) { const int32_t v = g.ci[c0 + i0]; a0 = g.rp[v + 1] - g.rp[v]; }
    if (i1 < cn) { const int32_t v = g.ci[c0 + i1]; a1 = g.rp[v + 1] - g.rp[v]; }
    int64_t ex, tot;
    Scan(scan_tmp).ExclusiveSum(a0 + a1, ex, tot);
    pre[i0] = ex;
    pre[i1] = ex + a0;
    if (threadIdx.x == 0) pre[PAIR_CHUNK] = tot;
    __syncthreads();
    const int64_t total = pre[PAIR_CHUNK];
    for (int64_t t = threadIdx.x; t < total; t += blockDim.x) {
      // largest k with pre[k] <= t
      int lo = 0, hi = cn;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (pre[mid] <= t) lo = mid; else hi = mid;
      }
      const int64_t s_uv = c0 + lo;
      const int32_t v = g.ci[s_uv];
      f(v, s_uv, g.rp[v] + (t - pre[lo]));
    }
    __syncthreads();
  }
}

// f(v, s_uv, r) for every full-list entry r of edge (u, v), v = ci[s_uv]
template <typename F>
__device__ __forceinline__ void flat_tri(const DGraph& g, const u32* __restrict__ Te, int64_t r0, int64_t r1,
                                         int64_t* pre, F f) {
  typedef cub::BlockScan<int64_t, PAIR_THREADS> Scan;
  __shared__ typename Scan::TempStorage scan_tmp2;
  for (int64_t c0 = r0; c0 < r1; c0 += PAIR_CHUNK) {
    const int cn = (int)min((int64_t)PAIR_CHUNK, r1 - c0);
    int64_t a0 = 0, a1 = 0;
    const int i0 = 2 * threadIdx.x, i1 = i0 + 1;
    if (i0 < cn) a0 = Te[g.eid[c0 + i0]];
    if (i1 < cn) a1 = Te[g.eid[c0 + i1]];
    int64_t ex, tot;
    Scan(scan_tmp2).ExclusiveSum(a0 + a1, ex, tot);
    pre[i0] = ex;
    pre[i1] = ex + a0;
    if (threadIdx.x == 0) pre[PAIR_CHUNK] = tot;
    __syncthreads();
    const int64_t total = pre[PAIR_CHUNK];
    for (int64_t t = threadIdx.x; t < total; t += blockDim.x) {
      int lo = 0, hi = cn;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (pre[mid] <= t) lo = mid; else hi = mid;
      }
      const int64_t s_uv = c0 + lo;
      const int32_t euv = g.eid[s_uv];
      f(g.ci[s_uv], s_uv, g.foff[euv] + (t - pre[lo]));
    }
    __syncthreads();
  }
}

// One source u, table type T.  All threads of the CTA call this together.
template <typename T>
__device__ void pair_source(const DGraph& g, const u32* __restrict__ Te, int32_t u, T& tab, int64_t* pre,
                            u64* red, const PairOut& o) {
  const int64_t r0 = g.rp[u], r1 = g.rp[u + 1];
  // ---- phase A: W(u,x) over all wedges u - v - x
  flat_wedges(g, r0, r1, pre, [&](int32_t v, int64_t s_uv, int64_t t) {
    const int32_t x = g.ci[t];
    if (x != u) tab.add_w(x);
  });
  // ---- phase B: D(u,x) over diamonds (u; v<w; x), chord (v,w) inside N(u)
  flat_tri(g, Te, r0, r1, pre, [&](int32_t v, int64_t s_uv, int64_t r) {
    const int32_t w = g.fx[r];
    if (w <= v) return;
    const int32_t euv = g.eid[s_uv];
    const int32_t evw = (g.esrc[euv] == v) ? g.fe1[r] : g.fe2[r];
    for (int64_t r2 = g.foff[evw]; r2 < g.foff[evw + 1]; r2++) {
      const int32_t x = g.fx[r2];
      if (x != u) tab.add_d(x);
    }
  });
  // ---- phase D (+ theta51 correction over N(u)): per wedge sums
  // E5(u,v), theta49(v), theta62(v) are per-v sums: accumulate in registers while the
  // flattened loop stays inside one v, flush with atomics when v changes.
  u64 s51 = 0;
  {
    int32_t cur_v = -1;
    int64_t cur_s = -1;
    u64 s5 = 0, s49 = 0, s62 = 0;
    auto flush = [&]() {
      if (cur_v < 0) return;
      const int32_t e = g.eid[cur_s];
      if (u < cur_v && s5) atomicAdd(&o.C4e[e], s5);
      if (s49) atomicAdd(&o.R49[cur_v], s49);
      if (s62) atomicAdd(&o.R62[cur_v], s62);
      s5 = s49 = s62 = 0;
    };
    flat_wedges(g, r0, r1, pre, [&](int32_t v, int64_t s_uv, int64_t t) {
      if (v != cur_v) { flush(); cur_v = v; cur_s = s_uv; }
      const int32_t x = g.ci[t];
      if (x == u) return;
      u64 w, d;
      tab.get(x, w, d);
      s5 += w - 1;
      s51 += (u64)Te[g.eid[t]] * (w - 1);
      if (x > u) {
        s49 += binom2(w - 1);
        s62 += d;
      }
    });
    flush();
  }
  for (int64_t s = r0 + threadIdx.x; s < r1; s += blockDim.x) {
    const u64 w = tab.get_w_or0(g.ci[s]);
    s51 -= w * (w - 1);
  }
  // ---- phase E: theta64(v) += W(u,x)-2 over diamonds (u; v, w; x), x > u
  {
    int32_t cur_v = -1;
    u64 acc = 0;
    flat_tri(g, Te, r0, r1, pre, [&](int32_t v, int64_t s_uv, int64_t r) {
      if (v != cur_v) {
        if (cur_v >= 0 && acc) atomicAdd(&o.R64[cur_v], acc);
        cur_v = v;
        acc = 0;
      }
      const int32_t euv = g.eid[s_uv];
      const int32_t evw = (g.esrc[euv] == v) ? g.fe1[r] : g.fe2[r];
      for (int64_t r2 = g.foff[evw]; r2 < g.foff[evw + 1]; r2++) {
        const int32_t x = g.fx[r2];
        if (x > u) acc += tab.get_w(x) - 2ull;
      }
    });
    if (cur_v >= 0 && acc) atomicAdd(&o.R64[cur_v], acc);
  }
  s51 = warp_sum(s51);
  if ((threadIdx.x & 31) == 0 && s51) atomicAdd(&red[3], s51);
}

// phase C contributions of one (x, W, D) pair
__device__ __forceinline__ void pair_c_terms(const DGraph& g, int32_t x, u64 w, u64 d, u64& a8, u64& a36,
                                             u64& a50, u64& a63) {
  const u64 c2 = binom2(w);
  a8 += c2;
  a36 += c2 * (u64)(int64_t)(dg_deg(g, x) - 2);
  a50 += binom3(w);
  a63 += d * (w - 2);
}

__device__ __forceinline__ void pair_flush_u(int32_t u, u64 a8, u64 a36, u64 a50, u64 a63, u64* red,
                                             const PairOut& o) {
  a8 = warp_sum(a8); a36 = warp_sum(a36); a50 = warp_sum(a50); a63 = warp_sum(a63);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&red[0], a8); atomicAdd(&red[1], a36); atomicAdd(&red[2], a50); atomicAdd(&red[4], a63);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    o.R8[u] += red[0]; o.R36[u] += red[1]; o.R50[u] += red[2]; o.R51[u] += red[3]; o.R63[u] += red[4];
    for (int i = 0; i < 5; i++) red[i] = 0;
  }
}

// Sources with a small 2-hop estimate: shared-memory hash, capacity per source.
__global__ void __launch_bounds__(PAIR_THREADS, 1) k_pairs_shared(DGraph g, const u32* __restrict__ Te,
                                                                   const int32_t* __restrict__ srcs,
                                                                   const u32* __restrict__ est, int nsrc,
                                                                   int* __restrict__ counter, PairOut o) {
  extern __shared__ int32_t sh_pairs[];
  __shared__ int64_t pre[PAIR_CHUNK + 1];
  __shared__ u64 red[5];
  __shared__ int s_idx;
  SharedHashTable tab;
  tab.keys = sh_pairs;
  tab.w = (u32*)(sh_pairs + PAIR_HASH_CAP);
  tab.d = tab.w + PAIR_HASH_CAP;
  if (threadIdx.x < 5) red[threadIdx.x] = 0;
  for (;;) {
    if (threadIdx.x == 0) s_idx = atomicAdd(counter, 1);
    __syncthreads();
    const int idx = s_idx;
    if (idx >= nsrc) break;
    const int32_t u = srcs[idx];
    u32 cap = 64;
    while (cap < 2u * est[idx] && cap < PAIR_HASH_CAP) cap <<= 1;
    tab.mask = cap - 1;
    for (u32 h = threadIdx.x; h < cap; h += blockDim.x) { tab.keys[h] = EMPTY_KEY; tab.w[h] = 0; tab.d[h] = 0; }
    __syncthreads();
    pair_source(g, Te, u, tab, pre, red, o);
    __syncthreads();
    u64 a8 = 0, a36 = 0, a50 = 0, a63 = 0;
    for (u32 h = threadIdx.x; h < cap; h += blockDim.x) {
      const int32_t x = tab.keys[h];
      if (x != EMPTY_KEY) pair_c_terms(g, x, tab.w[h], tab.d[h], a8, a36, a50, a63);
    }
    pair_flush_u(u, a8, a36, a50, a63, red, o);
    __syncthreads();
  }
}

// Sources with a large 2-hop set: dense packed table per CTA (L2-sized CTA count).
__global__ void __launch_bounds__(PAIR_THREADS, 1) k_pairs_global(DGraph g, const u32* __restrict__ Te,
                                                                   const int32_t* __restrict__ srcs, int nsrc,
                                                                   int* __restrict__ counter, u64* __restrict__ tabs,
                                                                   int32_t* __restrict__ lists, PairOut o) {
  __shared__ int64_t pre[PAIR_CHUNK + 1];
  __shared__ u64 red[5];
  __shared__ int s_idx, s_ntouch;
  GlobalDenseTable tab;
  tab.t = tabs + (size_t)blockIdx.x * g.n;
  tab.L = lists + (size_t)blockIdx.x * g.n;
  tab.ntouch = &s_ntouch;
  if (threadIdx.x < 5) red[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_ntouch = 0;
  for (;;) {
    if (threadIdx.x == 0) s_idx = atomicAdd(counter, 1);
    __syncthreads();
    const int idx = s_idx;
    if (idx >= nsrc) break;
    const int32_t u = srcs[idx];
    pair_source(g, Te, u, tab, pre, red, o);
    __syncthreads();
    const int nt = s_ntouch;
    u64 a8 = 0, a36 = 0, a50 = 0, a63 = 0;
    for (int i = threadIdx.x; i < nt; i += blockDim.x) {
      const int32_t x = tab.L[i];
      u64 w, d;
      tab.get(x, w, d);
      pair_c_terms(g, x, w, d, a8, a36, a50, a63);
    }
    pair_flush_u(u, a8, a36, a50, a63, red, o);
    for (int i = threadIdx.x; i < nt; i += blockDim.x) tab.t[tab.L[i]] = 0ull;
    if (threadIdx.x == 0) s_ntouch = 0;
    __syncthreads();
  }
}

// 2-hop estimate: est(u) = sum_{v in N(u)} d(v) - d(u) >= #distinct x at distance <= 2
__global__ void k_pair_est(DGraph g, u64* __restrict__ keys, int32_t* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t ui = gw; ui < g.n; ui += nw) {
    const int32_t u = (int32_t)ui;
    u64 s = 0;
    for (int64_t t = g.rp[u] + lane; t < g.rp[u + 1]; t += 32) s += (u64)dg_deg(g, g.ci[t]);
    s = warp_sum(s);
    if (lane == 0) {
      const u64 est = s - (u64)dg_deg(g, u);
      keys[u] = ~est;  // ascending sort = descending estimate
      vals[u] = u;
    }
  }
}

// shard filter of the sorted list + estimate per position
__global__ void k_pair_lists(const u64* __restrict__ skeys, const int32_t* __restrict__ svals, int32_t n,
                             int si, int ns, int32_t* __restrict__ list, u32* __restrict__ est) {
  for (int32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    if (p % ns == si) {
      const u64 e = ~skeys[p];
      list[p / ns] = svals[p];
      est[p / ns] = (u32)min(e, (u64)0xffffffffu);
    }
}
