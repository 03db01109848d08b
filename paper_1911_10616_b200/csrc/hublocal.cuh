// hublocal.cuh -- step a8 of SURVEY 8(a): the hub-local (diamond) pass for the wheel W4
// = H27 (theta68, theta69; Theorem B.1, readings R11, R13).
//
// Work item = ordered pair (v, a), a in N(v), T(v,a) >= 2.  A warp enumerates
//   b in N(v)&N(a) (full triangle list of edge (v,a)) and x in N(v)&N(b), x != a,
// i.e. c_v(a,x) = |N(v)&N(a)&N(x)| for every x in N(v), in a warp-private table
// indexed by x's position inside N(v).  Then
//   theta68(a) += sum_x C(c_v(a,x), 2)     (a rim vertex, v the hub, x the opposite rim)
//   theta69(v) += sum_x C(c'_v(a,x), 2)    where c' counts only b < a and x < a, i.e.
// every 4-cycle of G[N(v)] is counted once, by its maximum vertex a and its opposite x
// (this replaces the printed 1/2 of R13 without any division modulo 2^64).
#pragma once
#include "common.cuh"

__global__ void __launch_bounds__(256) k_hublocal(DGraph g, const u32* __restrict__ Te,
                                                  int* __restrict__ counter, int chunk,
                                                  int shard_index, int num_shards,
                                                  u64* __restrict__ tabs, int32_t* __restrict__ lists,
                                                  u64* __restrict__ R68, u64* __restrict__ R69) {
  __shared__ int s_cnt[8];
  __shared__ int64_t s_base[8];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  u64* tab = tabs + gw * (int64_t)g.max_deg;
  int32_t* L = lists + gw * (int64_t)g.max_deg;
  const int64_t nslots = 2 * g.m;
  if (lane == 0) s_cnt[wib] = 0;
  __syncwarp();
  for (;;) {
    if (lane == 0) s_base[wib] = (int64_t)atomicAdd(counter, 1) * chunk;
    __syncwarp();
    const int64_t base = s_base[wib];
    if (base >= nslots) break;
    const int64_t end = min(base + (int64_t)chunk, nslots);
    // vertex owning slot `base`
    int64_t lo = 0, hi = g.n;  // find v with rp[v] <= base < rp[v+1]
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (g.rp[mid] <= base) lo = mid; else hi = mid;
    }
    int32_t v = (int32_t)lo;
    for (int64_t s = base; s < end; s++) {
      while (g.rp[v + 1] <= s) v++;
      if ((v % num_shards) != shard_index) continue;
      const int32_t eva = g.eid[s];
      if (Te[eva] < 2) continue;
      const int32_t a = g.ci[s];
      const bool v_lo = g.esrc[eva] == v;
      const int64_t rpv = g.rp[v];
      for (int64_t r = g.foff[eva]; r < g.foff[eva + 1]; r++) {
        const int32_t b = g.fx[r];
        const int32_t evb = v_lo ? g.fe1[r] : g.fe2[r];
        const bool v_lo_b = g.esrc[evb] == v;
        for (int64_t r2 = g.foff[evb] + lane; r2 < g.foff[evb + 1]; r2 += 32) {
          const int32_t x = g.fx[r2];
          if (x == a) continue;
          const int32_t evx = v_lo_b ? g.fe1[r2] : g.fe2[r2];
          const int64_t p = (v < x) ? ((int64_t)g.dm[v] + (evx - g.orow[v])) : (g.eslot_hi[evx] - rpv);
          const u64 inc = 1ull + ((b < a && x < a) ? (1ull << 32) : 0ull);
          const u64 old = atomicAdd(&tab[p], inc);
          if (old == 0) L[atomicAdd(&s_cnt[wib], 1)] = (int32_t)p;
        }
      }
      __syncwarp();
      const int cnt = s_cnt[wib];
      u64 r68 = 0, r69 = 0;
      for (int t = lane; t < cnt; t += 32) {
        const int32_t p = L[t];
        const u64 val = tab[p];
        tab[p] = 0;
        r68 += binom2(val & 0xffffffffull);
        r69 += binom2(val >> 32);
      }
      r68 = warp_sum(r68);
      r69 = warp_sum(r69);
      if (lane == 0) {
        if (r68) atomicAdd(&R68[a], r68);
        if (r69) atomicAdd(&R69[v], r69);
        s_cnt[wib] = 0;
      }
      __syncwarp();
    }
  }
}
