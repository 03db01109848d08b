// hublocal.cuh -- step a8 of SURVEY 8(a): the hub-local (diamond) pass for the wheel W4
// = H27 (theta68, theta69; Theorem B.1, readings R11, R13).
//
//   theta68(a) = sum_{v in N(a)} sum_{x in N(v)\a} C(|N(v)&N(a)&N(x)|, 2)
//              = sum over hubs v in N(a) of the number of 4-cycles of G[N(v)] through a
//   theta69(v) = 1/2 sum_{a,x in N(v)} C(|N(v)&N(a)&N(x)|, 2) = #4-cycles of G[N(v)]
//
// Work item = ordered pair (v, a), a in N(v) with T(v,a) >= 2: a is the TOP (highest
// rank) vertex of the 4-cycles a-b-x-b' of G[N(v)] found from this item: a warp
// enumerates b in N(v)&N(a) with b < a and x in N(v)&N(b) with x < a and counts
// c(x) = #such b in a table indexed by x's position inside N(v) (shared memory when
// d(v) is small, a warp-private global region otherwise).  Each 4-cycle of G[N(v)] is
// found exactly once (from its top vertex, opposite x); its four corners are credited:
//   a, x    : C(c(x), 2) each           (theta68)
//   b (mid) : c(x) - 1 for every x      (theta68)
//   v       : C(c(x), 2)                (theta69)  -- no division modulo 2^64 needed.
// Restricting to cycles whose top is a (Chiba-Nishizeki) is what bounds the work.
#pragma once
#include "common.cuh"

#define HUB_SH_CAP 2048  // u32 table entries per warp in shared memory

__global__ void __launch_bounds__(256) k_hublocal(DGraph g, const u32* __restrict__ Te,
                                                  int* __restrict__ counter, int chunk,
                                                  int shard_index, int num_shards,
                                                  u32* __restrict__ gtabs, int32_t* __restrict__ glists,
                                                  u64* __restrict__ R68, u64* __restrict__ R69) {
  extern __shared__ u32 sh_tab[];  // 8 warps * HUB_SH_CAP (dynamic, 64 KB)
  __shared__ int s_cnt[8];
  __shared__ int64_t s_base[8];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  u32* stab = sh_tab + wib * HUB_SH_CAP;
  u32* gtab = gtabs + gw * (int64_t)g.max_deg;
  int32_t* L = glists + gw * (int64_t)g.max_deg;
  for (int t = lane; t < HUB_SH_CAP; t += 32) stab[t] = 0u;
  const int64_t nslots = 2 * g.m;
  if (lane == 0) s_cnt[wib] = 0;
  __syncwarp();
  for (;;) {
    if (lane == 0) s_base[wib] = (int64_t)atomicAdd(counter, 1) * chunk;
    __syncwarp();
    const int64_t base = s_base[wib];
    if (base >= nslots) break;
    const int64_t end = min(base + (int64_t)chunk, nslots);
    int64_t lo = 0, hi = g.n;  // v with rp[v] <= base < rp[v+1]
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
      const int32_t dv = (int32_t)(g.rp[v + 1] - rpv);
      u32* tab = (dv <= HUB_SH_CAP) ? stab : gtab;
      // pass 1: c(x) for x < a over b < a
      for (int64_t r = g.foff[eva]; r < g.foff[eva + 1]; r++) {
        const int32_t b = g.fx[r];
        if (b >= a) continue;
        const int32_t evb = v_lo ? g.fe1[r] : g.fe2[r];
        const bool v_lo_b = g.esrc[evb] == v;
        for (int64_t r2 = g.foff[evb] + lane; r2 < g.foff[evb + 1]; r2 += 32) {
          const int32_t x = g.fx[r2];
          if (x >= a) continue;
          const int32_t evx = v_lo_b ? g.fe1[r2] : g.fe2[r2];
          const int64_t p = (v < x) ? ((int64_t)g.dm[v] + (evx - g.orow[v])) : (g.eslot_hi[evx] - rpv);
          const u32 old = atomicAdd(&tab[p], 1u);
          if (old == 0) L[atomicAdd(&s_cnt[wib], 1)] = (int32_t)p;
        }
      }
      __syncwarp();
      const int cnt = s_cnt[wib];
      if (cnt == 0) continue;
      // pass 2: middles b get sum_x (c(x) - 1)
      for (int64_t r = g.foff[eva]; r < g.foff[eva + 1]; r++) {
        const int32_t b = g.fx[r];
        if (b >= a) continue;
        const int32_t evb = v_lo ? g.fe1[r] : g.fe2[r];
        const bool v_lo_b = g.esrc[evb] == v;
        u64 sb = 0;
        for (int64_t r2 = g.foff[evb] + lane; r2 < g.foff[evb + 1]; r2 += 32) {
          const int32_t x = g.fx[r2];
          if (x >= a) continue;
          const int32_t evx = v_lo_b ? g.fe1[r2] : g.fe2[r2];
          const int64_t p = (v < x) ? ((int64_t)g.dm[v] + (evx - g.orow[v])) : (g.eslot_hi[evx] - rpv);
          sb += (u64)tab[p] - 1ull;
        }
        sb = warp_sum(sb);
        if (lane == 0 && sb) atomicAdd(&R68[b], sb);
      }
      __syncwarp();
      // pass 3: corners a, x and the hub v
      u64 r69 = 0;
      for (int t = lane; t < cnt; t += 32) {
        const int32_t p = L[t];
        const u64 c2 = binom2(tab[p]);
        tab[p] = 0u;
        if (c2) {
          r69 += c2;
          atomicAdd(&R68[g.ci[rpv + p]], c2);
        }
      }
      r69 = warp_sum(r69);
      if (lane == 0) {
        if (r69) {
          atomicAdd(&R69[v], r69);
          atomicAdd(&R68[a], r69);
        }
        s_cnt[wib] = 0;
      }
      __syncwarp();
    }
  }
}
