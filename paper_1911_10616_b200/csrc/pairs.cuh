// pairs.cuh -- step a7 of SURVEY 8(a): the pair (wedge) pass.
//
// One CTA per source u holds, for every x at distance <= 2, the pair quantities of
// Theorem B.1 (readings R11, R14):
//   W(u,x)  = |N(u) & N(x)|                       (2-hop expansion, phase A)
//   D(u,x)  = #edges inside N(u) & N(x)            (diamond expansion, phase B)
// TT(u,x) = sum_{v in N(u)&N(x)} T(v,x) - W[u~x] (R14) enters theta51 only through
// sum_x TT(u,x)(W-1), which is summed per wedge in phase D once W is final (no table).
// and emits:  C4(u)=DM8, theta36, theta50, theta51, theta63 for u (phase C);
//   E5 = C4(u,v) = sum_{x in N(v)\u} (W(u,x)-1) per edge, and the centre credits
//   theta49(v) += C(W(u,x)-1,2), theta62(v) += D(u,x) for x>u in N(v) (phase D);
//   theta64(v) += sum over diamonds (u; v,w; x), x>u, of W(u,x)-2 (phase E):
//   DM64(v) = sum_{pairs {a,x} in N(v)} |N(v)&N(a)&N(x)| (W(a,x)-2) seen from the pair.
// Tables are dense per-CTA arrays over the vertex set, reset through a touched list.
#pragma once
#include "common.cuh"

struct PairOut {
  u64 *R8, *R36, *R50, *R51, *R63, *R49, *R62, *R64, *C4e;
};

__device__ __forceinline__ int64_t slot_of_lo_in_hi(const DGraph& g, int32_t e) { return g.eslot_hi[e]; }
__device__ __forceinline__ int64_t slot_of_hi_in_lo(const DGraph& g, int32_t e) {
  const int32_t a = g.esrc[e];
  return g.rp[a] + g.dm[a] + (e - g.orow[a]);
}

__global__ void __launch_bounds__(512) k_pairs(DGraph g, const u32* __restrict__ Te,
                                               const int32_t* __restrict__ srcs, int nsrc,
                                               int* __restrict__ counter, u32* __restrict__ Wt,
                                               u32* __restrict__ Dt, uint8_t* __restrict__ Ft,
                                               int32_t* __restrict__ Lt, PairOut o) {
  __shared__ int s_idx;
  __shared__ int s_ntouch;
  __shared__ u64 s_red[5];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  const size_t off = (size_t)blockIdx.x * (size_t)g.n;
  u32* W = Wt + off;
  u32* D = Dt + off;
  uint8_t* F = Ft + off;
  int32_t* L = Lt + off;
  if (threadIdx.x == 0) { s_ntouch = 0; for (int t = 0; t < 5; t++) s_red[t] = 0; }
  for (;;) {
    if (threadIdx.x == 0) s_idx = atomicAdd(counter, 1);
    __syncthreads();
    const int idx = s_idx;
    if (idx >= nsrc) break;
    const int32_t u = srcs[idx];
    const int64_t r0 = g.rp[u], r1 = g.rp[u + 1];
    for (int64_t s = r0 + threadIdx.x; s < r1; s += blockDim.x) F[g.ci[s]] = 1;
    // ---- phase A: 2-hop wedge expansion
    for (int64_t s = r0 + wib; s < r1; s += nwb) {
      const int32_t v = g.ci[s];
      for (int64_t t = g.rp[v] + lane; t < g.rp[v + 1]; t += 32) {
        const int32_t x = g.ci[t];
        if (x == u) continue;
        const u32 old = atomicAdd(&W[x], 1u);
        if (old == 0) L[atomicAdd(&s_ntouch, 1)] = x;
      }
    }
    // ---- phase B: diamonds with u and x off the chord (v,w), v<w
    for (int64_t s = r0 + wib; s < r1; s += nwb) {
      const int32_t v = g.ci[s];
      const int32_t euv = g.eid[s];
      const bool v_lo = g.esrc[euv] == v;
      for (int64_t r = g.foff[euv]; r < g.foff[euv + 1]; r++) {
        const int32_t w = g.fx[r];
        if (w <= v) continue;
        const int32_t evw = v_lo ? g.fe1[r] : g.fe2[r];
        for (int64_t r2 = g.foff[evw] + lane; r2 < g.foff[evw + 1]; r2 += 32) {
          const int32_t x = g.fx[r2];
          if (x != u) atomicAdd(&D[x], 1u);
        }
      }
    }
    __syncthreads();
    const int ntouch = s_ntouch;
    // ---- phase C: per-pair sums for u
    {
      u64 a8 = 0, a36 = 0, a50 = 0, a51 = 0, a63 = 0;
      for (int t = threadIdx.x; t < ntouch; t += blockDim.x) {
        const int32_t x = L[t];
        const u64 w = W[x];
        const u64 c2 = binom2(w);
        a8 += c2;
        a36 += c2 * (u64)(int64_t)(dg_deg(g, x) - 2);
        a50 += binom3(w);
        a51 -= (u64)F[x] * w * (w - 1);
        a63 += (u64)D[x] * (w - 2);
      }
      a8 = warp_sum(a8); a36 = warp_sum(a36); a50 = warp_sum(a50); a51 = warp_sum(a51); a63 = warp_sum(a63);
      if (lane == 0) {
        atomicAdd(&s_red[0], a8); atomicAdd(&s_red[1], a36); atomicAdd(&s_red[2], a50);
        atomicAdd(&s_red[3], a51); atomicAdd(&s_red[4], a63);
      }
    }
    // ---- phase D: per neighbour v: E5(u,v), theta49 / theta62 centre credits
    for (int64_t s = r0 + wib; s < r1; s += nwb) {
      const int32_t v = g.ci[s];
      const int32_t euv = g.eid[s];
      const int64_t rev = (u < v) ? slot_of_lo_in_hi(g, euv) : slot_of_hi_in_lo(g, euv);
      u64 s5 = 0, s49 = 0, s62 = 0, s51 = 0;
      for (int64_t t = g.rp[v] + lane; t < g.rp[v + 1]; t += 32) {
        if (t == rev) continue;
        const int32_t x = g.ci[t];
        const u64 w = W[x];
        s5 += w - 1;
        s51 += (u64)Te[g.eid[t]] * (w - 1);
        if (t > rev) {
          s49 += binom2(w - 1);
          s62 += D[x];
        }
      }
      s5 = warp_sum(s5); s49 = warp_sum(s49); s62 = warp_sum(s62); s51 = warp_sum(s51);
      if (lane == 0) {
        if (s51) atomicAdd(&s_red[3], s51);
        if (u < v) o.C4e[euv] = s5;
        if (s49) atomicAdd(&o.R49[v], s49);
        if (s62) atomicAdd(&o.R62[v], s62);
      }
    }
    // ---- phase E: theta64 credits to v
    for (int64_t s = r0 + wib; s < r1; s += nwb) {
      const int32_t v = g.ci[s];
      const int32_t euv = g.eid[s];
      const bool v_lo = g.esrc[euv] == v;
      u64 acc = 0;
      for (int64_t r = g.foff[euv]; r < g.foff[euv + 1]; r++) {
        const int32_t evw = v_lo ? g.fe1[r] : g.fe2[r];
        for (int64_t r2 = g.foff[evw] + lane; r2 < g.foff[evw + 1]; r2 += 32) {
          const int32_t x = g.fx[r2];
          if (x > u) acc += (u64)W[x] - 2ull;
        }
      }
      acc = warp_sum(acc);
      if (lane == 0 && acc) atomicAdd(&o.R64[v], acc);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      o.R8[u] += s_red[0]; o.R36[u] += s_red[1]; o.R50[u] += s_red[2];
      o.R51[u] += s_red[3]; o.R63[u] += s_red[4];
      for (int t = 0; t < 5; t++) s_red[t] = 0;
      s_ntouch = 0;
    }
    // ---- reset
    for (int t = threadIdx.x; t < ntouch; t += blockDim.x) {
      const int32_t x = L[t];
      W[x] = 0; D[x] = 0;
    }
    for (int64_t s = r0 + threadIdx.x; s < r1; s += blockDim.x) F[g.ci[s]] = 0;
    __syncthreads();
  }
}
