// cycles5.cuh -- step a10 of SURVEY 8(a): 5-cycle vertex orbit theta34, Theorem 3.3
// in the reading R16 of DESIGN.md.
//
// Orientation G-> (rank order).  Every 5-cycle has exactly one decomposition into a
// directed 3-path i <- j <- k -> l (k the path's source: k<j<i, k<l) and a wedge
// (i, w, l) that is not in-in (not w>i and w>l).  Pass 1 credits i,j,k,l
// with the number of such wedges between i and l minus the two cases w=k (i~k) and
// w=j (j~l); pass 2 credits w with P(i,l), the number of such paths from
// i to l, minus the tailed triangles where the path runs through w.
//
// B200 formulation: one CTA per endpoint l.  Instead of enumerating the DP(G->) paths
// one by one, the CTA builds dense tables keyed by vertex:
//   Wn[i]  = #non-in-in wedges (i, w, l)
//   Q[j]   = |N-(j) & N-(l)|   (out-out wedges k: j <- k -> l),  QT[j], QM[j] = the
//            same sum weighted by T_high(k,j), T_mid(k,j) (typed triangle counts)
//   P[i]   = sum_{j in N-(i), j != l} Q[j]   (= number of paths i <- j <- k -> l)
//   A[i]   = the part of P[i] with j ~ l;  S[j] = sum_{i in N+(j), i != l} Wn[i]
// and credits every role in closed form:
//   i : P[i] Wn[i] - A[i] - (QM[i] - Q[i][i>l, i~l])
//   j : Q[j] S[j] - Q[j][j~l](d+(j) - [l in N+(j)]) - (QT[j] - Q[j][l in N+(j)])
//   k : sum_{j in N+(k)\l} S[j] - [j~l](d+(j) - [l in N+(j)]) - (T_high(k,j) - [l in N+(j)])
//   l : sum of the i credits
//   w : sum over non-in-in wedges (i,w,l) of P[i] - [w<i] T_low(w,l)
//                                   - [w<l, w<i] (T_mid(w,i) - [l<i, l~i])
// Each (path, wedge) pair with distinct vertices is one 5-cycle; the tests check the
// identity against brute force (tests/test_gpu_parity.py) and the prototype derivation
// is written out in DESIGN.md.
#pragma once
#include "common.cuh"

struct C5Tables {
  u32* Wn; u32* Q; u64* P; u64* A; u64* QT; u64* QM; u64* S; u32* flag; int32_t* Li; int32_t* Lj;
};

__device__ __forceinline__ void c5_mark(u32* flag, int32_t* list, int* cnt, int32_t x, u32 bit) {
  const u32 old = atomicOr(&flag[x], bit);
  if (!(old & bit)) list[atomicAdd(cnt, 1)] = x;
}

__global__ void __launch_bounds__(512) k_cycles5(DGraph g, const u32* __restrict__ Tlow,
                                                 const u32* __restrict__ Tmid,
                                                 const u32* __restrict__ Thigh,
                                                 const int32_t* __restrict__ ls, int nl,
                                                 int* __restrict__ counter, C5Tables tb,
                                                 u64* __restrict__ C5) {
  __shared__ int s_idx, s_ni, s_nj;
  __shared__ u64 s_tot;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  const size_t off = (size_t)blockIdx.x * (size_t)g.n;
  u32* Wn = tb.Wn + off; u32* Q = tb.Q + off; u64* P = tb.P + off; u64* A = tb.A + off;
  u64* QT = tb.QT + off; u64* QM = tb.QM + off; u64* S = tb.S + off; u32* flag = tb.flag + off;
  int32_t* Li = tb.Li + off; int32_t* Lj = tb.Lj + off;
  if (threadIdx.x == 0) { s_ni = 0; s_nj = 0; s_tot = 0; }
  for (;;) {
    if (threadIdx.x == 0) s_idx = atomicAdd(counter, 1);
    __syncthreads();
    const int idx = s_idx;
    if (idx >= nl) break;
    const int32_t l = ls[idx];
    const int64_t r0 = g.rp[l], r1 = g.rp[l + 1], rmid = r0 + g.dm[l];
    for (int64_t s = r0 + threadIdx.x; s < r1; s += blockDim.x) flag[g.ci[s]] = 1u;
    __syncthreads();
    // step 1: non-in-in wedges (i, w, l)
    for (int64_t s = r0 + wib; s < r1; s += nwb) {
      const int32_t w = g.ci[s];
      const int64_t t0 = (w < l) ? g.rp[w] : g.rp[w] + g.dm[w];
      for (int64_t t = t0 + lane; t < g.rp[w + 1]; t += 32) {
        const int32_t i = g.ci[t];
        if (i == l) continue;
        atomicAdd(&Wn[i], 1u);
        c5_mark(flag, Li, &s_ni, i, 2u);
      }
    }
    // step 2: out-out wedges j <- k -> l, k in N-(l)
    for (int64_t s = r0 + wib; s < rmid; s += nwb) {
      const int32_t k = g.ci[s];
      const int64_t ok = g.orow[k];
      const int32_t dk = (int32_t)(g.orow[k + 1] - ok);
      for (int t = lane; t < dk; t += 32) {
        const int32_t j = g.ocol[ok + t];
        if (j == l) continue;
        atomicAdd(&Q[j], 1u);
        atomicAdd(&QT[j], (u64)Thigh[ok + t]);
        atomicAdd(&QM[j], (u64)Tmid[ok + t]);
        c5_mark(flag, Lj, &s_nj, j, 4u);
      }
    }
    __syncthreads();
    // step 3: paths through j: P, A, S and the j credits
    const int nj = s_nj;
    for (int t = wib; t < nj; t += nwb) {
      const int32_t j = Lj[t];
      const u64 q = Q[j];
      const bool adjj = flag[j] & 1u;
      const u64 lj = (l > j && adjj) ? 1ull : 0ull;
      const int64_t oj = g.orow[j];
      const int32_t dj = (int32_t)(g.orow[j + 1] - oj);
      u64 s = 0;
      for (int c = lane; c < dj; c += 32) {
        const int32_t i = g.ocol[oj + c];
        if (i == l) continue;
        s += Wn[i];
        atomicAdd(&P[i], q);
        if (adjj) atomicAdd(&A[i], q);
        c5_mark(flag, Li, &s_ni, i, 2u);
      }
      s = warp_sum(s);
      if (lane == 0) {
        S[j] = s;
        const u64 cj = q * s - q * (adjj ? 1ull : 0ull) * ((u64)dj - lj) - (QT[j] - q * lj);
        if (cj) atomicAdd(&C5[j], cj);
      }
    }
    __syncthreads();
    // step 4: k credits
    for (int64_t s = r0 + wib; s < rmid; s += nwb) {
      const int32_t k = g.ci[s];
      const int64_t ok = g.orow[k];
      const int32_t dk = (int32_t)(g.orow[k + 1] - ok);
      u64 ck = 0;
      for (int t = lane; t < dk; t += 32) {
        const int32_t j = g.ocol[ok + t];
        if (j == l) continue;
        const bool adjj = flag[j] & 1u;
        const u64 lj = (l > j && adjj) ? 1ull : 0ull;
        const u64 dj = (u64)(g.orow[j + 1] - g.orow[j]);
        ck += S[j] - (adjj ? (dj - lj) : 0ull) - ((u64)Thigh[ok + t] - lj);
      }
      ck = warp_sum(ck);
      if (lane == 0 && ck) atomicAdd(&C5[k], ck);
    }
    // step 5: i credits (and their sum for l)
    const int ni = s_ni;
    {
      u64 tot = 0;
      for (int t = threadIdx.x; t < ni; t += blockDim.x) {
        const int32_t i = Li[t];
        const bool adji = flag[i] & 1u;
        const u64 bi = QM[i] - (u64)Q[i] * ((i > l && adji) ? 1ull : 0ull);
        const u64 ci = P[i] * (u64)Wn[i] - A[i] - bi;
        if (ci) atomicAdd(&C5[i], ci);
        tot += ci;
      }
      tot = warp_sum(tot);
      if (lane == 0 && tot) atomicAdd(&s_tot, tot);
    }
    // step 6: wedge centres w
    for (int64_t s = r0 + wib; s < r1; s += nwb) {
      const int32_t w = g.ci[s];
      const u64 tlow = Tlow[g.eid[s]];
      const int64_t t0 = (w < l) ? g.rp[w] : g.rp[w] + g.dm[w];
      u64 acc = 0;
      for (int64_t t = t0 + lane; t < g.rp[w + 1]; t += 32) {
        const int32_t i = g.ci[t];
        if (i == l) continue;
        u64 corr = (w < i) ? tlow : 0ull;
        if (w < l && w < i) corr += (u64)Tmid[g.eid[t]] - ((l < i && (flag[i] & 1u)) ? 1ull : 0ull);
        acc += P[i] - corr;
      }
      acc = warp_sum(acc);
      if (lane == 0 && acc) atomicAdd(&C5[w], acc);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (s_tot) atomicAdd(&C5[l], s_tot);
      s_tot = 0; s_ni = 0; s_nj = 0;
    }
    // reset
    for (int t = threadIdx.x; t < ni; t += blockDim.x) {
      const int32_t i = Li[t];
      Wn[i] = 0; P[i] = 0; A[i] = 0; flag[i] = 0;
    }
    for (int t = threadIdx.x; t < nj; t += blockDim.x) {
      const int32_t j = Lj[t];
      Q[j] = 0; QT[j] = 0; QM[j] = 0; S[j] = 0; flag[j] = 0;
    }
    for (int64_t s = r0 + threadIdx.x; s < r1; s += blockDim.x) flag[g.ci[s]] = 0;
    __syncthreads();
  }
}
