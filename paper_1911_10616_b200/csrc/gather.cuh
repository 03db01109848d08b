// gather.cuh -- steps a11/a12 of SURVEY 8(a): neighbour sums (O(m)), triangle sums
// (O(#T)) and the per-vertex combination of Lemma 4vertexorbit and
// Theorem B.1 with the readings of DESIGN.md, followed by the induced
// transform DIM = A^-1 DM.
#pragma once
#include "common.cuh"

// Per-vertex fields, SoA: F[f * n + u].  Fields from F_R8 on are "sharded": they are
// produced by the passes whose work is split across shards and enter every equation
// linearly.
enum Field {
  F_T = 0, F_DM1, F_DM6, F_DM9, F_DM10, F_DM13, F_S22, F_S28, F_S31, F_S41, F_S55,
  F_DM12, F_K4,
  F_DM4, F_S18, F_S19, F_S24, F_S27, F_S39, F_S40, F_S45, F_S56, F_S57, F_S60, F_S67,
  F_S15,
  F_T25, F_T26, F_T29, F_T32, F_T43, F_T46, F_T48, F_T54, F_T59, F_T61, F_T65, F_T71,
  // ---- sharded
  F_R8, F_S35, F_S37, F_T52, F_T53, F_R36, F_R49, F_R50, F_R51, F_R62, F_R63, F_R64,
  F_R68, F_R69, F_C5, F_K5, F_R66, F_R70,
  F_COUNT
};
#define F_FIRST_SHARDED F_R8

struct EdgeVals {
  const u32* Te;
  const u64* E9f;   // E9<lo,hi>
  const u64* E9b;   // E9<hi,lo>
  const u64* K4e;   // E11
  const u64* C4e;   // E5
  const u64* E7;
  const u32* K4t;
};

#define FLD(f, u) F[(size_t)(f) * (size_t)n + (u)]

// ---- nbr1: needs d, T, Te
__global__ void k_nbr1(DGraph g, EdgeVals ev, u64* __restrict__ F) {
  const int32_t n = g.n;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u64i = gw; u64i < n; u64i += nw) {
    const int32_t u = (int32_t)u64i;
    u64 dm1 = 0, dm6 = 0, dm9 = 0, dm10 = 0, dm13 = 0, s22 = 0, s28 = 0, s31 = 0, s41 = 0, s55 = 0;
    for (int64_t s = g.rp[u] + lane; s < g.rp[u + 1]; s += 32) {
      const int32_t v = g.ci[s];
      const u64 dv = (u64)dg_deg(g, v);
      const u64 tv = FLD(F_T, v);
      const u64 te = ev.Te[g.eid[s]];
      dm1 += dv - 1;
      dm6 += binom2(dv - 1);
      dm9 += tv - te;
      dm10 += te * (dv - 2);
      dm13 += binom2(te);
      s22 += binom3(dv - 1);
      s28 += tv;
      s31 += (dv - 1) * tv;
      s41 += binom2(te) * (dv - 3);
      s55 += binom3(te);
    }
    dm1 = warp_sum(dm1); dm6 = warp_sum(dm6); dm9 = warp_sum(dm9); dm10 = warp_sum(dm10);
    dm13 = warp_sum(dm13); s22 = warp_sum(s22); s28 = warp_sum(s28); s31 = warp_sum(s31);
    s41 = warp_sum(s41); s55 = warp_sum(s55);
    if (lane == 0) {
      FLD(F_DM1, u) = dm1; FLD(F_DM6, u) = dm6; FLD(F_DM9, u) = dm9; FLD(F_DM10, u) = dm10;
      FLD(F_DM13, u) = dm13; FLD(F_S22, u) = s22; FLD(F_S28, u) = s28; FLD(F_S31, u) = s31;
      FLD(F_S41, u) = s41; FLD(F_S55, u) = s55;
    }
  }
}

// ---- nbr2: needs DM1, DM6, DM9, DM10, DM12, DM13, K4, R8 of neighbours and E5/E9/E11
__global__ void k_nbr2(DGraph g, EdgeVals ev, u64* __restrict__ F) {
  const int32_t n = g.n;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u64i = gw; u64i < n; u64i += nw) {
    const int32_t u = (int32_t)u64i;
    u64 s4 = 0, s18 = 0, s19 = 0, s24 = 0, s27 = 0, s39 = 0, s40 = 0, s45 = 0, s56 = 0, s57 = 0,
        s60 = 0, s67 = 0, s35 = 0, s37 = 0;
    for (int64_t s = g.rp[u] + lane; s < g.rp[u + 1]; s += 32) {
      const int32_t v = g.ci[s];
      const int32_t e = g.eid[s];
      const u64 dv = (u64)dg_deg(g, v);
      const u64 dm1v = FLD(F_DM1, v);
      const u64 te = ev.Te[e];
      const u64 e9vu = (v < u) ? ev.E9f[e] : ev.E9b[e];  // E9<v,u>
      const u64 k4e = ev.K4e[e];
      s4 += dm1v;
      s18 += FLD(F_DM6, v);
      s19 += dm1v * (dv - 1) - 2 * FLD(F_T, v);           // DM5(v)
      s24 += FLD(F_DM10, v);
      s27 += FLD(F_DM9, v);
      s39 += FLD(F_DM13, v);
      s40 += e9vu * (dv - 3);
      s45 += FLD(F_DM12, v);
      s56 += FLD(F_K4, v);
      s57 += k4e * (dv - 3);
      s60 += e9vu * (te - 1);
      s67 += k4e * (te - 2);
      s35 += FLD(F_R8, v);
      s37 += ev.C4e[e] * (dv - 2);
    }
    s4 = warp_sum(s4); s18 = warp_sum(s18); s19 = warp_sum(s19); s24 = warp_sum(s24);
    s27 = warp_sum(s27); s39 = warp_sum(s39); s40 = warp_sum(s40); s45 = warp_sum(s45);
    s56 = warp_sum(s56); s57 = warp_sum(s57); s60 = warp_sum(s60); s67 = warp_sum(s67);
    s35 = warp_sum(s35); s37 = warp_sum(s37);
    if (lane == 0) {
      const u64 d = (u64)dg_deg(g, u);
      FLD(F_DM4, u) = s4 - 2 * binom2(d) - 2 * FLD(F_T, u);
      FLD(F_S18, u) = s18; FLD(F_S19, u) = s19; FLD(F_S24, u) = s24; FLD(F_S27, u) = s27;
      FLD(F_S39, u) = s39; FLD(F_S40, u) = s40; FLD(F_S45, u) = s45; FLD(F_S56, u) = s56;
      FLD(F_S57, u) = s57; FLD(F_S60, u) = s60; FLD(F_S67, u) = s67;
      FLD(F_S35, u) = s35; FLD(F_S37, u) = s37;
    }
  }
}

// ---- nbr3: sum of DM4 over neighbours (theta15)
__global__ void k_nbr3(DGraph g, u64* __restrict__ F) {
  const int32_t n = g.n;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u64i = gw; u64i < n; u64i += nw) {
    const int32_t u = (int32_t)u64i;
    u64 s = 0;
    for (int64_t t = g.rp[u] + lane; t < g.rp[u + 1]; t += 32) s += FLD(F_DM4, g.ci[t]);
    s = warp_sum(s);
    if (lane == 0) FLD(F_S15, u) = s;
  }
}

// ---- triangle sums: thread per oriented triangle entry; each of the three vertices
// gets the summand of every triangle-sum equation with itself as u.
__device__ __forceinline__ void tri_credit(const DGraph& g, const EdgeVals& ev, u64* __restrict__ F,
                                           int32_t n, int32_t u, int32_t v, int32_t x, int32_t euv,
                                           int32_t eux, int32_t evx, u64 k4t) {
  const u64 du = dg_deg(g, u), dv = dg_deg(g, v), dx = dg_deg(g, x);
  const u64 tuv = ev.Te[euv], tux = ev.Te[eux], tvx = ev.Te[evx];
  atomicAdd(&FLD(F_T25, u), (dv - 2) * (dx - 2));
  atomicAdd(&FLD(F_T26, u), (du - 2) * ((dx - 2) + (dv - 2)));
  atomicAdd(&FLD(F_T29, u), FLD(F_DM1, v) + FLD(F_DM1, x));
  atomicAdd(&FLD(F_T32, u), binom2(dv - 2) + binom2(dx - 2));
  atomicAdd(&FLD(F_T43, u), (FLD(F_T, v) - 1) + (FLD(F_T, x) - 1));
  atomicAdd(&FLD(F_T46, u), ev.E7[evx]);
  atomicAdd(&FLD(F_T48, u), (tuv - 1) * (dx - 2) + (tux - 1) * (dv - 2));
  atomicAdd(&FLD(F_T54, u), binom2(tvx - 1));
  atomicAdd(&FLD(F_T59, u), ev.E9f[evx] + ev.E9b[evx]);
  atomicAdd(&FLD(F_T61, u), (tuv - 1) * (tux - 1));
  atomicAdd(&FLD(F_T65, u), ev.K4e[evx]);
  atomicAdd(&FLD(F_T71, u), binom2(k4t));
  atomicAdd(&FLD(F_T52, u), ev.C4e[evx]);
  atomicAdd(&FLD(F_T53, u), ev.C4e[euv] + ev.C4e[eux]);
}

__global__ void k_trigather(DGraph g, EdgeVals ev, u64* __restrict__ F) {
  const int32_t n = g.n;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < g.ntri;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int32_t eab = g.tab[q], eac = g.tac[q], ebc = g.tbc[q];
    const int32_t a = g.esrc[eab], b = g.edst[eab], c = g.tc[q];
    const u64 k4t = ev.K4t[q];
    tri_credit(g, ev, F, n, a, b, c, eab, eac, ebc, k4t);
    tri_credit(g, ev, F, n, b, a, c, eab, ebc, eac, k4t);
    tri_credit(g, ev, F, n, c, a, b, eac, ebc, eab, k4t);
  }
}

// ---- combine: DM per vertex (non-induced, Def. unlabeled-match), then
// DIM = A^-1 DM with A^-1 in constant memory (sparse rows).
#define AINV_MAX_NNZ 2048
__constant__ int c_ainv_rp[EVOKE_NUM_ORBITS_DEV + 1];
__constant__ uint8_t c_ainv_col[AINV_MAX_NNZ];
__constant__ long long c_ainv_val[AINV_MAX_NNZ];

__device__ void compute_dm(const DGraph& g, const u64* __restrict__ F, int32_t n, int32_t u,
                           bool zero_sharded, u64* DM) {
  auto f = [&](int fld) -> u64 {
    if (zero_sharded && fld >= F_FIRST_SHARDED) return 0ull;
    return FLD(fld, u);
  };
  const u64 d = (u64)dg_deg(g, u);
  const u64 T = f(F_T);
  DM[0] = d;
  DM[1] = f(F_DM1);
  DM[2] = binom2(d);
  DM[3] = T;
  DM[4] = f(F_DM4);
  DM[5] = DM[1] * (d - 1) - 2 * T;
  DM[6] = f(F_DM6);
  DM[7] = binom3(d);
  DM[8] = f(F_R8);
  DM[9] = f(F_DM9);
  DM[10] = f(F_DM10);
  DM[11] = T * (d - 2);
  DM[12] = f(F_DM12);
  DM[13] = f(F_DM13);
  DM[14] = f(F_K4);
  const u64 *D = DM;
  DM[15] = f(F_S15) - D[5] - 2 * D[11] - 2 * D[8];
  DM[16] = D[4] * (d - 1) - D[10] - 2 * D[8];
  DM[17] = binom2(D[1]) - D[3] - D[6] - D[8] - D[10];
  DM[18] = f(F_S18) - 3 * D[7] - D[10];
  DM[19] = f(F_S19) - D[4] - D[5] - D[10];                 // R6
  DM[20] = (d - 1) * D[6] - D[10];                          // R7
  DM[21] = binom2(d - 1) * D[1] - 2 * D[11];                // R7
  DM[22] = f(F_S22);
  DM[23] = binom4(d);
  DM[24] = f(F_S24) - D[10] - 2 * D[11] - 2 * D[12];
  DM[25] = f(F_T25) - D[12];
  DM[26] = f(F_T26) - 2 * D[13];
  DM[27] = f(F_S27) - D[11] - 2 * D[13];
  DM[28] = (d - 1) * f(F_S28) - 2 * D[3] - 2 * D[11] - 2 * D[12];
  DM[29] = f(F_T29) - 4 * D[3] - D[10] - 2 * D[11] - 2 * D[12] - 2 * D[13];
  DM[30] = T * D[1] - 2 * D[3] - D[10] - 2 * D[13];
  DM[31] = f(F_S31) - 2 * D[9] - D[10] - 2 * D[3];
  DM[32] = f(F_T32);
  DM[33] = T * binom2(d - 2);
  DM[34] = f(F_C5);
  DM[35] = f(F_S35) - 2 * D[8] - D[13];                     // R9
  DM[36] = f(F_R36) - D[13];
  DM[37] = f(F_S37) - 2 * D[12];
  DM[38] = D[8] * (d - 2) - D[13];
  DM[39] = f(F_S39) - D[13] - 2 * D[12];
  DM[40] = f(F_S40);                                        // R10
  DM[41] = f(F_S41);
  DM[42] = D[13] * (d - 3);
  DM[43] = f(F_T43) - 2 * D[12] - 2 * D[13];
  DM[44] = binom2(T) - D[13];
  DM[45] = f(F_S45) - 2 * D[13] - 3 * D[14];
  DM[46] = f(F_T46) - D[11] - 3 * D[14];
  DM[47] = D[12] * (d - 2) - 3 * D[14];
  DM[48] = f(F_T48) - 6 * D[14];
  DM[49] = f(F_R49);
  DM[50] = f(F_R50);
  DM[51] = f(F_R51) - 2 * D[12];                            // R14
  DM[52] = f(F_T52) - 2 * D[13];
  DM[53] = f(F_T53) - 2 * D[13] - 2 * D[12];
  DM[54] = f(F_T54);
  DM[55] = f(F_S55);
  DM[56] = f(F_S56) - 3 * D[14];
  DM[57] = f(F_S57);
  DM[58] = D[14] * (d - 3);
  DM[59] = f(F_T59) - 2 * D[13] - 6 * D[14];
  DM[60] = f(F_S60) - 6 * D[14];
  DM[61] = f(F_T61) - 3 * D[14];
  DM[62] = f(F_R62) - D[13];
  DM[63] = f(F_R63);                                        // R11
  DM[64] = f(F_R64);                                        // R11
  DM[65] = f(F_T65) - 3 * D[14];
  DM[66] = f(F_R66) - 6 * D[14];                            // R12
  DM[67] = f(F_S67);
  DM[68] = f(F_R68);                                        // R11
  DM[69] = f(F_R69);                                        // R13
  DM[70] = f(F_R70);
  DM[71] = f(F_T71);
  DM[72] = f(F_K5);
}

// ncols = 73, or 15 for the 4-vertex orbits only (the 5-vertex columns are written as 0;
// A is block diagonal by pattern size, so DIM 0..14 needs DM 0..14 only)
__global__ void k_combine(DGraph g, const u64* __restrict__ F, const int32_t* __restrict__ perm,
                          int induced, int primary, int ncols, u64* __restrict__ out) {
  const int32_t n = g.n;
  for (int32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
    u64 DM[EVOKE_NUM_ORBITS_DEV];
    compute_dm(g, F, n, u, false, DM);
    if (!primary) {
      u64 DM0[EVOKE_NUM_ORBITS_DEV];
      compute_dm(g, F, n, u, true, DM0);
      for (int i = 0; i < EVOKE_NUM_ORBITS_DEV; i++) DM[i] -= DM0[i];
    }
    u64* row = out + (size_t)perm[u] * EVOKE_NUM_ORBITS_DEV;
    if (!induced) {
      for (int i = 0; i < EVOKE_NUM_ORBITS_DEV; i++) row[i] = i < ncols ? DM[i] : 0ull;
    } else {
      for (int i = 0; i < EVOKE_NUM_ORBITS_DEV; i++) {
        u64 acc = 0;
        if (i < ncols)
          for (int p = c_ainv_rp[i]; p < c_ainv_rp[i + 1]; p++)
            acc += (u64)c_ainv_val[p] * DM[c_ainv_col[p]];
        row[i] = acc;
      }
    }
  }
}
