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
  // packed rows for the late gathers (k_pack_rows): per vertex V2[v][V2_W], per edge EV[e][EV_W]
  const u64* V2 = nullptr;
  const u64* EV = nullptr;
};

// The late gathers (nbr2, the triangle gather) read, for every neighbour v / triangle corner,
// about ten per-vertex fields and five per-edge values at random places: one 32-byte sector
// per field in the field-major layout.  k_pack_rows copies them once (coalesced) into rows --
// per vertex 96 bytes (the values of v the gathers read; the first sector holds what the
// triangle gather needs), per edge 64 bytes -- so a random visit reads 1-3 sectors.
enum { V2_D = 0, V2_DM1, V2_T, V2_DM5, V2_DM6, V2_DM10, V2_DM9, V2_DM13, V2_DM12, V2_K4, V2_R8, V2_W = 12 };
enum { EV_E9F = 0, EV_E9B, EV_K4E, EV_C4E, EV_E7, EV_TE, EV_W = 8 };

#define FLD(f, u) F[(size_t)(f) * (size_t)n + (u)]

// Neighbour gathers.  Vertices of degree <= NBR_HEAVY: one warp each (warp reduction);
// the others (hubs) are appended to a list by the warp kernel and summed by a second kernel
// with one CTA per hub (block reduction), so a hub's list is not walked by a single warp.
#define NBR_HEAVY 2048

// block-wide sum of NS values (blockDim.x = 1024 or 256); result valid in thread 0
template <int NS>
__device__ __forceinline__ void block_sum_vals(u64 (&a)[NS], u64* sh) {
#pragma unroll
  for (int i = 0; i < NS; i++) a[i] = warp_sum(a[i]);
  if (threadIdx.x < NS) sh[threadIdx.x] = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int i = 0; i < NS; i++)
      if (a[i]) atomicAdd(&sh[i], a[i]);
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NS; i++) a[i] = sh[i];
  __syncthreads();
}

// ---- nbr1: needs d, T, Te
__device__ __forceinline__ void nbr1_acc(const DGraph& g, const EdgeVals& ev, const u64* __restrict__ F, int32_t n,
                                         int32_t u, int64_t start, int stride, u64 (&a)[10]) {
  for (int64_t s = g.rp[u] + start; s < g.rp[u + 1]; s += stride) {
    const int32_t v = g.ci[s];
    const u64 dv = (u64)dg_deg(g, v);
    const u64 tv = FLD(F_T, v);
    const u64 te = g.tes[s];
    a[0] += dv - 1;
    a[1] += binom2(dv - 1);
    a[2] += tv - te;
    a[3] += te * (dv - 2);
    a[4] += binom2(te);
    a[5] += binom3(dv - 1);
    a[6] += tv;
    a[7] += (dv - 1) * tv;
    a[8] += binom2(te) * (dv - 3);
    a[9] += binom3(te);
  }
}
__device__ __forceinline__ void nbr1_store(u64* __restrict__ F, int32_t n, int32_t u, const u64 (&a)[10]) {
  FLD(F_DM1, u) = a[0]; FLD(F_DM6, u) = a[1]; FLD(F_DM9, u) = a[2]; FLD(F_DM10, u) = a[3];
  FLD(F_DM13, u) = a[4]; FLD(F_S22, u) = a[5]; FLD(F_S28, u) = a[6]; FLD(F_S31, u) = a[7];
  FLD(F_S41, u) = a[8]; FLD(F_S55, u) = a[9];
}

__global__ void k_pack_rows(DGraph g, EdgeVals ev, const u64* __restrict__ F, u64* __restrict__ V2,
                            u64* __restrict__ EV) {
  const int32_t n = g.n;
  const int64_t N = max((int64_t)n, g.m);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < N; q += (int64_t)gridDim.x * blockDim.x) {
    if (q < n) {
      const int32_t v = (int32_t)q;
      const u64 d = (u64)dg_deg(g, v), dm1 = FLD(F_DM1, v), t = FLD(F_T, v);
      ulonglong2* r = reinterpret_cast<ulonglong2*>(V2 + (size_t)v * V2_W);
      r[0] = make_ulonglong2(d, dm1);
      r[1] = make_ulonglong2(t, dm1 * (d - 1) - 2 * t);  // DM5(v)
      r[2] = make_ulonglong2(FLD(F_DM6, v), FLD(F_DM10, v));
      r[3] = make_ulonglong2(FLD(F_DM9, v), FLD(F_DM13, v));
      r[4] = make_ulonglong2(FLD(F_DM12, v), FLD(F_K4, v));
      r[5] = make_ulonglong2(FLD(F_R8, v), 0ull);
    }
    if (q < g.m) {
      ulonglong2* r = reinterpret_cast<ulonglong2*>(EV + (size_t)q * EV_W);
      r[0] = make_ulonglong2(ev.E9f[q], ev.E9b[q]);
      r[1] = make_ulonglong2(ev.K4e[q], ev.C4e[q]);
      r[2] = make_ulonglong2(ev.E7[q], (u64)ev.Te[q]);
    }
  }
}

// ---- nbr2: needs DM1, DM6, DM9, DM10, DM12, DM13, K4, R8 of neighbours and E5/E9/E11
// (from the packed rows)
__device__ __forceinline__ void nbr2_acc(const DGraph& g, const EdgeVals& ev, const u64* __restrict__ F, int32_t n,
                                         int32_t u, int64_t start, int stride, u64 (&a)[14]) {
  for (int64_t s = g.rp[u] + start; s < g.rp[u + 1]; s += stride) {
    const int32_t v = g.ci[s];
    const int32_t e = g.eid[s];
    const u64 te = g.tes[s];
    const ulonglong2* r = reinterpret_cast<const ulonglong2*>(ev.V2 + (size_t)v * V2_W);
    const ulonglong2* q = reinterpret_cast<const ulonglong2*>(ev.EV + (size_t)e * EV_W);
    const ulonglong2 r0 = r[0], r1 = r[1], r2 = r[2], r3 = r[3], r4 = r[4], r5 = r[5];
    const ulonglong2 q0 = q[0], q1 = q[1];
    const u64 dv = r0.x;
    const u64 e9vu = (v < u) ? q0.x : q0.y;  // E9<v,u>
    const u64 k4e = q1.x;
    a[0] += r0.y;            // DM1(v)
    a[1] += r2.x;            // DM6(v)
    a[2] += r1.y;            // DM5(v)
    a[3] += r2.y;            // DM10(v)
    a[4] += r3.x;            // DM9(v)
    a[5] += r3.y;            // DM13(v)
    a[6] += e9vu * (dv - 3);
    a[7] += r4.x;            // DM12(v)
    a[8] += r4.y;            // K4(v)
    a[9] += k4e * (dv - 3);
    a[10] += e9vu * (te - 1);
    a[11] += k4e * (te - 2);
    a[12] += r5.x;           // R8(v)
    a[13] += q1.y * (dv - 2);  // C4e
  }
}
__device__ __forceinline__ void nbr2_store(const DGraph& g, u64* __restrict__ F, int32_t n, int32_t u,
                                           const u64 (&a)[14]) {
  const u64 d = (u64)dg_deg(g, u);
  FLD(F_DM4, u) = a[0] - 2 * binom2(d) - 2 * FLD(F_T, u);
  FLD(F_S18, u) = a[1]; FLD(F_S19, u) = a[2]; FLD(F_S24, u) = a[3]; FLD(F_S27, u) = a[4];
  FLD(F_S39, u) = a[5]; FLD(F_S40, u) = a[6]; FLD(F_S45, u) = a[7]; FLD(F_S56, u) = a[8];
  FLD(F_S57, u) = a[9]; FLD(F_S60, u) = a[10]; FLD(F_S67, u) = a[11];
  FLD(F_S35, u) = a[12]; FLD(F_S37, u) = a[13];
}

// ---- nbr3: sum of DM4 over neighbours (theta15)
__device__ __forceinline__ void nbr3_acc(const DGraph& g, const EdgeVals&, const u64* __restrict__ F, int32_t n,
                                         int32_t u, int64_t start, int stride, u64 (&a)[1]) {
  for (int64_t t = g.rp[u] + start; t < g.rp[u + 1]; t += stride) a[0] += FLD(F_DM4, g.ci[t]);
}
__device__ __forceinline__ void nbr3_store(const DGraph&, u64* __restrict__ F, int32_t n, int32_t u,
                                           const u64 (&a)[1]) {
  FLD(F_S15, u) = a[0];
}

template <int K>
struct NbrK;
template <>
struct NbrK<1> {
  static constexpr int NS = 10;
  __device__ static void acc(const DGraph& g, const EdgeVals& ev, const u64* F, int32_t n, int32_t u, int64_t st,
                             int sd, u64 (&a)[NS]) { nbr1_acc(g, ev, F, n, u, st, sd, a); }
  __device__ static void store(const DGraph&, u64* F, int32_t n, int32_t u, const u64 (&a)[NS]) {
    nbr1_store(F, n, u, a);
  }
};
template <>
struct NbrK<2> {
  static constexpr int NS = 14;
  __device__ static void acc(const DGraph& g, const EdgeVals& ev, const u64* F, int32_t n, int32_t u, int64_t st,
                             int sd, u64 (&a)[NS]) { nbr2_acc(g, ev, F, n, u, st, sd, a); }
  __device__ static void store(const DGraph& g, u64* F, int32_t n, int32_t u, const u64 (&a)[NS]) {
    nbr2_store(g, F, n, u, a);
  }
};
template <>
struct NbrK<3> {
  static constexpr int NS = 1;
  __device__ static void acc(const DGraph& g, const EdgeVals& ev, const u64* F, int32_t n, int32_t u, int64_t st,
                             int sd, u64 (&a)[NS]) { nbr3_acc(g, ev, F, n, u, st, sd, a); }
  __device__ static void store(const DGraph& g, u64* F, int32_t n, int32_t u, const u64 (&a)[NS]) {
    nbr3_store(g, F, n, u, a);
  }
};

// Vertices of degree <= NBR_SMALL: eight lanes each (four vertices per warp; a warp per
// vertex left half the lanes idle at mean degree 16 and spent 70 shuffles on its 14 sums);
// degree <= NBR_HEAVY: appended to `mid` (a warp each, k_nbr_mid); heavier: to `heavy` (a CTA
// each).  Counts *nmid, *nheavy.
#define NBR_SMALL 64
#ifndef NBR_MINB
#define NBR_MINB 4  // resident 256-thread CTAs per SM the register budget must allow (config 4: gather 1
                    // 1.00 -> 0.95 ms, gather 2 2.87 -> 2.78 ms; the triangle gather at 4 was slower, 2.70 vs 2.50)
#endif
template <int K>
__global__ void __launch_bounds__(256, NBR_MINB) k_nbr(DGraph g, EdgeVals ev, u64* __restrict__ F, int32_t* __restrict__ heavy,
                      int* __restrict__ nheavy, int32_t* __restrict__ mid, int* __restrict__ nmid) {
  constexpr int NS = NbrK<K>::NS;
  const int32_t n = g.n;
  const int lane = threadIdx.x & 31, sub = lane & 7;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = gw * 4; base < n; base += nw * 4) {  // warp-uniform
    const int64_t uq = base + (lane >> 3);
    const int32_t u = (int32_t)min(uq, (int64_t)n - 1);
    const int d = uq < n ? dg_deg(g, u) : 0;
    u64 a[NS];
#pragma unroll
    for (int i = 0; i < NS; i++) a[i] = 0;
    if (uq < n && d <= NBR_SMALL) NbrK<K>::acc(g, ev, F, n, u, sub, 8, a);
#pragma unroll
    for (int i = 0; i < NS; i++) {
      a[i] += __shfl_xor_sync(FULL_MASK, a[i], 4);
      a[i] += __shfl_xor_sync(FULL_MASK, a[i], 2);
      a[i] += __shfl_xor_sync(FULL_MASK, a[i], 1);
    }
    if (uq < n && sub == 0) {
      if (d <= NBR_SMALL) NbrK<K>::store(g, F, n, u, a);
      else if (d <= NBR_HEAVY) mid[atomicAdd(nmid, 1)] = u;
      else heavy[atomicAdd(nheavy, 1)] = u;
    }
  }
}

// a warp per vertex of the mid list
template <int K>
__global__ void k_nbr_mid(DGraph g, EdgeVals ev, u64* __restrict__ F, const int32_t* __restrict__ mid,
                          const int* __restrict__ nmid) {
  constexpr int NS = NbrK<K>::NS;
  const int32_t n = g.n;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int cnt = *nmid;
  for (int64_t q = gw; q < cnt; q += nw) {
    const int32_t u = mid[q];
    u64 a[NS];
#pragma unroll
    for (int i = 0; i < NS; i++) a[i] = 0;
    NbrK<K>::acc(g, ev, F, n, u, lane, 32, a);
#pragma unroll
    for (int i = 0; i < NS; i++) a[i] = warp_sum(a[i]);
    if (lane == 0) NbrK<K>::store(g, F, n, u, a);
  }
}

// one CTA per hub of the list
template <int K>
__global__ void __launch_bounds__(1024) k_nbr_heavy(DGraph g, EdgeVals ev, u64* __restrict__ F,
                                                    const int32_t* __restrict__ heavy, const int* __restrict__ nheavy) {
  constexpr int NS = NbrK<K>::NS;
  __shared__ u64 sh[NS];
  const int32_t n = g.n;
  const int nh = *nheavy;
  for (int q = blockIdx.x; q < nh; q += gridDim.x) {
    const int32_t u = heavy[q];
    u64 a[NS];
#pragma unroll
    for (int i = 0; i < NS; i++) a[i] = 0;
    NbrK<K>::acc(g, ev, F, n, u, threadIdx.x, blockDim.x, a);
    block_sum_vals<NS>(a, sh);
    if (threadIdx.x == 0) NbrK<K>::store(g, F, n, u, a);
  }
}

// ---- triangle sums: thread per oriented triangle entry; each of the three vertices
// gets the summand of every triangle-sum equation with itself as u, into per-vertex rows of
// TG_W accumulators (one vertex's 14 sums in four sectors instead of 14 fields; k_tg_fields
// copies them into F).  Corner and edge values from the packed rows.
#define TG_ROWS_MAX_TPV 64  // triangle gather in rows while 3 #T <= this x n (triangle corners per vertex)
enum { TG_T25 = 0, TG_T26, TG_T29, TG_T32, TG_T43, TG_T46, TG_T48, TG_T54, TG_T59, TG_T61, TG_T65, TG_T71,
       TG_T52, TG_T53, TG_W = 16 };
struct TriCorner {  // the first sector of a vertex row
  u64 d, dm1, t;
};
__device__ __forceinline__ TriCorner tri_corner(const EdgeVals& ev, int32_t v) {
  const ulonglong2* r = reinterpret_cast<const ulonglong2*>(ev.V2 + (size_t)v * V2_W);
  const ulonglong2 a = r[0], b = r[1];
  return TriCorner{a.x, a.y, b.x};
}
struct TriEdge {
  u64 e9f, e9b, k4e, c4e, e7, te;
};
__device__ __forceinline__ TriEdge tri_edge(const EdgeVals& ev, int32_t e) {
  const ulonglong2* r = reinterpret_cast<const ulonglong2*>(ev.EV + (size_t)e * EV_W);
  const ulonglong2 a = r[0], b = r[1], c = r[2];
  return TriEdge{a.x, a.y, b.x, b.y, c.x, c.y};
}
// corner u with the other corners v, x; edges uv, ux and the opposite edge vx.  ROWS: into
// u's row of TG; else straight into the fields of F (triangle-heavy graphs: a hub's credits
// spread over 14 lines instead of queueing on the 4 lines of its row)
template <bool ROWS>
__device__ __forceinline__ void tri_credit(u64* __restrict__ TG, int32_t n, int32_t u, const TriCorner& U,
                                           const TriCorner& V, const TriCorner& X, const TriEdge& Euv,
                                           const TriEdge& Eux, const TriEdge& Evx, u64 k4t) {
  const u64 du = U.d, dv = V.d, dx = X.d;
  const u64 tuv = Euv.te, tux = Eux.te, tvx = Evx.te;
  u64* F = TG;
  auto at = [&](int j, int fld) -> u64* { return ROWS ? &TG[(size_t)u * TG_W + j] : &FLD(fld, u); };
  atomicAdd(at(TG_T25, F_T25), (dv - 2) * (dx - 2));
  atomicAdd(at(TG_T26, F_T26), (du - 2) * ((dx - 2) + (dv - 2)));
  atomicAdd(at(TG_T29, F_T29), V.dm1 + X.dm1);
  atomicAdd(at(TG_T32, F_T32), binom2(dv - 2) + binom2(dx - 2));
  atomicAdd(at(TG_T43, F_T43), (V.t - 1) + (X.t - 1));
  atomicAdd(at(TG_T46, F_T46), Evx.e7);
  atomicAdd(at(TG_T48, F_T48), (tuv - 1) * (dx - 2) + (tux - 1) * (dv - 2));
  atomicAdd(at(TG_T54, F_T54), binom2(tvx - 1));
  atomicAdd(at(TG_T59, F_T59), Evx.e9f + Evx.e9b);
  atomicAdd(at(TG_T61, F_T61), (tuv - 1) * (tux - 1));
  atomicAdd(at(TG_T65, F_T65), Evx.k4e);
  atomicAdd(at(TG_T71, F_T71), binom2(k4t));
  atomicAdd(at(TG_T52, F_T52), Evx.c4e);
  atomicAdd(at(TG_T53, F_T53), Euv.c4e + Eux.c4e);
}

// ROWS: TG = the row accumulators (k_tg_fields copies them); else TG = F
#ifndef TRIG_MINB
#define TRIG_MINB 1  // (developer variant: resident 256-thread CTAs per SM for the register budget)
#endif
template <bool ROWS>
__global__ void __launch_bounds__(256, TRIG_MINB) k_trigather(DGraph g, EdgeVals ev, u64* __restrict__ TG) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < g.ntri;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int32_t eab = g.tab[q], eac = g.tac[q], ebc = g.tbc[q];
    const int32_t a = g.esrc[eab], b = g.edst[eab], c = g.tc[q];
    const u64 k4t = ev.K4t[q];
    const TriCorner A = tri_corner(ev, a), B = tri_corner(ev, b), C = tri_corner(ev, c);
    const TriEdge Eab = tri_edge(ev, eab), Eac = tri_edge(ev, eac), Ebc = tri_edge(ev, ebc);
    tri_credit<ROWS>(TG, g.n, a, A, B, C, Eab, Eac, Ebc, k4t);
    tri_credit<ROWS>(TG, g.n, b, B, A, C, Eab, Ebc, Eac, k4t);
    tri_credit<ROWS>(TG, g.n, c, C, A, B, Eac, Ebc, Eab, k4t);
  }
}

// the triangle sums into their fields
__global__ void k_tg_fields(const u64* __restrict__ TG, int32_t n, u64* __restrict__ F) {
  const int fld[14] = {F_T25, F_T26, F_T29, F_T32, F_T43, F_T46, F_T48, F_T54, F_T59, F_T61, F_T65, F_T71,
                       F_T52, F_T53};
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < (int64_t)n * TG_W;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(q % TG_W);
    if (j < 14) F[(size_t)fld[j] * (size_t)n + (size_t)(q / TG_W)] = TG[q];
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
// A is block diagonal by pattern size, so DIM 0..14 needs DM 0..14 only).  Each thread's DM
// row lives in shared memory (a local array indexed by the A^-1 column list spilled to local
// memory), the transform runs in place (A^-1 is unit upper triangular: DIM_i reads DM_j, j >=
// i, so row i may overwrite DM_i once computed), and the warp then writes its 32 output rows
// (scattered by perm) one row at a time, consecutive lanes on consecutive words.
#define COMBINE_BT 128
__global__ void __launch_bounds__(COMBINE_BT) k_combine(DGraph g, const u64* __restrict__ F,
                                                        const int32_t* __restrict__ perm, int induced, int primary,
                                                        int ncols, u64* __restrict__ out) {
  extern __shared__ u64 comb_sh[];  // [COMBINE_BT][73]
  const int32_t n = g.n;
  const int lane = threadIdx.x & 31;
  u64* tile = comb_sh + (size_t)(threadIdx.x & ~31) * EVOKE_NUM_ORBITS_DEV;  // this warp's 32 rows
  u64* DM = tile + (size_t)lane * EVOKE_NUM_ORBITS_DEV;
  for (int32_t base = (blockIdx.x * blockDim.x + threadIdx.x) & ~31; base < n; base += gridDim.x * blockDim.x) {
    const int32_t u = base + lane;
    if (u < n) {
      compute_dm(g, F, n, u, false, DM);
      if (!primary) {
        u64 DM0[EVOKE_NUM_ORBITS_DEV];
        compute_dm(g, F, n, u, true, DM0);
        for (int i = 0; i < EVOKE_NUM_ORBITS_DEV; i++) DM[i] -= DM0[i];
      }
      if (!induced) {
        for (int i = ncols; i < EVOKE_NUM_ORBITS_DEV; i++) DM[i] = 0ull;
      } else {
        for (int i = 0; i < EVOKE_NUM_ORBITS_DEV; i++) {
          u64 acc = 0;
          if (i < ncols)
            for (int p = c_ainv_rp[i]; p < c_ainv_rp[i + 1]; p++)
              acc += (u64)c_ainv_val[p] * DM[c_ainv_col[p]];
          DM[i] = acc;  // in place: rows > i read only DM_j, j > i
        }
      }
    }
    __syncwarp();
    const int rows = min(32, n - base);
    for (int r = 0; r < rows; r++) {
      u64* dst = out + (size_t)perm[base + r] * EVOKE_NUM_ORBITS_DEV;
      const u64* src = tile + (size_t)r * EVOKE_NUM_ORBITS_DEV;
      for (int i = lane; i < EVOKE_NUM_ORBITS_DEV; i += 32) dst[i] = src[i];
    }
    __syncwarp();
  }
}
