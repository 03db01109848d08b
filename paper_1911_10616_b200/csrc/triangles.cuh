// triangles.cuh -- step a4 + a6 of SURVEY 8(a): triangle pass over the oriented graph
// (each triangle a<b<c found once as c in N+(a) & N+(b)), per-vertex T(v) (=DM3,
// P:716), per-edge T(e) (=E1), typed counts (third vertex below/between/above
// the edge's endpoints; used by the 5-cycle corrections), E7, the
// oriented triangle lists, then E9, DM12 and the full per-edge
// triangle lists.
#pragma once
#include "common.cuh"

// Warp per vertex a: N+(a) staged in shared memory; for every b in N+(a), the lanes
// stream N+(b) and binary-search each c in N+(a).
// PASS 0: Thigh[e_ab] = |N+(a) & N+(b)|.
// PASS 1: write oriented lists (sorted by c because N+(b) is sorted and the ballot
//         compaction keeps lane order) and credit T, Te, Tlow, Tmid, E7.
template <int PASS>
__global__ void __launch_bounds__(256) k_triangles(
    DGraph g, int smem_per_warp, u32* __restrict__ Thigh, u32* __restrict__ Tmid,
    u32* __restrict__ Tlow, u32* __restrict__ Te, u64* __restrict__ Tv, u64* __restrict__ E7,
    int32_t* __restrict__ tc, int32_t* __restrict__ tab, int32_t* __restrict__ tac,
    int32_t* __restrict__ tbc) {
  extern __shared__ int32_t sh_tri[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  int32_t* La = sh_tri + wib * smem_per_warp;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t a64 = gw; a64 < g.n; a64 += nw) {
    const int32_t a = (int32_t)a64;
    const int64_t oa = g.orow[a];
    const int32_t da = (int32_t)(g.orow[a + 1] - oa);
    if (da < 2) continue;
    const int32_t* L = g.ocol + oa;
    if (da <= smem_per_warp) {
      for (int i = lane; i < da; i += 32) La[i] = L[i];
      __syncwarp();
      L = La;
    }
    u64 ta = 0;
    const int32_t dga = dg_deg(g, a);
    for (int ib = 0; ib < da - 1; ib++) {
      const int32_t b = L[ib];
      const int64_t eab = oa + ib;
      const int64_t ob = g.orow[b];
      const int32_t db = (int32_t)(g.orow[b + 1] - ob);
      int64_t base = 0;
      if (PASS == 1) base = g.toff[eab];
      u32 cnt = 0;
      u64 e7ab = 0;
      const int32_t dgb = dg_deg(g, b);
      for (int j0 = 0; j0 < db; j0 += 32) {
        const int j = j0 + lane;
        bool found = false;
        int32_t c = 0;
        int64_t pos = 0;
        if (j < db) {
          c = g.ocol[ob + j];
          pos = lower_bound_dev<int32_t>(L, ib + 1, da, c);
          found = pos < da && L[pos] == c;
        }
        const u32 bal = __ballot_sync(FULL_MASK, found);
        if (PASS == 1 && found) {
          const int64_t q = base + cnt + __popc(bal & ((1u << lane) - 1u));
          const int32_t eac = (int32_t)(oa + pos), ebc = (int32_t)(ob + j);
          tc[q] = c; tab[q] = (int32_t)eab; tac[q] = eac; tbc[q] = ebc;
          atomicAdd(&Tv[c], 1ull);
          atomicAdd(&Te[eac], 1u);
          atomicAdd(&Te[ebc], 1u);
          atomicAdd(&Tmid[eac], 1u);
          atomicAdd(&Tlow[ebc], 1u);
          const int32_t dgc = dg_deg(g, c);
          e7ab += (u64)(dgc - 2);
          atomicAdd(&E7[eac], (u64)(dgb - 2));
          atomicAdd(&E7[ebc], (u64)(dga - 2));
        }
        cnt += __popc(bal);
      }
      if (PASS == 0) {
        if (lane == 0) Thigh[eab] = cnt;
      } else {
        e7ab = warp_sum(e7ab);
        if (lane == 0 && cnt) {
          atomicAdd(&Te[eab], cnt);
          atomicAdd(&Tv[b], (u64)cnt);
          atomicAdd(&E7[eab], e7ab);
        }
        ta += cnt;
      }
    }
    if (PASS == 1 && lane == 0 && ta) atomicAdd(&Tv[a], ta);
    __syncwarp();
  }
}

// Graphs whose out-lists are all short (max d+ <= 32): the same pass with the (b, c) pairs
// of a vertex flattened over the lanes (warp_flat over the items b in N+(a)), so a warp does
// not walk N+(a) one b at a time with most lanes idle (config 4: d+ <= 8).  The lanes of one
// item are consecutive, so a found c's rank inside its list is the item's count so far
// (per-warp shared) plus the found lanes below it among the item's lanes (match_any mask);
// the lists stay sorted by c.
#ifndef TRIFLAT_MINB
#define TRIFLAT_MINB 8  // resident CTAs per SM the register budget must allow (config 4: 2.57 -> 2.44 ms)
#endif
template <int PASS>
__global__ void __launch_bounds__(256, TRIFLAT_MINB) k_triangles_flat(
    DGraph g, u32* __restrict__ Thigh, u32* __restrict__ Tmid, u32* __restrict__ Tlow, u32* __restrict__ Te,
    u64* __restrict__ Tv, u64* __restrict__ E7, int32_t* __restrict__ tc, int32_t* __restrict__ tab,
    int32_t* __restrict__ tac, int32_t* __restrict__ tbc) {
  __shared__ int32_t sh_L[8][32];
  __shared__ u32 sh_cnt[8][32];
  __shared__ u64 sh_e7[8][32];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  int32_t* La = sh_L[wib];
  u32* cnt = sh_cnt[wib];
  u64* e7 = sh_e7[wib];
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t a64 = gw; a64 < g.n; a64 += nw) {
    const int32_t a = (int32_t)a64;
    const int64_t oa = g.orow[a];
    const int32_t da = (int32_t)(g.orow[a + 1] - oa);  // <= 32
    if (da < 2) continue;
    const int32_t dga = dg_deg(g, a);
    // item lane i < da - 1: b = N+(a)[i], its out-list
    int32_t b = 0, db = 0, dgb = 0;
    int64_t ob = 0, base = 0;
    if (lane < da) {
      b = g.ocol[oa + lane];
      La[lane] = b;
    }
    if (lane < da - 1) {
      ob = g.orow[b];
      db = (int32_t)(g.orow[b + 1] - ob);
      dgb = dg_deg(g, b);
      if (PASS == 1) base = g.toff[oa + lane];
    }
    cnt[lane] = 0u;
    if (PASS == 1) e7[lane] = 0ull;
    __syncwarp();
    warp_flat(db, [&](int j, int k, bool valid) {
      const int64_t obj = __shfl_sync(FULL_MASK, ob, j);
      const int64_t basej = __shfl_sync(FULL_MASK, base, j);
      const int32_t dgbj = __shfl_sync(FULL_MASK, dgb, j);
      bool found = false;
      int32_t c = 0;
      int64_t pos = 0;
      if (valid) {
        c = g.ocol[obj + k];
        pos = lower_bound_dev<int32_t>(La, j + 1, da, c);
        found = pos < da && La[pos] == c;
      }
      const unsigned same = __match_any_sync(FULL_MASK, valid ? j : -1);
      const unsigned bal = __ballot_sync(FULL_MASK, found) & same;
      const u32 before = cnt[j];  // (every lane of the group reads it before the leader adds)
      __syncwarp();
      if (valid && lane == __ffs(same) - 1) cnt[j] = before + __popc(bal);
      if (PASS == 1 && found) {
        const int64_t q = basej + before + __popc(bal & ((1u << lane) - 1u));
        const int32_t eac = (int32_t)(oa + pos), ebc = (int32_t)(obj + k);
        tc[q] = c; tab[q] = (int32_t)(oa + j); tac[q] = eac; tbc[q] = ebc;
        atomicAdd(&Tv[c], 1ull);
        atomicAdd(&Te[eac], 1u);
        atomicAdd(&Te[ebc], 1u);
        atomicAdd(&Tmid[eac], 1u);
        atomicAdd(&Tlow[ebc], 1u);
        atomicAdd(&e7[j], (u64)(dg_deg(g, c) - 2));
        atomicAdd(&E7[eac], (u64)(dgbj - 2));
        atomicAdd(&E7[ebc], (u64)(dga - 2));
      }
      __syncwarp();
    });
    __syncwarp();
    const u32 cb = lane < da - 1 ? cnt[lane] : 0u;
    if (PASS == 0) {
      if (lane < da - 1) Thigh[oa + lane] = cb;
    } else {
      if (cb) {
        atomicAdd(&Te[oa + lane], cb);
        atomicAdd(&Tv[b], (u64)cb);
        atomicAdd(&E7[oa + lane], e7[lane]);
      }
      const u64 ta = warp_sum((u64)cb);
      if (lane == 0 && ta) atomicAdd(&Tv[a], ta);
    }
    __syncwarp();
  }
}

__global__ void k_fcur_init(int64_t m, const int64_t* __restrict__ foff, const u32* __restrict__ Thigh,
                            int64_t* __restrict__ fcur) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x)
    fcur[e] = foff[e] + Thigh[e];
}

// Thread per oriented triangle entry q (a<b<c): E9 for the six ordered edges
// (E9<x,y> = sum over triangles (x,y,z) of E1(x,z)-1), DM12 for the three
// vertices (sum over triangles (u,v,x) of T(v,x)-1), and the full per-edge
// lists: for edge e=(lo,hi) entries (x, e(lo,x), e(hi,x)).
#ifndef SWEEP1_MINB
#define SWEEP1_MINB 1  // (developer variant: resident 256-thread CTAs per SM for the register budget)
#endif
__global__ void __launch_bounds__(256, SWEEP1_MINB) k_tri_sweep1(DGraph g, const u32* __restrict__ Te, u64* __restrict__ E9f,
                             u64* __restrict__ E9b, u64* __restrict__ DM12,
                             int64_t* __restrict__ fcur, int32_t* __restrict__ fx,
                             int32_t* __restrict__ fe1, int32_t* __restrict__ fe2) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < g.ntri;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int32_t eab = g.tab[q], eac = g.tac[q], ebc = g.tbc[q];
    const int32_t a = g.esrc[eab], b = g.edst[eab], c = g.tc[q];
    const u64 tab_ = Te[eab], tac_ = Te[eac], tbc_ = Te[ebc];
    atomicAdd(&E9f[eab], tac_ - 1);  // <a,b>
    atomicAdd(&E9b[eab], tbc_ - 1);  // <b,a>
    atomicAdd(&E9f[eac], tab_ - 1);  // <a,c>
    atomicAdd(&E9b[eac], tbc_ - 1);  // <c,a>
    atomicAdd(&E9f[ebc], tab_ - 1);  // <b,c>
    atomicAdd(&E9b[ebc], tac_ - 1);  // <c,b>
    atomicAdd(&DM12[a], tbc_ - 1);
    atomicAdd(&DM12[b], tac_ - 1);
    atomicAdd(&DM12[c], tab_ - 1);
    int64_t r;
    // the owner edge's entries come first, in oriented-list order (no atomic); the two other
    // roles append after them (fcur starts at foff + Thigh)
    r = g.foff[eab] + (q - g.toff[eab]);
    fx[r] = c; fe1[r] = eac; fe2[r] = ebc;
    r = (int64_t)atomicAdd((unsigned long long*)&fcur[eac], 1ull);
    fx[r] = b; fe1[r] = eab; fe2[r] = ebc;
    r = (int64_t)atomicAdd((unsigned long long*)&fcur[ebc], 1ull);
    fx[r] = a; fe1[r] = eab; fe2[r] = eac;
  }
}

// Sorting the full per-edge triangle lists by third vertex (once, for triangle-heavy graphs):
// key = (edge id << 32) | x for every entry, then one radix sort of (key, entry) pairs.
__global__ void k_full_keys(DGraph g, u64* __restrict__ keys, int32_t* __restrict__ idx) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < g.m; e += (int64_t)gridDim.x * blockDim.x)
    for (int64_t r = g.foff[e]; r < g.foff[e + 1]; r++) {
      keys[r] = ((u64)e << 32) | (u32)g.fx[r];
      idx[r] = (int32_t)r;
    }
}
__global__ void k_full_apply(int64_t N, const u64* __restrict__ skeys, const int32_t* __restrict__ sidx,
                             const int32_t* __restrict__ fe1_old, const int32_t* __restrict__ fe2_old,
                             int32_t* __restrict__ fx, int32_t* __restrict__ fe1, int32_t* __restrict__ fe2) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < N; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t q = sidx[r];
    fx[r] = (int32_t)(u32)(skeys[r] & 0xffffffffull);
    fe1[r] = fe1_old[q];
    fe2[r] = fe2_old[q];
  }
}
