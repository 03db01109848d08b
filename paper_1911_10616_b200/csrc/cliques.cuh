// cliques.cuh -- steps a5 and a9 of SURVEY 8(a).
//
// One CTA per vertex u.  L = N+(u) (k = d+(u) <= degeneracy vertices, sorted), the
// local graph G[L] is held as a symmetric k x k bitmap S in shared memory, built from
// the oriented triangle lists of the edges (u, L_i) (a triangle (u, L_i, L_j) is local
// edge (i, j)).  Every clique is counted once, from its lowest vertex u:
//   4-cliques {u,i,j,l}   = triangles of G[L]      -> K4(v), K4(e)=E11, K4(t)
//   5-cliques {u,i,j,l,p} = 4-cliques of G[L]      -> K5(v) = DM72
// Per local vertex i the counts are popcounts of ANDed rows, so no per-clique atomics
// are needed for vertex and (u, L_i) edge credits.  K4(t) of a triangle t=(a<b<c) is
// (apexes above a, counted in a's frame) + (apexes below a: +1 from each lower u).
//
// MODE 1 (after K4(t) and E1 are final) credits theta66 (reading R12) and
// theta70 per 4-clique without enumerating cliques one by one for u's own
// theta66 credit.
#pragma once
#include "common.cuh"

template <typename F>
__device__ __forceinline__ void for_each_bit(u32 x, int base, F f) {
  while (x) {
    int b = __ffs(x) - 1;
    x &= x - 1;
    f(base + b);
  }
}

// rank of local j among the set bits of row R (restricted to bits > i): number of set
// bits of (R & GT(i)) strictly below j
__device__ __forceinline__ int row_rank(const u32* __restrict__ R, int W, int i, int j) {
  int r = 0;
  const int jw = j >> 5;
  for (int w = (i >> 5); w <= jw && w < W; w++) r += __popc(R[w] & gt_mask(i, w) & lt_mask(j, w));
  return r;
}

// One row i of the bitmap S of G[N+(u)] (k local vertices, W words per row): lanes take the
// columns j; the credits of L_i, of the local edges and triangles through i, and u's own
// sums (acc_u0, acc_u1; per lane, the caller reduces them).
template <int MODE>
__device__ __forceinline__ void clique_row(const DGraph& g, const u32* S, int W, int k, int64_t ou, int i,
                                           int lane, bool do_k4, bool do_k5, bool rows66, const u32* __restrict__ Te,
                                           u32* __restrict__ K4t, u64* __restrict__ K4v, u64* __restrict__ K4e,
                                           u64* __restrict__ K5v, u64* __restrict__ R66, u64* __restrict__ R70,
                                           u64& acc_u0, u64& acc_u1) {
  const u32* Si = S + (int64_t)i * W;
  const int32_t Li = g.ocol[ou + i];
  u64 a0 = 0, a1 = 0, a2 = 0;  // per-i accumulators
  const int64_t qi0 = g.toff[ou + i];
  for (int j = lane; j < k; j += 32) {
    if (!((Si[j >> 5] >> (j & 31)) & 1u)) continue;
    const u32* Sj = S + (int64_t)j * W;
    if (MODE == 0) {
      for (int w = (j >> 5); w < W; w++) {
        const u32 x = Si[w] & Sj[w] & gt_mask(j, w);
        if (do_k4) a0 += __popc(x);
        if (do_k5)
          for_each_bit(x, w << 5, [&](int l) {
            const u32* Sl = S + (int64_t)l * W;
            u64 c = 0;
            for (int w2 = (l >> 5); w2 < W; w2++) c += __popc(Si[w2] & Sj[w2] & Sl[w2] & gt_mask(l, w2));
            a1 += c;
          });
      }
      if (do_k4 && j > i) {
        u32 c = 0;
        for (int w = 0; w < W; w++) c += __popc(Si[w] & Sj[w]);
        const int64_t qij = qi0 + row_rank(Si, W, i, j);
        const int32_t eij = g.tbc[qij];
        if (c) {
          atomicAdd(&K4e[eij], (u64)c);
          atomicAdd(&K4t[qij], c);
        }
        // local triangles (i<j<l): triangle (L_i, L_j, L_l) gets apex u below it
        int64_t lo = g.toff[eij];
        const int64_t hi = g.toff[eij + 1];
        for (int w = (j >> 5); w < W; w++) {
          const u32 x = Si[w] & Sj[w] & gt_mask(j, w);
          for_each_bit(x, w << 5, [&](int l) {
            const int32_t Ll = g.ocol[ou + l];
            const int64_t pos = lower_bound_dev<int32_t>(g.tc, lo, hi, Ll);
            atomicAdd(&K4t[pos], 1u);
            lo = pos + 1;
          });
        }
      }
    } else {
      // theta66 / theta70 credits to L_i over the local edges (j,l) inside S_i (rows66; else
      // credited per local edge by clique_edges66)
      const u64 te_uj = Te[ou + j];
      const int64_t qj0 = g.toff[ou + j];
      for (int w = (j >> 5); rows66 && w < W; w++) {
        const u32 x = Si[w] & Sj[w] & gt_mask(j, w);
        for_each_bit(x, w << 5, [&](int l) {
          const int64_t qjl = qj0 + row_rank(Sj, W, j, l);
          a0 += te_uj + (u64)Te[ou + l] + (u64)Te[g.tbc[qjl]];
          a1 += (u64)K4t[qjl] - 1ull;
        });
      }
      if (j > i) {
        u32 c = 0;
        for (int w = 0; w < W; w++) c += __popc(Si[w] & Sj[w]);
        const int64_t qij = qi0 + row_rank(Si, W, i, j);
        const int32_t eij = g.tbc[qij];
        acc_u0 += (u64)Te[eij] * (u64)c;
        int64_t lo = g.toff[eij];
        const int64_t hi = g.toff[eij + 1];
        for (int w = (j >> 5); w < W; w++) {
          const u32 x = Si[w] & Sj[w] & gt_mask(j, w);
          for_each_bit(x, w << 5, [&](int l) {
            const int32_t Ll = g.ocol[ou + l];
            const int64_t pos = lower_bound_dev<int32_t>(g.tc, lo, hi, Ll);
            acc_u1 += (u64)K4t[pos] - 1ull;
            lo = pos + 1;
          });
        }
      }
    }
  }
  a0 = warp_sum(a0);
  a1 = warp_sum(a1);
  (void)a2;
  if (lane == 0) {
    if (MODE == 0) {
      if (do_k4 && a0) {
        atomicAdd(&K4v[Li], a0);
        atomicAdd(&K4e[ou + i], a0);
      }
      if (do_k5 && a1) atomicAdd(&K5v[Li], a1);
      acc_u0 += a0;
      acc_u1 += a1;
    } else {
      if (a0) atomicAdd(&R66[Li], a0);
      if (a1) atomicAdd(&R70[Li], a1);
    }
  }
}

// theta66 / theta70 credits of the local vertices, one local edge (j, l) at a time: the local
// edge is the oriented triangle q = (u, L_j, L_l) of u's out-edges, and every local i adjacent
// to both closes the 4-clique {u, L_i, L_j, L_l}; L_i gets T(u,L_j) + T(u,L_l) + T(L_j,L_l) for
// theta66 and K4(q) - 1 for theta70.  The per-q values are read once, coalesced over q, and
// the credits go to shared accumulators acc66/acc70 [k] (flushed by the caller) instead of a
// per-(i, j, l) rank search and three dependent global loads.
__device__ __forceinline__ void clique_edges66(const DGraph& g, const u32* S, int W, int64_t ou, int64_t q0,
                                               int64_t q1, int t, int nt, const u32* __restrict__ Te,
                                               const u32* __restrict__ K4t, u64* acc66, u64* acc70) {
  for (int64_t q = q0 + t; q < q1; q += nt) {
    const int32_t ej = g.tab[q], el = g.tac[q];
    const u64 f66 = (u64)Te[ej] + (u64)Te[el] + (u64)Te[g.tbc[q]];
    const u64 f70 = (u64)K4t[q] - 1ull;
    const u32* Sj = S + (int64_t)(ej - ou) * W;
    const u32* Sl = S + (int64_t)(el - ou) * W;
    for (int w = 0; w < W; w++)
      for_each_bit(Sj[w] & Sl[w], w << 5, [&](int i) {
        atomicAdd(&acc66[i], f66);
        if (f70) atomicAdd(&acc70[i], f70);
      });
  }
}

template <int MODE>
__global__ void __launch_bounds__(256) k_cliques(
    DGraph g, const int32_t* __restrict__ ulist, int nu, int smem_words, int acc66_words, int acc_k,
    u32* __restrict__ gscratch,
    int64_t gscratch_words, int do_k4, const uint8_t* __restrict__ mine,
    const u32* __restrict__ Te, u32* __restrict__ K4t, u64* __restrict__ K4v, u64* __restrict__ K4e,
    u64* __restrict__ K5v, u64* __restrict__ R66, u64* __restrict__ R70) {
  extern __shared__ u32 sh_bits[];
  __shared__ u64 red[1][2];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  if (threadIdx.x == 0) { red[0][0] = 0; red[0][1] = 0; }
  if (MODE == 1 && acc66_words > 0) {  // 2 x acc_k accumulators, kept zero between units by the flush
    u64* acc = reinterpret_cast<u64*>(sh_bits + acc66_words);
    for (int i = threadIdx.x; i < 2 * acc_k; i += blockDim.x) acc[i] = 0;
  }
  __syncthreads();
  for (int idx = blockIdx.x; idx < nu; idx += gridDim.x) {
    const int32_t u = ulist[idx];
    const bool in_shard = !mine || mine[u];  // this shard's units (work-balanced, deterministic)
    const bool do_k5 = (MODE == 0) && in_shard;
    if (MODE == 0 && !do_k4 && !do_k5) continue;
    if (MODE == 1 && !in_shard) continue;
    const int64_t ou = g.orow[u];
    const int k = (int)(g.orow[u + 1] - ou);
    const int W = (k + 31) >> 5;
    u32* S = ((int64_t)k * W <= smem_words) ? sh_bits : (gscratch + (int64_t)blockIdx.x * gscratch_words);
    for (int64_t t = threadIdx.x; t < (int64_t)k * W; t += blockDim.x) S[t] = 0u;
    __syncthreads();
    const int64_t q0 = g.toff[ou], q1 = g.toff[ou + k];
    for (int64_t q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
      const int i = (int)(g.tab[q] - ou), j = (int)(g.tac[q] - ou);
      atomicOr(&S[(int64_t)i * W + (j >> 5)], 1u << (j & 31));
      atomicOr(&S[(int64_t)j * W + (i >> 5)], 1u << (i & 31));
    }
    __syncthreads();
    u64 acc_u0 = 0, acc_u1 = 0;  // u's own credits (MODE 0: 3*#K4 and 4*#K5; MODE 1: th66, th70)
    // MODE 1, bitmap in shared memory: the local vertices' credits per local edge, into shared
    // accumulators after the bitmap (the launch sizes them; k <= the bin's kmax)
    const bool edges66 = MODE == 1 && S == sh_bits && acc66_words > 0;
    if (edges66) {
      u64* acc66 = reinterpret_cast<u64*>(sh_bits + acc66_words);
      u64* acc70 = acc66 + k;
      clique_edges66(g, S, W, ou, q0, q1, threadIdx.x, blockDim.x, Te, K4t, acc66, acc70);
      __syncthreads();
      for (int i = threadIdx.x; i < k; i += blockDim.x) {
        const int32_t Li = g.ocol[ou + i];
        if (acc66[i]) atomicAdd(&R66[Li], acc66[i]);
        if (acc70[i]) atomicAdd(&R70[Li], acc70[i]);
        acc66[i] = 0;
        acc70[i] = 0;
      }
    }
    for (int i = wib; i < k; i += nwb)
      clique_row<MODE>(g, S, W, k, ou, i, lane, do_k4, do_k5, !edges66, Te, K4t, K4v, K4e, K5v, R66, R70, acc_u0,
                       acc_u1);
    // block reduction of u's credits
    acc_u0 = warp_sum(acc_u0);
    acc_u1 = warp_sum(acc_u1);
    if (lane == 0) {
      atomicAdd(&red[0][0], acc_u0);
      atomicAdd(&red[0][1], acc_u1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const u64 s0 = red[0][0], s1 = red[0][1];
      if (MODE == 0) {
        if (do_k4 && s0) atomicAdd(&K4v[u], s0 / 3);  // each local triangle counted at its 3 vertices
        if (do_k5 && s1) atomicAdd(&K5v[u], s1 / 4);  // each local 4-clique counted at its 4 vertices
      } else {
        if (s0) atomicAdd(&R66[u], s0);
        if (s1) atomicAdd(&R70[u], s1);
      }
      red[0][0] = 0; red[0][1] = 0;
    }
    __syncthreads();
  }
}

// The rows of a one-word bitmap (k <= 32) with the (i, j) pairs, j in S_i, flattened over the
// lanes (warp_flat over the rows; __fns finds the pair's column): the same per-pair work as
// clique_row, but a warp no longer walks the k rows one after the other with only the k
// lanes of a row busy (config 4: k <= 8).  Per-row sums go to the warp's shared acc0/acc1
// [32] (MODE 0; flushed here), u's own sums to acc_u0/acc_u1 (per lane).
template <int MODE>
__device__ __forceinline__ void clique_pairs_w1(const DGraph& g, const u32* S, int k, int64_t ou, int lane,
                                                bool do_k4, bool do_k5, const u32* __restrict__ Te,
                                                u32* __restrict__ K4t, u64* __restrict__ K4v, u64* __restrict__ K4e,
                                                u64* __restrict__ K5v, u64* acc0, u64* acc1, u64& acc_u0,
                                                u64& acc_u1) {
  const u32 Sl_own = lane < k ? S[lane] : 0u;
  const int len = __popc(Sl_own);
  const int64_t qi0_own = lane < k ? g.toff[ou + lane] : 0;
  if (MODE == 0) { acc0[lane] = 0; acc1[lane] = 0; }
  __syncwarp();
  warp_flat(len, [&](int i, int kk, bool valid) {
    const u32 Si = __shfl_sync(FULL_MASK, Sl_own, i);
    const int64_t qi0 = __shfl_sync(FULL_MASK, qi0_own, i);
    if (!valid) return;
    const int j = __fns(Si, 0, kk + 1);  // the kk-th column of row i
    const u32 Sj = S[j];
    const u32 gtj = j == 31 ? 0u : (FULL_MASK << (j + 1));
    const u32 x = Si & Sj & gtj;  // local triangles (i, j, l), l > j
    if (MODE == 0) {
      if (do_k4 && x) atomicAdd(&acc0[i], (u64)__popc(x));
      if (do_k5) {
        u64 c5 = 0;
        for_each_bit(x, 0, [&](int l) {
          const u32 gtl = l == 31 ? 0u : (FULL_MASK << (l + 1));
          c5 += __popc(Si & Sj & S[l] & gtl);
        });
        if (c5) atomicAdd(&acc1[i], c5);
      }
    }
    if (j > i && (MODE == 1 || do_k4)) {
      const u32 c = __popc(Si & Sj);
      const u32 gti = i == 31 ? 0u : (FULL_MASK << (i + 1));
      const int64_t qij = qi0 + __popc(Si & gti & ((1u << j) - 1u));
      const int32_t eij = g.tbc[qij];
      if (MODE == 0) {
        if (c) {
          atomicAdd(&K4e[eij], (u64)c);
          atomicAdd(&K4t[qij], c);
        }
      } else {
        acc_u0 += (u64)Te[eij] * (u64)c;
      }
      int64_t lo = g.toff[eij];
      const int64_t hi = g.toff[eij + 1];
      for_each_bit(x, 0, [&](int l) {
        const int32_t Ll = g.ocol[ou + l];
        const int64_t pos = lower_bound_dev<int32_t>(g.tc, lo, hi, Ll);
        if (MODE == 0) atomicAdd(&K4t[pos], 1u);
        else acc_u1 += (u64)K4t[pos] - 1ull;
        lo = pos + 1;
      });
    }
  });
  __syncwarp();
  if (MODE == 0 && lane < k) {
    const u64 a0 = acc0[lane], a1 = acc1[lane];
    const int32_t Li = g.ocol[ou + lane];
    if (do_k4 && a0) {
      atomicAdd(&K4v[Li], a0);
      atomicAdd(&K4e[ou + lane], a0);
    }
    if (do_k5 && a1) atomicAdd(&K5v[Li], a1);
    acc_u0 += a0;
    acc_u1 += a1;
  }
  __syncwarp();
}

// Units with k = d+(u) <= 32 (one bitmap word per row): one WARP per unit instead of a CTA,
// the rows in a per-warp 32-word slice of shared memory (most units of a sparse graph:
// config 4 has degeneracy 8, so every unit is this small and a CTA per unit spent its time
// in barriers).
template <int MODE>
__global__ void __launch_bounds__(256) k_cliques_warp(
    DGraph g, const int32_t* __restrict__ ulist, int nu, int do_k4, const uint8_t* __restrict__ mine,
    const u32* __restrict__ Te, u32* __restrict__ K4t, u64* __restrict__ K4v, u64* __restrict__ K4e,
    u64* __restrict__ K5v, u64* __restrict__ R66, u64* __restrict__ R70) {
  __shared__ u32 sh_rows[8][32];
  __shared__ u64 sh_acc[8][64];  // per warp: theta66 / theta70 (MODE 1) or per-row K4 / K5 sums (MODE 0)
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  u32* S = sh_rows[wib & 7];
  u64* acc66 = sh_acc[wib & 7];
  u64* acc70 = acc66 + 32;
  if (MODE == 1) { acc66[lane] = 0; acc70[lane] = 0; }
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t idx = gw; idx < nu; idx += nw) {
    const int32_t u = ulist[idx];
    const bool in_shard = !mine || mine[u];
    const bool do_k5 = (MODE == 0) && in_shard;
    if (MODE == 0 && !do_k4 && !do_k5) continue;
    if (MODE == 1 && !in_shard) continue;
    const int64_t ou = g.orow[u];
    const int k = (int)(g.orow[u + 1] - ou);  // <= 32
    S[lane] = 0u;
    __syncwarp();
    const int64_t q0 = g.toff[ou], q1 = g.toff[ou + k];
    for (int64_t q = q0 + lane; q < q1; q += 32) {
      const int i = (int)(g.tab[q] - ou), j = (int)(g.tac[q] - ou);
      atomicOr(&S[i], 1u << j);
      atomicOr(&S[j], 1u << i);
    }
    __syncwarp();
    u64 acc_u0 = 0, acc_u1 = 0;
    if (MODE == 1) {
      clique_edges66(g, S, 1, ou, q0, q1, lane, 32, Te, K4t, acc66, acc70);
      __syncwarp();
      if (lane < k) {
        const int32_t Li = g.ocol[ou + lane];
        if (acc66[lane]) atomicAdd(&R66[Li], acc66[lane]);
        if (acc70[lane]) atomicAdd(&R70[Li], acc70[lane]);
        acc66[lane] = 0;
        acc70[lane] = 0;
      }
      __syncwarp();
    }
    clique_pairs_w1<MODE>(g, S, k, ou, lane, do_k4, do_k5, Te, K4t, K4v, K4e, K5v, acc66, acc70, acc_u0, acc_u1);
    acc_u0 = warp_sum(acc_u0);
    acc_u1 = warp_sum(acc_u1);
    if (lane == 0) {
      if (MODE == 0) {
        if (do_k4 && acc_u0) atomicAdd(&K4v[u], acc_u0 / 3);  // each local triangle counted at its 3 vertices
        if (do_k5 && acc_u1) atomicAdd(&K5v[u], acc_u1 / 4);  // each local 4-clique counted at its 4 vertices
      } else {
        if (acc_u0) atomicAdd(&R66[u], acc_u0);
        if (acc_u1) atomicAdd(&R70[u], acc_u1);
      }
    }
    __syncwarp();
  }
}
