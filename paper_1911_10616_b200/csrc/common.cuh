// common.cuh -- shared device helpers for the EVOKE sm_100a kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

typedef unsigned long long u64;
typedef unsigned int u32;

#define EV_WARP 32
#define EVOKE_NUM_ORBITS_DEV 73
#define FULL_MASK 0xffffffffu

// ---------------------------------------------------------------------------
// Exact binomials modulo 2^64 (reading R20).  The argument x is an exact
// non-negative count (< 2^63); the factor divisible by k! is divided before the
// multiplications, so every product is a ring product and the result is
// C(x,k) mod 2^64 exactly, also when C(x,k) >= 2^64.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ u64 binom2(u64 x) {
  if (x < 2) return 0;
  u64 a = x, b = x - 1;
  if (a & 1) b >>= 1; else a >>= 1;
  return a * b;
}
__host__ __device__ __forceinline__ u64 binom3(u64 x) {
  if (x < 3) return 0;
  u64 f[3] = {x, x - 1, x - 2};
  for (int i = 0; i < 3; i++) if (f[i] % 3 == 0) { f[i] /= 3; break; }
  for (int i = 0; i < 3; i++) if ((f[i] & 1) == 0) { f[i] >>= 1; break; }
  return f[0] * f[1] * f[2];
}
__host__ __device__ __forceinline__ u64 binom4(u64 x) {
  if (x < 4) return 0;
  u64 f[4] = {x, x - 1, x - 2, x - 3};
  // of four consecutive integers one is = 0 (mod 4), one is = 2 (mod 4), and at least
  // one is = 0 (mod 3); 3 and 4 are coprime so the divisions commute
  for (int i = 0; i < 4; i++) if ((x - i) % 3 == 0) { f[i] /= 3; break; }
  for (int i = 0; i < 4; i++) {
    if (((x - i) & 3) == 0) f[i] >>= 2;
    else if (((x - i) & 3) == 2) f[i] >>= 1;
  }
  return f[0] * f[1] * f[2] * f[3];
}

// ---------------------------------------------------------------------------
// warp helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ u64 warp_sum(u64 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
  return v;
}
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ void atomic_add_u64(u64* p, u64 v) {
  if (v) atomicAdd(p, v);
}

// lower_bound of key in sorted a[lo, hi)
template <typename T>
__device__ __forceinline__ int64_t lower_bound_dev(const T* a, int64_t lo, int64_t hi, T key) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// bits strictly above position j within word w (word index w, 32-bit words)
__device__ __forceinline__ u32 gt_mask(int j, int w) {
  int jw = j >> 5;
  if (w < jw) return 0u;
  if (w > jw) return FULL_MASK;
  int b = j & 31;
  return b == 31 ? 0u : (FULL_MASK << (b + 1));
}
// bits strictly below position j within word w
__device__ __forceinline__ u32 lt_mask(int j, int w) {
  int jw = j >> 5;
  if (w < jw) return FULL_MASK;
  if (w > jw) return 0u;
  int b = j & 31;
  return b == 0 ? 0u : (FULL_MASK >> (32 - b));
}

// ---------------------------------------------------------------------------
// Device graph view (relabelled ids = degeneracy rank).
// ---------------------------------------------------------------------------
#define OUT8 8
#define OUT8_LONG (-2)
struct DGraph {
  int32_t n;
  int64_t m;            // undirected edges
  int64_t ntri;         // triangles
  int32_t max_deg, max_out;
  // undirected CSR, lists sorted ascending
  const int64_t* rp;    // [n+1]
  const int32_t* ci;    // [2m]
  const int32_t* dm;    // [n]  number of lower neighbours (in-degree in G->)
  const int32_t* deg;   // [n]  d(u) (one 4-byte load instead of two rowptr loads)
  const int32_t* eid;   // [2m] edge id of each slot
  // oriented out-CSR = edge ids
  const int64_t* orow;  // [n+1]
  const int32_t* ocol;  // [m]
  const int32_t* esrc;  // [m] lower endpoint
  const int32_t* edst;  // [m] higher endpoint
  const int64_t* eslot_hi; // [m] slot of esrc inside edst's list
  const int32_t* twin;  // [2m] for the slot of v in N(u): the slot of u in N(v)
  // out-lists of at most OUT8 vertices in one 32-byte row each: out8[8 j + t] = N+(j)[t],
  // -1 past the end; out8[8 j] = OUT8_LONG when d+(j) > OUT8 (then orow / ocol).  Built only
  // when every out-list is that short (nullptr otherwise)
  const int32_t* out8;
  // pair pass: for the slot of v in N(u), |N(v) above u| (written by k_pair_est)
  const int32_t* plen;
  // 5-cycle pass: for the slot of w in N(l), {start, length} of w's wedge list Nsel(w) (N(w) if
  // w < l, N+(w) if w > l) and, for w < l, of w's out-list in edge ids (k_c5_slots)
  const int4* c5s;
  // oriented triangle lists: edge e=(a->b): third vertices c > b, sorted
  const int64_t* toff;  // [m+1]
  const int32_t* tc;    // [ntri]
  const int32_t* tab;   // [ntri] owner edge (a,b)
  const int32_t* tac;   // [ntri] edge (a,c)
  const int32_t* tbc;   // [ntri] edge (b,c)
  // full triangle lists per undirected edge e=(lo,hi): (x, e(lo,x), e(hi,x))
  const int64_t* foff;  // [m+1]
  const int32_t* fx;    // [3 ntri]
  const int32_t* fe1;   // [3 ntri]
  const int32_t* fe2;   // [3 ntri]
  int32_t full_sorted;  // 1: every full list is sorted by x (prefix / suffix bounds by search)
  // per-slot copies of per-edge triangle counts, aligned with ci (streamed with the list
  // instead of a dependent load through eid): T(e), T_low(e), T_mid(e) of e = eid[s]
  const u32* tes;       // [2m]
  const u32* tlows;     // [2m]
  const u32* tmids;     // [2m]
};

__device__ __forceinline__ int32_t dg_deg(const DGraph& g, int32_t u) { return g.deg[u]; }
__device__ __forceinline__ int32_t dg_dplus(const DGraph& g, int32_t u) {
  return (int32_t)(g.orow[u + 1] - g.orow[u]);
}
// edge id between u and v given that x is the third vertex entry of the full list of
// edge e=(lo,hi): returns e(w, x) for w in {lo, hi}
__device__ __forceinline__ int32_t full_other_edge(const DGraph& g, int64_t r, int32_t e, int32_t w) {
  return (g.esrc[e] == w) ? g.fe1[r] : g.fe2[r];
}

// developer unit timers (EVOKE_DEBUG): per heavy persistent kernel ([0] pair heavy, [1]
// hub-local heavy, [2] 5-cycle big), SM cycles of the longest single unit, its list index,
// and the cycles summed over all units (thread 0 of the CTA)
__device__ unsigned long long g_unit_max[4], g_unit_sum[4];
__device__ int g_unit_arg[4];
__device__ int g_unit_prof;
__device__ __forceinline__ long long unit_t0() { return g_unit_prof && threadIdx.x == 0 ? clock64() : 0; }
__device__ __forceinline__ void unit_t1(int k, long long t0, int idx) {
  if (g_unit_prof && threadIdx.x == 0) {
    const unsigned long long d = (unsigned long long)(clock64() - t0);
    atomicAdd(&g_unit_sum[k], d);
    if (atomicMax(&g_unit_max[k], d) < d) g_unit_arg[k] = idx;
  }
}
