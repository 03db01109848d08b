// hublocal.cuh -- step a8 of SURVEY 8(a): the hub-local (diamond) pass for the wheel W4
// = H27 (theta68, theta69; Theorem B.1, readings R11, R13).
//
//   theta68(a) = sum_{v in N(a)} sum_{x in N(v)\a} C(|N(v)&N(a)&N(x)|, 2)
//              = sum over hubs v in N(a) of the number of 4-cycles of G[N(v)] through a
//   theta69(v) = 1/2 sum_{a,x in N(v)} C(|N(v)&N(a)&N(x)|, 2) = #4-cycles of G[N(v)]
//
// Work item = slot (v, a), a in N(v) with T(v,a) >= 2: a is the TOP (highest rank)
// vertex of the 4-cycles a-b-x-b' of G[N(v)] found from this item: the item enumerates
// b in N(v)&N(a) with b < a and x in N(v)&N(b) with x < a and counts c(x) = #such b.
// Each 4-cycle of G[N(v)] is found exactly once (from its top vertex, opposite x); its
// four corners are credited:
//   a, x    : C(c(x), 2) each           (theta68)
//   b (mid) : c(x) - 1 for every x      (theta68)
//   v       : C(c(x), 2)                (theta69)  -- no division modulo 2^64 needed.
// Restricting to cycles whose top is a (Chiba-Nishizeki) is what bounds the work.
//
// Scheduling (B200): k_hub_est measures every item's inner work
//   est(v,a) = sum_{b in tri(v,a), b<a} T(v,b)
// (one thread per triangle) and k_hub_bin splits the items into a heavy list
// (est > HUB_WARP_MAX, sorted by est, descending) and a light list.  k_hub_process is
// persistent: its CTAs first take heavy items one CTA per item (block-flattened (b, x)
// loop, c(x) in a dense shared table indexed by x's position in N(v), or a per-CTA
// global one for hubs beyond the shared capacity), then every warp takes light items
// (warp-flattened loop, c(x) in a per-warp shared hash keyed by x).  Work per lane is
// balanced no matter how heavy-tailed T(e) is.
#pragma once
#include "common.cuh"
#include "sched.cuh"

#define HUB_BT 256                                   // threads per CTA of the light-item kernel (8 warps)
#define HUB_WARP_CAP 1024                            // per-warp hash capacity (light items)
#define HUB_WARP_MAX (HUB_WARP_CAP / 2)              // light item: est <= this
#define HUB_SMEM (HUB_BT / 32 * HUB_WARP_CAP * 12)   // 96 KB dynamic shared memory
#define HUB_GSMEM (200 << 10)                        // giant items: 1024-thread CTA (one per SM), this much shared memory
#define HUB_HSMEM (44 << 10)                         // heavy items: 256-thread CTAs (four per SM), this much each
#define HUB_GIANT (1u << 20)                         // item est above this: giant
#define HUB_SH_DENSE (HUB_GSMEM / 2)                 // shared 16-bit counts by position if d(v) <= min(this, smem / 2)
#define HUB_HASH_MAX (((HUB_GSMEM / 6) & ~1) * 3 / 4)  // x-keyed shared hash if min(d(v)-1, est) <= min(this, 3/4 slots)
#define HUB_FEW_ITEMS 262144                         // at most this many items: one CTA per SM
#define HUB_LONG 32                                  // heavy item: x-lists this long are streamed by a whole warp
#define HUB_ILP 4                                    // ... with this many loads per lane in flight
#define HUB_SPLIT 256                                // heavy item: longer x-lists are chunked over the CTA
#define HUB_MICRO_MAX 16                             // micro item: est <= this, one THREAD per item

// number of entries of the full list [f, f+len) with third vertex < bound: a binary search
// when the lists are sorted (g.full_sorted), else the whole list (callers then filter)
__device__ __forceinline__ int full_prefix(const DGraph& g, int64_t f, int len, int32_t bound) {
  if (!g.full_sorted) return len;
  return (int)(lower_bound_dev<int32_t>(g.fx, f, f + len, bound) - f);
}

// position of x inside N(v) given the edge id e(v,x)
__device__ __forceinline__ int64_t pos_in_list(const DGraph& g, int32_t v, int32_t x, int32_t evx) {
  return (v < x) ? ((int64_t)g.dm[v] + (evx - g.orow[v])) : (g.eslot_hi[evx] - g.rp[v]);
}

// ---- item measurement and binning ---------------------------------------------------
// est(v,a) = sum_{b in tri(v,a), b<a} T(v,b) summed per triangle instead of per item: a
// triangle a<b<c (ranks) has a third vertex below the item's far end exactly for the items
// (a,c) [b<c], (b,c) [a<c] and (c,b) [a<b], which receive T(a,b), T(b,a) and T(c,a).  One
// thread per triangle, three atomics: balanced however heavy-tailed the lists are (a warp
// per item would leave the hub edges' thousands of entries to single warps).
__global__ void k_hub_est(DGraph g, const u32* __restrict__ Te, u64* __restrict__ est) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < g.ntri;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int32_t eab = g.tab[q], eac = g.tac[q], ebc = g.tbc[q];
    const u64 tab_ = Te[eab], tac_ = Te[eac];
    atomicAdd((unsigned long long*)&est[slot_of_hi_in_lo(g, eac)], tab_);  // item (a, c)
    atomicAdd((unsigned long long*)&est[slot_of_hi_in_lo(g, ebc)], tab_);  // item (b, c)
    atomicAdd((unsigned long long*)&est[g.eslot_hi[ebc]], tac_);          // item (c, b)
  }
}

// items (slot s of a in N(v)) with T(v,a) >= 2 and est > 0, of this shard (mine[s], nullptr:
// every item): micro (est <= micro_max <= HUB_MICRO_MAX), light (est <= warp_max <=
// HUB_WARP_MAX) or heavy (with est for the sort)
__global__ void k_hub_bin(DGraph g, const u32* __restrict__ Te, const u64* __restrict__ est,
                          const uint8_t* __restrict__ mine, u64 micro_max, u64 warp_max, int32_t* __restrict__ micro,
                          int* n_micro, int32_t* __restrict__ light, int* n_light, int32_t* __restrict__ heavy,
                          u32* __restrict__ heavy_est, int* n_heavy, u64 giant_min, int* n_giant) {
  const int lane = threadIdx.x & 31;
  const int64_t m2 = 2 * g.m;
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll; base < m2;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = base + lane;
    u64 e = 0;
    if (s < m2 && g.tes[s] >= 2 && (!mine || mine[s])) e = est[s];  // (T(v,a) per slot: no edge-id load)
    warp_append(e > 0 && e <= micro_max, (int32_t)s, micro, n_micro);
    warp_append(e > micro_max && e <= warp_max, (int32_t)s, light, n_light);
    const bool is_heavy = e > warp_max;
    {
      const u32 gb = __ballot_sync(FULL_MASK, is_heavy && e > giant_min);
      if (lane == 0 && gb) atomicAdd(n_giant, __popc(gb));
    }
    const u32 bal = __ballot_sync(FULL_MASK, is_heavy);
    if (bal) {
      int hb = 0;
      const int leader = __ffs(bal) - 1;
      if (lane == leader) hb = atomicAdd(n_heavy, __popc(bal));
      hb = __shfl_sync(FULL_MASK, hb, leader);
      if (is_heavy) {
        const int q = hb + __popc(bal & ((1u << lane) - 1u));
        heavy[q] = (int32_t)s;
        heavy_est[q] = (u32)min(e, (u64)0xffffffffu);
      }
    }
  }
}

// ---- micro item: one thread ------------------------------------------------------------
// Items with est <= HUB_MICRO_MAX (most items of a sparse graph: config 4 averages 4.5 inner
// visits per item) are too small for a warp: one lane per item keeps its (b, x) pairs in a
// local array and counts c(x) by comparison, so a warp works on 32 items at once.
__global__ void k_hub_micro(DGraph g, const int32_t* __restrict__ items, int n_items, u64* __restrict__ R68,
                            u64* __restrict__ R69) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_items; q += gridDim.x * blockDim.x) {
    const int32_t s = items[q];
    const int32_t eva = g.eid[s];
    const int32_t a = g.ci[s];
    const int32_t lo_ = g.esrc[eva];
    const int32_t v = lo_ + g.edst[eva] - a;
    const bool v_lo = lo_ == v;
    const int64_t fa = g.foff[eva];
    const int na = full_prefix(g, fa, (int)(g.foff[eva + 1] - fa), a);  // b < a (or all, filtered)
    int32_t xs[HUB_MICRO_MAX];
    int8_t xb[HUB_MICRO_MAX];
    int32_t bs[HUB_MICRO_MAX];
    int cnt = 0, nb = 0;
    for (int i = 0; i < na; i++) {
      const int64_t r = fa + i;
      const int32_t b = g.fx[r];
      if (b >= a) continue;
      const int32_t evb = v_lo ? g.fe1[r] : g.fe2[r];
      const int64_t fb = g.foff[evb];
      const int len = full_prefix(g, fb, (int)(g.foff[evb + 1] - fb), a);  // x < a
      for (int k = 0; k < len; k++) {
        const int32_t x = g.fx[fb + k];
        if (x >= a) continue;
        xs[cnt] = x;  // cnt <= est(v,a) <= HUB_MICRO_MAX
        xb[cnt] = (int8_t)nb;
        cnt++;
      }
      bs[nb++] = b;  // T(v,b) >= 1 (a is a common neighbour), so nb <= est
    }
    u64 sb[HUB_MICRO_MAX];
    for (int t = 0; t < nb; t++) sb[t] = 0;
    u64 r69 = 0;
    for (int p = 0; p < cnt; p++) {
      int c = 0;
      bool first = true;
      for (int t = 0; t < cnt; t++) {
        if (xs[t] == xs[p]) {
          c++;
          if (t < p) first = false;
        }
      }
      sb[xb[p]] += (u64)(c - 1);  // R68[b] += c(x) - 1 for every x of b
      if (first && c >= 2) {
        const u64 c2 = binom2((u64)c);
        r69 += c2;
        atomicAdd(&R68[xs[p]], c2);
      }
    }
    for (int t = 0; t < nb; t++)
      if (sb[t]) atomicAdd(&R68[bs[t]], sb[t]);
    if (r69) {
      atomicAdd(&R69[v], r69);
      atomicAdd(&R68[a], r69);
    }
  }
}

// ---- heavy item: one CTA ----------------------------------------------------------------
// The CTA's warps take the item's middles b in groups of 32 (a shared counter) and flatten
// their short x-lists over the lanes (warp_flat): no per-element search, and the pass-2 sums
// of a middle stay in a lane's register while the lane stays on it.  Lists of HUB_LONG or
// more elements are streamed by a whole warp (HUB_ILP loads per lane in flight); lists longer
// than HUB_SPLIT go to a CTA queue and are cut into HUB_SPLIT-element chunks that all warps
// share, so one hub middle does not keep the other warps waiting at the pass barrier.
// c(x) lives in one of three tables, chosen per item:
//   HUB_T_HASH : shared open-addressing hash keyed by x (x+1, 0 = empty) when the number of
//                distinct x, at most min(d(v)-1, est(v,a)), fits hash_max -- no per-element
//                position lookup (fe1/fe2 and the slot map of x in N(v) are never read);
//   HUB_T_SHPOS: shared counts dense by x's position in N(v) (d(v) <= sh_dense_max), swept;
//   HUB_T_GLPOS: a per-CTA global u32 table by position with a touched list (larger hubs).
// The shared tables hold 16-bit counts, two per word: c(x) <= #middles <= T(v,a) < 2^16
// (checked per item), so an increment never carries into the neighbouring count.  All three
// are left zeroed (shared memory is zero between items in every mode).
enum { HUB_T_HASH = 0, HUB_T_SHPOS = 1, HUB_T_GLPOS = 2 };
#define HUB_QCAP 256   // queued long lists per CTA and pass
template <int BT>
struct HubCtaSharedT {
  int next;   // group counter of the current pass
  int cnt;    // touched entries (global table)
  int qn;     // queued long lists
  int qnext;  // chunk counter of the queue
  u64 r69;
  u64 acc[BT / 32][32];  // per-warp sums of the current 32 middles (pass 2)
  int64_t qfb[HUB_QCAP];
  int qlen[HUB_QCAP];
  int32_t qb[HUB_QCAP];
  int qc0[HUB_QCAP + 1];  // first chunk of every queued list
  bool qvl[HUB_QCAP];
};

__device__ __forceinline__ u32 hub_h0(int32_t x, u32 cap) { return __umulhi((u32)x * 0x9E3779B1u, cap); }

template <int MODE, int BT>
__device__ void hub_item_cta(const DGraph& g, int32_t s, u32 cap, u32* shm, HubCtaSharedT<BT>& S,
                             u32* __restrict__ gtab, int32_t* __restrict__ glist, u64* __restrict__ R68,
                             u64* __restrict__ R69, int split) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int32_t eva = g.eid[s];
  const int32_t a = g.ci[s];
  const int32_t lo_ = g.esrc[eva];
  const int32_t v = lo_ + g.edst[eva] - a;
  const bool v_lo = lo_ == v;
  const int64_t rpv = g.rp[v];
  const int32_t dv = (int32_t)(g.rp[v + 1] - rpv);
  const int64_t fa = g.foff[eva];
  const int na = full_prefix(g, fa, (int)(g.foff[eva + 1] - fa), a);  // b < a (or all, filtered)
  int32_t* hkeys = reinterpret_cast<int32_t*>(shm);                 // HUB_T_HASH: x + 1
  u32* c16 = MODE == HUB_T_HASH ? shm + cap : shm;                   // shared 16-bit counts
  u32* tab = gtab;                                                   // HUB_T_GLPOS
  u64* acc = S.acc[wib];
  if (threadIdx.x == 0) { S.cnt = 0; S.r69 = 0; }
  acc[lane] = 0;
  // the count slot of x (pass 1: found or claimed; pass 2: found -- every x of pass 2 was
  // inserted by pass 1); r2 = x's entry in the full list, vlj: fe1 holds e(v,x)
  auto slot_of = [&](int pass, int32_t x, int64_t r2, bool vlj) -> u32 {
    if (MODE == HUB_T_HASH) {
      u32 h = hub_h0(x, cap);
      if (pass == 1) {
        for (;;) {
          const int32_t kk = hkeys[h];
          if (kk == x + 1) break;
          if (kk == 0) {
            const int32_t o = atomicCAS(&hkeys[h], 0, x + 1);
            if (o == 0 || o == x + 1) break;
          }
          h = (h + 1 == cap) ? 0 : h + 1;
        }
      } else {
        while (hkeys[h] != x + 1) h = (h + 1 == cap) ? 0 : h + 1;
      }
      return h;
    }
    const int32_t evx = vlj ? g.fe1[r2] : g.fe2[r2];
    return (u32)pos_in_list(g, v, x, evx);
  };
  auto bump = [&](u32 h) {
    if (MODE == HUB_T_GLPOS) {
      if (atomicAdd(&tab[h], 1u) == 0u) glist[atomicAdd(&S.cnt, 1)] = (int32_t)h;
    } else {
      atomicAdd(&c16[h >> 1], 1u << ((h & 1) * 16));
    }
  };
  auto count = [&](u32 h) -> u64 {
    if (MODE == HUB_T_GLPOS) return (u64)tab[h];
    return (u64)((c16[h >> 1] >> ((h & 1) * 16)) & 0xffffu);
  };
  // the whole warp streams elements [k0, k1) of one list; returns the lane's pass-2 sum
  auto stream = [&](int pass, int64_t fbj, int k0, int k1, bool vlj) -> u64 {
    u64 sum = 0;
    for (int kb = k0; kb < k1; kb += 32 * HUB_ILP) {
      int32_t xs[HUB_ILP];
#pragma unroll
      for (int u = 0; u < HUB_ILP; u++) {
        const int k = kb + 32 * u + lane;
        xs[u] = k < k1 ? g.fx[fbj + k] : a;
      }
#pragma unroll
      for (int u = 0; u < HUB_ILP; u++) {
        if (xs[u] >= a) continue;
        const u32 h = slot_of(pass, xs[u], fbj + kb + 32 * u + lane, vlj);
        if (pass == 1) bump(h);
        else sum += count(h) - 1ull;
      }
    }
    return sum;
  };
#pragma unroll 1
  for (int pass = 1; pass <= 2; pass++) {
    if (threadIdx.x == 0) { S.next = 0; S.qn = 0; S.qnext = 0; }
    __syncthreads();
    for (;;) {
      int i0 = 0;
      if (lane == 0) i0 = atomicAdd(&S.next, 32);
      i0 = __shfl_sync(FULL_MASK, i0, 0);
      if (i0 >= na) break;
      const int i = i0 + lane;
      int len = 0;
      int64_t fb = 0;
      int32_t b = 0;
      bool vl = false;  // v is the lower end of e(v,b): fe1 holds e(v,x)
      if (i < na) {
        const int64_t r = fa + i;
        b = g.fx[r];
        if (b < a) {
          const int32_t evb = v_lo ? g.fe1[r] : g.fe2[r];
          fb = g.foff[evb];
          len = full_prefix(g, fb, (int)(g.foff[evb + 1] - fb), a);  // x < a
          if (MODE != HUB_T_HASH) vl = g.esrc[evb] == v;
        }
      }
      // very long lists: to the CTA queue (chunks shared by all warps) while it has room
      if (len > split) {
        const int q = atomicAdd(&S.qn, 1);
        if (q < HUB_QCAP) {
          S.qfb[q] = fb; S.qlen[q] = len; S.qb[q] = b; S.qvl[q] = vl;
          len = 0;
        }
      }
      // long lists: the whole warp streams one list at a time
      unsigned lm = __ballot_sync(FULL_MASK, len >= HUB_LONG);
      while (lm) {
        const int j = __ffs(lm) - 1;
        lm &= lm - 1;
        const int64_t fbj = __shfl_sync(FULL_MASK, fb, j);
        const int lenj = __shfl_sync(FULL_MASK, len, j);
        const bool vlj = MODE != HUB_T_HASH && __shfl_sync(FULL_MASK, vl, j);
        const int32_t bj = __shfl_sync(FULL_MASK, b, j);
        const u64 sum = warp_sum(stream(pass, fbj, 0, lenj, vlj));
        if (pass == 2 && lane == 0 && sum) atomicAdd(&R68[bj], sum);
        if (lane == j) len = 0;
      }
      int cur = -1;
      u64 cacc = 0;
      warp_flat(len, [&](int j, int k, bool valid) {
        const int64_t fbj = __shfl_sync(FULL_MASK, fb, j);
        const bool vlj = MODE != HUB_T_HASH && __shfl_sync(FULL_MASK, vl, j);
        if (!valid) return;
        const int64_t r2 = fbj + k;
        const int32_t x = g.fx[r2];
        if (x >= a) return;
        const u32 h = slot_of(pass, x, r2, vlj);
        if (pass == 1) {
          bump(h);
        } else {
          if (j != cur) {
            if (cur >= 0 && cacc) atomicAdd(&acc[cur], cacc);
            cur = j;
            cacc = 0;
          }
          cacc += count(h) - 1ull;  // middles b get sum over their x of c(x) - 1
        }
      });
      if (pass == 2) {
        if (cur >= 0 && cacc) atomicAdd(&acc[cur], cacc);
        __syncwarp();
        const u64 sb = acc[lane];
        acc[lane] = 0;
        if (sb) atomicAdd(&R68[b], sb);
        __syncwarp();
      }
    }
    __syncthreads();
    // the queued lists, in HUB_SPLIT-element chunks over all warps
    const int nq = min(S.qn, HUB_QCAP);
    if (nq > 0) {
      if (threadIdx.x == 0) {
        int c = 0;
        for (int q = 0; q < nq; q++) { S.qc0[q] = c; c += (S.qlen[q] + split - 1) / split; }
        S.qc0[nq] = c;
      }
      __syncthreads();
      const int nchunks = S.qc0[nq];
      for (;;) {
        int c = 0;
        if (lane == 0) c = atomicAdd(&S.qnext, 1);
        c = __shfl_sync(FULL_MASK, c, 0);
        if (c >= nchunks) break;
        int lo = 0, hi = nq;  // the list of chunk c: largest lo with qc0[lo] <= c
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (S.qc0[mid] <= c) lo = mid; else hi = mid;
        }
        const int k0 = (c - S.qc0[lo]) * split;
        const int k1 = min(S.qlen[lo], k0 + split);
        const u64 sum = warp_sum(stream(pass, S.qfb[lo], k0, k1, S.qvl[lo]));
        if (pass == 2 && lane == 0 && sum) atomicAdd(&R68[S.qb[lo]], sum);
      }
      __syncthreads();
    }
  }
  // pass 3: corners a, x and the hub v; clear the table
  u64 r69 = 0;
  if (MODE == HUB_T_HASH) {
    for (u32 h = threadIdx.x; h < cap; h += BT) {
      const int32_t kk = hkeys[h];
      if (kk == 0) continue;
      const u64 c2 = binom2(count(h));
      hkeys[h] = 0;
      if (c2) {
        r69 += c2;
        atomicAdd(&R68[kk - 1], c2);
      }
    }
    __syncthreads();
    for (u32 w = threadIdx.x; w < (cap + 1) / 2; w += BT) c16[w] = 0u;
  } else if (MODE == HUB_T_SHPOS) {
    for (int32_t p = threadIdx.x; p < dv; p += BT) {
      const u64 c2 = binom2(count((u32)p));
      if (c2) {
        r69 += c2;
        atomicAdd(&R68[g.ci[rpv + p]], c2);
      }
    }
    __syncthreads();
    for (int32_t w = threadIdx.x; w < (dv + 1) / 2; w += BT) c16[w] = 0u;
  } else {
    const int cnt = S.cnt;
    for (int t = threadIdx.x; t < cnt; t += BT) {
      const int32_t p = glist[t];
      const u64 c2 = binom2(tab[p]);
      tab[p] = 0u;
      if (c2) {
        r69 += c2;
        atomicAdd(&R68[g.ci[rpv + p]], c2);
      }
    }
  }
  r69 = warp_sum(r69);
  if (lane == 0 && r69) atomicAdd(&S.r69, r69);
  __syncthreads();
  if (threadIdx.x == 0 && S.r69) {
    atomicAdd(&R69[v], S.r69);
    atomicAdd(&R68[a], S.r69);
  }
  __syncthreads();
}

// ---- light item: one warp, per-warp shared hash keyed by x ----------------------------
__device__ void hub_item_warp(const DGraph& g, const u32* __restrict__ Te, int32_t s, ShCount& H, int32_t* L,
                              int* cnt, u64* acc, u64* __restrict__ R68, u64* __restrict__ R69) {
  const int lane = threadIdx.x & 31;
  const int32_t eva = g.eid[s];
  const int32_t a = g.ci[s];
  const int32_t lo_ = g.esrc[eva];
  const int32_t v = lo_ + g.edst[eva] - a;
  const bool v_lo = lo_ == v;
  const int64_t fa = g.foff[eva];
  const int na = full_prefix(g, fa, (int)(g.foff[eva + 1] - fa), a);  // b < a (or all, filtered)
  for (int o0 = 0; o0 < na; o0 += 32) {
    const int i = o0 + lane;
    int len = 0;
    int64_t fb = 0;
    int32_t b = 0;
    if (i < na) {
      const int64_t r = fa + i;
      b = g.fx[r];
      if (b < a) {
        const int32_t evb = v_lo ? g.fe1[r] : g.fe2[r];
        fb = g.foff[evb];
        len = full_prefix(g, fb, (int)(g.foff[evb + 1] - fb), a);  // x < a
      }
    }
    warp_flat(len, [&](int j, int k, bool valid) {
      const int64_t fbj = __shfl_sync(FULL_MASK, fb, j);
      if (!valid) return;
      const int32_t x = g.fx[fbj + k];
      if (x >= a) return;
      const u32 h = H.insert(x);
      if (atomicAdd(&H.val[h], 1u) == 0u) L[atomicAdd(cnt, 1)] = (int32_t)h;
    });
  }
  __syncwarp();
  for (int o0 = 0; o0 < na; o0 += 32) {
    const int i = o0 + lane;
    int len = 0;
    int64_t fb = 0;
    int32_t b = 0;
    if (i < na) {
      const int64_t r = fa + i;
      b = g.fx[r];
      if (b < a) {
        const int32_t evb = v_lo ? g.fe1[r] : g.fe2[r];
        fb = g.foff[evb];
        len = full_prefix(g, fb, (int)(g.foff[evb + 1] - fb), a);  // x < a
      }
    }
    int cur = -1;
    u64 cacc = 0;
    warp_flat(len, [&](int j, int k, bool valid) {
      const int64_t fbj = __shfl_sync(FULL_MASK, fb, j);
      if (!valid) return;
      if (j != cur) {
        if (cur >= 0 && cacc) atomicAdd(&acc[cur], cacc);
        cur = j;
        cacc = 0;
      }
      const int32_t x = g.fx[fbj + k];
      if (x >= a) return;
      cacc += (u64)H.val[H.find(x)] - 1ull;
    });
    if (cur >= 0 && cacc) atomicAdd(&acc[cur], cacc);
    __syncwarp();
    const u64 sb = acc[lane];
    acc[lane] = 0;
    if (sb) atomicAdd(&R68[b], sb);
    __syncwarp();
  }
  const int c = *cnt;
  u64 r69 = 0;
  for (int t = lane; t < c; t += 32) {
    const int32_t h = L[t];
    const u64 c2 = binom2(H.val[h]);
    if (c2) {
      r69 += c2;
      atomicAdd(&R68[H.keys[h]], c2);
    }
    H.keys[h] = SH_EMPTY;
    H.val[h] = 0u;
  }
  r69 = warp_sum(r69);
  if (lane == 0) {
    if (r69) {
      atomicAdd(&R69[v], r69);
      atomicAdd(&R68[a], r69);
    }
    *cnt = 0;
  }
  __syncwarp();
}

// ---- persistent kernels -------------------------------------------------------------------
// Heavy items: one BT-thread CTA per item (persistent, est-sorted list), c(x) table chosen per
// item (hash / shared by position / global by position).
template <int BT, int SMEM>
__global__ void __launch_bounds__(BT) k_hub_heavy(DGraph g, const int32_t* __restrict__ heavy,
                                                  const u32* __restrict__ heavy_est, int n_heavy,
                                                  int* __restrict__ counter, u32* __restrict__ gtabs,
                                                  int32_t* __restrict__ glists, u64* __restrict__ R68,
                                                  u64* __restrict__ R69, int sh_dense_max, int hash_max, int split) {
  extern __shared__ u32 hub_sh[];
  __shared__ HubCtaSharedT<BT> S;
  __shared__ int s_idx;
  constexpr u32 kSlots = (SMEM / 6) & ~1u;  // (x+1, 16-bit count) hash slots
  u32* gtab = gtabs ? gtabs + (size_t)blockIdx.x * g.max_deg : nullptr;
  int32_t* glist = glists ? glists + (size_t)blockIdx.x * g.max_deg : nullptr;
  for (int i = threadIdx.x; i < SMEM / 4; i += BT) hub_sh[i] = 0u;  // cleared by pass 3 after use
  __syncthreads();
  for (;;) {
    if (threadIdx.x == 0) s_idx = atomicAdd(counter, 1);
    __syncthreads();
    const int idx = s_idx;
    __syncthreads();
    if (idx >= n_heavy) break;
    const int32_t s = heavy[idx];
    const int32_t a = g.ci[s];
    const int32_t eva = g.eid[s];
    const int32_t v = g.esrc[eva] + g.edst[eva] - a;
    const u64 dv = (u64)g.deg[v];
    const u64 bound = min(dv - 1, (u64)heavy_est[idx]);  // distinct x of the item
    const bool c16 = g.foff[eva + 1] - g.foff[eva] < 65536;  // T(v,a) bounds every c(x)
    const long long ut = unit_t0();
    if (c16 && bound <= (u64)min(hash_max, (int)(kSlots * 3 / 4))) {
      const u32 cap = (u32)min((u64)kSlots, bound + bound / 3 + 64);
      hub_item_cta<HUB_T_HASH, BT>(g, s, cap, hub_sh, S, gtab, glist, R68, R69, split);
    } else if (c16 && dv <= (u64)min(sh_dense_max, SMEM / 2)) {
      hub_item_cta<HUB_T_SHPOS, BT>(g, s, 0, hub_sh, S, gtab, glist, R68, R69, split);
    } else {
      hub_item_cta<HUB_T_GLPOS, BT>(g, s, 0, hub_sh, S, gtab, glist, R68, R69, split);
    }
    unit_t1(1, ut, idx);
  }
}

// Light items: every warp takes items from a counter (per-warp hash keyed by x in the
// dynamic shared memory: keys, counts, touched list).
__global__ void __launch_bounds__(HUB_BT) k_hub_light(DGraph g, const u32* __restrict__ Te,
                                                      const int32_t* __restrict__ light, int n_light,
                                                      int* __restrict__ counter, u64* __restrict__ R68,
                                                      u64* __restrict__ R69) {
  extern __shared__ u32 hub_sh[];
  __shared__ int s_cnt[HUB_BT / 32];
  __shared__ u64 s_acc[HUB_BT / 32][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  ShCount H;
  H.keys = (int32_t*)hub_sh + wib * (3 * HUB_WARP_CAP);
  H.val = (u32*)(H.keys + HUB_WARP_CAP);
  H.mask = HUB_WARP_CAP - 1;
  int32_t* L = H.keys + 2 * HUB_WARP_CAP;
  for (int t = lane; t < HUB_WARP_CAP; t += 32) { H.keys[t] = SH_EMPTY; H.val[t] = 0u; }
  s_acc[wib][lane] = 0;
  if (lane == 0) s_cnt[wib] = 0;
  __syncwarp();
  for (;;) {
    int idx = 0;
    if (lane == 0) idx = atomicAdd(counter, 4);
    idx = __shfl_sync(FULL_MASK, idx, 0);
    if (idx >= n_light) break;
    const int end = min(idx + 4, n_light);
    for (int q = idx; q < end; q++)
      hub_item_warp(g, Te, light[q], H, L, &s_cnt[wib], s_acc[wib], R68, R69);
  }
}
