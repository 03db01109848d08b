// sched.cuh -- load-balancing building blocks shared by the enumeration passes.
//
// The passes are nested loops "for every outer item i, for every k < len(i)" whose inner
// lengths are heavy-tailed (adjacency and triangle lists of hubs).  These helpers flatten
// such a loop over the 32 lanes of a warp (warp_flat) or the threads of a CTA
// (block_flat), so every lane gets one (i, k) pair per step no matter how the lengths
// are distributed, and give small per-warp / per-CTA open-addressing tables in shared
// memory for the pair-keyed counts (W, D, c(x), ...) the passes join on.
#pragma once
#include <cub/block/block_scan.cuh>
#include "common.cuh"

// ---------------------------------------------------------------------------------
// warp_flat: the warp visits every (j, k) where j is a lane owning an outer item with
// len_j = the lane's `len` argument and k < len_j.  All lanes call body(j, k, valid) in
// lock-step (warp-uniform control flow), so the body may shuffle the owner's registers
// (__shfl_sync(FULL_MASK, reg, j)) before testing `valid`.
// ---------------------------------------------------------------------------------
template <typename Body>
__device__ __forceinline__ void warp_flat(int len, Body body) {
  const int lane = threadIdx.x & 31;
  int incl = len;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(FULL_MASK, incl, d);
    if (lane >= d) incl += y;
  }
  const int total = __shfl_sync(FULL_MASK, incl, 31);
  for (int t0 = 0; t0 < total; t0 += 32) {
    const int t = t0 + lane;
    // owner = number of lanes whose inclusive prefix is <= t (binary lifting)
    int j = 0;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      const int c = __shfl_sync(FULL_MASK, incl, j + s - 1);
      if (c <= t) j += s;
    }
    const int start = __shfl_sync(FULL_MASK, incl - len, j);
    body(j, t - start, t < total);
  }
}

// ---------------------------------------------------------------------------------
// block_flat: the CTA visits every (i, k), i in [0, n_outer), k in [0, len(i)), in chunks
// of BT outer items (one per thread).  pre[] is shared scratch of BT+1 int64 entries.
//   load(i) -> len(i) (thread threadIdx.x loads outer item c0 + threadIdx.x and may stash
//   payload in shared arrays indexed by threadIdx.x);  body(li, k) with li = i - c0;
//   after(c0, cn) runs (all threads) after each chunk, between two barriers; flush() runs
//   in every thread before the first of them (to spill per-thread register sums).
// ---------------------------------------------------------------------------------
struct NoFlush {
  __device__ __forceinline__ void operator()() const {}
};
template <int BT, typename Load, typename Body, typename After, typename Flush = NoFlush>
__device__ __forceinline__ void block_flat(int64_t n_outer, int64_t* pre, Load load, Body body, After after,
                                           Flush flush = Flush()) {
  typedef cub::BlockScan<int64_t, BT> Scan;
  __shared__ typename Scan::TempStorage scan_tmp;
  for (int64_t c0 = 0; c0 < n_outer; c0 += BT) {
    const int cn = (int)min((int64_t)BT, n_outer - c0);
    int64_t a = 0;
    if ((int)threadIdx.x < cn) a = load(c0 + threadIdx.x);
    int64_t ex, tot;
    Scan(scan_tmp).ExclusiveSum(a, ex, tot);
    pre[threadIdx.x] = ex;
    if (threadIdx.x == 0) pre[BT] = tot;
    __syncthreads();
    const int64_t total = pre[BT];
    for (int64_t t = threadIdx.x; t < total; t += BT) {
      int lo = 0, hi = cn;  // largest lo with pre[lo] <= t
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (pre[mid] <= t) lo = mid; else hi = mid;
      }
      body(lo, t - pre[lo]);
    }
    flush();
    __syncthreads();
    after(c0, cn);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------
// Open-addressing counter table in shared memory (keys int32, -1 = empty; one u32 count).
// Linear probing; capacity is a power of two >= 2 x the number of distinct keys.
// ---------------------------------------------------------------------------------
#define SH_EMPTY (-1)
struct ShCount {
  int32_t* keys;
  u32* val;
  u32 mask;
  __device__ __forceinline__ u32 h0(int32_t x) const { return ((u32)x * 0x9E3779B1u) >> 7 & mask; }
  __device__ __forceinline__ u32 insert(int32_t x) {
    u32 h = h0(x);
    for (;;) {
      const int32_t k = keys[h];
      if (k == x) return h;
      if (k == SH_EMPTY) {
        const int32_t old = atomicCAS(&keys[h], SH_EMPTY, x);
        if (old == SH_EMPTY || old == x) return h;
      }
      h = (h + 1) & mask;
    }
  }
  __device__ __forceinline__ u32 find(int32_t x) const {
    u32 h = h0(x);
    while (keys[h] != x) h = (h + 1) & mask;
    return h;
  }
  __device__ __forceinline__ u32 find_or_miss(int32_t x) const {  // mask+1 if absent
    u32 h = h0(x);
    for (;;) {
      const int32_t k = keys[h];
      if (k == x) return h;
      if (k == SH_EMPTY) return mask + 1;
      h = (h + 1) & mask;
    }
  }
};

__device__ __forceinline__ u32 pow2_at_least(u32 x, u32 lo) {
  u32 c = lo;
  while (c < x) c <<= 1;
  return c;
}

// Append x to list (counter in shared memory) with one atomic per group of active lanes.
__device__ __forceinline__ void append_active(bool pred, int32_t x, int32_t* list, int* counter) {
  const unsigned act = __activemask();
  const unsigned m = __ballot_sync(act, pred);
  if (!pred) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(m) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(counter, __popc(m));
  base = __shfl_sync(m, base, leader);
  list[base + __popc(m & ((1u << lane) - 1u))] = x;
}

// warp-aggregated append to a global list (one atomic per warp per call)
__device__ __forceinline__ void warp_append(bool pred, int32_t val, int32_t* list, int* counter) {
  const u32 bal = __ballot_sync(FULL_MASK, pred);
  if (!bal) return;
  const int lane = threadIdx.x & 31;
  int base = 0;
  const int leader = __ffs(bal) - 1;
  if (lane == leader) base = atomicAdd(counter, __popc(bal));
  base = __shfl_sync(FULL_MASK, base, leader);
  if (pred) list[base + __popc(bal & ((1u << lane) - 1u))] = val;
}

// ---------------------------------------------------------------------------------
// Generic list engines.  Items i in [0, n_items); item i is the list [base, base + len)
// (info(i, base, len) fills both); elem(i, base, k) visits element k of item i and
// returns its contribution to the item's sum; flush(i, sum) receives non-zero partial
// sums (several per item are possible: callers accumulate with atomics).
// ---------------------------------------------------------------------------------
#define LE_LONG 32      // item longer than this: queued and cut in chunks (CTA engine)
#define LE_CHUNK 256    // elements per chunk (8 per lane)

// warp engine: the warp walks all items, 32 at a time, flattened over the lanes
template <typename Info, typename Elem, typename Flush>
__device__ __forceinline__ void warp_lists(int n_items, Info info, Elem elem, Flush flush) {
  const int lane = threadIdx.x & 31;
  for (int o0 = 0; o0 < n_items; o0 += 32) {
    const int i = o0 + lane;
    int64_t base = 0;
    int len = 0;
    if (i < n_items) info(i, base, len);
    int cur = -1;
    u64 acc = 0;
    warp_flat(len, [&](int j, int k, bool valid) {
      const int64_t bj = __shfl_sync(FULL_MASK, base, j);
      if (!valid) return;
      if (j != cur) {
        if (cur >= 0 && acc) flush(o0 + cur, acc);
        cur = j;
        acc = 0;
      }
      acc += elem(o0 + j, bj, k);
    });
    if (cur >= 0 && acc) flush(o0 + cur, acc);
  }
}

struct ListEng {
  int next;
  int qn;
  int next_chunk;
  int nchunks;
  int32_t* qi;   // queued items (global memory, one region per CTA)
  int32_t* lc0;  // first chunk of each queued item (+1 entry)
  int qcap;
};

// CTA-wide exclusive scan of one int per thread (any blockDim that is a multiple of 32,
// <= 1024); returns the exclusive prefix, *total gets the sum.  Contains barriers.
__device__ __forceinline__ int block_exclusive_scan(int x, int* total) {
  __shared__ int ws[32];
  __shared__ int wtot;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int incl = x;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(FULL_MASK, incl, d);
    if (lane >= d) incl += y;
  }
  if (lane == 31) ws[w] = incl;
  __syncthreads();
  if (w == 0) {
    int v = lane < nw ? ws[lane] : 0;
    int iv = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(FULL_MASK, iv, d);
      if (lane >= d) iv += y;
    }
    if (lane < nw) ws[lane] = iv - v;  // exclusive prefix of warp sums
    if (lane == 31) wtot = iv;         // total (lane 31 holds the full sum)
  }
  __syncthreads();
  const int ex = ws[w] + incl - x;
  *total = wtot;
  __syncthreads();
  return ex;
}

// CTA engine: warps take items (a few per grab when items are few, up to 32), walk
// short ones with warp_flat and queue long ones; queued items are then cut into
// LE_CHUNK-element chunks taken by whole warps.  Ends with a barrier.
template <typename Info, typename Elem, typename Flush>
__device__ void cta_lists(int n_items, ListEng& E, Info info, Elem elem, Flush flush) {
  const int lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  if (threadIdx.x == 0) { E.next = 0; E.qn = 0; E.next_chunk = 0; }
  __syncthreads();
  const int grab = max(1, min(32, n_items / (4 * nw)));  // ~4 grabs per warp: dynamic balance
  for (;;) {
    int b = 0;
    if (lane == 0) b = atomicAdd(&E.next, grab);
    b = __shfl_sync(FULL_MASK, b, 0);
    if (b >= n_items) break;
    const int i = b + lane;
    int64_t base = 0;
    int len = 0;
    if (lane < grab && i < n_items) info(i, base, len);
    if (len > LE_LONG) {
      const int q = atomicAdd(&E.qn, 1);
      if (q < E.qcap) { E.qi[q] = i; len = 0; }
    }
    int cur = -1;
    u64 acc = 0;
    warp_flat(len, [&](int j, int k, bool valid) {
      const int64_t bj = __shfl_sync(FULL_MASK, base, j);
      if (!valid) return;
      if (j != cur) {
        if (cur >= 0 && acc) flush(b + cur, acc);
        cur = j;
        acc = 0;
      }
      acc += elem(b + j, bj, k);
    });
    if (cur >= 0 && acc) flush(b + cur, acc);
  }
  __syncthreads();
  const int nq = min(E.qn, E.qcap);
  if (nq == 0) return;  // uniform
  {
    __shared__ int s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int q0 = 0; q0 < nq; q0 += blockDim.x) {
      const int q = q0 + threadIdx.x;
      int nc = 0;
      if (q < nq) {
        int64_t base;
        int len;
        info(E.qi[q], base, len);
        nc = (len + LE_CHUNK - 1) / LE_CHUNK;
      }
      int tot = 0;
      const int ex = block_exclusive_scan(nc, &tot);
      if (q < nq) E.lc0[q] = s_carry + ex;
      __syncthreads();
      if (threadIdx.x == 0) s_carry += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) { E.lc0[nq] = s_carry; E.nchunks = s_carry; }
  }
  __syncthreads();
  const int nchunks = E.nchunks;
  for (;;) {
    int c = 0;
    if (lane == 0) c = atomicAdd(&E.next_chunk, 1);
    c = __shfl_sync(FULL_MASK, c, 0);
    if (c >= nchunks) break;
    int lo = 0, hi = nq;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (E.lc0[mid] <= c) lo = mid; else hi = mid;
    }
    const int i = E.qi[lo];
    int64_t base;
    int len;
    info(i, base, len);
    const int k0 = (c - E.lc0[lo]) * LE_CHUNK;
    const int k1 = min(len, k0 + LE_CHUNK);
    u64 acc = 0;
    for (int k = k0 + lane; k < k1; k += 32) acc += elem(i, base, k);
    acc = warp_sum(acc);
    if (lane == 0 && acc) flush(i, acc);
  }
  __syncthreads();
}
