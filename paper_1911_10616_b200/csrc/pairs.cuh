// pairs.cuh -- step a7 of SURVEY 8(a): the pair (wedge) pass.
//
// For every source u the pass holds, for every x at distance <= 2, the pair quantities
// of Theorem B.1 (readings R11, R14):
//   W(u,x)  = |N(u) & N(x)|                       (2-hop expansion)
//   D(u,x)  = #edges inside N(u) & N(x)            (diamond expansion)
// TT(u,x) = sum_{v in N(u)&N(x)} T(v,x) - W[u~x] (R14) enters theta51 only through
// sum_x TT(u,x)(W-1), which is summed per wedge once W is final (no table).
// Emits:  C4(u)=DM8, theta36, theta50, theta51, theta63 for u;
//   E5 = C4(u,v) = sum_{x in N(v)\u} (W(u,x)-1) per edge, and the centre credits
//   theta49(v) += C(W(u,x)-1,2), theta62(v) += D(u,x) for x>u in N(v);
//   theta64(v) += sum over diamonds (u; v,w; x), x>u, of W(u,x)-2:
//   DM64(v) = sum_{pairs {a,x} in N(v)} |N(v)&N(a)&N(x)| (W(a,x)-2) seen from the pair.
//
// Two passes per source over the same items (the neighbours v of u; item v has the wedge
// elements u-v-x with x > u and T(u,v) chord elements (u; v, w)): pass 1 builds the table
// (W from wedges, D from the diamonds behind chords w > v), pass 2 reads it (per-pair
// terms over the table entries, per-wedge and per-diamond sums over the items).
//
// Each unordered pair {u, x} is formed once, from its lower end u (rank order; N(v) is
// sorted, so the x > u part of N(v) is the suffix after u's own slot, found in O(1) from the
// edge's slot map): the wedge walks are half of sum_v d(v)(d(v)-1).  A pair's terms are
// credited to both ends (the x side with atomics, only for pairs with W >= 2), and so are
// the per-wedge terms of both wedge edges (E5 of e(x,v), theta51 of x).
//
// Scheduling (B200): sources are sorted by their 2-hop estimate est(u) = sum_{v in N(u)}
// d(v) - d(u) (>= the number of distinct x) and split in tiers:
//   light (est <= PAIR_WARP_MAX): one WARP per source, per-warp packed shared hash;
//   mid   (est <= PAIR_MID_MAX) : one CTA per source, packed shared hash;
//   heavy                       : one CTA per source, dense per-CTA table in global
//                                 memory (u32 W|D<<16, or u64 W|D<<32 for sources past the
//                                 16-bit bounds), CTA count sized so the tables stay in L2.
// Inside a CTA, short items are flattened over the 32 lanes of a warp (warp_flat) and
// long items (hub neighbours) are cut into fixed chunks that whole warps take from a
// shared queue, so lanes stay busy however heavy-tailed the degrees are, every element
// is found without a search, and reads stay coalesced along each adjacency list.
#pragma once
#include <cub/block/block_scan.cuh>
#include "common.cuh"
#include "sched.cuh"

// The pair pass's per-vertex credits, interleaved by vertex (PO_STRIDE u64 per vertex, the
// four per-pair terms of a vertex in one 32-byte sector): the x-side credits of a pair are
// scattered atomics, one sector each instead of one per field.  k_pair_fields copies them into
// the per-field arrays F afterwards.
enum PairField { PO_R8 = 0, PO_R36, PO_R50, PO_R63, PO_R51, PO_R49, PO_R62, PO_R64, PO_STRIDE };
struct PairOut {
  u64* pa;  // [n][PO_STRIDE]
  u64* C4e;
  const int32_t* hstar;     // per source: its heaviest neighbour h* (wedges through h* are not walked)
  const int32_t* hstar_s;   // per source: the slot of h* in N(u)
  const int32_t* hub_slot;  // per vertex: row of its position map, or -1
  const int32_t* hub_pos;   // [slot][x]: position of x in N(hub) if x ~ hub, else -1
};
__device__ __forceinline__ void xadd(const PairOut& o, int f, int32_t x, u64 v) {
  atomicAdd(&o.pa[(size_t)x * PO_STRIDE + f], v);
}
__device__ __forceinline__ int64_t slot_of_lo_in_hi(const DGraph& g, int32_t e) { return g.eslot_hi[e]; }
__device__ __forceinline__ int64_t slot_of_hi_in_lo(const DGraph& g, int32_t e) {
  const int32_t a = g.esrc[e];
  return g.rp[a] + g.dm[a] + (e - g.orow[a]);
}

#define PAIR_BT 256              // mid-tier CTA (and light-tier warps) kernel
#define PAIR_MID_CAP 8192        // mid tier: packed shared hash entries (key + W|D<<16)
#define PAIR_SMEM (PAIR_MID_CAP * 8)     // dynamic shared memory of the mid / light kernel
#define PAIR_MID_MAX 6144        // mid tier: est <= this (load <= 0.75)
#define PAIR_MIDS_BT 128         // small-mid tier: CTA of 4 warps per source ...
#define PAIR_MIDS_CAP 4096       // ... with a 32 KB packed shared hash: five sources share an SM
#define PAIR_MIDS_MAX 2048       // small-mid tier: est <= this
#define PAIR_WARP_CAP 1024       // light tier: per-warp packed hash entries (8 warps x 8 KB)
#define PAIR_WARP_MAX 512        // light tier: est <= this
#define PAIR_TINY_CAP 256        // tiny tier (k_pairs_tiny): per-warp packed hash entries ...
#define PAIR_TINY_MAX 128        // ... for est <= this (load <= 0.5)
#ifndef PAIR_TINY_MINB
#define PAIR_TINY_MINB 4         // resident CTAs per SM the tiny kernel's register budget must allow
#endif
#define PAIR_HBT 1024            // heavy tier CTA
#define PAIR_HOT_BYTES (192 << 10)  // heavy tier: shared table entries of the top ranks (hot x)

#define PAIR_LONG 64             // item part longer than this: chunked, shared queue
#define PAIR_CHUNK 256           // elements per long-item chunk (8 per lane)
#define PAIR_ILP 4               // independent wedge chains per lane in the pass-2 walk
#define PAIR_DIAM_DEFER 256      // diamond list longer than this: queued by the CTA engine
#define PAIR_HUBMAP_MIN 1024     // vertices of degree >= this get a position map (budgeted)
#define EMPTY_KEY (-1)

// Packed variant (one u32 per key: W | D << 16).  Valid for sources with d(u) < 2^16
// (W(u,x) <= d(u)) and T(u) < 2^16 (D(u,x) counts edges inside N(u)&N(x), at most T(u)).
struct SharedPackedHash {
  static constexpr bool kDense = false;
  typedef u32 WordT;
  int32_t* keys;
  u32* val;
  u32 mask;
  __device__ __forceinline__ u32 h0(int32_t x) const { return ((u32)x * 0x9E3779B1u) >> 7 & mask; }
  __device__ __forceinline__ u32 insert(int32_t x) {
    u32 h = h0(x);
    for (;;) {
      const int32_t k = keys[h];
      if (k == x) return h;
      if (k == EMPTY_KEY) {
        const int32_t old = atomicCAS(&keys[h], EMPTY_KEY, x);
        if (old == EMPTY_KEY || old == x) return h;
      }
      h = (h + 1) & mask;
    }
  }
  __device__ __forceinline__ u32 find(int32_t x) const {
    u32 h = h0(x);
    while (keys[h] != x) h = (h + 1) & mask;
    return h;
  }
  __device__ __forceinline__ void add_w(int32_t x) { atomicAdd(&val[insert(x)], 1u); }
  // insert, not find: pass 1 visits wedges and diamonds concurrently
  __device__ __forceinline__ void add_d(int32_t x) { atomicAdd(&val[insert(x)], 1u << 16); }
  __device__ __forceinline__ void get(int32_t x, u64& wv, u64& dv) const {
    const u32 v = val[find(x)];
    wv = v & 0xffffu;
    dv = v >> 16;
  }
  __device__ __forceinline__ u64 get_w(int32_t x) const { return val[find(x)] & 0xffffu; }
  __device__ __forceinline__ u64 get_w_or0(int32_t x) const {
    u32 h = h0(x);
    for (;;) {
      const int32_t k = keys[h];
      if (k == x) return val[h] & 0xffffu;
      if (k == EMPTY_KEY) return 0;
      h = (h + 1) & mask;
    }
  }
  __device__ __forceinline__ u32* word_if(int32_t x) const {
    u32 h = h0(x);
    for (;;) {
      const int32_t k = keys[h];
      if (k == x) return &val[h];
      if (k == EMPTY_KEY) return nullptr;
      h = (h + 1) & mask;
    }
  }
  __device__ __forceinline__ static u64 wfield(u32 v) { return (u64)(v & 0xffffu); }
  __device__ __forceinline__ static u64 dfield(u32 v) { return (u64)(v >> 16); }
  template <typename F>
  __device__ __forceinline__ void for_each_mut(int tid, int nthr, F f) {
    for (u32 h = tid; h <= mask; h += nthr) {
      const int32_t x = keys[h];
      if (x == EMPTY_KEY) continue;
      const u32 v = val[h];
      const u64 w = f(x, (u64)(v & 0xffffu), (u64)(v >> 16));
      if (w != (u64)(v & 0xffffu)) val[h] = (v & 0xffff0000u) | (u32)w;
    }
  }
  __device__ __forceinline__ void reset(int tid, int nthr) {
    for (u32 h = tid; h <= mask; h += nthr) { keys[h] = EMPTY_KEY; val[h] = 0u; }
  }
};

// Dense per-CTA table in global memory indexed by x; W in the low half of the word,
// D in the high half; touched list for the entry sweep and the reset.
template <typename Word, bool SCAN>
struct GlobalDense {
  // SCAN (2-hop set a sizeable part of n): updates are fire-and-forget reductions and the
  // entries are found by sweeping the whole table (16-byte loads).  Otherwise the first
  // update of an entry appends x to the touched list L (entry sweep, reset).
  // Reads go through L2 (__ldcg): the entries are updated by L2 atomics.
  // Hot entries: x >= hot0 (the hotK highest ranks, where the 2-hop ends of a hub source
  // concentrate in the degeneracy order) live in shared memory instead (hot[x - hot0]):
  // shared atomics, swept by for_each_mut / reset, never on the touched list.
  static constexpr bool kDense = true;
  typedef Word WordT;
  Word* t;
  int32_t* L;
  int* ntouch;  // shared counter
  int32_t n;
  Word* hot = nullptr;
  int32_t hot0 = 0x7fffffff;
  int hotK = 0;
  static constexpr int SH = (int)sizeof(Word) * 4;
  static constexpr Word LOW = (Word)(((u64)1 << SH) - 1);
  static constexpr int PER = 16 / (int)sizeof(Word);
  __device__ __forceinline__ Word raw_add(int32_t x, Word inc) {
    if (x >= hot0) return atomicAdd(&hot[x - hot0], inc);
    if (SCAN) {
      atomicAdd(&t[x], inc);
      return (Word)1;
    }
    return atomicAdd(&t[x], inc);
  }
  __device__ __forceinline__ void after_w(int32_t x, Word old) {
    if (!SCAN && x < hot0) append_active(old == 0, x, L, ntouch);
  }
  __device__ __forceinline__ void add_w(int32_t x) { after_w(x, raw_add(x, (Word)1)); }
  __device__ __forceinline__ void add_d(int32_t x) { after_w(x, raw_add(x, (Word)((Word)1 << SH))); }
  __device__ __forceinline__ Word load(int32_t x) const { return x >= hot0 ? hot[x - hot0] : __ldcg(&t[x]); }
  __device__ __forceinline__ void get(int32_t x, u64& wv, u64& dv) const {
    const Word v = load(x);
    wv = (u64)(v & LOW);
    dv = (u64)(v >> SH);
  }
  __device__ __forceinline__ u64 get_w(int32_t x) const { return (u64)(load(x) & LOW); }
  __device__ __forceinline__ u64 get_w_or0(int32_t x) const { return (u64)(load(x) & LOW); }
  // entry word of x if x has an entry, else nullptr (single-writer update by the caller)
  __device__ __forceinline__ Word* word_if(int32_t x) const {
    Word* p = x >= hot0 ? &hot[x - hot0] : &t[x];
    return load(x) != 0 ? p : nullptr;
  }
  __device__ __forceinline__ static u64 wfield(Word v) { return (u64)(v & LOW); }
  __device__ __forceinline__ static u64 dfield(Word v) { return (u64)(v >> SH); }
  // f(x, w, d) -> new w, for every entry (strided over `nthr` threads from `tid`)
  template <typename F>
  __device__ __forceinline__ void for_each_mut(int tid, int nthr, F f) {
    for (int i = tid; i < hotK; i += nthr) {
      const Word v = hot[i];
      if (v == 0) continue;
      const u64 w = f(hot0 + i, (u64)(v & LOW), (u64)(v >> SH));
      if (w != (u64)(v & LOW)) hot[i] = (Word)((v & ~LOW) | (Word)w);
    }
    if (SCAN) {
      const int32_t nvec = (min(n, hot0) + PER - 1) / PER;  // (a vector across hot0 holds no hot entry)
      const uint4* tv = reinterpret_cast<const uint4*>(t);
      for (int32_t v0 = tid; v0 < nvec; v0 += nthr * 4) {
        uint4 q[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
          const int32_t vi = v0 + i * nthr;
          q[i] = vi < nvec ? __ldcg(&tv[vi]) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int i = 0; i < 4; i++) {
          if ((q[i].x | q[i].y | q[i].z | q[i].w) == 0) continue;
          const int32_t vi = v0 + i * nthr;
          const Word* e = reinterpret_cast<const Word*>(&q[i]);
#pragma unroll
          for (int c = 0; c < PER; c++) {
            if (e[c] == 0) continue;
            const u64 w = f(vi * PER + c, (u64)(e[c] & LOW), (u64)(e[c] >> SH));
            if (w != (u64)(e[c] & LOW)) t[vi * PER + c] = (Word)((e[c] & ~LOW) | (Word)w);
          }
        }
      }
      return;
    }
    const int nt = *ntouch;
    for (int i = tid; i < nt; i += nthr) {
      const int32_t x = L[i];
      const Word v = __ldcg(&t[x]);
      const u64 w = f(x, (u64)(v & LOW), (u64)(v >> SH));
      if (w != (u64)(v & LOW)) t[x] = (Word)((v & ~LOW) | (Word)w);
    }
  }
  __device__ __forceinline__ void reset(int tid, int nthr) {
    for (int i = tid; i < hotK; i += nthr) hot[i] = (Word)0;
    if (SCAN) {
      const int32_t nvec = (min(n, hot0) + PER - 1) / PER;
      uint4* tv = reinterpret_cast<uint4*>(t);
      for (int32_t v0 = tid; v0 < nvec; v0 += nthr * 4) {
        uint4 q[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
          const int32_t vi = v0 + i * nthr;
          q[i] = vi < nvec ? __ldcg(&tv[vi]) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int i = 0; i < 4; i++)
          if ((q[i].x | q[i].y | q[i].z | q[i].w) != 0) tv[v0 + i * nthr] = make_uint4(0, 0, 0, 0);
      }
      return;
    }
    const int nt = *ntouch;
    for (int i = tid; i < nt; i += nthr) t[L[i]] = (Word)0;
  }
};

// phase C contributions of one (x, W, D) pair {u, x}, x > u: to u (summed by the caller)
// and to x (atomics; du = d(u))
__device__ __forceinline__ void pair_c_terms(const DGraph& g, const PairOut& o, u64 du, int32_t x, u64 w, u64 d,
                                             u64& a8, u64& a36, u64& a50, u64& a63) {
  if (w < 2) return;  // W = 1: every term is 0 (and D = 0)
  const u64 c2 = binom2(w), c3 = binom3(w), t63 = d * (w - 2);
  a8 += c2;
  a36 += c2 * (u64)(int64_t)(dg_deg(g, x) - 2);
  a50 += c3;
  a63 += t63;
  xadd(o, PO_R8, x, c2);
  xadd(o, PO_R36, x, c2 * (du - 2));  // du >= w >= 2
  if (c3) xadd(o, PO_R50, x, c3);
  if (t63) xadd(o, PO_R63, x, t63);
}

// ---- per-element work (shared by the warp and CTA engines) --------------------------
// Item v of source u.  Wedge element k: x = N(v)[k].  Chord element k: the k-th entry of
// the full triangle list of e(u,v), i.e. w with (u, v, w) a triangle.
struct PairItem {
  int32_t v;
  int32_t e;        // e(u, v)
  int64_t rb;       // rp[v]
  int64_t fo;       // foff[e]
  int32_t dv;       // d(v)
  int32_t tv;       // T(u, v)
  bool vlo;         // v is the lower endpoint of e
};

// slot of u in N(v) for the edge e = e(u, v) (vlo: v is its lower endpoint)
__device__ __forceinline__ int64_t slot_in_other(const DGraph& g, int32_t v, int32_t e, bool vlo) {
  return vlo ? g.rp[v] + g.dm[v] + (e - g.orow[v]) : g.eslot_hi[e];
}
// Item v of source u: its wedge part is the suffix of N(v) after u (x > u); the wedge part of
// item h* is empty: W(u,x) gets the h* contribution from a membership test over the table
// keys instead (see hstar_and_terms)
// (u: the source; the slot's twin, T(u,v) per slot and the rank order give the item with two
// random loads, rp[v+1] and, for items with chords, foff[e])
__device__ __forceinline__ PairItem pair_item(const DGraph& g, int32_t u, int64_t s_uv, int32_t hs) {
  PairItem it;
  it.v = g.ci[s_uv];
  it.e = g.eid[s_uv];
  it.vlo = it.v < u;  // ranks: the lower endpoint of e(u,v)
  it.rb = (int64_t)g.twin[s_uv] + 1;
  it.dv = it.v == hs ? 0 : g.plen[s_uv];  // (= rp[v+1] - rb, from the estimates)
  it.tv = (int32_t)g.tes[s_uv];
  it.fo = it.tv ? g.foff[it.e] : 0;
  return it;
}

// pass-2 per-item accumulators (flushed to global counters)
struct PairAcc {
  u64 c5, c49, c62, c64;
  __device__ __forceinline__ void zero() { c5 = c49 = c62 = c64 = 0; }
  __device__ __forceinline__ void flush(int32_t u, int32_t v, int32_t e, const PairOut& o) {
    if (u < v && c5) atomicAdd(&o.C4e[e], c5);
    if (c49) xadd(o, PO_R49, v, c49);
    if (c62) xadd(o, PO_R62, v, c62);
    if (c64) xadd(o, PO_R64, v, c64);
    zero();
  }
};

template <typename Tab>
__device__ __forceinline__ void pass1_wedge(const DGraph& g, int64_t rb, int k, Tab& tab) {
  tab.add_w(g.ci[rb + k]);  // x > u: the item's list is the suffix after u
}
// The x-side terms of a wedge u - v - x (x > u, W = W(u,x) >= 2, t = the slot of x in N(v),
// tuv = T(u,v)): E5 of e(x,v) (counted from its lower end, as PairAcc::flush does for e(u,v))
// and theta51 of x.
__device__ __forceinline__ void wedge_x_side(const DGraph& g, const PairOut& o, int32_t x, int32_t v, int64_t t,
                                             int tuv, u64 w) {
  if (x < v) atomicAdd(&o.C4e[g.eid[t]], w - 1);
  if (tuv) xadd(o, PO_R51, x, (u64)tuv * (w - 1));
}

// Chords and diamonds, flattened on two levels.  Every lane brings at most one chord
// (v, w): the k-th third vertex of e(u,v), kept only for w > v -- each unordered chord once:
// PASS 1 adds it to D(u,x) once, and PASS 2's theta64 sum over its diamond list,
// sum_{x in tri(v,w), x > u} (W(u,x) - 2), is the same for both chord ends (tri(v,w) =
// tri(w,v)), so it is computed once and credited to v (acc[owner], per-warp shared
// accumulators, one per item owner) and to w (o->pa).  The diamond lists tri(v,w) of the (up
// to 32) chords of the warp are flattened over the lanes with a second warp_flat.
// Warp-uniform call.
struct NoDefer {
  __device__ __forceinline__ bool operator()(int64_t, int32_t, bool) const { return false; }
};
template <int PASS, typename Tab, typename Defer = NoDefer>
__device__ __forceinline__ void chords_step(const DGraph& g, int32_t u, bool valid, int32_t v, int64_t fo, bool vlo,
                                            int k, int owner, Tab& tab, u64* acc, const PairOut* o,
                                            Defer defer = Defer()) {
  int64_t f0 = 0;
  int len2 = 0;
  int32_t w = 0;
  if (valid) {
    const int64_t r = fo + k;
    w = g.fx[r];
    if (w > v) {
      const int32_t evw = vlo ? g.fe1[r] : g.fe2[r];
      f0 = g.foff[evw];
      len2 = (int)(g.foff[evw + 1] - f0);
      if (g.full_sorted) {  // both passes need x > u only: the suffix of a sorted list
        const int64_t s0 = lower_bound_dev<int32_t>(g.fx, f0, f0 + len2, u + 1);
        len2 -= (int)(s0 - f0);
        f0 = s0;
      }
      // a long diamond list goes to the CTA's queue (chunked over whole warps) instead
      if (len2 > PAIR_DIAM_DEFER && defer(r, v, vlo)) len2 = 0;
    }
  }
  int cur = -1, cown = 0;
  int32_t cw = 0;
  u64 c = 0;
  warp_flat(len2, [&](int j2, int k2, bool v2) {
    const int64_t f0j = __shfl_sync(FULL_MASK, f0, j2);
    const int own = __shfl_sync(FULL_MASK, owner, j2);
    const int32_t wj = __shfl_sync(FULL_MASK, w, j2);
    if (!v2) return;
    const int32_t x = g.fx[f0j + k2];
    if (PASS == 1) {
      if (x > u) tab.add_d(x);
    } else {
      if (j2 != cur) {
        if (cur >= 0 && c) { atomicAdd(&acc[cown], c); xadd(*o, PO_R64, cw, c); }
        cur = j2;
        cown = own;
        cw = wj;
        c = 0;
      }
      if (x > u) c += tab.get_w(x) - 2ull;
    }
  });
  if (PASS == 2 && cur >= 0 && c) { atomicAdd(&acc[cown], c); xadd(*o, PO_R64, cw, c); }
}

// Pass-2 wedge walk of up to 32 items (lane's item: list [rb, rb+len), vertex v, edge e),
// flattened like warp_flat but PAIR_ILP steps at a time with every load of a step issued
// before the dependent ones (list entry -> table entry -> edge id / T): a lane keeps
// PAIR_ILP dependent chains in flight instead of one.
template <typename Tab>
__device__ __forceinline__ void wedges_pass2_ilp(const DGraph& g, const u32* __restrict__ Te, int32_t u, int len,
                                                 int64_t rb, int32_t v, int32_t e, int tv, const Tab& tab, u64& s51,
                                                 const PairOut& o) {
  const int lane = threadIdx.x & 31;
  int incl = len;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(FULL_MASK, incl, d);
    if (lane >= d) incl += y;
  }
  const int total = __shfl_sync(FULL_MASK, incl, 31);
  PairAcc A;
  A.zero();
  int cur = -1;
  int32_t cv = 0, ce = 0;
  for (int t0 = 0; t0 < total; t0 += 32 * PAIR_ILP) {
    int32_t xs[PAIR_ILP], js[PAIR_ILP], vs[PAIR_ILP], es[PAIR_ILP], tvs[PAIR_ILP];
    int64_t ts[PAIR_ILP];
#pragma unroll
    for (int i = 0; i < PAIR_ILP; i++) {
      const int t = t0 + 32 * i + lane;
      int j = 0;
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) {
        const int c = __shfl_sync(FULL_MASK, incl, j + s - 1);
        if (c <= t) j += s;
      }
      const int start = __shfl_sync(FULL_MASK, incl - len, j);
      const int64_t rbj = __shfl_sync(FULL_MASK, rb, j);
      vs[i] = __shfl_sync(FULL_MASK, v, j);
      es[i] = __shfl_sync(FULL_MASK, e, j);
      tvs[i] = __shfl_sync(FULL_MASK, tv, j);
      const bool valid = t < total;
      js[i] = valid ? j : -1;
      ts[i] = rbj + (t - start);
      xs[i] = valid ? g.ci[ts[i]] : u;
    }
    u64 wv[PAIR_ILP], dv[PAIR_ILP];
#pragma unroll
    for (int i = 0; i < PAIR_ILP; i++) {
      wv[i] = 0; dv[i] = 0;
      if (xs[i] != u) tab.get(xs[i], wv[i], dv[i]);
    }
    u32 te[PAIR_ILP];
#pragma unroll
    for (int i = 0; i < PAIR_ILP; i++) te[i] = wv[i] >= 2 ? g.tes[ts[i]] : 0u;
#pragma unroll
    for (int i = 0; i < PAIR_ILP; i++) {
      if (js[i] < 0) continue;
      if (js[i] != cur) {
        if (cur >= 0) A.flush(u, cv, ce, o);
        cur = js[i]; cv = vs[i]; ce = es[i];
      }
      if (wv[i] < 2) continue;  // W(u,x) = 1 (hence D = 0) contributes nothing
      const u64 w = wv[i];
      A.c5 += w - 1;
      s51 += (u64)te[i] * (w - 1);
      A.c49 += binom2(w - 1);
      A.c62 += dv[i];
      wedge_x_side(g, o, xs[i], vs[i], ts[i], tvs[i], w);
    }
  }
  if (cur >= 0) A.flush(u, cv, ce, o);
}

// ---- warp engine: the warp runs one pass over items s_uv in [r0, r1) --------------------
// Every part (wedges, chords) of 32 items at a time is flattened over the lanes.
template <int PASS, typename Tab>
__device__ __forceinline__ void warp_pass(const DGraph& g, const u32* __restrict__ Te, int32_t u, int32_t hs,
                                          int64_t r0, int64_t r1, Tab& tab, u64& s51, const PairOut& o, u64* acc) {
  const int lane = threadIdx.x & 31;
  for (int64_t o0 = r0; o0 < r1; o0 += 32) {
    PairItem it;
    const bool have = o0 + lane < r1;
    if (have) it = pair_item(g, u, o0 + lane, hs);
    else { it.v = 0; it.e = 0; it.rb = 0; it.fo = 0; it.dv = 0; it.tv = 0; it.vlo = false; }
    PairAcc A;
    A.zero();
    int cur = -1;
    int32_t cv = 0, ce = 0;
    auto flush = [&]() {
      if (PASS == 2 && cur >= 0) A.flush(u, cv, ce, o);
    };
    // wedges
    if (PASS == 2) {
      wedges_pass2_ilp(g, Te, u, it.dv, it.rb, it.v, it.e, it.tv, tab, s51, o);
    } else {
      warp_flat(it.dv, [&](int j, int k, bool valid) {
        const int64_t rbj = __shfl_sync(FULL_MASK, it.rb, j);
        if (!valid) return;
        pass1_wedge(g, rbj, k, tab);
      });
    }
    flush();
    cur = -1;
    // chords (two-level flattening); theta64 sums per item in acc[lane]
    warp_flat(it.tv, [&](int j, int k, bool valid) {
      const int64_t foj = __shfl_sync(FULL_MASK, it.fo, j);
      const bool vloj = __shfl_sync(FULL_MASK, it.vlo, j);
      const int32_t vj = __shfl_sync(FULL_MASK, it.v, j);
      chords_step<PASS>(g, u, valid, vj, foj, vloj, k, j, tab, acc, &o);
    });
    __syncwarp();
    if (PASS == 2) {
      if (have && acc[lane]) xadd(o, PO_R64, it.v, acc[lane]);
      acc[lane] = 0;
      __syncwarp();
    }
  }
}

// developer phase timers (EVOKE_DEBUG sets g_pair_prof): SM cycles per phase summed over
// sources, CTA tiers
__device__ unsigned long long g_pair_phase[2][8];
__device__ int g_pair_prof;
#define PAIR_PHASE(i)                                                                     \
  do {                                                                                    \
    if (g_pair_prof && threadIdx.x == 0) {                                                \
      const long long t_ = clock64();                                                     \
      atomicAdd(&g_pair_phase[Tab::kDense ? 1 : 0][i], (unsigned long long)(t_ - t_prev)); \
      t_prev = t_;                                                                        \
    }                                                                                     \
  } while (0)

// ---- CTA engine ------------------------------------------------------------------------
// Sweep: warps take a few items at a time from a shared counter and flatten their short
// parts over the lanes (chords and their diamond lists on two levels, chords_step).  Wedge
// or chord parts longer than PAIR_LONG go to a shared queue; they are then cut into
// PAIR_CHUNK-element chunks that whole warps take from a second counter.  Every element is
// visited exactly once; no per-element search.
enum { PK_WEDGE = 0, PK_CHORD = 1, PK_DIAM = 2 };
// The queue of long parts lives in global memory (one region per CTA, capacity qcap): a hub
// source can have thousands of long parts, and an overflowing queue would push them back
// onto single warps.
struct EngQueue {
  int64_t* qslot;   // item slot s_uv (wedge / chord parts) or chord entry r (diamond)
  int32_t* qv;      // v (diamond parts)
  int8_t* qkind;
  int8_t* qvlo;
  int32_t* lc0;     // first chunk of each part of the current round (+1 entry)
  int qcap;
};
template <int NW>
struct EngSharedT {
  int next;
  int qn;
  int next_chunk;
  int nchunks;
  EngQueue Q;
  u64 acc[NW][32];  // per-warp theta64 accumulators (chords_step)
};
// bytes of one queue region of capacity qcap
__host__ __device__ __forceinline__ size_t eng_queue_bytes(int qcap) {
  const size_t b = (size_t)qcap * (8 + 4 + 1 + 1) + (size_t)(qcap + 1) * 4 + 64;
  return (b + 255) & ~(size_t)255;  // every region starts 256-byte aligned (int64 slots first)
}
__device__ __forceinline__ EngQueue eng_queue_at(char* base, int qcap) {
  EngQueue q;
  q.qslot = reinterpret_cast<int64_t*>(base);
  q.qv = reinterpret_cast<int32_t*>(base + (size_t)qcap * 8);
  q.lc0 = q.qv + qcap;
  q.qkind = reinterpret_cast<int8_t*>(q.lc0 + qcap + 1);
  q.qvlo = q.qkind + qcap;
  q.qcap = qcap;
  return q;
}
template <typename ES>
struct CtaDefer {
  ES* E;
  __device__ __forceinline__ bool operator()(int64_t r, int32_t v, bool vlo) const {
    const int q = atomicAdd(&E->qn, 1);
    if (q >= E->Q.qcap) return false;
    E->Q.qslot[q] = r; E->Q.qv[q] = v; E->Q.qkind[q] = PK_DIAM; E->Q.qvlo[q] = vlo;
    return true;
  }
};
__device__ __forceinline__ int part_len(const DGraph& g, const EngQueue& Q, int q, int32_t u, int32_t hs) {
  const int kind = Q.qkind[q];
  if (kind == PK_DIAM) {
    const int64_t r = Q.qslot[q];
    const int32_t evw = Q.qvlo[q] ? g.fe1[r] : g.fe2[r];
    return (int)(g.foff[evw + 1] - g.foff[evw]);
  }
  const PairItem it = pair_item(g, u, Q.qslot[q], hs);
  return kind == PK_WEDGE ? it.dv : it.tv;
}

template <int PASS, int BT, typename Tab, typename ES>
__device__ void cta_pass(const DGraph& g, const u32* __restrict__ Te, int32_t u, int32_t hs, int64_t r0, int64_t r1,
                         Tab& tab, ES& E, u64& s51, const PairOut& o) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  u64* acc = E.acc[wib];
  long long t_prev = clock64();
  if (threadIdx.x == 0) { E.next = 0; E.qn = 0; }
  acc[lane] = 0;
  __syncthreads();
  const int64_t nitems = r1 - r0;
  // items per warp grab: about four grabs per warp (dynamic balance), at most 32
  const int grab = (int)min((int64_t)32, max((int64_t)1, nitems / (4 * (int64_t)(blockDim.x >> 5))));
  for (;;) {
    int base = 0;
    if (lane == 0) base = atomicAdd(&E.next, grab);
    base = __shfl_sync(FULL_MASK, base, 0);
    if (base >= nitems) break;
    PairItem it;
    const bool have = lane < grab && base + lane < nitems;
    if (have) it = pair_item(g, u, r0 + base + lane, hs);
    else { it.v = 0; it.e = 0; it.rb = 0; it.fo = 0; it.dv = 0; it.tv = 0; it.vlo = false; }
    const int tuv = it.tv;  // T(u,v) for the wedges' x-side terms (it.tv is zeroed if the chords are queued)
    // defer long parts to the queue (if it has room)
    const int long_min = PAIR_LONG;
    if (it.dv > long_min) {
      const int q = atomicAdd(&E.qn, 1);
      if (q < E.Q.qcap) { E.Q.qslot[q] = r0 + base + lane; E.Q.qkind[q] = PK_WEDGE; it.dv = 0; }
    }
    if (it.tv > long_min) {
      const int q = atomicAdd(&E.qn, 1);
      if (q < E.Q.qcap) { E.Q.qslot[q] = r0 + base + lane; E.Q.qkind[q] = PK_CHORD; it.tv = 0; }
    }
    PairAcc A;
    A.zero();
    int cur = -1;
    int32_t cv = 0, ce = 0;
    auto flush = [&]() {
      if (PASS == 2 && cur >= 0) A.flush(u, cv, ce, o);
    };
    if (PASS == 2) {
      wedges_pass2_ilp(g, Te, u, it.dv, it.rb, it.v, it.e, tuv, tab, s51, o);
    } else {
      warp_flat(it.dv, [&](int j, int k, bool valid) {
        const int64_t rbj = __shfl_sync(FULL_MASK, it.rb, j);
        if (!valid) return;
        pass1_wedge(g, rbj, k, tab);
      });
    }
    flush();
    warp_flat(it.tv, [&](int j, int k, bool valid) {
      const int64_t foj = __shfl_sync(FULL_MASK, it.fo, j);
      const bool vloj = __shfl_sync(FULL_MASK, it.vlo, j);
      const int32_t vj = __shfl_sync(FULL_MASK, it.v, j);
      chords_step<PASS>(g, u, valid, vj, foj, vloj, k, j, tab, acc, &o, CtaDefer<ES>{&E});
    });
    __syncwarp();
    if (PASS == 2) {
      if (have && acc[lane]) xadd(o, PO_R64, it.v, acc[lane]);
      acc[lane] = 0;
      __syncwarp();
    }
  }
  __syncthreads();
  PAIR_PHASE(5);
  // rounds over the queued parts, cut in chunks (chord chunks may queue diamond lists)
  int qb = 0;
  for (;;) {
  const int qe = min(E.qn, E.Q.qcap);
  if (qb >= qe) break;  // uniform (E.qn read after a barrier)
  const int nq = qe - qb;
  {
    // chunk table of the round: CTA-wide exclusive scan of the parts' chunk counts
    typedef cub::BlockScan<int, BT> CScan;
    __shared__ typename CScan::TempStorage cscan;
    __shared__ int s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int q0 = 0; q0 < nq; q0 += blockDim.x) {
      const int q = q0 + threadIdx.x;
      const int nc = (q < nq) ? (part_len(g, E.Q, qb + q, u, hs) + PAIR_CHUNK - 1) / PAIR_CHUNK : 0;
      int ex = 0, tot = 0;
      if (blockDim.x == BT) {
        CScan(cscan).ExclusiveSum(nc, ex, tot);
      } else {
        // smaller CTA: warp scans chained through shared memory
        __shared__ int wsum[BT / 32];
        int incl = nc;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int y = __shfl_up_sync(FULL_MASK, incl, d);
          if (lane >= d) incl += y;
        }
        if (lane == 31) wsum[wib] = incl;
        __syncthreads();
        int before = 0;
        tot = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
          if (w < wib) before += wsum[w];
          tot += wsum[w];
        }
        ex = before + incl - nc;
        __syncthreads();
      }
      if (q < nq) E.Q.lc0[q] = s_carry + ex;
      __syncthreads();
      if (threadIdx.x == 0) s_carry += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) { E.Q.lc0[nq] = s_carry; E.nchunks = s_carry; E.next_chunk = 0; }
  }
  __syncthreads();
  const int nchunks = E.nchunks;
  for (;;) {
    int c = 0;
    if (lane == 0) c = atomicAdd(&E.next_chunk, 1);
    c = __shfl_sync(FULL_MASK, c, 0);
    if (c >= nchunks) break;
    int ql = 0;
    if (lane == 0) {
      int lo = 0, hi = nq;  // largest part with lc0 <= c
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (E.Q.lc0[mid] <= c) lo = mid; else hi = mid;
      }
      ql = lo;
    }
    ql = __shfl_sync(FULL_MASK, ql, 0);
    const int q = qb + ql;
    const int kind = E.Q.qkind[q];
    const int k0 = (c - E.Q.lc0[ql]) * PAIR_CHUNK;
    PairAcc A;
    A.zero();
    if (kind == PK_DIAM) {
      const int64_t r = E.Q.qslot[q];
      const int32_t evw = E.Q.qvlo[q] ? g.fe1[r] : g.fe2[r];
      const int64_t f0 = g.foff[evw];
      const int k1 = min((int)(g.foff[evw + 1] - f0), k0 + PAIR_CHUNK);
      for (int k = k0 + lane; k < k1; k += 32) {
        const int32_t x = g.fx[f0 + k];
        if (PASS == 1) {
          if (x > u) tab.add_d(x);
        } else {
          if (x > u) A.c64 += tab.get_w(x) - 2ull;
        }
      }
      if (PASS == 2) {  // both chord ends: v (queued) and w = fx[r]
        A.c64 = warp_sum(A.c64);
        if (lane == 0 && A.c64) {
          xadd(o, PO_R64, E.Q.qv[q], A.c64);
          xadd(o, PO_R64, g.fx[r], A.c64);
        }
      }
      continue;
    }
    const PairItem it = pair_item(g, u, E.Q.qslot[q], hs);
    if (kind == PK_WEDGE) {
      // PAIR_CHUNK / 32 elements per lane, all loads issued before the table updates
      constexpr int U = PAIR_CHUNK / 32;
      const int k1 = min(it.dv, k0 + PAIR_CHUNK);
      int32_t xs[U];
#pragma unroll
      for (int i = 0; i < U; i++) {
        const int k = k0 + lane + 32 * i;
        xs[i] = k < k1 ? g.ci[it.rb + k] : u;
      }
      if (PASS == 1) {
        if constexpr (Tab::kDense) {
          typename Tab::WordT olds[U];
#pragma unroll
          for (int i = 0; i < U; i++) olds[i] = xs[i] != u ? tab.raw_add(xs[i], 1) : 1;
#pragma unroll
          for (int i = 0; i < U; i++)
            if (xs[i] != u) tab.after_w(xs[i], olds[i]);
        } else {
#pragma unroll
          for (int i = 0; i < U; i++)
            if (xs[i] != u) tab.add_w(xs[i]);
        }
      } else {
        u32 te[U];
        u64 wv[U], dv[U];
#pragma unroll
        for (int i = 0; i < U; i++) {
          wv[i] = 0; dv[i] = 0;
          if (xs[i] > u) tab.get(xs[i], wv[i], dv[i]);
        }
#pragma unroll
        for (int i = 0; i < U; i++) {
          const int k = k0 + lane + 32 * i;
          te[i] = wv[i] >= 2 ? g.tes[it.rb + k] : 0u;  // W = 1 pairs contribute nothing
        }
#pragma unroll
        for (int i = 0; i < U; i++) {
          if (wv[i] < 2) continue;
          const u64 w = wv[i];
          A.c5 += w - 1;
          s51 += (u64)te[i] * (w - 1);
          A.c49 += binom2(w - 1);
          A.c62 += dv[i];
          wedge_x_side(g, o, xs[i], it.v, it.rb + k0 + lane + 32 * i, it.tv, w);
        }
      }
    } else {
      const int k1 = min(it.tv, k0 + PAIR_CHUNK);
      for (int i = 0; i < PAIR_CHUNK / 32; i++) {
        const int k = k0 + lane + 32 * i;
        chords_step<PASS>(g, u, k < k1, it.v, it.fo, it.vlo, k, 0, tab, acc, &o, CtaDefer<ES>{&E});
      }
      __syncwarp();
      if (PASS == 2 && lane == 0) {
        A.c64 = acc[0];
        acc[0] = 0;
      }
      __syncwarp();
    }
    if (PASS == 2) {
      A.c5 = warp_sum(A.c5); A.c49 = warp_sum(A.c49); A.c62 = warp_sum(A.c62);
      if (lane == 0) A.flush(u, it.v, it.e, o);
    }
  }
  __syncthreads();
  qb = qe;
  }
  PAIR_PHASE(6);
}

// ---- the h* contribution ----------------------------------------------------------------
// After pass 1 the table holds W_R(u,x), the common neighbours other than h*.  Then
// W(u,x) = W_R + [x in N(h*)] for every key, and keys absent from the table have W <= 1 and
// contribute nothing, so the wedges u - h* - x are never inserted.  Two ways to add the
// h* term, chosen per source by cost: walk N(h*) and look every x up in the table
// (hstar_walk, cost d(h*)), or binary-search every key in the sorted N(h*) (hstar_search,
// cost #keys * log d(h*)).  Both also emit the terms of the wedges u - h* - x with W >= 2
// (E5 of e(u,h*), theta49/62 of h*, theta51 of u) into H / s51.
template <typename Tab>
__device__ __forceinline__ void hstar_walk(const DGraph& g, const PairOut& o, int32_t u, int32_t hs, int64_t hfrom,
                                           int tuh, const Tab& tab, int tid, int nthr, PairAcc& H, u64& s51) {
  const int64_t he = g.rp[hs + 1];
  for (int64_t p = hfrom + tid; p < he; p += nthr) {  // x > u: the suffix of N(h*) after u
    const int32_t x = g.ci[p];
    auto* wp = tab.word_if(x);
    if (!wp) continue;
    const auto v = *wp + 1;  // x is visited once: plain update
    *wp = v;
    const u64 w = Tab::wfield(v), d = Tab::dfield(v);
    if (w < 2) continue;
    H.c5 += w - 1;
    s51 += (u64)g.tes[p] * (w - 1);
    H.c49 += binom2(w - 1);
    H.c62 += d;
    wedge_x_side(g, o, x, hs, p, tuh, w);
  }
}

// The h* term by the cheapest available way, fused with the per-pair terms when the table
// is swept anyway (map / key search): returns true when a8..a63 were already added.
// hfrom = the first slot of N(h*) above u; tuh = T(u, h*)
template <typename Tab>
__device__ __forceinline__ bool hstar_and_terms(const DGraph& g, int32_t u, int32_t hs, int64_t hfrom, int tuh,
                                                const PairOut& o, Tab& tab, int tid, int nthr, u64 nkeys_bound,
                                                PairAcc& H, u64& s51, u64& a8, u64& a36, u64& a50, u64& a63) {
  if (hs < 0) return false;
  const int32_t slot = o.hub_slot[hs];
  const int64_t hb = g.rp[hs], he = g.rp[hs + 1];
  const bool walk = Tab::kDense || (slot < 0 && (u64)(he - hfrom) <= 12ull * nkeys_bound);
  if (walk) {
    hstar_walk(g, o, u, hs, hfrom, tuh, tab, tid, nthr, H, s51);
    return false;
  }
  const int32_t* pmap = slot >= 0 ? o.hub_pos + (size_t)slot * (size_t)g.n : nullptr;
  const u64 du = (u64)dg_deg(g, u);
  tab.for_each_mut(tid, nthr, [&](int32_t x, u64 w, u64 d) -> u64 {
    int64_t p = -1;  // slot of x in N(h*) when x ~ h*
    if (pmap) {
      const int32_t q = pmap[x];  // position of x in N(h*), or -1
      if (q >= 0) p = hb + q;
    } else {
      const int64_t q = lower_bound_dev<int32_t>(g.ci, hfrom, he, x);
      if (q < he && g.ci[q] == x) p = q;
    }
    if (p >= 0) {
      w += 1;
      if (w >= 2) {
        H.c5 += w - 1;
        s51 += (u64)g.tes[p] * (w - 1);
        H.c49 += binom2(w - 1);
        H.c62 += d;
        wedge_x_side(g, o, x, hs, p, tuh, w);
      }
    }
    pair_c_terms(g, o, du, x, w, d, a8, a36, a50, a63);
    return w;
  });
  return true;
}

// adjacency maps of the hubs (d >= PAIR_HUBMAP_MIN) up to max_slots rows
__global__ void k_hub_slots(DGraph g, int max_slots, int32_t* __restrict__ slot, int32_t* __restrict__ hubs,
                            int* __restrict__ cnt) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < g.n; v += gridDim.x * blockDim.x) {
    int32_t sl = -1;
    if (dg_deg(g, v) >= PAIR_HUBMAP_MIN) {
      const int q = atomicAdd(cnt, 1);
      if (q < max_slots) {
        sl = q;
        hubs[q] = v;
      }
    }
    slot[v] = sl;
  }
}
// block per hub: row[x] = position of x in N(hub) for x in N(hub) (the rows start at -1)
__global__ void k_hub_maps(DGraph g, const u32* __restrict__ Te, const int32_t* __restrict__ hubs, int nhubs,
                           int32_t* __restrict__ pos) {
  for (int q = blockIdx.x; q < nhubs; q += gridDim.x) {
    const int32_t v = hubs[q];
    int32_t* row = pos + (size_t)q * (size_t)g.n;
    const int64_t b = g.rp[v], e = g.rp[v + 1];
    for (int64_t k = b + threadIdx.x; k < e; k += blockDim.x) row[g.ci[k]] = (int32_t)(k - b);
  }
}

// per-pair terms over the final table (keys with W >= 2)
template <typename Tab>
__device__ __forceinline__ void entry_terms(const DGraph& g, const PairOut& o, int32_t u, Tab& tab, int tid,
                                            int nthr, u64& a8, u64& a36, u64& a50, u64& a63) {
  const u64 du = (u64)dg_deg(g, u);
  tab.for_each_mut(tid, nthr, [&](int32_t x, u64 w, u64 d) -> u64 {
    pair_c_terms(g, o, du, x, w, d, a8, a36, a50, a63);
    return w;
  });
}

// theta51 correction sum_{x in N(u)} W(u,x)(W(u,x)-1), from the pairs' lower ends: the
// neighbours x > u of u (the suffix of N(u) after its dm(u) lower neighbours)
template <typename Tab>
__device__ __forceinline__ void s51_adjacent(const DGraph& g, const PairOut& o, int32_t u, const Tab& tab, int tid,
                                             int nthr, u64& s51) {
  for (int64_t s = g.rp[u] + g.dm[u] + tid; s < g.rp[u + 1]; s += nthr) {
    const int32_t x = g.ci[s];
    const u64 w = tab.get_w_or0(x);
    if (w < 2) continue;
    s51 -= w * (w - 1);
    xadd(o, PO_R51, x, (u64)0 - w * (w - 1));
  }
}

// h* of u: the first slot of N(h*) above u, and T(u, h*)
// (p: the slot of h* in N(u), from k_pair_est; its twin is u's slot in N(h*))
__device__ __forceinline__ void hstar_info(const DGraph& g, int32_t hs, int32_t p, int64_t& hfrom, int& tuh,
                                           int32_t& euh) {
  hfrom = 0; tuh = 0; euh = -1;
  if (hs < 0) return;
  euh = g.eid[p];
  tuh = (int)g.tes[p];
  hfrom = (int64_t)g.twin[p] + 1;
}

// slot of h* in N(u) -> edge id e(u, h*)
__device__ __forceinline__ int32_t edge_of(const DGraph& g, int32_t u, int32_t v) {
  const int64_t p = lower_bound_dev<int32_t>(g.ci, g.rp[u], g.rp[u + 1], v);
  return g.eid[p];
}

// ---- one source on a CTA (mid and heavy tiers) ------------------------------------------
template <int BT, typename Tab, typename ES>
__device__ void pair_source_cta(const DGraph& g, const u32* __restrict__ Te, int32_t u, Tab& tab, ES& E,
                                u64* red, const PairOut& o, u32 tab_keys_bound) {
  const int64_t r0 = g.rp[u], r1 = g.rp[u + 1];
  const int32_t hs = o.hstar[u];
  int64_t hfrom;
  int tuh;
  int32_t euh;
  hstar_info(g, hs, hs >= 0 ? o.hstar_s[u] : 0, hfrom, tuh, euh);
  u64 s51 = 0;
  long long t_prev = clock64();
  cta_pass<1, BT>(g, Te, u, hs, r0, r1, tab, E, s51, o);
  PAIR_PHASE(0);
  u64 a8 = 0, a36 = 0, a50 = 0, a63 = 0;
  PairAcc H;
  H.zero();
  const bool fused = hstar_and_terms(g, u, hs, hfrom, tuh, o, tab, threadIdx.x, BT, (u64)tab_keys_bound, H, s51, a8,
                                     a36, a50, a63);
  H.c5 = warp_sum(H.c5); H.c49 = warp_sum(H.c49); H.c62 = warp_sum(H.c62);
  if ((threadIdx.x & 31) == 0) {
    if (H.c5) atomicAdd(&red[5], H.c5);
    if (H.c49) atomicAdd(&red[6], H.c49);
    if (H.c62) atomicAdd(&red[7], H.c62);
  }
  __syncthreads();
  PAIR_PHASE(1);
  if (!fused) {
    entry_terms(g, o, u, tab, threadIdx.x, BT, a8, a36, a50, a63);
    __syncthreads();  // W final
  }
  PAIR_PHASE(2);
  cta_pass<2, BT>(g, Te, u, hs, r0, r1, tab, E, s51, o);
  PAIR_PHASE(3);
  s51_adjacent(g, o, u, tab, threadIdx.x, BT, s51);
  a8 = warp_sum(a8); a36 = warp_sum(a36); a50 = warp_sum(a50); a63 = warp_sum(a63); s51 = warp_sum(s51);
  if ((threadIdx.x & 31) == 0) {
    if (a8) atomicAdd(&red[0], a8);
    if (a36) atomicAdd(&red[1], a36);
    if (a50) atomicAdd(&red[2], a50);
    if (s51) atomicAdd(&red[3], s51);
    if (a63) atomicAdd(&red[4], a63);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // atomics: the pairs' lower ends credit their upper ends concurrently
    if (red[0]) xadd(o, PO_R8, u, red[0]);
    if (red[1]) xadd(o, PO_R36, u, red[1]);
    if (red[2]) xadd(o, PO_R50, u, red[2]);
    if (red[3]) xadd(o, PO_R51, u, red[3]);
    if (red[4]) xadd(o, PO_R63, u, red[4]);
    if (hs >= 0) {
      H.c5 = red[5]; H.c49 = red[6]; H.c62 = red[7]; H.c64 = 0;
      H.flush(u, hs, euh, o);
    }
    for (int i = 0; i < 8; i++) red[i] = 0;
  }
  tab.reset(threadIdx.x, BT);
  __syncthreads();
  PAIR_PHASE(4);
}

// ---- light tier: one warp per source --------------------------------------------------
__device__ void pair_source_warp(const DGraph& g, const u32* __restrict__ Te, int32_t u, u32 cap,
                                 SharedPackedHash& tab, const PairOut& o, u64* acc) {
  const int lane = threadIdx.x & 31;
  const int64_t r0 = g.rp[u], r1 = g.rp[u + 1];
  const int32_t hs = o.hstar[u];
  int64_t hfrom;
  int tuh;
  int32_t euh;
  hstar_info(g, hs, hs >= 0 ? o.hstar_s[u] : 0, hfrom, tuh, euh);
  tab.mask = cap - 1;
  u64 s51 = 0;
  warp_pass<1>(g, Te, u, hs, r0, r1, tab, s51, o, acc);
  __syncwarp();
  u64 a8 = 0, a36 = 0, a50 = 0, a63 = 0;
  PairAcc H;
  H.zero();
  const bool fused = hstar_and_terms(g, u, hs, hfrom, tuh, o, tab, lane, 32, (u64)(cap / 2), H, s51, a8, a36, a50,
                                     a63);
  __syncwarp();
  if (!fused) {
    entry_terms(g, o, u, tab, lane, 32, a8, a36, a50, a63);
    __syncwarp();
  }
  warp_pass<2>(g, Te, u, hs, r0, r1, tab, s51, o, acc);
  s51_adjacent(g, o, u, tab, lane, 32, s51);
  a8 = warp_sum(a8); a36 = warp_sum(a36); a50 = warp_sum(a50); a63 = warp_sum(a63); s51 = warp_sum(s51);
  H.c5 = warp_sum(H.c5); H.c49 = warp_sum(H.c49); H.c62 = warp_sum(H.c62);
  if (lane == 0) {
    if (a8) xadd(o, PO_R8, u, a8);
    if (a36) xadd(o, PO_R36, u, a36);
    if (a50) xadd(o, PO_R50, u, a50);
    if (s51) xadd(o, PO_R51, u, s51);
    if (a63) xadd(o, PO_R63, u, a63);
    if (hs >= 0) H.flush(u, hs, euh, o);
  }
  __syncwarp();
  tab.reset(lane, 32);
  __syncwarp();
}

// Mid and light tiers: persistent CTAs take mid sources (one CTA each, packed shared
// hash) from mid[0, n_mid), then each warp takes light sources from light[0, n_light).
#ifndef PAIR_MAIN_MINB
#define PAIR_MAIN_MINB 3  // resident CTAs per SM the register budget must allow (shared memory allows 3)
#endif
__global__ void __launch_bounds__(PAIR_BT, PAIR_MAIN_MINB) k_pairs_main(DGraph g, const u32* __restrict__ Te,
                                                        const int32_t* __restrict__ mid, int n_mid,
                                                        const int32_t* __restrict__ light, int n_light,
                                                        const u32* __restrict__ est, int* __restrict__ counters,
                                                        PairOut o_, char* __restrict__ qmem, int qcap) {
  extern __shared__ int32_t sh_pairs[];
  __shared__ EngSharedT<PAIR_BT / 32> E;
  __shared__ u64 red[8];
  __shared__ int s_idx;
  const PairOut& o = o_;
  if (threadIdx.x < 8) red[threadIdx.x] = 0;
  if (threadIdx.x == 0) E.Q = eng_queue_at(qmem + (size_t)blockIdx.x * eng_queue_bytes(qcap), qcap);
  {
    SharedPackedHash tab;
    tab.keys = sh_pairs;
    tab.val = (u32*)(sh_pairs + PAIR_MID_CAP);
    for (u32 h = threadIdx.x; h < PAIR_MID_CAP; h += PAIR_BT) { tab.keys[h] = EMPTY_KEY; tab.val[h] = 0u; }
    for (;;) {
      if (threadIdx.x == 0) s_idx = atomicAdd(&counters[0], 1);
      __syncthreads();
      const int idx = s_idx;
      __syncthreads();
      if (idx >= n_mid) break;
      const int32_t u = mid[idx];
      tab.mask = min(pow2_at_least(2u * est[u], 64u), (u32)PAIR_MID_CAP) - 1;
      pair_source_cta<PAIR_BT>(g, Te, u, tab, E, red, o, est[u]);  // leaves the table clean
    }
  }
  // light tier: per-warp packed hash in the dynamic shared memory
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  SharedPackedHash tab;
  tab.keys = sh_pairs + wib * (2 * PAIR_WARP_CAP);
  tab.val = (u32*)(tab.keys + PAIR_WARP_CAP);
  for (int h = lane; h < PAIR_WARP_CAP; h += 32) { tab.keys[h] = EMPTY_KEY; tab.val[h] = 0u; }
  u64* acc = E.acc[wib];
  acc[lane] = 0;
  __syncwarp();
  for (;;) {
    int idx = 0;
    if (lane == 0) idx = atomicAdd(&counters[1], 2);
    idx = __shfl_sync(FULL_MASK, idx, 0);
    if (idx >= n_light) break;
    const int end = min(idx + 2, n_light);
    for (int q = idx; q < end; q++) {
      const int32_t u = light[q];
      const u32 cap = pow2_at_least(2u * est[u], 32u);
      pair_source_warp(g, Te, u, cap, tab, o, acc);
    }
  }
}

// Tiny tier (est <= PAIR_TINY_MAX): the light tier's warp per source with a per-warp hash of
// PAIR_TINY_CAP entries (2 KB instead of 8 KB) in a kernel of its own, so the shared memory
// and a smaller register budget let PAIR_TINY_MINB CTAs share an SM (the main kernel's mid
// tier holds it to three)
template <int WCAP>
__global__ void __launch_bounds__(PAIR_BT, PAIR_TINY_MINB) k_pairs_tiny(DGraph g, const u32* __restrict__ Te,
                                                                       const int32_t* __restrict__ light, int n_light,
                                                                       const u32* __restrict__ est,
                                                                       int* __restrict__ counter, PairOut o_) {
  __shared__ int32_t sh_tiny[PAIR_BT / 32][2 * WCAP];
  __shared__ u64 sh_acc[PAIR_BT / 32][32];
  const PairOut& o = o_;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  SharedPackedHash tab;
  tab.keys = sh_tiny[wib];
  tab.val = (u32*)(tab.keys + WCAP);
  for (int h = lane; h < WCAP; h += 32) { tab.keys[h] = EMPTY_KEY; tab.val[h] = 0u; }
  u64* acc = sh_acc[wib];
  acc[lane] = 0;
  __syncwarp();
  for (;;) {
    int idx = 0;
    if (lane == 0) idx = atomicAdd(counter, 2);
    idx = __shfl_sync(FULL_MASK, idx, 0);
    if (idx >= n_light) break;
    const int end = min(idx + 2, n_light);
    for (int q = idx; q < end; q++) {
      const int32_t u = light[q];
      const u32 cap = pow2_at_least(2u * est[u], 32u);  // <= WCAP (est <= PAIR_TINY_MAX)
      pair_source_warp(g, Te, u, cap, tab, o, acc);
    }
  }
}

// Small-mid tier: persistent CTAs of PAIR_MIDS_BT threads take one source each (packed
// shared hash of PAIR_MIDS_CAP entries).  Smaller CTAs than the mid tier: a source's phases
// are latency-bound and separated by CTA barriers, so more sources in flight per SM (five
// instead of three) hide more of the latency than more threads per source would.
#ifndef PAIR_MIDS_MINB
#define PAIR_MIDS_MINB 5  // resident small-mid CTAs per SM the register budget must allow (96 registers: config 4
                          // pair pass 40.9 -> 38.7 ms against 126 registers / 4 CTAs; 6 CTAs: 39.0 ms)
#endif
__global__ void __launch_bounds__(PAIR_MIDS_BT, PAIR_MIDS_MINB) k_pairs_mids(DGraph g, const u32* __restrict__ Te,
                                                             const int32_t* __restrict__ mids, int n_mids,
                                                             const u32* __restrict__ est, int* __restrict__ counter,
                                                             PairOut o_, char* __restrict__ qmem, int qcap) {
  extern __shared__ int32_t sh_pairs[];
  __shared__ EngSharedT<PAIR_MIDS_BT / 32> E;
  __shared__ u64 red[8];
  __shared__ int s_idx;
  const PairOut& o = o_;
  if (threadIdx.x < 8) red[threadIdx.x] = 0;
  if (threadIdx.x == 0) E.Q = eng_queue_at(qmem + (size_t)blockIdx.x * eng_queue_bytes(qcap), qcap);
  SharedPackedHash tab;
  tab.keys = sh_pairs;
  tab.val = (u32*)(sh_pairs + PAIR_MIDS_CAP);
  for (u32 h = threadIdx.x; h < PAIR_MIDS_CAP; h += PAIR_MIDS_BT) { tab.keys[h] = EMPTY_KEY; tab.val[h] = 0u; }
  for (;;) {
    if (threadIdx.x == 0) s_idx = atomicAdd(counter, 1);
    __syncthreads();
    const int idx = s_idx;
    __syncthreads();
    if (idx >= n_mids) break;
    const int32_t u = mids[idx];
    tab.mask = min(pow2_at_least(2u * est[u], 64u), (u32)PAIR_MIDS_CAP) - 1;
    pair_source_cta<PAIR_MIDS_BT>(g, Te, u, tab, E, red, o, est[u]);  // leaves the table clean
  }
}

// Heavy tier: one CTA per source, dense per-CTA table in global memory (Word = u32
// packed W|D<<16, or u64 W|D<<32 for sources past the 16-bit bounds).
template <typename Word, bool SCAN>
__global__ void __launch_bounds__(PAIR_HBT) k_pairs_heavy(DGraph g, const u32* __restrict__ Te,
                                                          const int32_t* __restrict__ srcs, int nsrc,
                                                          int* __restrict__ counter, Word* __restrict__ tabs,
                                                          int32_t* __restrict__ lists, PairOut o_,
                                                          char* __restrict__ qmem, int qcap, int hot_k) {
  extern __shared__ __align__(16) unsigned char pair_hot_sh[];
  __shared__ EngSharedT<PAIR_HBT / 32> E;
  __shared__ u64 red[8];
  __shared__ int s_idx, s_ntouch;
  const PairOut& o = o_;
  if (threadIdx.x == 0) E.Q = eng_queue_at(qmem + (size_t)blockIdx.x * eng_queue_bytes(qcap), qcap);
  GlobalDense<Word, SCAN> tab;
  constexpr int PER = GlobalDense<Word, SCAN>::PER;
  const size_t stride = (size_t)((g.n + PER - 1) / PER * PER);  // 16-byte aligned rows
  tab.t = tabs + (size_t)blockIdx.x * stride;
  tab.L = SCAN ? nullptr : lists + (size_t)blockIdx.x * g.n;
  tab.ntouch = &s_ntouch;
  tab.n = g.n;
  if (hot_k > 0) {
    tab.hot = reinterpret_cast<Word*>(pair_hot_sh);
    tab.hot0 = g.n - hot_k;
    tab.hotK = hot_k;
    for (int i = threadIdx.x; i < hot_k; i += PAIR_HBT) tab.hot[i] = (Word)0;
    __syncthreads();
  }
  if (threadIdx.x < 8) red[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_ntouch = 0;
  for (;;) {
    if (threadIdx.x == 0) s_idx = atomicAdd(counter, 1);
    __syncthreads();
    const int idx = s_idx;
    __syncthreads();
    if (idx >= nsrc) break;
    const long long ut = unit_t0();
    pair_source_cta<PAIR_HBT>(g, Te, srcs[idx], tab, E, red, o, 0u);
    unit_t1(0, ut, idx);
    if (threadIdx.x == 0) s_ntouch = 0;
  }
}

// Diamond work of every source u: D(u) = sum over the triangles (u, v, w) of T(v, w), the
// diamond elements its chords lead to.  One thread per triangle, three atomics (a triangle
// a, b, c gives T(b,c) to a, T(a,c) to b and T(a,b) to c).
__global__ void k_pair_dwork(DGraph g, const u32* __restrict__ Te, u64* __restrict__ dwork) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < g.ntri; q += (int64_t)gridDim.x * blockDim.x) {
    const int32_t eab = g.tab[q], eac = g.tac[q], ebc = g.tbc[q];
    atomicAdd((unsigned long long*)&dwork[g.esrc[eab]], (u64)Te[ebc]);
    atomicAdd((unsigned long long*)&dwork[g.edst[eab]], (u64)Te[eac]);
    atomicAdd((unsigned long long*)&dwork[g.tc[q]], (u64)Te[eab]);
  }
}

// Work estimate of source u: west(u) = sum_{v in N(u), v != h*} |{x in N(v) : x > u}|, the
// wedge elements walked (>= the number of table keys: every diamond end is also the end of a
// walked wedge), and the sort key ~(west + D(u)) (D: the diamond work, nullptr: none), so
// the tiers and the heaviest-first order see the chords' diamond lists too (a source with
// few wedges can own long diamond lists).  h*(u) = the neighbour with the longest such suffix
// (ties: lower id).
__global__ void k_pair_est(DGraph g, const u64* __restrict__ dwork, u32* __restrict__ keys,
                           int32_t* __restrict__ vals, u32* __restrict__ west, int32_t* __restrict__ hstar,
                           int32_t* __restrict__ hstar_s, int32_t* __restrict__ plen) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t ui = gw; ui < g.n; ui += nw) {
    const int32_t u = (int32_t)ui;
    u64 s = 0;
    int32_t best = -1, bestl = -1, bests = 0;
    for (int64_t t = g.rp[u] + lane; t < g.rp[u + 1]; t += 32) {
      const int32_t v = g.ci[t];
      const int32_t len = (int32_t)(g.rp[v + 1] - g.twin[t] - 1);  // N(v) above u
      plen[t] = len;
      s += (u64)len;
      if (len > bestl || (len == bestl && v < best)) { bestl = len; best = v; bests = (int32_t)t; }
    }
    s = warp_sum(s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const int32_t ol = __shfl_xor_sync(FULL_MASK, bestl, o);
      const int32_t ob = __shfl_xor_sync(FULL_MASK, best, o);
      const int32_t os = __shfl_xor_sync(FULL_MASK, bests, o);
      if (ol > bestl || (ol == bestl && ob < best)) { bestl = ol; best = ob; bests = os; }
    }
    if (lane == 0) {
      const u64 est = best >= 0 ? s - (u64)bestl : 0;
      const u64 tot = est > 0 ? est + (dwork ? dwork[u] : 0) : 0;
      keys[u] = ~(u32)min(tot, (u64)0xffffffffu);  // ascending sort = descending estimate
      vals[u] = u;
      west[u] = (u32)min(est, (u64)0xffffffffu);
      hstar[u] = best;
      hstar_s[u] = bests;
    }
  }
}


// Shard filter of the est-sorted (descending) vertex list and tier classification.
// Lists keep the descending order approximately (warp-aggregated appends in list order).
enum { PT_G64 = 0, PT_G32, PT_G32S, PT_MID, PT_LIGHT, PT_MIDS, PT_TINY, PT_COUNT };
// tier limits: the defaults are the capacities of each tier's tables; tests lower them (env
// EVOKE_PAIR_*) to force sources onto the heavier tiers' code paths on small graphs
struct PairTiers {
  u64 packed_lim;  // d(u) and T(u) below this: packed 16-bit W | D (<= 65536)
  u64 light_max, mids_max, mid_max;  // <= PAIR_WARP_MAX, PAIR_MIDS_MAX, PAIR_MID_MAX
  u64 tiny_max;                       // <= PAIR_TINY_MAX (light sources this small: the tiny tier)
  int sweep;       // -1: by size (2-hop set >= n/16), 0: never, 1: always sweep the table
};
__global__ void k_pair_classify(DGraph g, const u32* __restrict__ skeys, const int32_t* __restrict__ svals,
                                int si, int ns, PairTiers pt, const u64* __restrict__ Tv, const u32* __restrict__ west,
                                u32* __restrict__ est_v, int32_t* __restrict__ lists, int* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = gw * 32; base < g.n; base += nw * 32) {
    const int64_t p = base + lane;
    int tier = -1;
    int32_t u = 0;
    if (p < g.n && p % ns == si) {
      u = svals[p];
      const u64 e = (u64)(u32)~skeys[p];  // wedges + diamonds: the tier
      const u64 ew = west[u];             // wedges: bounds the table keys
      est_v[u] = (u32)ew;
      if (ew > 0) {
        const bool packed_ok = (u64)dg_deg(g, u) < pt.packed_lim && Tv[u] < pt.packed_lim;
        const bool sweep = pt.sweep < 0 ? ew * 16 >= (u64)g.n : pt.sweep > 0;
        tier = !packed_ok ? PT_G64
             : (e <= pt.tiny_max && ew <= PAIR_TINY_MAX) ? PT_TINY
             : e <= pt.light_max ? PT_LIGHT
             : e <= pt.mids_max ? PT_MIDS
             : e <= pt.mid_max ? PT_MID
             : sweep ? PT_G32S  // 2-hop set a sizeable part of n: sweep the table
             : PT_G32;
      }
    }
    for (int t = 0; t < PT_COUNT; t++) warp_append(tier == t, u, lists + (size_t)t * g.n, counts + t);
  }
}

// the interleaved pair credits into the per-field arrays (fields f0.. in PairField order)
struct PairFields { u64* f[PO_STRIDE]; };
__global__ void k_pair_fields(const u64* __restrict__ pa, int32_t n, PairFields fields) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < (int64_t)n * PO_STRIDE;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = (int32_t)(q / PO_STRIDE);
    const int f = (int)(q % PO_STRIDE);
    fields.f[f][u] = pa[q];
  }
}
