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
// B200 formulation: one work unit per endpoint l.  Instead of enumerating the DP(G->)
// paths one by one, the unit builds records keyed by vertex:
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
// identity against brute force (tests/test_gpu_parity.py).
//
// Scheduling (B200): k_c5_splus / k_c5_work give every endpoint its exact work W(l) and
// record bound R(l) in O(m) total; k_c5_bin splits this shard's endpoints into light ones
// (one WARP each, packed records in a per-warp open-addressing region, shared memory when
// small), mid ones (one 128-thread CTA each, packed records in a per-CTA hash region) and
// big ones (one 1024-thread CTA each, sorted by W descending, records dense by vertex id).
// All list walks go through the load-balanced engines of sched.cuh (warp_lists / cta_lists).
#pragma once
#include "common.cuh"
#include "sched.cuh"

// Record of one vertex for one endpoint.  wf = Wn | flags << 28 (Wn < 2^28 because Wn(i)
// <= d(l) and max degree < 2^28 is checked); V = u32 when the endpoint's work bound W(l) <
// 2^32 (every field is at most W(l)), else u64.  32 or 64 bytes.
template <typename V>
struct __align__(16) C5RecT {
  int32_t key;   // hash regions: x + 1 (0 = empty); unused in dense tables
  u32 wf;        // Wn (low 28 bits) | C5_* flags (high 4 bits)
  V Q, P, A, QT, QM, S;
};
typedef C5RecT<u64> C5Rec;
// Packed record of the light and mid endpoints (W(l) <= C5_MID_MAX < 2^16, so every field
// fits 16 bits and two share a word: the additions of one never carry into the other).
// 20 bytes instead of 32, and step 2 needs two atomics instead of three.
struct __align__(4) C5RecP {
  int32_t key;
  u32 wf;
  u32 qp;   // Q | P << 16
  u32 as;   // A | S << 16
  u32 qtm;  // QT | QM << 16
};
// field access for both layouts
// Q += 1, QT += th, QM += tm, returning whether this was the record's first j-mark (Q was 0)
template <typename V>
__device__ __forceinline__ bool rec_add_q_first(C5RecT<V>* r, u32 th, u32 tm) {
  const V old = atomicAdd(&r->Q, (V)1);
  atomicAdd(&r->QT, (V)th);
  atomicAdd(&r->QM, (V)tm);
  return old == 0;
}
__device__ __forceinline__ bool rec_add_q_first(C5RecP* r, u32 th, u32 tm) {
  const u32 old = atomicAdd(&r->qp, 1u);
  atomicAdd(&r->qtm, th | (tm << 16));
  return (old & 0xffffu) == 0;
}
template <typename V>
__device__ __forceinline__ void rec_add_q(C5RecT<V>* r, u32 th, u32 tm) {
  atomicAdd(&r->Q, (V)1);
  atomicAdd(&r->QT, (V)th);
  atomicAdd(&r->QM, (V)tm);
}
__device__ __forceinline__ void rec_add_q(C5RecP* r, u32 th, u32 tm) {
  atomicAdd(&r->qp, 1u);
  atomicAdd(&r->qtm, th | (tm << 16));
}
template <typename V> __device__ __forceinline__ u64 rec_q(const C5RecT<V>* r) { return (u64)r->Q; }
template <typename V> __device__ __forceinline__ u64 rec_p(const C5RecT<V>* r) { return (u64)r->P; }
template <typename V> __device__ __forceinline__ u64 rec_a(const C5RecT<V>* r) { return (u64)r->A; }
template <typename V> __device__ __forceinline__ u64 rec_s(const C5RecT<V>* r) { return (u64)r->S; }
template <typename V> __device__ __forceinline__ u64 rec_qt(const C5RecT<V>* r) { return (u64)r->QT; }
template <typename V> __device__ __forceinline__ u64 rec_qm(const C5RecT<V>* r) { return (u64)r->QM; }
__device__ __forceinline__ u64 rec_q(const C5RecP* r) { return (u64)(r->qp & 0xffffu); }
__device__ __forceinline__ u64 rec_p(const C5RecP* r) { return (u64)(r->qp >> 16); }
__device__ __forceinline__ u64 rec_a(const C5RecP* r) { return (u64)(r->as & 0xffffu); }
__device__ __forceinline__ u64 rec_s(const C5RecP* r) { return (u64)(r->as >> 16); }
__device__ __forceinline__ u64 rec_qt(const C5RecP* r) { return (u64)(r->qtm & 0xffffu); }
__device__ __forceinline__ u64 rec_qm(const C5RecP* r) { return (u64)(r->qtm >> 16); }
template <typename V>
__device__ __forceinline__ void rec_add_pa(C5RecT<V>* r, u64 q, bool adj) {
  atomicAdd(&r->P, (V)q);
  if (adj) atomicAdd(&r->A, (V)q);
}
__device__ __forceinline__ void rec_add_pa(C5RecP* r, u64 q, bool adj) {
  atomicAdd(&r->qp, (u32)q << 16);
  if (adj) atomicAdd(&r->as, (u32)q);
}
template <typename V>
__device__ __forceinline__ void rec_add_s(C5RecT<V>* r, u64 s) { atomicAdd(&r->S, (V)s); }
__device__ __forceinline__ void rec_add_s(C5RecP* r, u64 s) { atomicAdd(&r->as, (u32)s << 16); }
template <typename V>
__device__ __forceinline__ void rec_zero(C5RecT<V>* r) {
  uint4* q = reinterpret_cast<uint4*>(r);
  const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(*r) / 16); i++) q[i] = z;
}
__device__ __forceinline__ void rec_zero(C5RecP* r) {
  r->key = 0; r->wf = 0u; r->qp = 0u; r->as = 0u; r->qtm = 0u;
}
// Record of the light endpoints (W(l) < 2^12, so every field fits 12 bits): 16 bytes, one
// aligned half-sector, instead of 20 (which straddles sectors).  wf = Wn | Q << 12 | flags << 28;
// rest = P | A << 12 | S << 24 | QT << 36 | QM << 48; step 3's P and A in one 64-bit atomic.
struct __align__(16) C5RecL {
  int32_t key;
  u32 wf;
  unsigned long long rest;
};
#define C5L_BITS 12
#define C5L_MASK 0xfffull
__device__ __forceinline__ void rec_add_q(C5RecL* r, u32 th, u32 tm) {
  atomicAdd(&r->wf, 1u << C5L_BITS);
  atomicAdd(&r->rest, ((u64)th << 36) | ((u64)tm << 48));
}
__device__ __forceinline__ bool rec_add_q_first(C5RecL* r, u32 th, u32 tm) {
  const u32 old = atomicAdd(&r->wf, 1u << C5L_BITS);
  atomicAdd(&r->rest, ((u64)th << 36) | ((u64)tm << 48));
  return ((old >> C5L_BITS) & (u32)C5L_MASK) == 0;
}
__device__ __forceinline__ u64 rec_q(const C5RecL* r) { return (u64)(r->wf >> C5L_BITS) & C5L_MASK; }
__device__ __forceinline__ u64 rec_p(const C5RecL* r) { return r->rest & C5L_MASK; }
__device__ __forceinline__ u64 rec_a(const C5RecL* r) { return (r->rest >> 12) & C5L_MASK; }
__device__ __forceinline__ u64 rec_s(const C5RecL* r) { return (r->rest >> 24) & C5L_MASK; }
__device__ __forceinline__ u64 rec_qt(const C5RecL* r) { return (r->rest >> 36) & C5L_MASK; }
__device__ __forceinline__ u64 rec_qm(const C5RecL* r) { return (r->rest >> 48) & C5L_MASK; }
__device__ __forceinline__ void rec_add_pa(C5RecL* r, u64 q, bool adj) {
  atomicAdd(&r->rest, adj ? (q | (q << 12)) : q);
}
__device__ __forceinline__ void rec_add_s(C5RecL* r, u64 s) { atomicAdd(&r->rest, s << 24); }
__device__ __forceinline__ void rec_zero(C5RecL* r) { *reinterpret_cast<uint4*>(r) = make_uint4(0, 0, 0, 0); }

#define C5_WN_MASK 0x0fffffffu
template <typename R>
__device__ __forceinline__ u32 c5_flags(const R* r) { return r->wf >> 28; }
template <typename R>
__device__ __forceinline__ u64 c5_wn(const R* r) { return (u64)(r->wf & C5_WN_MASK); }
__device__ __forceinline__ u64 c5_wn(const C5RecL* r) { return (u64)(r->wf & (u32)C5L_MASK); }
#define C5_ADJ 1u      // vertex is a neighbour of l
#define C5_I 2u        // i-key: Wn > 0 (dense records; hashed records test Wn itself)
#define C5_J 4u        // j-key (step 2)
#define C5_PRESENT 8u  // record in use (touched list)

#define C5_BT 256
#define C5_WARP_MAX 1024          // light endpoint: record bound R(l) <= this ...
#define C5_WARP_WORK 4095         // ... and work W(l) <= this (12-bit record fields)
#define C5_WARP_CAP (2 * C5_WARP_MAX)  // records per warp region (load <= 0.5; global only when EVOKE_C5_SHCAP < it)
#define C5_SH_CAP 512             // light endpoints with a region of <= sh_cap (<= this) slots: shared memory
#define C5_SH_CAP_DEFAULT 256
#define C5_SH_WARP_BYTES(cap) ((size_t)(cap) * (sizeof(C5RecL) + 2 * 4))   // records + touched + J lists
#define C5_SH_BYTES(cap) ((C5_BT / 32) * (C5_SH_WARP_BYTES(cap) + C5_FB_WARP * 4))
#define C5_HBT 1024               // heavy-endpoint CTA
#define C5_MID_MAX 4096           // mid endpoint: R(l) <= this ...
#define C5_MID_WORK 65535         // ... and W(l) <= this (packed 16-bit record fields)
#define C5_MID_CAP (2 * C5_MID_MAX)  // hashed records in a per-CTA global region (load <= 0.5)
#define C5_MBT 128                // mid-endpoint CTA (several endpoints in flight per SM)
#define C5_BITS_SMEM_MAX (160 << 10)  // heavy CTAs: shared first-touch bitmaps up to this size
#define C5_HOT_MAX 16384              // heavy CTAs (u32 records): hot-vertex cache of up to this many top ranks
#define C5_SMEM_MAX (208 << 10)       // heavy CTAs: bitmaps + hot cache within this
#define C5_HOT_MIN_W (1ull << 22)     // hot cache only when the largest big endpoint's W(l) reaches this
#define C5_GIANT_W (1ull << 32)   // endpoints with W(l) >= this: whole-GPU kernels (k_c5_giant)
#define C5_FB_WARP 128            // i-key filter words per light warp (4096 bits)
#define C5_FB_CTA 256             // i-key filter words per mid CTA (8192 bits)

// dense records indexed by vertex id; touched list holds vertex ids
template <typename Rec>
struct C5Dense {
  typedef Rec RecT;
  Rec* R;
  int32_t* L;
  int* nL;
  // optional shared-memory bitmaps by vertex id (present, j-key): first-touch detection by a
  // shared atomic, so the record's flag update becomes a fire-and-forget global atomic and
  // no element waits for a global round trip to learn whether to append (nullptr: the
  // record's own atomicOr decides, for graphs whose bitmaps do not fit)
  u32* bP = nullptr;
  u32* bJ = nullptr;
  // old = the flags before; word = the whole wf word before (its Wn bits are unchanged by
  // the Or, so callers that need Wn take it from here instead of loading it again)
  __device__ __forceinline__ Rec* mark(int32_t x, u32 bits, u32& old, u32& word) {
    Rec* r = &R[x];
    word = atomicOr(&r->wf, (bits | C5_PRESENT) << 28);
    old = word >> 28;
    append_active(!(old & C5_PRESENT), x, L, nL);
    return r;
  }
  __device__ __forceinline__ Rec* mark(int32_t x, u32 bits, u32& old) {
    u32 word;
    return mark(x, bits, old, word);
  }
  // mark without needing the old flags
  __device__ __forceinline__ Rec* mark_nr(int32_t x, u32 bits) {
    if (!bP) {
      u32 old;
      return mark(x, bits, old);
    }
    Rec* r = &R[x];
    const u32 bit = 1u << (x & 31);
    const u32 ob = atomicOr(&bP[x >> 5], bit);
    append_active(!(ob & bit), x, L, nL);
    atomicOr(&r->wf, (bits | C5_PRESENT) << 28);  // result unused: a reduction
    return r;
  }
  // Hot-vertex cache (big endpoints of large graphs, u32 records): the step-3 path ends i
  // are out-neighbours of out-neighbours, which in the degeneracy order concentrate on the
  // highest ranks (the dense core).  For i >= hot0, Wn[i] is mirrored in shared memory by
  // step 1 and step 3 adds P[i] and A[i] with shared atomics, flushed into the records once
  // per endpoint (hot_flush) -- instead of an L2 load and one or two L2 atomics per path.
  u32* hWn = nullptr;
  u32* hP = nullptr;
  u32* hA = nullptr;
  int32_t hot0 = 0x7fffffff;
  int hotK = 0;
  // step-1 mark of a wedge end: Wn += 1 (its first mark makes it an i-key: Wn > 0)
  __device__ __forceinline__ Rec* mark_wedge(int32_t x) {
    Rec* r = mark_nr(x, C5_I);
    atomicAdd(&r->wf, 1u);
    if (x >= hot0) atomicAdd(&hWn[x - hot0], 1u);
    return r;
  }
  // step 3 for a hot path end i: true if i is hot (wn = Wn[i]; P, A added when wn > 0)
  __device__ __forceinline__ bool hot_pa(int32_t i, u64 q, bool adj, u64& wn) {
    if (i < hot0) return false;
    const int x = i - hot0;
    wn = hWn[x];
    if (wn) {
      atomicAdd(&hP[x], (u32)q);
      if (adj) atomicAdd(&hA[x], (u32)q);
    }
    return true;
  }
  // after step 3 (all threads, between barriers): P, A of the hot records; clear the cache
  template <typename Eng>
  __device__ __forceinline__ void hot_flush(const Eng& eng) {
    if constexpr (sizeof(Rec) == sizeof(C5RecT<u32>)) {
      for (int x = eng.tid(); x < hotK; x += eng.nthr()) {
        const u32 p = hP[x], a = hA[x];
        if (p | a) {
          Rec* r = &R[hot0 + x];
          r->P += p;  // this thread is the records' only writer now
          r->A += a;
          hP[x] = 0u;
          hA[x] = 0u;
        }
        hWn[x] = 0u;
      }
    }
  }
  // step-2 mark of a j-key with its Q, QT, QM updates
  __device__ __forceinline__ Rec* mark_j_q(int32_t x, u32 th, u32 tm, bool& newj) {
    Rec* r = mark_j(x, newj);
    rec_add_q(r, th, tm);
    return r;
  }
  // j-key mark: newj = first C5_J mark of x
  __device__ __forceinline__ Rec* mark_j(int32_t x, bool& newj) {
    if (!bP) {
      u32 old;
      Rec* r = mark(x, C5_J, old);
      newj = !(old & C5_J);
      return r;
    }
    const u32 bit = 1u << (x & 31);
    newj = !(atomicOr(&bJ[x >> 5], bit) & bit);
    return mark_nr(x, C5_J);
  }
  __device__ __forceinline__ void note_i(int32_t) const {}
  // record of x if Wn[x] > 0 (step 3; Wn is final since step 1), else nullptr
  __device__ __forceinline__ Rec* peek_i(int32_t x) const {
    Rec* r = &R[x];
    return (__ldcg(&r->wf) & C5_WN_MASK) ? r : nullptr;
  }
  __device__ __forceinline__ Rec* peek(int32_t x) const { return &R[x]; }
  __device__ __forceinline__ int32_t id_of(int32_t idx) const { return idx; }  // record index -> vertex
  __device__ __forceinline__ Rec* touched(int t, int32_t& x) const {
    x = L[t];
    return &R[x];
  }
  __device__ __forceinline__ void clear_bits(int32_t x) const {
    if (bP) { bP[x >> 5] = 0u; bJ[x >> 5] = 0u; }
  }
};

// open-addressing records (key = x + 1); touched list holds slots
template <typename Rec>
struct C5Hash {
  typedef Rec RecT;
  Rec* R;
  u32 mask;
  int32_t* L;
  int* nL;
  // Bit filter of the i-keys (vertices with Wn > 0), in shared memory: step 3 looks up every
  // path end i, most of which have no record (or Wn = 0), and a clear bit answers those
  // without a probe of the (L2-resident) region.  fb == nullptr: no filter.
  u32* fb = nullptr;
  int fshift = 0;  // 32 - log2(filter bits)
  __device__ __forceinline__ u32 hf(int32_t x) const { return ((u32)x * 0x85EBCA6Bu) >> fshift; }
  __device__ __forceinline__ void note_i(int32_t x) {
    if (fb) {
      const u32 b = hf(x);
      atomicOr(&fb[b >> 5], 1u << (b & 31));
    }
  }
  __device__ __forceinline__ u32 h0(int32_t x) const { return ((u32)x * 0x9E3779B1u) >> 7 & mask; }
  // find or claim the slot of x; the thread whose CAS claims it appends the slot to the
  // touched list (so no mark has to wait for the flags' old value to decide that)
  __device__ __forceinline__ Rec* probe(int32_t x) {
    u32 h = h0(x);
    bool claimed = false;
    for (;;) {
      const int32_t k = R[h].key;
      if (k == x + 1) break;
      if (k == 0) {
        const int32_t o = atomicCAS(&R[h].key, 0, x + 1);
        if (o == 0) { claimed = true; break; }
        if (o == x + 1) break;
      }
      h = (h + 1) & mask;
    }
    append_active(claimed, (int32_t)h, L, nL);
    return &R[h];
  }
  __device__ __forceinline__ Rec* mark_nr(int32_t x, u32 bits) {
    Rec* r = probe(x);
    atomicOr(&r->wf, (bits | C5_PRESENT) << 28);  // result unused: a reduction
    return r;
  }
  // step-1 mark of a wedge end: Wn += 1, one atomic (a claimed key is present, and Wn > 0 is
  // what makes it an i-key, so no flag update is needed)
  __device__ __forceinline__ Rec* mark_wedge(int32_t x) {
    Rec* r = probe(x);
    atomicAdd(&r->wf, 1u);
    return r;
  }
  // step-2 mark of a j-key: the Q increment's old value tells a new j-key (Q was 0), so no
  // flag update is needed either
  __device__ __forceinline__ Rec* mark_j_q(int32_t x, u32 th, u32 tm, bool& newj) {
    Rec* r = probe(x);
    newj = rec_add_q_first(r, th, tm);
    return r;
  }
  __device__ __forceinline__ void clear_bits(int32_t) const {}
  __device__ __forceinline__ Rec* peek(int32_t x) const {
    u32 h = h0(x);
    for (;;) {
      const int32_t k = R[h].key;
      if (k == x + 1) return &R[h];
      if (k == 0) return nullptr;
      h = (h + 1) & mask;
    }
  }
  __device__ __forceinline__ Rec* peek_i(int32_t x) const {
    if (fb) {
      const u32 b = hf(x);
      if (!(fb[b >> 5] & (1u << (b & 31)))) return nullptr;
    }
    Rec* r = peek(x);
    return (r && c5_wn(r)) ? r : nullptr;
  }
  __device__ __forceinline__ Rec* touched(int t, int32_t& x) const {
    Rec* r = &R[L[t]];
    x = r->key - 1;
    return r;
  }
  __device__ __forceinline__ bool hot_pa(int32_t, u64, bool, u64&) const { return false; }
  template <typename Eng>
  __device__ __forceinline__ void hot_flush(const Eng&) const {}
  __device__ __forceinline__ int32_t id_of(int32_t idx) const { return R[idx].key - 1; }  // slot -> vertex
};

// Engine adaptors: warp (light endpoints) and CTA (heavy endpoints)
struct WarpEng {
  static constexpr bool kCta = false;
  static constexpr bool kGrid = false;
  __device__ __forceinline__ void sync() const { __syncwarp(); }
  __device__ __forceinline__ int tid() const { return threadIdx.x & 31; }
  __device__ __forceinline__ int nthr() const { return 32; }
  template <typename I, typename E, typename F>
  __device__ __forceinline__ void lists(int n, I info, E elem, F flush) const { warp_lists(n, info, elem, flush); }
};
struct CtaEng {
  static constexpr bool kCta = true;
  static constexpr bool kGrid = false;
  ListEng* E;
  __device__ __forceinline__ void sync() const { __syncthreads(); }
  __device__ __forceinline__ int tid() const { return threadIdx.x; }
  __device__ __forceinline__ int nthr() const { return blockDim.x; }
  template <typename I, typename E2, typename F>
  __device__ __forceinline__ void lists(int n, I info, E2 elem, F flush) const { cta_lists(n, *E, info, elem, flush); }
};

// Whole-grid engine (giant endpoints): list items are dealt round robin to the CTAs, each
// walks its share with the CTA engine; flat loops run over every thread of the grid.  There
// is no grid barrier: the step groups are separate kernels.
struct GridEng {
  static constexpr bool kCta = true;
  static constexpr bool kGrid = true;
  ListEng* E;
  __device__ __forceinline__ void sync() const { __syncthreads(); }
  __device__ __forceinline__ int tid() const { return blockIdx.x * blockDim.x + threadIdx.x; }
  __device__ __forceinline__ int nthr() const { return gridDim.x * blockDim.x; }
  template <typename I, typename E2, typename F>
  __device__ __forceinline__ void lists(int n, I info, E2 elem, F flush) const {
    const int G = gridDim.x, b = blockIdx.x;
    const int cnt = n > b ? (n - b + G - 1) / G : 0;
    cta_lists(cnt, *E, [&](int i, int64_t& base, int& len) { info(i * G + b, base, len); },
              [&](int i, int64_t base, int k) -> u64 { return elem(i * G + b, base, k); },
              [&](int i, u64 v) { flush(i * G + b, v); });
  }
};

template <typename R>
__device__ __forceinline__ bool c5_adj(const R* r) { return r && (c5_flags(r) & C5_ADJ); }

// developer step timers (EVOKE_DEBUG): SM cycles of thread 0 per step, summed over the
// endpoints of the CTA engines ([0] heavy 1024-thread CTAs, [1] mid CTAs)
// developer step timers (EVOKE_DEBUG sets g_c5_prof): SM cycles per step summed over the
// endpoints, [0] heavy 1024-thread CTAs, [1] mid CTAs (thread 0), [2] light warps (lane 0)
__device__ unsigned long long g_c5_phase[3][8];
__device__ int g_c5_prof;
#define C5_PHASE(i)                                                                              \
  do {                                                                                           \
    if (g_c5_prof && !Eng::kGrid && (Eng::kCta ? threadIdx.x == 0 : (threadIdx.x & 31) == 0)) {  \
      const long long t_ = clock64();                                                            \
      atomicAdd(&g_c5_phase[!Eng::kCta ? 2 : blockDim.x == C5_HBT ? 0 : 1][i],                   \
                (unsigned long long)(t_ - t_prev));                                              \
      t_prev = t_;                                                                               \
    }                                                                                            \
  } while (0)

// One endpoint l, in three step groups separated by barriers (the giant endpoints run each
// group as a whole-GPU kernel, k_c5_giant_*).  J: list of j-keys (counter *nJ); tot: u64
// accumulator of the l credit (zeroed).  Step 3 is the only step whose work is split across
// shards for a giant endpoint: its outputs P, A, S enter every credit linearly, so shard si of
// ns takes the j-keys with j % ns == si, and the constant terms (those not multiplied by P, A
// or S) are added by shard 0 alone (consts).
struct C5Split {
  int ns = 1, si = 0;
  __device__ __forceinline__ bool mine(int32_t j) const { return ns == 1 || j % ns == si; }
  __device__ __forceinline__ bool consts() const { return si == 0; }
};

// wedge lists of steps 1/6: w = N(l)[t], i in N(w) (w < l) or N+(w) (w > l); from the slot's
// precomputed row (coalesced along N(l), no dependent load through w)
struct C5WInfo {
  const DGraph& g;
  int64_t r0;
  int32_t l;
  __device__ __forceinline__ void operator()(int t, int64_t& base, int& len) const {
    const int4 si = g.c5s[r0 + t];
    base = si.x;
    len = si.y;
  }
};
// out-out lists of steps 2/4: k = N-(l)[t], j in N+(k) (edge ids orow[k] + .)
struct C5KInfo {
  const DGraph& g;
  int64_t r0;
  __device__ __forceinline__ void operator()(int t, int64_t& base, int& len) const {
    const int4 si = g.c5s[r0 + t];
    base = si.z;
    len = si.w;
  }
};

// the slot rows of C5WInfo / C5KInfo, one warp per vertex l
__global__ void k_c5_slots(DGraph g, int4* __restrict__ c5s) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = gw; q < g.n; q += nw) {
    const int32_t l = (int32_t)q;
    for (int64_t s = g.rp[l] + lane; s < g.rp[l + 1]; s += 32) {
      const int32_t w = g.ci[s];
      const int64_t rw = g.rp[w];
      const int dw = g.deg[w], dmw = g.dm[w];
      int4 r;
      if (w < l) {
        const int64_t ow = g.orow[w];
        r = make_int4((int)rw, dw, (int)ow, dw - dmw);  // d+(w) = d(w) - d-(w)
      } else {
        r = make_int4((int)(rw + dmw), dw - dmw, 0, 0);
      }
      c5s[s] = r;
    }
  }
}

// steps 0-2: ADJ flags, Wn, Q/QT/QM and the j-key list
template <typename Eng, typename Loc>
__device__ __forceinline__ void c5_steps012(const DGraph& g, const u32* __restrict__ Tmid,
                                            const u32* __restrict__ Thigh, int32_t l, const Eng& eng, Loc& loc,
                                            int32_t* J, int* nJ, long long& t_prev) {
  const int64_t r0 = g.rp[l];
  const int dl = g.deg[l];
  const int dml = g.dm[l];
  // ---- step 0: neighbours of l
  for (int t = eng.tid(); t < dl; t += eng.nthr()) loc.mark_nr(g.ci[r0 + t], C5_ADJ);
  C5_PHASE(0);
  // ---- step 1: Wn over non-in-in wedges (i, w, l)
  eng.lists(dl, C5WInfo{g, r0, l},
      [&](int, int64_t base, int k) -> u64 {
        const int32_t i = g.ci[base + k];
        if (i == l) return 0;
        loc.mark_wedge(i);  // Wn += 1
        loc.note_i(i);
        return 0;
      },
      [&](int, u64) {});
  C5_PHASE(1);
  // ---- step 2: Q, QT, QM over out-out wedges j <- k -> l
  eng.lists(dml, C5KInfo{g, r0},
      [&](int, int64_t base, int k) -> u64 {
        const int64_t e = base + k;
        const int32_t j = g.ocol[e];
        if (j == l) return 0;
        bool newj;
        auto* r = loc.mark_j_q(j, Thigh[e], Tmid[e], newj);
        append_active(newj, (int32_t)(r - loc.R), J, nJ);  // J holds record indices (no lookups later)
        return 0;
      },
      [&](int, u64) {});
}

// step 3: paths through j: P, A (to i), S and the j credits
template <typename Eng, typename Loc>
__device__ __forceinline__ void c5_step3(const DGraph& g, int32_t l, const Eng& eng, Loc& loc, const int32_t* J,
                                         int nj, u64* __restrict__ C5, C5Split sp) {
  eng.lists(nj,
      [&](int t, int64_t& base, int& len) {
        // N+(j) from j's out8 row (one sector) when it is short; base < 0 encodes the row
        const int32_t j = loc.id_of(J[t]);
        if (g.out8) {  // (every out-list is short: max d+ <= OUT8)
          const int4* r = reinterpret_cast<const int4*>(g.out8 + (size_t)OUT8 * j);
          const int4 a = r[0];
          const int4 b = r[1];
          len = (a.x >= 0) + (a.y >= 0) + (a.z >= 0) + (a.w >= 0) + (b.x >= 0) + (b.y >= 0) + (b.z >= 0) + (b.w >= 0);
          base = ~((int64_t)OUT8 * j);
        } else {  // (a graph with longer out-lists: an extra load for every j was slower, config 3)
          base = g.orow[j];
          len = (int)(g.orow[j + 1] - base);
        }
        if (!sp.mine(j)) len = 0;
      },
      [&](int t, int64_t base, int k) -> u64 {
        // Only i with Wn[i] > 0 can close a 5-cycle: a path i <- j <- k -> l with Wn[i] = 0
        // has j !~ l and i !~ k (both would be wedges (i, w, l)), so its every term (P Wn,
        // A, the QM correction, its share of S[j]) is zero.  The lookup is read-only: no
        // record is created for such i (Wn is final after step 1).
        const int32_t i = base >= 0 ? g.ocol[base + k] : g.out8[~base + k];
        if (i == l) return 0;
        const auto* rj = &loc.R[J[t]];
        u64 wn;
        if (loc.hot_pa(i, rec_q(rj), c5_flags(rj) & C5_ADJ, wn)) return wn;
        auto* ri = loc.peek_i(i);
        if (!ri) return 0;
        rec_add_pa(ri, rec_q(rj), c5_flags(rj) & C5_ADJ);
        return c5_wn(ri);
      },
      [&](int t, u64 s) {
        auto* rj = &loc.R[J[t]];
        rec_add_s(rj, s);
        atomicAdd(&C5[loc.id_of(J[t])], rec_q(rj) * s);  // the j credit is linear in S
      });
  // constant part of the j credits
  if (sp.consts())
    for (int t = eng.tid(); t < nj; t += eng.nthr()) {
      const int32_t j = loc.id_of(J[t]);
      const auto* rj = &loc.R[J[t]];
      const u64 q = rec_q(rj);
      const bool adjj = c5_flags(rj) & C5_ADJ;
      const u64 lj = (l > j && adjj) ? 1ull : 0ull;
      u64 c = rec_qt(rj) - q * lj;
      if (adjj) c += q * ((u64)(g.orow[j + 1] - g.orow[j]) - lj);
      if (c) atomicAdd(&C5[j], (u64)0 - c);
    }
}

// steps 4-6: k, i (and l) and w credits; every record is final
template <typename Eng, typename Loc>
__device__ __forceinline__ void c5_steps456(const DGraph& g, const u32* __restrict__ Thigh, int32_t l,
                                            const Eng& eng, Loc& loc, u64* tot, u64* __restrict__ C5,
                                            C5Split sp, long long& t_prev) {
  const int64_t r0 = g.rp[l];
  const int dl = g.deg[l];
  const int dml = g.dm[l];
  const u64 cm = sp.consts() ? ~0ull : 0ull;  // constant terms: shard 0 only
  // ---- step 4: k credits
  eng.lists(dml, C5KInfo{g, r0},
      [&](int, int64_t base, int k) -> u64 {
        const int64_t e = base + k;
        const int32_t j = g.ocol[e];
        if (j == l) return 0;
        const auto* rj = loc.peek(j);
        const bool adjj = c5_flags(rj) & C5_ADJ;
        const u64 lj = (l > j && adjj) ? 1ull : 0ull;
        u64 c = (u64)Thigh[e] - lj;
        if (adjj) c += (u64)(g.orow[j + 1] - g.orow[j]) - lj;  // d+(j): read for neighbours of l only
        return rec_s(rj) - (c & cm);
      },
      [&](int t, u64 s) { atomicAdd(&C5[g.ci[r0 + t]], s); });
  C5_PHASE(4);
  // ---- step 5: i credits (and their sum for l)
  {
    const int nt = *loc.nL;
    u64 acc = 0;
    for (int t = eng.tid(); t < nt; t += eng.nthr()) {
      int32_t x;
      const auto* r = loc.touched(t, x);
      const u32 fl = c5_flags(r);
      if (!c5_wn(r)) continue;  // not an i-key
      const bool adji = fl & C5_ADJ;
      const u64 bi = (rec_qm(r) - rec_q(r) * ((x > l && adji) ? 1ull : 0ull)) & cm;
      const u64 ci = rec_p(r) * c5_wn(r) - rec_a(r) - bi;
      if (ci) atomicAdd(&C5[x], ci);
      acc += ci;
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(tot, acc);
  }
  C5_PHASE(5);
  // ---- step 6: wedge centres w
  eng.lists(dl, C5WInfo{g, r0, l},
      [&](int t, int64_t base, int k) -> u64 {
        const int64_t s = base + k;
        const int32_t i = g.ci[s];
        if (i == l) return 0;
        const int32_t w = g.ci[r0 + t];
        const auto* ri = loc.peek(i);
        u64 corr = 0;
        if (w < i) {  // (the typed triangle counts are read only where they enter)
          corr = (u64)g.tlows[r0 + t];
          if (w < l) corr += (u64)g.tmids[s] - ((l < i && c5_adj(ri)) ? 1ull : 0ull);
        }
        return rec_p(ri) - (corr & cm);
      },
      [&](int t, u64 s) { atomicAdd(&C5[g.ci[r0 + t]], s); });
}

template <typename Eng, typename Loc>
__device__ void c5_endpoint(const DGraph& g, const u32* __restrict__ Tlow, const u32* __restrict__ Tmid,
                            const u32* __restrict__ Thigh, int32_t l, const Eng& eng, Loc& loc, int32_t* J,
                            int* nJ, u64* tot, u64* __restrict__ C5) {
  long long t_prev = clock64();
  c5_steps012(g, Tmid, Thigh, l, eng, loc, J, nJ, t_prev);
  eng.sync();
  C5_PHASE(2);
  c5_step3(g, l, eng, loc, J, *nJ, C5, C5Split{});
  eng.sync();
  loc.hot_flush(eng);
  eng.sync();
  C5_PHASE(3);
  c5_steps456(g, Thigh, l, eng, loc, tot, C5, C5Split{}, t_prev);
  eng.sync();
  C5_PHASE(6);
}

// reset every touched record (and the counters) of one endpoint
template <typename Eng, typename Loc>
__device__ __forceinline__ void c5_reset(const Eng& eng, Loc& loc) {
  const int nt = *loc.nL;
  for (int t = eng.tid(); t < nt; t += eng.nthr()) {
    int32_t x;
    auto* r = loc.touched(t, x);
    loc.clear_bits(x);
    rec_zero(r);
  }
}

// ---- per-endpoint work, binning -----------------------------------------------------------
// Work of endpoint l (every element its steps visit):
//   W(l) = d(l) + sum_{w in N(l)} |Nsel(w)| + sum_{k in N-(l)} (d+(k) + s+(k)),
//   s+(k) = sum_{j in N+(k)} d+(j)     (step-3 path elements through k),
// and the bound on the records it creates (steps 0-2; step 3 creates none):
//   R(l) = d(l) + sum_{w in N(l)} |Nsel(w)| + sum_{k in N-(l)} d+(k).
// Every record field is at most W(l) (Wn <= d(l), Q <= d-(l), QT and QM <= sum d+(k),
// P and A <= #paths, S <= #wedges), which decides the record width.
__global__ void k_c5_splus(DGraph g, u32* __restrict__ splus) {
  for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < g.n; k += gridDim.x * blockDim.x) {
    u32 s = 0;  // <= kappa^2 < 2^31 (kappa <= sqrt(2m), m < 2^30)
    for (int64_t e = g.orow[k]; e < g.orow[k + 1]; e++) {
      const int32_t j = g.ocol[e];
      s += (u32)(g.orow[j + 1] - g.orow[j]);
    }
    splus[k] = s;
  }
}

// W(l) and R(l) of every vertex, one warp per vertex (hubs' lists split over the lanes)
__global__ void k_c5_work(DGraph g, const u32* __restrict__ splus, u64* __restrict__ W, u64* __restrict__ R) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = gw; q < g.n; q += nw) {
    const int32_t l = (int32_t)q;
    const int64_t r0 = g.rp[l], r1 = g.rp[l + 1], rm = r0 + g.dm[l];
    u64 w = 0, r = 0;
    for (int64_t s = r0 + lane; s < r1; s += 32) {
      const int4 si = g.c5s[s];  // the slot's |Nsel(x)| and, for x < l, d+(x)
      const u64 sel = (u64)si.y;
      w += sel;
      r += sel;
      if (s < rm) {
        const u64 dpx = (u64)si.w;
        w += dpx + (u64)splus[g.ci[s]];
        r += dpx;
      }
    }
    w = warp_sum(w);
    r = warp_sum(r);
    if (lane == 0) {
      const u64 d = (u64)(r1 - r0);
      W[l] = d > 0 ? w + d : 0;
      R[l] = d > 0 ? r + d : 0;
    }
  }
}

// Tiers of this shard's endpoints (mine == nullptr: every endpoint), and the giants (W >=
// giant_w, tier 3, list order = vertex order, on every shard):
//   light (one warp):    R <= rec_light and W <= work_light (packed records, per-warp hash;
//                        shared memory when 2R fits the warp's shared region, else global)
//   mid (128 threads):   R <= rec_mid   and W <= work_mid   (packed records, per-CTA hash in global memory)
//   big (1024 threads):  the rest (dense records by vertex id, sorted by W descending)
// Packed 16-bit record fields need W < 2^16 for the hashed tiers (work_mid < 2^16).  Measured
// on config 4: a warp per endpoint with its records in an L2 region beats a CTA per endpoint
// with the records in shared memory (78 vs 124 ms): the CTA engine's barriers and idle warps
// cost more than the region's L2 round trips, which many resident warps hide.
// Lists: tier t in lists[t * n ...], with R (t < 2) or W (big) beside it.
__global__ void k_c5_bin(DGraph g, const u64* __restrict__ W, const u64* __restrict__ R,
                         const uint8_t* __restrict__ mine, u64 rec_light, u64 work_light, u64 rec_mid,
                         u64 work_mid, u64 giant_w, int32_t* __restrict__ lists, u32* __restrict__ rbs,
                         u64* __restrict__ big_w, int* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll; base < g.n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int32_t l = (int32_t)min(base + lane, (int64_t)g.n - 1);
    const bool any = base + lane < g.n && W[l] > 0;
    const u64 w = any ? W[l] : 0, r = any ? R[l] : 0;
    // giants: every shard (their step 3 is split by j-key); the rest: this shard's own
    const int tier = !any ? -1
                   : w >= giant_w ? 3
                   : (mine && !mine[l]) ? -1
                   : (r <= rec_light && w <= work_light) ? 0
                   : (r <= rec_mid && w <= work_mid) ? 1 : 2;
    for (int t = 0; t < 4; t++) {
      const u32 bal = __ballot_sync(FULL_MASK, tier == t);
      if (!bal) continue;
      int b0 = 0;
      const int leader = __ffs(bal) - 1;
      if (lane == leader) b0 = atomicAdd(&counts[t], __popc(bal));
      b0 = __shfl_sync(FULL_MASK, b0, leader);
      if (tier != t) continue;
      const int q = b0 + __popc(bal & ((1u << lane) - 1u));
      lists[(size_t)t * g.n + q] = l;
      if (t < 2) rbs[(size_t)t * g.n + q] = (u32)r;
      else if (t == 2) big_w[q] = w;
    }
  }
}

// Heavy endpoints: one CTA each, dense records per CTA (persistent, W-sorted list).
template <typename V>
__global__ void __launch_bounds__(C5_HBT) k_c5_heavy(DGraph g, const u32* __restrict__ Tlow,
                                                    const u32* __restrict__ Tmid, const u32* __restrict__ Thigh,
                                                    const int32_t* __restrict__ heavy, int n_heavy,
                                                    int* __restrict__ counter, C5RecT<V>* __restrict__ dense,
                                                    int32_t* __restrict__ dlists, u64* __restrict__ C5,
                                                    int32_t* __restrict__ qmem, int use_bits, int hot_k) {
  __shared__ ListEng E;
  if (threadIdx.x == 0) {
    E.qcap = g.max_deg;
    E.qi = qmem + (size_t)blockIdx.x * (2 * (size_t)g.max_deg + 1);
    E.lc0 = E.qi + g.max_deg;
  }
  __shared__ int s_idx, s_nL, s_nJ;
  __shared__ u64 s_tot;
  extern __shared__ u32 c5_bits[];  // 2 x ceil(n/32) words when the launch provides them
  CtaEng eng{&E};
  C5Dense<C5RecT<V>> loc;
  if (use_bits) {
    const int nwd = (g.n + 31) >> 5;
    for (int i = threadIdx.x; i < 2 * nwd; i += blockDim.x) c5_bits[i] = 0u;
    loc.bP = c5_bits;
    loc.bJ = c5_bits + nwd;
    __syncthreads();
  }
  if (hot_k > 0) {  // (u32 records only; the host passes 0 otherwise)
    u32* hb = c5_bits + (use_bits ? 2 * ((g.n + 31) >> 5) : 0);
    for (int i = threadIdx.x; i < 3 * hot_k; i += blockDim.x) hb[i] = 0u;
    loc.hWn = hb;
    loc.hP = hb + hot_k;
    loc.hA = hb + 2 * hot_k;
    loc.hot0 = g.n - hot_k;
    loc.hotK = hot_k;
    __syncthreads();
  }
  loc.R = dense + (size_t)blockIdx.x * g.n;
  loc.L = dlists + (size_t)blockIdx.x * 2 * g.n;
  loc.nL = &s_nL;
  int32_t* J = loc.L + g.n;
  for (;;) {
    if (threadIdx.x == 0) { s_idx = atomicAdd(counter, 1); s_nL = 0; s_nJ = 0; s_tot = 0; }
    __syncthreads();
    const int idx = s_idx;
    if (idx >= n_heavy) break;
    const int32_t l = heavy[idx];
    const long long ut = unit_t0();
    c5_endpoint(g, Tlow, Tmid, Thigh, l, eng, loc, J, &s_nJ, &s_tot, C5);
    if (threadIdx.x == 0 && s_tot) atomicAdd(&C5[l], s_tot);
    c5_reset(eng, loc);
    __syncthreads();
    unit_t1(2, ut, idx);
  }
}

// Giant endpoints (W(l) past C5_GIANT_W, or any W(l) >= 2^32): one endpoint at a time on the
// whole GPU, one kernel per step group (part 0: steps 0-2, 1: step 3, 2: steps 4-6, 3: reset
// and the l credit), u64 records dense by vertex id.  Counters per giant: cnt[2 gi] = touched
// records, cnt[2 gi + 1] = j-keys; tot[gi] = the l credit (all zeroed before the first part).
// With shards, step 3's j-keys are split by j % ns (C5Split) and every shard runs the other
// parts, so one hub's endpoint is spread over every rank.
__global__ void __launch_bounds__(C5_HBT) k_c5_giant(int part, DGraph g, const u32* __restrict__ Tmid,
                                                    const u32* __restrict__ Thigh, const int32_t* __restrict__ giants,
                                                    int gi, C5Rec* __restrict__ dense, int32_t* __restrict__ dlist,
                                                    int* __restrict__ cnt, u64* __restrict__ tot,
                                                    u64* __restrict__ C5, int32_t* __restrict__ qmem, int ns, int si) {
  __shared__ ListEng E;
  if (threadIdx.x == 0) {
    E.qcap = g.max_deg;
    E.qi = qmem + (size_t)blockIdx.x * (2 * (size_t)g.max_deg + 1);
    E.lc0 = E.qi + g.max_deg;
  }
  __syncthreads();
  GridEng eng{&E};
  C5Dense<C5Rec> loc;
  loc.R = dense;
  loc.L = dlist;
  loc.nL = &cnt[2 * gi];
  int32_t* J = dlist + g.n;
  int* nJ = &cnt[2 * gi + 1];
  C5Split sp;
  sp.ns = ns;
  sp.si = si;
  const int32_t l = giants[gi];
  long long t_prev = 0;
  if (part == 0) {
    c5_steps012(g, Tmid, Thigh, l, eng, loc, J, nJ, t_prev);
  } else if (part == 1) {
    c5_step3(g, l, eng, loc, J, *nJ, C5, sp);
  } else if (part == 2) {
    c5_steps456(g, Thigh, l, eng, loc, &tot[gi], C5, sp, t_prev);
  } else {
    c5_reset(eng, loc);
    if (blockIdx.x == 0 && threadIdx.x == 0 && tot[gi]) atomicAdd(&C5[l], tot[gi]);
  }
}

// Light endpoints: one warp each, 16-byte records in a per-warp open-addressing region whose
// used part is sized per endpoint (2 x its record bound, so the records stay L2-resident).
#ifndef C5_LIGHT_MINB
#define C5_LIGHT_MINB 6  // resident CTAs per SM the register budget must allow (40 registers: config 4 light
                         // endpoints 48.8 ms vs 50.4 at 48 registers / 5 CTAs, 49.7 at 32 registers / 8 CTAs)
#endif
__global__ void __launch_bounds__(C5_BT, C5_LIGHT_MINB) k_c5_light(DGraph g, const u32* __restrict__ Tlow,
                                                    const u32* __restrict__ Tmid, const u32* __restrict__ Thigh,
                                                    const int32_t* __restrict__ light, const u32* __restrict__ lw,
                                                    int n_light, int* __restrict__ counter,
                                                    C5RecL* __restrict__ wregions, int32_t* __restrict__ wlists,
                                                    u64* __restrict__ C5, int sh_cap) {
  // endpoints whose region needs at most sh_cap (<= C5_SH_CAP) slots keep records and lists in shared
  // memory (per warp); larger ones use the warp's global region
  extern __shared__ unsigned char c5_sh[];
  __shared__ int w_nL[C5_BT / 32], w_nJ[C5_BT / 32];
  __shared__ u64 w_tot[C5_BT / 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const size_t gw = (size_t)blockIdx.x * (C5_BT / 32) + wib;
  WarpEng eng;
  C5RecL* shR = reinterpret_cast<C5RecL*>(c5_sh + (size_t)wib * C5_SH_WARP_BYTES(sh_cap));
  int32_t* shL = reinterpret_cast<int32_t*>(shR + sh_cap);
  u32* fb = reinterpret_cast<u32*>(c5_sh + (size_t)(C5_BT / 32) * C5_SH_WARP_BYTES(sh_cap)) + wib * C5_FB_WARP;
  {
    uint4* z = reinterpret_cast<uint4*>(shR);
    for (int i = lane; i < (int)(sh_cap * sizeof(C5RecL) / 16); i += 32) z[i] = make_uint4(0, 0, 0, 0);
    for (int i = lane; i < C5_FB_WARP; i += 32) fb[i] = 0u;
  }
  __syncwarp();
  C5Hash<C5RecL> loc;
  loc.nL = &w_nL[wib];
  loc.fb = fb;
  loc.fshift = 32 - 12;  // 4096 bits
  for (;;) {
    int idx = 0;
    if (lane == 0) idx = atomicAdd(counter, 1);
    idx = __shfl_sync(FULL_MASK, idx, 0);
    if (idx >= n_light) break;
    const int32_t l = light[idx];
    // region of at least 1.25 R(l) + 1 slots: R(l) bounds the records (typically a quarter of
    // it are distinct), so the load stays <= 0.8 and the probes terminate; a smaller region
    // keeps more of the warps' records in L2 (config 4: 23 % of 2R slots were used)
    const u32 cap = pow2_at_least(lw[idx] + lw[idx] / 4 + 1, 64u);  // <= C5_WARP_CAP
    int32_t* J;
    if (cap <= (u32)sh_cap) {
      loc.R = shR;
      loc.L = shL;
      J = shL + sh_cap;
    } else {
      loc.R = wregions + gw * C5_WARP_CAP;
      loc.L = wlists + gw * 2 * C5_WARP_CAP;
      J = loc.L + C5_WARP_CAP;
    }
    loc.mask = cap - 1;
    if (lane == 0) { w_nL[wib] = 0; w_nJ[wib] = 0; w_tot[wib] = 0; }
    __syncwarp();
    c5_endpoint(g, Tlow, Tmid, Thigh, l, eng, loc, J, &w_nJ[wib], &w_tot[wib], C5);
    if (lane == 0 && w_tot[wib]) atomicAdd(&C5[l], w_tot[wib]);
    if (g_c5_prof && lane == 0) {  // developer: records used vs region slots
      atomicAdd(&g_c5_phase[2][7], (unsigned long long)w_nL[wib]);
      atomicAdd(&g_c5_phase[1][7], (unsigned long long)cap);
    }
    c5_reset(eng, loc);
    for (int i = lane; i < C5_FB_WARP; i += 32) fb[i] = 0u;
    __syncwarp();
  }
}

// Mid endpoints: one C5_MBT-thread CTA each, records in a per-CTA open-addressing region of
// 2 x R(l) slots in global memory (the region is reused endpoint after endpoint, so it stays
// in L2).  A 1024-thread CTA per such endpoint would spend its time in barriers and dependent
// round trips with most warps idle.
#ifndef C5_MID_MINB
#define C5_MID_MINB 16  // resident mid-endpoint CTAs per SM the register budget must allow (32 registers:
                        // config 4 5-cycle pass 47.9 -> 46.2 ms against 40 registers / 12 CTAs)
#endif
__global__ void __launch_bounds__(C5_MBT, C5_MID_MINB) k_c5_mid(DGraph g, const u32* __restrict__ Tlow,
                                                   const u32* __restrict__ Tmid, const u32* __restrict__ Thigh,
                                                   const int32_t* __restrict__ list, const u32* __restrict__ rb,
                                                   int n_mid, int* __restrict__ counter, C5RecP* __restrict__ regions,
                                                   int32_t* __restrict__ rlists, u64* __restrict__ C5,
                                                   int32_t* __restrict__ qmem) {
  __shared__ ListEng E;
  if (threadIdx.x == 0) {
    E.qcap = g.max_deg;
    E.qi = qmem + (size_t)blockIdx.x * (2 * (size_t)g.max_deg + 1);
    E.lc0 = E.qi + g.max_deg;
  }
  __shared__ int s_idx, s_nL, s_nJ;
  __shared__ u64 s_tot;
  CtaEng eng{&E};
  C5Hash<C5RecP> loc;
  loc.R = regions + (size_t)blockIdx.x * C5_MID_CAP;
  loc.L = rlists + (size_t)blockIdx.x * 2 * C5_MID_CAP;
  int32_t* J = loc.L + C5_MID_CAP;
  loc.nL = &s_nL;
  __shared__ u32 s_fb[C5_FB_CTA];
  for (int i = threadIdx.x; i < C5_FB_CTA; i += blockDim.x) s_fb[i] = 0u;
  loc.fb = s_fb;
  loc.fshift = 32 - 13;  // 8192 bits
  for (;;) {
    if (threadIdx.x == 0) { s_idx = atomicAdd(counter, 1); s_nL = 0; s_nJ = 0; s_tot = 0; }
    __syncthreads();
    const int idx = s_idx;
    if (idx >= n_mid) break;
    const int32_t l = list[idx];
    loc.mask = pow2_at_least(rb[idx] + rb[idx] / 4 + 1, 64u) - 1;  // rb[idx] = R(l) <= C5_MID_MAX (load <= 0.8)
    c5_endpoint(g, Tlow, Tmid, Thigh, l, eng, loc, J, &s_nJ, &s_tot, C5);
    if (threadIdx.x == 0 && s_tot) atomicAdd(&C5[l], s_tot);
    c5_reset(eng, loc);
    for (int i = threadIdx.x; i < C5_FB_CTA; i += blockDim.x) s_fb[i] = 0u;
    __syncthreads();
  }
}
