// evoke.cu -- host orchestration and the C ABI (include/evoke.h) of the B200-native
// EVOKE vertex-orbit counter.  One translation unit: the kernels live in the .cuh
// files included below; this file sequences them on one stream (SURVEY 8(a) rows
// a1..a12).
#include <cub/cub.cuh>

#include <chrono>
#include <cstdlib>
#include <algorithm>
#include <functional>
#include <mutex>
#include <utility>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/evoke.h"
#include "common.cuh"
#include "graph_build.cuh"
#include "triangles.cuh"
#include "cliques.cuh"
#include "pairs.cuh"
#include "hublocal.cuh"
#include "cycles5.cuh"
#include "gather.cuh"
#include "transform.cuh"
#include "workmodel.cuh"
#include "ccd.cuh"

#define EVOKE_VERSION "0.1.0-sm100a"
#define EVOKE_SORT_FULL_MIN (3ll << 20)  // full triangle lists sorted when 3 #T >= this

namespace {

thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

struct EvokeError {
  int code;
};

// EVOKE_HOSTPROF=1: report every CUDA API call that blocks the host for more than 2 ms
inline bool hostprof() {
  static const bool on = std::getenv("EVOKE_HOSTPROF") != nullptr;
  return on;
}
struct HostTimer {
  const char* what; int line; std::chrono::steady_clock::time_point t0;
  HostTimer(const char* w, int l) : what(w), line(l) { if (hostprof()) t0 = std::chrono::steady_clock::now(); }
  ~HostTimer() {
    if (!hostprof()) return;
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (ms > 2.0) fprintf(stderr, "[evoke hostprof] %.2f ms line %d: %.80s\n", ms, line, what);
  }
};

#define CK(call)                                                                        \
  do {                                                                                  \
    HostTimer _ht(#call, __LINE__);                                                     \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess) {                                                            \
      set_error("%s failed: %s (%s:%d)", #call, cudaGetErrorString(_e), __FILE__, __LINE__); \
      throw EvokeError{_e == cudaErrorMemoryAllocation ? EVOKE_ENOMEM : EVOKE_ECUDA};   \
    }                                                                                   \
  } while (0)

static const char* kPassNames[] = {
    "h2d",        "canonicalise", "kcore_order", "csr_build",  "triangles",  "tri_lists",
    "cliques_k4k5", "nbr_gather1", "pair_pass",  "hub_local",  "cycles5",    "cliques_66_70",
    "nbr_gather2", "tri_gather",  "combine",    "d2h"};
enum { P_H2D = 0, P_CANON, P_KCORE, P_CSR, P_TRI, P_TRILIST, P_CLIQ, P_NBR1, P_PAIR, P_HUB, P_C5,
       P_CLIQ2, P_NBR2, P_TRIG, P_COMB, P_D2H, P_COUNT };

// ---- the library's own stream-ordered memory pool (one per device) -------------------
// Scratch comes from a private pool whose release threshold keeps freed memory mapped
// between calls (the default threshold of 0 would unmap and remap gigabytes of tables on
// every call).  Private, so the process-wide default pool that other libraries use keeps
// its own settings; evoke_release_scratch trims it back to nothing.
std::mutex g_pool_mu;
cudaMemPool_t g_pools[256] = {};
cudaMemPool_t evoke_pool(int dev) {
  cudaMemPool_t* pools = g_pools;
  if (dev < 0 || dev >= 256) { set_error("device ordinal out of range"); throw EvokeError{EVOKE_EINTERNAL}; }
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!pools[dev]) {
    cudaMemPoolProps props;
    std::memset(&props, 0, sizeof(props));
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    CK(cudaMemPoolCreate(&pools[dev], &props));
    uint64_t thr = ~0ull;
    CK(cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr));
  }
  return pools[dev];
}
cudaMemPool_t evoke_pool_if_any(int dev) {  // the pool if one was created (never creates)
  if (dev < 0 || dev >= 256) return nullptr;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  return g_pools[dev];
}

// ---- zero-invariant scratch, kept between calls --------------------------------------
// The per-CTA tables of the pair, hub-local and 5-cycle passes start zeroed and every kernel
// that uses them resets what it touched before it finishes (touched lists / sweeps), so at
// the end of a successful call they are all zero again.  One buffer per device keeps them
// between calls: a call leases it (exclusively; a concurrent call on the same device falls
// back to fresh zeroed allocations), carves its tables out of it, and the next call skips
// the memsets (≈ 0.9 GB at config 2).  A call that fails leaves the buffer marked dirty and
// the next lease zeroes it again; a call that needed more than the buffer holds got fresh
// allocations for the rest, and the next lease grows the buffer to that size.
// The kept buffer is worth its memory where the memsets it saves are a visible part of the
// call (0.9 GB of a 9 ms call at config 2, ~25 GB of a 109 ms call at config 4); at config 5 a
// call's tables pass 100 GB, zeroing them is 0.05 % of the call, and a kept buffer of that size
// starved the next call's budgets (avail_bytes counts it as used) and had to be re-carved out
// of a fragmented pool: the test suite's second config-5 call ran its heavy pair tier on a
// handful of CTAs, 760 s instead of 28 s.  So the buffer never grows past a quarter of the
// device; tables that do not fit get fresh zeroed allocations, as without a lease.
size_t zero_pool_cap(int dev) {
  static std::mutex mu;
  static size_t cap[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 0 || dev >= 64) return 0;
  if (!cap[dev]) {
    int cur = 0;
    size_t freeb = 0, totalb = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && cudaSetDevice(dev) == cudaSuccess &&
        cudaMemGetInfo(&freeb, &totalb) == cudaSuccess)
      cap[dev] = totalb / 4;
    else
      cap[dev] = (size_t)16 << 30;
    (void)cudaGetLastError();
    (void)cudaSetDevice(cur);
  }
  return cap[dev];
}
struct ZeroPool {
  std::mutex mu;
  char* p = nullptr;
  size_t bytes = 0;
  size_t target = 0;
  bool dirty = false;
};
ZeroPool& zero_pool(int dev) {
  static ZeroPool pools[64];
  if (dev < 0 || dev >= 64) { set_error("device ordinal out of range"); throw EvokeError{EVOKE_EINTERNAL}; }
  return pools[dev];
}
struct ZeroLease {
  ZeroPool* zp = nullptr;
  size_t used = 0, need = 0, cap = 0;
  bool ok = false;  // set when the call completed (the tables are zero again)
  void acquire(int dev, cudaStream_t st) {
    ZeroPool& z = zero_pool(dev);
    if (std::getenv("EVOKE_NO_ZERO_POOL") || !z.mu.try_lock()) return;
    zp = &z;
    cap = zero_pool_cap(dev);
    if (z.target > z.bytes) {
      if (z.p) CK(cudaFreeAsync(z.p, st));
      z.p = nullptr;
      z.bytes = 0;
      void* q = nullptr;
      if (cudaMallocFromPoolAsync(&q, z.target, evoke_pool(dev), st) != cudaSuccess) {
        (void)cudaGetLastError();
        z.target = 0;
        return;
      }
      z.p = (char*)q;
      z.bytes = z.target;
      z.dirty = true;
    }
    if (z.dirty && z.p) {
      CK(cudaMemsetAsync(z.p, 0, z.bytes, st));
      z.dirty = false;
    }
  }
  // what is left of the leased buffer: the pool counts the whole buffer as used, but this
  // much of it is still there for the call's tables (added to avail_bytes by the budgets)
  size_t room() const { return (zp && zp->p && zp->bytes > used) ? zp->bytes - used : 0; }
  // zeroed region of `bytes` from the lease, or nullptr (the caller allocates)
  void* take(size_t bytes) {
    bytes = (bytes + 255) & ~(size_t)255;
    need += bytes;
    if (!zp || !zp->p || used + bytes > zp->bytes) return nullptr;
    void* q = zp->p + used;
    used += bytes;
    return q;
  }
  ~ZeroLease() {
    if (!zp) return;
    if (!ok) {
      // a failed call may leave kernels writing into the buffer on any of its streams
      (void)cudaDeviceSynchronize();
      (void)cudaGetLastError();
      zp->dirty = true;
    }
    if (std::min(need, cap) > zp->target) zp->target = std::min(need, cap);
    zp->mu.unlock();
  }
};

// Device allocations of one call; everything is freed (stream-ordered) at the end.
struct Arena {
  cudaStream_t st;
  cudaMemPool_t pool;
  std::vector<void*> ptrs;
  Arena(cudaStream_t s, int dev) : st(s), pool(evoke_pool(dev)) {}
  template <typename T>
  T* alloc(size_t count, bool zero = false) {
    T* p = try_alloc<T>(count, zero);
    if (!p) throw EvokeError{EVOKE_ENOMEM};
    return p;
  }
  // nullptr (and the error recorded) when the pool cannot grow by `count` elements
  template <typename T>
  T* try_alloc(size_t count, bool zero = false) {
    void* p = nullptr;
    size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, pool, st);
    if (e == cudaErrorMemoryAllocation) {
      // the pool keeps every block this process ever freed (release threshold = never): hand
      // the unused ones back to the device so that the request can be met with fresh memory
      // whatever the cached blocks' sizes, and try once more
      (void)cudaGetLastError();
      if (cudaStreamSynchronize(st) == cudaSuccess && cudaMemPoolTrimTo(pool, 0) == cudaSuccess)
        e = cudaMallocFromPoolAsync(&p, bytes, pool, st);
    }
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      set_error("cudaMallocFromPoolAsync(%zu bytes): %s", bytes, cudaGetErrorString(e));
      return nullptr;
    }
    ptrs.push_back(p);
    if (zero) CK(cudaMemsetAsync(p, 0, bytes, st));
    return (T*)p;
  }
  ZeroLease* lease = nullptr;
  // zero-invariant table (see ZeroPool): from the lease when it has room, else a fresh
  // zeroed allocation
  template <typename T>
  T* zalloc(size_t count) {
    T* p = try_zalloc<T>(count);
    if (!p) throw EvokeError{EVOKE_ENOMEM};
    return p;
  }
  template <typename T>
  T* try_zalloc(size_t count) {
    const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    if (lease) {
      if (void* q = lease->take(bytes)) return (T*)q;
    }
    return try_alloc<T>(count, true);
  }
  void release(void* p) {
    for (auto& q : ptrs)
      if (q == p) { cudaFreeAsync(q, st); q = nullptr; }
  }
  ~Arena() {
    for (void* p : ptrs)
      if (p) cudaFreeAsync(p, st);
  }
};

struct Ctx {
  cudaStream_t st;
  int dev, num_sms;
  double sm_mhz = 1965.0;  // (developer timers only)
  int launches = 0;
  int lib_launches = 0;
  cudaEvent_t ev[P_COUNT + 1];
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_pre = nullptr, ev_side = nullptr;  // side stream of a5/a9 + gather 1
  cudaEvent_t sev[3] = {};                          // side timing: start, after cliques, end
  bool side_used = false;
  cudaEvent_t gev[3] = {};  // early tail gathers: start, after gathers 2/3, after the triangle gather
  bool gathers_early = false;
  bool serial_run = false;  // the concurrent passes ran one after the other on the main stream
  cudaStream_t side_st = nullptr;
  static const int MAXJOBS = 16;
  cudaStream_t jst[MAXJOBS] = {};
  cudaEvent_t pev[MAXJOBS][2] = {};
  int njobs = 0;
  int job_pass[MAXJOBS] = {};
  int job_rank[MAXJOBS] = {};
  bool timing;
  // stream for job i with the priority of its rank (rank 0 = the device's greatest priority).
  // Streams are created once per (device, rank) and kept for the process lifetime: creating
  // and destroying them on every call costs more than the calls' shorter passes.
  cudaStream_t stream(size_t i, int rank) {
    if (i >= (size_t)MAXJOBS) { set_error("too many concurrent jobs"); throw EvokeError{EVOKE_EINTERNAL}; }
    static std::mutex mu;
    static cudaStream_t pool[64][MAXJOBS] = {};
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 0 || dev >= 64) { set_error("device ordinal out of range"); throw EvokeError{EVOKE_EINTERNAL}; }
    if (!pool[dev][i]) {
      int lo = 0, hi = 0;  // lo = least priority (numerically greatest), hi = greatest
      CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      const int prio = std::min(lo, hi + rank);
      CK(cudaStreamCreateWithPriority(&pool[dev][i], cudaStreamNonBlocking, prio));
    }
    return pool[dev][i];
  }
  cudaStream_t side() {
    if (!side_st) CK(cudaStreamCreateWithFlags(&side_st, cudaStreamNonBlocking));
    return side_st;
  }
  std::chrono::steady_clock::time_point hts[P_COUNT + 1];
  bool hset[P_COUNT + 1] = {};
  // developer timeline (EVOKE_TICKS=1): named events on the main stream, printed at the end
  std::vector<std::pair<const char*, cudaEvent_t>> ticks;
  void tick(const char* what) {
    static const bool on = std::getenv("EVOKE_TICKS") != nullptr;
    if (!on) return;
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    CK(cudaEventRecord(e, st));
    ticks.emplace_back(what, e);
  }
  void print_ticks() {
    if (ticks.empty()) return;
    std::string line;
    for (size_t i = 1; i < ticks.size(); i++) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, ticks[i - 1].second, ticks[i].second));
      char b[96];
      snprintf(b, sizeof(b), " %s %.3f", ticks[i].first, ms);
      line += b;
    }
    for (auto& t : ticks) cudaEventDestroy(t.second);
    ticks.clear();
    fprintf(stderr, "[evoke ticks]%s\n", line.c_str());
  }
  void mark(int pass) {
    if (timing) CK(cudaEventRecord(ev[pass], st));
    if (hostprof()) { hts[pass] = std::chrono::steady_clock::now(); hset[pass] = true; }
  }
  void host_report() {
    if (!hostprof() || !hset[0]) return;
    std::string line;
    int prev = 0;
    for (int p = 1; p <= P_COUNT; p++) {
      if (!hset[p]) continue;
      const double ms = std::chrono::duration<double, std::milli>(hts[p] - hts[prev]).count();
      char b[64];
      snprintf(b, sizeof(b), " %s=%.1f", kPassNames[prev], ms);
      line += b;
      prev = p;
    }
    fprintf(stderr, "[evoke hostprof] host segments:%s\n", line.c_str());
  }
};

inline int grid_for(int64_t work, int block, int num_sms) {
  int64_t g = (work + block - 1) / block;
  int64_t cap = (int64_t)num_sms * 32;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// Device memory this call may still take.  cudaMemGetInfo can block the host for tens of
// milliseconds while stream-ordered frees are in flight, so it is read once per device;
// afterwards the estimate is that first reading minus what the stream-ordered pool (which
// keeps its memory between calls, see run()) currently has in use:
// avail = free0 + reserved0 - used_now.
size_t avail_bytes(int dev) {
  static std::mutex mu;
  static size_t base[256] = {};
  static bool have[256] = {};
  cudaMemPool_t pool = evoke_pool(dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 0 || dev >= 256) { set_error("device ordinal out of range"); throw EvokeError{EVOKE_EINTERNAL}; }
    if (!have[dev]) {
      size_t freeb = 0, totalb = 0;
      uint64_t reserved = 0;
      CK(cudaMemGetInfo(&freeb, &totalb));
      CK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
      base[dev] = freeb + (size_t)reserved;
      have[dev] = true;
    }
  }
  uint64_t used = 0;
  CK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
  return base[dev] > used ? base[dev] - (size_t)used : 0;
}

template <typename T>
T d2h_scalar(const T* dptr, cudaStream_t st) {
  T v;
  CK(cudaMemcpyAsync(&v, dptr, sizeof(T), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return v;
}

// ---- CUB wrappers (stream-ordered temp storage)
void sort_keys_u64(Arena& A, Ctx& C, const u64* in, u64* out, int64_t N, int end_bit) {
  size_t tb = 0;
  CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, in, out, (int64_t)N, 0, end_bit, C.st));
  void* t = A.alloc<char>(tb);
  CK(cub::DeviceRadixSort::SortKeys(t, tb, in, out, (int64_t)N, 0, end_bit, C.st));
  A.release(t);
  C.lib_launches += 4;
}

template <typename Tin, typename Tout>
void inclusive_sum(Arena& A, Ctx& C, const Tin* in, Tout* out, int64_t N) {
  size_t tb = 0;
  CK(cub::DeviceScan::InclusiveSum(nullptr, tb, in, out, N, C.st));
  void* t = A.alloc<char>(tb);
  CK(cub::DeviceScan::InclusiveSum(t, tb, in, out, N, C.st));
  A.release(t);
  C.lib_launches += 2;
}

// Work-balanced shard membership (north star: units "partitioned by balanced work
// estimate"; the paper's parallel orbit groups): the N items sorted by estimate,
// descending (CUB's radix sort is stable, so ties keep index order and every rank computes
// the same list), and position p belongs to shard p mod ns.  Returns nullptr (every item is
// this shard's) when ns == 1; sums[0..1] (device) receive this shard's and all estimates.
__global__ void k_iota_i32(int32_t* __restrict__ a, int64_t n);
__global__ void k_shard_mask(const u64* __restrict__ skeys, const int32_t* __restrict__ sidx, int64_t n, int si,
                             int ns, uint8_t* __restrict__ mine, u64* __restrict__ sums);
uint8_t* shard_mask(Arena& A, Ctx& C, const u64* est, int64_t N, int si, int ns, u64* sums);

int bits_for(int64_t x) {
  int b = 1;
  while ((1ll << b) <= x) b++;
  return b;
}

// Test / developer override of a tier limit: the compiled default, or a LOWER value from the
// environment (a lower limit only moves work items onto a heavier tier's code path, whose
// tables are sized for anything; a higher one could overflow a lighter tier's tables).
u64 env_cap(const char* name, u64 dflt) {
  const char* e = getenv(name);
  if (!e || !*e) return dflt;
  const long long v = atoll(e);
  return v < 0 ? 0 : std::min<u64>((u64)v, dflt);
}

__global__ void k_iota_i32(int32_t* __restrict__ a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (int32_t)i;
}
// position p of the estimate-sorted (descending) item list belongs to shard p mod ns;
// sums[0] += the estimates of this shard's items, sums[1] += all estimates
__global__ void k_shard_mask(const u64* __restrict__ skeys, const int32_t* __restrict__ sidx, int64_t n, int si,
                             int ns, uint8_t* __restrict__ mine, u64* __restrict__ sums) {
  u64 own = 0, all = 0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const bool m = (p % ns) == si;
    mine[sidx[p]] = m ? 1 : 0;
    all += skeys[p];
    if (m) own += skeys[p];
  }
  own = warp_sum(own);
  all = warp_sum(all);
  if ((threadIdx.x & 31) == 0) {
    if (own) atomicAdd(&sums[0], own);
    if (all) atomicAdd(&sums[1], all);
  }
}
// the pair pass's own sorted list (keys = ~est, u32): this shard's and all estimates
__global__ void k_shard_sum_u32(const u32* __restrict__ skeys, int64_t n, int si, int ns, u64* __restrict__ sums) {
  u64 own = 0, all = 0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const u64 e = (u64)(u32)~skeys[p];
    all += e;
    if ((p % ns) == si) own += e;
  }
  own = warp_sum(own);
  all = warp_sum(all);
  if ((threadIdx.x & 31) == 0) {
    if (own) atomicAdd(&sums[0], own);
    if (all) atomicAdd(&sums[1], all);
  }
}
// the 5-cycle endpoints' work for the position split: giants (every shard takes 1/ns of their
// step 3) are left out of it and counted here, W / ns for this shard
__global__ void k_c5_giant_mask(const u64* __restrict__ W, int32_t n, u64 giant_w, int ns, u64* __restrict__ Wm,
                                u64* __restrict__ sums) {
  u64 own = 0, all = 0;
  for (int32_t l = blockIdx.x * blockDim.x + threadIdx.x; l < n; l += gridDim.x * blockDim.x) {
    const u64 w = W[l];
    const bool giant = w >= giant_w;
    Wm[l] = giant ? 0 : w;
    if (giant) { own += w / (u64)ns; all += w; }
  }
  own = warp_sum(own);
  all = warp_sum(all);
  if ((threadIdx.x & 31) == 0) {
    if (own) atomicAdd(&sums[0], own);
    if (all) atomicAdd(&sums[1], all);
  }
}
// (k = d+(u))^3: the 4/5-clique unit's work estimate
__global__ void k_clique_est(const int64_t* __restrict__ orow, int32_t n, u64* __restrict__ est) {
  for (int32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
    const u64 k = (u64)(orow[u + 1] - orow[u]);
    est[u] = k >= 3 ? k * k * k : 0;
  }
}

__global__ void k_gather_u64(const u64* __restrict__ src, const int32_t* __restrict__ idx, int64_t n,
                             u64* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = src[idx[i]];
}
__global__ void k_permute_c5(const int32_t* __restrict__ perm, int64_t n, const int32_t* __restrict__ l,
                             const u32* __restrict__ r, int32_t* __restrict__ lo, u32* __restrict__ ro) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    lo[i] = l[perm[i]];
    ro[i] = r[perm[i]];
  }
}
__global__ void k_u32_to_i64(const u32* __restrict__ a, int64_t n, int64_t* __restrict__ b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}
__global__ void k_i32_to_i64(const int32_t* __restrict__ a, int64_t n, int64_t* __restrict__ b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}
__global__ void k_set_i64(int64_t* p, int64_t v) { *p = v; }
__global__ void k_max_i32(const int32_t* __restrict__ a, int64_t n, int* out) {
  int m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, a[i]);
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(FULL_MASK, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}
__global__ void k_max_diff_i64(const int64_t* __restrict__ a, int64_t n, int* out) {
  int m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, (int)(a[i + 1] - a[i]));
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(FULL_MASK, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}
// EVOKE_CHECK_ZERO: flag any nonzero 16-byte word of a zero-invariant region
__global__ void k_check_zero(const uint4* __restrict__ p, size_t n16, int* flag) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 q = p[i];
    if (q.x | q.y | q.z | q.w) { *flag = 1; return; }
  }
}
// per-slot copies of the per-edge triangle counts (DGraph::tes, tlows, tmids)
__global__ void k_slot_counts(const int32_t* __restrict__ eid, int64_t m2, const u32* __restrict__ Te,
                              const u32* __restrict__ Tlow, const u32* __restrict__ Tmid, u32* __restrict__ tes,
                              u32* __restrict__ tlows, u32* __restrict__ tmids) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m2; s += (int64_t)gridDim.x * blockDim.x) {
    const int32_t e = eid[s];
    tes[s] = Te[e];
    tlows[s] = Tlow[e];
    tmids[s] = Tmid[e];
  }
}
// wedge total W(G) = sum C(d,2)
__global__ void k_wedges(const int64_t* __restrict__ rp, int32_t n, u64* out) {
  u64 s = 0;
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    s += binom2((u64)(rp[v + 1] - rp[v]));
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

// clique bins by k = d+(u): bin 0: 3..32, 1: 33..128, 2: 129..512, 3: 513..1024, 4: >1024
__global__ void k_clique_bins(const int64_t* __restrict__ orow, int32_t n, int32_t* __restrict__ lists,
                              int* __restrict__ counts) {
  // warp-aggregated appends (one atomic per warp and bin, not per vertex: 2M vertices
  // appending to one counter serialise on it)
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll; base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = (int32_t)(base + (threadIdx.x & 31));
    int b = -1;
    if (u < n) {
      const int64_t k = orow[u + 1] - orow[u];
      if (k >= 3) b = k <= 32 ? 0 : k <= 128 ? 1 : k <= 512 ? 2 : k <= 1024 ? 3 : 4;
    }
    for (int t = 0; t < 5; t++) warp_append(b == t, u, lists + (int64_t)t * n, counts + t);
  }
}

uint8_t* shard_mask(Arena& A, Ctx& C, const u64* est, int64_t N, int si, int ns, u64* sums) {
  if (ns <= 1 || N <= 0) return nullptr;
  const int B = 256;
  int32_t* idx = A.alloc<int32_t>(N);
  int32_t* sidx = A.alloc<int32_t>(N);
  u64* skeys = A.alloc<u64>(N);
  uint8_t* mine = A.alloc<uint8_t>(N);
  k_iota_i32<<<grid_for(N, B, C.num_sms), B, 0, C.st>>>(idx, N);
  size_t tb = 0;
  CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, est, skeys, idx, sidx, N, 0, 64, C.st));
  void* t = A.alloc<char>(tb);
  CK(cub::DeviceRadixSort::SortPairsDescending(t, tb, est, skeys, idx, sidx, N, 0, 64, C.st));
  k_shard_mask<<<grid_for(N, B, C.num_sms), B, 0, C.st>>>(skeys, sidx, N, si, ns, mine, sums);
  C.launches += 2;
  C.lib_launches += 4;
  A.release(idx); A.release(sidx); A.release(skeys); A.release(t);
  return mine;
}

struct Input {
  int kind;  // 0 edges, 1 csr
  int64_t n, m;
  const int32_t* edges;
  const int64_t* rowptr;
  const int32_t* col;
};

void run(const Input& in, uint64_t* out, const evoke_options& o) {
  int dev = o.device;
  if (dev < 0) CK(cudaGetDevice(&dev));
  CK(cudaSetDevice(dev));
  Ctx C;
  C.dev = dev;
  CK(cudaDeviceGetAttribute(&C.num_sms, cudaDevAttrMultiProcessorCount, dev));
  if (getenv("EVOKE_DEBUG")) {
    int khz = 0;
    if (cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev) == cudaSuccess && khz > 0) C.sm_mhz = khz / 1e3;
  }
  if (o.stream) {
    C.st = (cudaStream_t)o.stream;
  } else {
    // no caller stream (torch's default stream also arrives as NULL): the device's kept
    // non-blocking stream, ordered after all work already queued on the legacy default
    // stream (device-pointer inputs may still be in production there, and the caching
    // allocator may have handed `out` over from work still queued on it)
    C.st = C.stream(Ctx::MAXJOBS - 3, 0);
    cudaEvent_t e0;
    CK(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
    CK(cudaEventRecord(e0, cudaStreamLegacy));
    CK(cudaStreamWaitEvent(C.st, e0, 0));
    CK(cudaEventDestroy(e0));
  }
  C.timing = true;
  for (int i = 0; i <= P_COUNT; i++) CK(cudaEventCreate(&C.ev[i]));
  CK(cudaEventCreateWithFlags(&C.ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&C.ev_pre, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&C.ev_side, cudaEventDisableTiming));
  for (int i = 0; i < 3; i++) CK(cudaEventCreate(&C.sev[i]));
  for (int i = 0; i < 3; i++) CK(cudaEventCreate(&C.gev[i]));
  CK(cudaEventCreateWithFlags(&C.ev_join, cudaEventDisableTiming));
  for (int i = 0; i < Ctx::MAXJOBS; i++)
    for (int j = 0; j < 2; j++) CK(cudaEventCreate(&C.pev[i][j]));
  struct Cleanup {
    Ctx& C;
    ~Cleanup() {
      for (int i = 0; i <= P_COUNT; i++) cudaEventDestroy(C.ev[i]);
      cudaEventDestroy(C.ev_fork);
      cudaEventDestroy(C.ev_pre);
      cudaEventDestroy(C.ev_side);
      for (int i = 0; i < 3; i++) cudaEventDestroy(C.sev[i]);
      for (int i = 0; i < 3; i++) cudaEventDestroy(C.gev[i]);
      cudaEventDestroy(C.ev_join);
      for (int i = 0; i < Ctx::MAXJOBS; i++)
        for (int j = 0; j < 2; j++) cudaEventDestroy(C.pev[i][j]);
      if (C.side_st) { cudaStreamSynchronize(C.side_st); cudaStreamDestroy(C.side_st); }
    }
  } cleanup{C};

  const auto& TF = evoke_host::transform();
  {
    int rp[74];
    uint8_t col[AINV_MAX_NNZ];
    long long val[AINV_MAX_NNZ];
    if ((int)TF.col.size() > AINV_MAX_NNZ) { set_error("A^-1 too dense"); throw EvokeError{EVOKE_EINTERNAL}; }
    for (int i = 0; i < 74; i++) rp[i] = TF.rp[i];
    for (size_t i = 0; i < TF.col.size(); i++) { col[i] = (uint8_t)TF.col[i]; val[i] = TF.val[i]; }
    CK(cudaMemcpyToSymbolAsync(c_ainv_rp, rp, sizeof(rp), 0, cudaMemcpyHostToDevice, C.st));
    CK(cudaMemcpyToSymbolAsync(c_ainv_col, col, TF.col.size(), 0, cudaMemcpyHostToDevice, C.st));
    CK(cudaMemcpyToSymbolAsync(c_ainv_val, val, TF.col.size() * sizeof(long long), 0,
                               cudaMemcpyHostToDevice, C.st));
  }

  {
    const int prof = getenv("EVOKE_DEBUG") ? 1 : 0;  // developer step / phase timers
    CK(cudaMemcpyToSymbolAsync(g_c5_prof, &prof, sizeof(int), 0, cudaMemcpyHostToDevice, C.st));
    CK(cudaMemcpyToSymbolAsync(g_pair_prof, &prof, sizeof(int), 0, cudaMemcpyHostToDevice, C.st));
    CK(cudaMemcpyToSymbolAsync(g_unit_prof, &prof, sizeof(int), 0, cudaMemcpyHostToDevice, C.st));
  }
  Arena A(C.st, dev);
  ZeroLease lease;  // destroyed before A (its buffer is not A's)
  lease.acquire(dev, C.st);
  A.lease = &lease;
  const int32_t n = (int32_t)in.n;
  const int B = 256;
  const int SM = C.num_sms;
  C.mark(0);
  // ------------------------------------------------------------------ a1: input
  int* d_bad = A.alloc<int>(1, true);
  int64_t mraw = 0;
  u64* keys = nullptr;
  if (in.kind == 0) {
    mraw = in.m;
    const int32_t* d_edges = in.edges;
    if (!o.device_pointers && mraw > 0) {
      int32_t* t = A.alloc<int32_t>(2 * mraw);
      CK(cudaMemcpyAsync(t, in.edges, sizeof(int32_t) * 2 * mraw, cudaMemcpyHostToDevice, C.st));
      d_edges = t;
    }
    C.mark(P_CANON);
    keys = A.alloc<u64>(mraw + 1);
    if (mraw > 0) {
      k_make_keys<<<grid_for(mraw, B, SM), B, 0, C.st>>>(d_edges, mraw, n, keys, d_bad);
      C.launches++;
    }
  } else {
    const int64_t* d_rp = in.rowptr;
    const int32_t* d_col = in.col;
    if (!o.device_pointers) {
      mraw = in.rowptr[n];
      int64_t* t1 = A.alloc<int64_t>(n + 1);
      CK(cudaMemcpyAsync(t1, in.rowptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, C.st));
      int32_t* t2 = A.alloc<int32_t>(mraw + 1);
      if (mraw) CK(cudaMemcpyAsync(t2, in.col, sizeof(int32_t) * mraw, cudaMemcpyHostToDevice, C.st));
      d_rp = t1; d_col = t2;
    } else {
      mraw = d2h_scalar<int64_t>(in.rowptr + n, C.st);
    }
    C.mark(P_CANON);
    k_check_rowptr<<<grid_for(n, B, SM), B, 0, C.st>>>(d_rp, n, d_bad);
    if (d2h_scalar<int>(d_bad, C.st)) { set_error("malformed CSR rowptr"); throw EvokeError{EVOKE_EINVAL}; }
    keys = A.alloc<u64>(mraw + 1);
    if (mraw > 0) k_make_keys_csr<<<grid_for(n, B, SM), B, 0, C.st>>>(d_rp, d_col, n, keys, d_bad);
    C.launches += 2;
  }
  if (d2h_scalar<int>(d_bad, C.st)) { set_error("vertex id outside [0, n)"); throw EvokeError{EVOKE_EINVAL}; }
  int64_t m = 0;
  u64* ukeys = A.alloc<u64>(mraw + 1);
  if (mraw > 0) {
    u64* sk = A.alloc<u64>(mraw);
    // keys (min << 32) | max < 2^(32 + bits(n)); the self-loop sentinel ~0 is still above every
    // key in those bits, so it sorts last
    sort_keys_u64(A, C, keys, sk, mraw, std::min(64, 32 + bits_for(n)));
    int64_t* d_nsel = A.alloc<int64_t>(1);
    size_t tb = 0;
    CK(cub::DeviceSelect::Unique(nullptr, tb, sk, ukeys, d_nsel, mraw, C.st));
    void* t = A.alloc<char>(tb);
    CK(cub::DeviceSelect::Unique(t, tb, sk, ukeys, d_nsel, mraw, C.st));
    C.launches += 2;
    int64_t nsel = d2h_scalar<int64_t>(d_nsel, C.st);
    // drop the self-loop sentinel (sorted last)
    u64 last = 0;
    if (nsel > 0) last = d2h_scalar<u64>(ukeys + nsel - 1, C.st);
    m = (nsel > 0 && last == ~0ull) ? nsel - 1 : nsel;
    A.release(sk); A.release(t); A.release(keys);
  }
  if (m >= (1ll << 30)) { set_error("graph too large: m = %lld (limit 2^30: slot ids are int32)", (long long)m); throw EvokeError{EVOKE_EINVAL}; }
  const int64_t m2 = 2 * m;

  // ------------------------------------------------------------------ a2: k-core order
  C.mark(P_KCORE);
  int32_t* deg0 = A.alloc<int32_t>(n, true);
  int64_t* rp0 = A.alloc<int64_t>(n + 1);
  int32_t* adj0 = A.alloc<int32_t>(m2 + 1);
  int32_t* perm = A.alloc<int32_t>(n);
  int32_t* inv = A.alloc<int32_t>(n);
  int peel_rounds = 0, degeneracy_level = 0;
  if (n > 0) {
    if (m > 0) { k_degrees<<<grid_for(m, B, SM), B, 0, C.st>>>(ukeys, m, deg0); C.launches++; }
    int64_t* deg64 = A.alloc<int64_t>(n);
    k_i32_to_i64<<<grid_for(n, B, SM), B, 0, C.st>>>(deg0, n, deg64);
    k_set_i64<<<1, 1, 0, C.st>>>(rp0, 0);
    inclusive_sum(A, C, deg64, rp0 + 1, n);
    C.launches += 2;
    int64_t* cursor = A.alloc<int64_t>(n);
    CK(cudaMemcpyAsync(cursor, rp0, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, C.st));
    if (m > 0) { k_fill_adj0<<<grid_for(m, B, SM), B, 0, C.st>>>(ukeys, m, cursor, adj0); C.launches++; }
    int32_t* rnd = A.alloc<int32_t>(n);
    int32_t* l0 = A.alloc<int32_t>(n);
    int32_t* l1 = A.alloc<int32_t>(n);
    PeelCtl* ctl = A.alloc<PeelCtl>(1, true);
    const char* psw_env = getenv("EVOKE_PEEL_SWITCH");  // developer knob (<= PEEL_SWITCH)
    int peel_switch = (int)std::min<int64_t>(n, psw_env ? std::max(64, std::min(PEEL_SWITCH, atoi(psw_env))) : PEEL_SWITCH);
    int32_t* lidmap = A.alloc<int32_t>(n);
    int32_t* loc = A.alloc<int32_t>(peel_switch + 1);
    int32_t* lcnt = A.alloc<int32_t>(peel_switch + 1);
    uint16_t* ladj = A.alloc<uint16_t>(2 * m + 1);
    const size_t peel_smem = (size_t)peel_switch * PEEL_LOCAL_BYTES;
    CK(cudaFuncSetAttribute(k_peel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)peel_smem));
    CK(cudaFuncSetAttribute(k_peel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)peel_smem));
    void* args[] = {(void*)&n, (void*)&rp0, (void*)&adj0, (void*)&deg0, (void*)&rnd, (void*)&l0,
                    (void*)&l1, (void*)&lidmap, (void*)&loc, (void*)&lcnt, (void*)&ladj, (void*)&ctl,
                    (void*)&peel_switch};
    // graphs up to PEEL_CLUSTER_MAXN vertices: one 16-CTA cluster with hardware cluster
    // barriers between rounds; larger: a cooperative grid (one CTA per SM)
    bool launched = false;
    if (n <= PEEL_CLUSTER_MAXN && n > peel_switch) {
      if (cudaFuncSetAttribute(k_peel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(PEEL_CLUSTER, 1, 1);
        cfg.blockDim = dim3(PEEL_BT, 1, 1);
        cfg.dynamicSmemBytes = peel_smem;
        cfg.stream = C.st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = PEEL_CLUSTER;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        launched = cudaLaunchKernelExC(&cfg, (const void*)k_peel<true>, args) == cudaSuccess;
      }
      if (!launched) (void)cudaGetLastError();  // fall back to the cooperative grid
    }
    if (!launched) {
      int bps = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_peel<false>, PEEL_BT, peel_smem));
      const char* pg_env = getenv("EVOKE_PEEL_GRID");  // developer knob: CTAs of the grid-wide phase
      // (every SM: config 4's first rounds are large -- 3.53 ms at 64 CTAs, 3.17 ms at 148; the
      // grid barrier of the small rounds costs no more at 148: config 3 6.26 vs 6.25 ms)
      const int pg_want = pg_env ? std::max(1, atoi(pg_env)) : SM;
      const int pgrid = n <= peel_switch ? 1 : std::max(1, std::min(std::max(bps, 1) * SM, pg_want));
      CK(cudaLaunchCooperativeKernel((void*)k_peel<false>, pgrid, PEEL_BT, args, peel_smem, C.st));
    }
    C.launches++;
    PeelCtl hc = d2h_scalar<PeelCtl>(ctl, C.st);
    peel_rounds = hc.rounds;
    if (getenv("EVOKE_DEBUG"))
      fprintf(stderr, "[evoke] peel: %d rounds (%d grid-wide, %.3f ms; %d in one CTA, %.3f ms), level %d\n",
              hc.rounds, hc.rounds1, (hc.t1 - hc.t0) * 1e-6, hc.rounds - hc.rounds1, (hc.t2 - hc.t1) * 1e-6,
              hc.level);
    degeneracy_level = hc.level;
    u64* okeys = A.alloc<u64>(n);
    u64* osorted = A.alloc<u64>(n);
    k_order_keys<<<grid_for(n, B, SM), B, 0, C.st>>>(rnd, n, okeys);
    C.launches++;
    sort_keys_u64(A, C, okeys, osorted, n, 32 + bits_for(std::max(peel_rounds, 1)));
    k_perm<<<grid_for(n, B, SM), B, 0, C.st>>>(osorted, n, perm, inv);
    C.launches++;
    A.release(okeys); A.release(osorted); A.release(rnd); A.release(l0); A.release(l1); A.release(lidmap);
    A.release(loc); A.release(lcnt); A.release(ladj);
    A.release(cursor); A.release(deg64);
  }
  A.release(adj0); A.release(rp0); A.release(deg0);
  (void)degeneracy_level;

  // ------------------------------------------------------------------ a3: CSR + edges
  C.mark(P_CSR);
  int64_t* rp = A.alloc<int64_t>(n + 1);
  int32_t* ci = A.alloc<int32_t>(m2 + 1);
  int32_t* dmv = A.alloc<int32_t>(n + 1);
  int32_t* degv = A.alloc<int32_t>(n + 1);
  int64_t* orow = A.alloc<int64_t>(n + 1);
  int32_t* eid = A.alloc<int32_t>(m2 + 1);
  int32_t* ocol = A.alloc<int32_t>(m + 1);
  int32_t* esrc = A.alloc<int32_t>(m + 1);
  int32_t* edst = A.alloc<int32_t>(m + 1);
  int64_t* eslot_hi = A.alloc<int64_t>(m + 1);
  int32_t* twin = A.alloc<int32_t>(m2 + 1);
  int max_deg = 0, max_out = 0;
  const int kb = bits_for(std::max(n, 1));  // bits of a vertex id in the directed CSR keys
  if (n > 0) {
    int32_t* degc = A.alloc<int32_t>(n, true);
    int64_t* tmp64 = A.alloc<int64_t>(n);
    u64* dk = A.alloc<u64>(m2 + 1);
    u64* dks = A.alloc<u64>(m2 + 1);
    if (m > 0) {
      k_relabel_keys<<<grid_for(m, B, SM), B, 0, C.st>>>(ukeys, m, inv, dk, kb);
      C.launches++;
      sort_keys_u64(A, C, dk, dks, m2, 2 * kb);
      k_split_keys<<<grid_for(m2, B, SM), B, 0, C.st>>>(dks, m2, ci, degc, kb);
      C.launches++;
    }
    k_i32_to_i64<<<grid_for(n, B, SM), B, 0, C.st>>>(degc, n, tmp64);
    k_set_i64<<<1, 1, 0, C.st>>>(rp, 0);
    inclusive_sum(A, C, tmp64, rp + 1, n);
    k_split_counts<<<grid_for(n, B, SM), B, 0, C.st>>>(n, rp, ci, dmv, tmp64, degv);
    k_set_i64<<<1, 1, 0, C.st>>>(orow, 0);
    inclusive_sum(A, C, tmp64, orow + 1, n);
    C.launches += 4;
    if (m > 0) {
      k_edge_arrays<<<grid_for(m2, B, SM), B, 0, C.st>>>(dks, m2, rp, ci, dmv, orow, eid, ocol, esrc, edst,
                                                         eslot_hi, twin, kb);
      k_twin_hi<<<grid_for(m2, B, SM), B, 0, C.st>>>(n, rp, dmv, orow, eslot_hi, eid, m2, dks, twin, kb);
      C.launches += 2;
    }
    int* d_mx = A.alloc<int>(2, true);
    k_max_diff_i64<<<grid_for(n, B, SM), B, 0, C.st>>>(rp, n, d_mx);
    k_max_diff_i64<<<grid_for(n, B, SM), B, 0, C.st>>>(orow, n, d_mx + 1);
    C.launches += 2;
    int hm[2];
    CK(cudaMemcpyAsync(hm, d_mx, sizeof(hm), cudaMemcpyDeviceToHost, C.st));
    CK(cudaStreamSynchronize(C.st));
    max_deg = hm[0]; max_out = hm[1];
    if (max_deg >= (1 << 28)) {  // 5-cycle records pack Wn (<= d(l)) in 28 bits
      set_error("maximum degree %d >= 2^28 is not supported", max_deg);
      throw EvokeError{EVOKE_EINVAL};
    }
    A.release(dk); A.release(dks); A.release(degc); A.release(tmp64);
  }
  A.release(ukeys);

  DGraph g;
  std::memset(&g, 0, sizeof(g));
  g.n = n; g.m = m; g.max_deg = std::max(max_deg, 1); g.max_out = max_out;
  g.rp = rp; g.ci = ci; g.dm = dmv; g.deg = degv; g.eid = eid; g.orow = orow; g.ocol = ocol; g.esrc = esrc;
  g.edst = edst; g.eslot_hi = eslot_hi; g.twin = twin;
  if (n > 0 && max_out <= OUT8) {  // out8 rows only when every out-list fits one (no fallback loads)
    int32_t* out8 = A.alloc<int32_t>((size_t)OUT8 * n);
    k_out8<<<grid_for(n, B, SM), B, 0, C.st>>>(n, orow, ocol, reinterpret_cast<int4*>(out8));
    C.launches++;
    g.out8 = out8;
  }

  // per-vertex fields and per-edge arrays
  u64* F = A.alloc<u64>((size_t)F_COUNT * std::max(n, 1), true);
  u32* Te = A.alloc<u32>(m + 1, true);
  u32* Tlow = A.alloc<u32>(m + 1, true);
  u32* Tmid = A.alloc<u32>(m + 1, true);
  u32* Thigh = A.alloc<u32>(m + 1, true);
  u64* E7 = A.alloc<u64>(m + 1, true);
  u64* E9f = A.alloc<u64>(m + 1, true);
  u64* E9b = A.alloc<u64>(m + 1, true);
  u64* K4e = A.alloc<u64>(m + 1, true);
  u64* C4e = A.alloc<u64>(m + 1, true);
  auto Fp = [&](int f) { return F + (size_t)f * (size_t)n; };

  // ------------------------------------------------------------------ a4: triangles
  C.mark(P_TRI);
  int64_t* toff = A.alloc<int64_t>(m + 1);
  int64_t ntri = 0;
  const int tri_smem_per_warp = std::min(std::max(max_out, 1), 2048);
  const int tri_block = 256;
  const size_t tri_smem = (size_t)(tri_block / 32) * tri_smem_per_warp * sizeof(int32_t);
  if (tri_smem > 48 * 1024)
    CK(cudaFuncSetAttribute(k_triangles<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tri_smem));
  if (tri_smem > 48 * 1024)
    CK(cudaFuncSetAttribute(k_triangles<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tri_smem));
  const int tri_grid = grid_for((int64_t)n * 32, tri_block, SM);
  int32_t *tc = nullptr, *tab = nullptr, *tac = nullptr, *tbc = nullptr;
  if (m > 0) {
    // out-lists of at most 32: the (b, c) pairs of a vertex flattened over the lanes
    const bool tri_flat = max_out <= 32 && !getenv("EVOKE_TRI_NO_FLAT");  // (env: tests / A/B)
    if (tri_flat)
      k_triangles_flat<0><<<tri_grid, tri_block, 0, C.st>>>(g, Thigh, Tmid, Tlow, Te, Fp(F_T), E7, nullptr, nullptr,
                                                            nullptr, nullptr);
    else
      k_triangles<0><<<tri_grid, tri_block, tri_smem, C.st>>>(g, tri_smem_per_warp, Thigh, Tmid, Tlow, Te,
                                                             Fp(F_T), E7, nullptr, nullptr, nullptr, nullptr);
    int64_t* th64 = A.alloc<int64_t>(m);
    k_u32_to_i64<<<grid_for(m, B, SM), B, 0, C.st>>>(Thigh, m, th64);
    k_set_i64<<<1, 1, 0, C.st>>>(toff, 0);
    inclusive_sum(A, C, th64, toff + 1, m);
    C.launches += 3;
    A.release(th64);
    ntri = d2h_scalar<int64_t>(toff + m, C.st);
    tc = A.alloc<int32_t>(ntri + 1);
    tab = A.alloc<int32_t>(ntri + 1);
    tac = A.alloc<int32_t>(ntri + 1);
    tbc = A.alloc<int32_t>(ntri + 1);
    g.toff = toff; g.ntri = ntri; g.tc = tc; g.tab = tab; g.tac = tac; g.tbc = tbc;
    if (tri_flat)
      k_triangles_flat<1><<<tri_grid, tri_block, 0, C.st>>>(g, Thigh, Tmid, Tlow, Te, Fp(F_T), E7, tc, tab, tac, tbc);
    else
      k_triangles<1><<<tri_grid, tri_block, tri_smem, C.st>>>(g, tri_smem_per_warp, Thigh, Tmid, Tlow, Te,
                                                             Fp(F_T), E7, tc, tab, tac, tbc);
    C.launches++;
  } else {
    CK(cudaMemsetAsync(toff, 0, sizeof(int64_t) * (m + 1), C.st));
    g.toff = toff;
  }

  // ------------------------------------------------------------------ a6: tri lists, E9, DM12
  C.mark(P_TRILIST);
  int64_t* foff = A.alloc<int64_t>(m + 1);
  int32_t *fx = nullptr, *fe1 = nullptr, *fe2 = nullptr;
  u32* K4t = A.alloc<u32>(ntri + 1, true);
  if (ntri > 0) {
    int64_t* te64 = A.alloc<int64_t>(m);
    k_u32_to_i64<<<grid_for(m, B, SM), B, 0, C.st>>>(Te, m, te64);
    k_set_i64<<<1, 1, 0, C.st>>>(foff, 0);
    inclusive_sum(A, C, te64, foff + 1, m);
    A.release(te64);
    int64_t* fcur = A.alloc<int64_t>(m + 1);
    k_fcur_init<<<grid_for(m, B, SM), B, 0, C.st>>>(m, foff, Thigh, fcur);
    fx = A.alloc<int32_t>(3 * ntri);
    fe1 = A.alloc<int32_t>(3 * ntri);
    fe2 = A.alloc<int32_t>(3 * ntri);
    g.foff = foff; g.fx = fx; g.fe1 = fe1; g.fe2 = fe2;
    k_tri_sweep1<<<grid_for(ntri, B, SM), B, 0, C.st>>>(g, Te, E9f, E9b, Fp(F_DM12), fcur, fx, fe1, fe2);
    C.launches += 3;
    A.release(fcur);
    // triangle-heavy graphs: sort every full list by third vertex, so the passes that need
    // only x < a (hub-local) or x > u (pair pass 2) read a prefix / suffix instead of filtering
    const int64_t N3 = 3 * ntri;
    const size_t freeb = avail_bytes(C.dev) + lease.room();
    const char* sort_env = getenv("EVOKE_SORT_FULL_MIN");  // test hook: force / disable the sort
    const int64_t sort_min = sort_env ? atoll(sort_env) : EVOKE_SORT_FULL_MIN;
    // (and only when the lists are long on average: 3 #T >= 8 m; config 4's 1.4 entries per
    // list gained nothing from the 1.6 ms sort)
    if (N3 >= sort_min && (sort_env || N3 >= 8 * m) && (size_t)N3 * 40 < freeb / 2) {
      u64* k0 = A.alloc<u64>(N3);
      u64* k1 = A.alloc<u64>(N3);
      int32_t* i0 = A.alloc<int32_t>(N3);
      int32_t* i1 = A.alloc<int32_t>(N3);
      k_full_keys<<<grid_for(m, B, SM), B, 0, C.st>>>(g, k0, i0);
      size_t tb = 0;
      CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, i0, i1, N3, 0, 32 + bits_for(m), C.st));
      void* t = A.alloc<char>(tb);
      CK(cub::DeviceRadixSort::SortPairs(t, tb, k0, k1, i0, i1, N3, 0, 32 + bits_for(m), C.st));
      int32_t* ofe1 = A.alloc<int32_t>(N3);
      int32_t* ofe2 = A.alloc<int32_t>(N3);
      CK(cudaMemcpyAsync(ofe1, fe1, sizeof(int32_t) * N3, cudaMemcpyDeviceToDevice, C.st));
      CK(cudaMemcpyAsync(ofe2, fe2, sizeof(int32_t) * N3, cudaMemcpyDeviceToDevice, C.st));
      k_full_apply<<<grid_for(N3, B, SM), B, 0, C.st>>>(N3, k1, i1, ofe1, ofe2, fx, fe1, fe2);
      C.launches += 2;
      C.lib_launches += 4;
      A.release(k0); A.release(k1); A.release(i0); A.release(i1); A.release(t); A.release(ofe1); A.release(ofe2);
      g.full_sorted = 1;
    }
  } else {
    CK(cudaMemsetAsync(foff, 0, sizeof(int64_t) * (m + 1), C.st));
    g.foff = foff;
  }

  {
    u32* tes = A.alloc<u32>(m2 + 1);
    u32* tlows = A.alloc<u32>(m2 + 1);
    u32* tmids = A.alloc<u32>(m2 + 1);
    if (m2 > 0) {
      k_slot_counts<<<grid_for(m2, B, SM), B, 0, C.st>>>(g.eid, m2, Te, Tlow, Tmid, tes, tlows, tmids);
      C.launches++;
    }
    g.tes = tes; g.tlows = tlows; g.tmids = tmids;
  }
  const int si = o.shard_index, ns = o.num_shards;
  // Concurrent passes pay off while the passes are short (their tails and the host-visible
  // preparations overlap); on large graphs every pass fills the GPU by itself and running
  // them side by side only splits L2 between their tables (config 4: 190 ms serial, 209 ms
  // concurrent), so from EVOKE_CONCURRENT_MAX_M edges on they run one after the other, and
  // each takes every SM at the occupancy that hides most latency (config 4, 5-cycles: 78 ms
  // at the concurrent-mode grids, 63 ms at full occupancy).
  const char* cmax_env = getenv("EVOKE_CONCURRENT_MAX_M");
  const int64_t concurrent_max_m = cmax_env ? atoll(cmax_env) : (4ll << 20);
  const bool whole_gpu_passes = m > concurrent_max_m;
  // per sharded pass (pair, hub-local, 5-cycle, cliques): this shard's and all work estimates
  u64* d_work = A.alloc<u64>(8, true);
  // rows of the late gathers (k_pack_rows, k_trigather): allocated here, before the passes
  // run (a pool allocation while the random-access passes run slowed them: TLB updates)
  u64* V2rows = n > 0 ? A.alloc<u64>((size_t)n * V2_W) : nullptr;
  u64* EVrows = n > 0 ? A.alloc<u64>((size_t)std::max<int64_t>(m, 1) * EV_W) : nullptr;
  u64* TGrows = (ntri > 0 && !(o.flags & EVOKE_FLAG_FOUR) && 3 * ntri <= TG_ROWS_MAX_TPV * (int64_t)n)
                    ? A.alloc<u64>((size_t)n * TG_W) : nullptr;
  // ------------------------------------------------------------------ a5/a9: cliques
  C.mark(P_CLIQ);
  const uint8_t* cmine = nullptr;
  if (ns > 1 && n > 0) {
    u64* cest = A.alloc<u64>(n);
    k_clique_est<<<grid_for(n, B, SM), B, 0, C.st>>>(orow, n, cest);
    C.launches++;
    cmine = shard_mask(A, C, cest, n, si, ns, d_work + 6);
  }
  int32_t* cbins = A.alloc<int32_t>((size_t)5 * std::max(n, 1));
  int* ccounts = A.alloc<int>(5, true);
  int hcounts[5] = {0, 0, 0, 0, 0};
  const int bin_k[5] = {32, 128, 512, 1024, 0};
  u32* cscratch = nullptr;
  int64_t cscratch_words = 0;
  int cscratch_grid = 0;
  if (n > 0) {
    k_clique_bins<<<grid_for(n, B, SM), B, 0, C.st>>>(orow, n, cbins, ccounts);
    C.launches++;
    CK(cudaMemcpyAsync(hcounts, ccounts, sizeof(hcounts), cudaMemcpyDeviceToHost, C.st));
    CK(cudaStreamSynchronize(C.st));
    if (hcounts[4] > 0) {
      const int64_t kk = max_out, W = (kk + 31) / 32;
      cscratch_words = kk * W;
      cscratch_grid = std::min(hcounts[4], 2 * SM);
      cscratch = A.alloc<u32>((size_t)cscratch_words * cscratch_grid);
    }
  }
  auto launch_cliques = [&](int mode, cudaStream_t lst) {
    for (int b = 0; b < 5; b++) {
      if (hcounts[b] == 0) continue;
      const int kmax = b < 4 ? bin_k[b] : 0;
      const int W = (kmax + 31) / 32;
      const int words = kmax * W;
      const size_t smem = (size_t)words * sizeof(u32);
      const int block = b == 0 ? 64 : (b == 1 ? 128 : 256);
      int grid = b < 4 ? std::min(hcounts[b], SM * 16) : cscratch_grid;
      if (b == 0) {  // k <= 32: a warp per unit
        const int wg = std::max(1, std::min((hcounts[0] + 7) / 8, SM * 8));
        if (mode == 0)
          k_cliques_warp<0><<<wg, 256, 0, lst>>>(g, cbins, hcounts[0], 1, cmine, Te, K4t, Fp(F_K4), K4e, Fp(F_K5),
                                                 nullptr, nullptr);
        else
          k_cliques_warp<1><<<wg, 256, 0, lst>>>(g, cbins, hcounts[0], 0, cmine, Te, K4t, nullptr, nullptr, nullptr,
                                                 Fp(F_R66), Fp(F_R70));
        C.launches++;
        continue;
      }
      if (mode == 0) {
        if (smem > 48 * 1024)
          CK(cudaFuncSetAttribute(k_cliques<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_cliques<0><<<grid, block, smem, lst>>>(g, cbins + (size_t)b * n, hcounts[b], words, 0, 0, cscratch,
                                                 cscratch_words, 1, cmine, Te, K4t, Fp(F_K4), K4e, Fp(F_K5),
                                                 nullptr, nullptr);
      } else {
        // theta66 / theta70 per local edge: 2 x kmax u64 accumulators after the bitmap (shared-memory bins)
        const int accw = b < 4 ? (words + 1) & ~1 : 0;
        const size_t smem1 = b < 4 ? (size_t)accw * sizeof(u32) + (size_t)2 * kmax * sizeof(u64) : smem;
        if (smem1 > 48 * 1024)
          CK(cudaFuncSetAttribute(k_cliques<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1));
        k_cliques<1><<<grid, block, smem1, lst>>>(g, cbins + (size_t)b * n, hcounts[b], words, accw, kmax, cscratch,
                                                  cscratch_words, 0, cmine, Te, K4t, nullptr, nullptr, nullptr,
                                                  Fp(F_R66), Fp(F_R70));
      }
      C.launches++;
    }
  };
  // a5/a9 and the first neighbour gather feed none of the pass preparations below, so they
  // run on a side stream while the main stream prepares the passes (whose host reads of tier
  // counts would otherwise leave the GPU idle); the passes start after both (ev_fork)
  EdgeVals ev{Te, E9f, E9b, K4e, C4e, E7, K4t};
  const int warp_grid = grid_for((int64_t)n * 32, B, SM);
  int32_t* nbr_heavy = A.alloc<int32_t>(std::max(n, 1));
  int32_t* nbr_mid = A.alloc<int32_t>(std::max(n, 1));
  int* nbr_nh = A.alloc<int>(8, true);  // [slot] heavy, [4 + slot] mid counts of gather `slot`
  const int group_grid = grid_for(((int64_t)n + 3) / 4 * 32, B, SM);
  auto gather_on = [&](cudaStream_t gs, auto kw, auto km, auto kh, int slot) {
    kw<<<group_grid, B, 0, gs>>>(g, ev, F, nbr_heavy, nbr_nh + slot, nbr_mid, nbr_nh + 4 + slot);
    km<<<4 * SM, B, 0, gs>>>(g, ev, F, nbr_mid, nbr_nh + 4 + slot);
    kh<<<SM, 1024, 0, gs>>>(g, ev, F, nbr_heavy, nbr_nh + slot);
    C.launches += 3;
  };
  const bool serial_flag = (o.flags & EVOKE_FLAG_SERIAL) != 0;
  cudaStream_t pre = C.st;
  if (!serial_flag && n > 0 && !getenv("EVOKE_NO_SIDE")) {  // (EVOKE_NO_SIDE: developer A/B)
    pre = C.stream(Ctx::MAXJOBS - 1, 0);
    C.side_used = true;
    CK(cudaEventRecord(C.ev_pre, C.st));
    CK(cudaStreamWaitEvent(pre, C.ev_pre, 0));
    CK(cudaEventRecord(C.sev[0], pre));
  }
  if (ntri > 0) launch_cliques(0, pre);
  if (C.side_used) CK(cudaEventRecord(C.sev[1], pre));
  // ------------------------------------------------------------------ nbr gather 1
  C.mark(P_NBR1);
  if (n > 0) gather_on(pre, k_nbr<1>, k_nbr_mid<1>, k_nbr_heavy<1>, 0);
  if (C.side_used) {
    CK(cudaEventRecord(C.sev[2], pre));
    CK(cudaEventRecord(C.ev_side, pre));
  }

  // ------------------------------------------------------------------ a7, a8, a10, theta66/70
  // The four passes are independent (disjoint outputs; inputs from a1-a6).  Their
  // preparations (work estimates, sorts, tier counts: host syncs) run first on the main
  // stream; then each pass's persistent kernels are launched on a stream of its own so the
  // passes overlap (the GPU analogue of the paper's concurrent orbit groups).
  struct Job { int pass; int rank; std::function<void(cudaStream_t)> fn; };
  std::vector<Job> jobs;  // rank: launch order / stream priority (long single-item tails first)
  u64* pair_pa = nullptr;  // the pair pass's per-vertex credits (PairField order, interleaved)
  C.mark(P_PAIR);
  C.tick("start");
  if (n > 0 && m > 0) {
    // source lists by 2-hop estimate (descending), sharded by position, split in tiers
    u32* pk = A.alloc<u32>(n);
    u32* pk2 = A.alloc<u32>(n);
    int32_t* pv = A.alloc<int32_t>(n);
    int32_t* pv2 = A.alloc<int32_t>(n);
    u32* pest = A.alloc<u32>(n);
    int32_t* plists = A.alloc<int32_t>((size_t)PT_COUNT * n);
    int* tiers = A.alloc<int>(8, true);
    int32_t* hstar = A.alloc<int32_t>(n);
    int32_t* hstar_s = A.alloc<int32_t>(n);
    u32* pwest = A.alloc<u32>(n);
    u64* dwork = nullptr;
    if (ntri > 0 && !getenv("EVOKE_PAIR_NO_DWORK")) {  // (env: developer A/B)
      dwork = A.alloc<u64>(n, true);
      k_pair_dwork<<<grid_for(ntri, B, SM), B, 0, C.st>>>(g, Te, dwork);
      C.launches++;
    }
    int32_t* plen = A.alloc<int32_t>(m2 + 1);
    k_pair_est<<<warp_grid, B, 0, C.st>>>(g, dwork, pk, pv, pwest, hstar, hstar_s, plen);
    g.plen = plen;  // (the pair jobs capture g after this)
    C.tick("pair_est");
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, pk, pk2, pv, pv2, (int64_t)n, 0, 32, C.st));
    void* t = A.alloc<char>(tb);
    CK(cub::DeviceRadixSort::SortPairs(t, tb, pk, pk2, pv, pv2, (int64_t)n, 0, 32, C.st));
    C.tick("pair_sort");
    PairTiers ptiers;
    ptiers.packed_lim = env_cap("EVOKE_PAIR_PACKED_LIM", 65536);
    ptiers.light_max = env_cap("EVOKE_PAIR_LIGHT_MAX", PAIR_WARP_MAX);
    ptiers.mids_max = env_cap("EVOKE_PAIR_MIDS_MAX", PAIR_MIDS_MAX);
    ptiers.mid_max = env_cap("EVOKE_PAIR_MID_MAX", PAIR_MID_MAX);
    ptiers.tiny_max = env_cap("EVOKE_PAIR_TINY_MAX", PAIR_TINY_MAX);
    ptiers.sweep = getenv("EVOKE_PAIR_SWEEP") ? atoi(getenv("EVOKE_PAIR_SWEEP")) : -1;
    k_pair_classify<<<warp_grid, B, 0, C.st>>>(g, pk2, pv2, si, ns, ptiers, Fp(F_T), pwest, pest, plists, tiers);
    k_shard_sum_u32<<<grid_for(n, B, SM), B, 0, C.st>>>(pk2, n, si, ns, d_work + 0);
    C.launches += 3;
    C.lib_launches += 4;
    int ht[PT_COUNT];
    CK(cudaMemcpyAsync(ht, tiers, sizeof(ht), cudaMemcpyDeviceToHost, C.st));
    CK(cudaStreamSynchronize(C.st));
    C.tick("pair_classify+sync");
    auto plist = [&](int tier) { return plists + (size_t)tier * n; };
    if (getenv("EVOKE_DEBUG"))
      fprintf(stderr, "[evoke] pair tiers: g64 %d g32 %d g32s %d mid %d small-mid %d light %d tiny %d\n", ht[PT_G64],
              ht[PT_G32], ht[PT_G32S], ht[PT_MID], ht[PT_MIDS], ht[PT_LIGHT], ht[PT_TINY]);
    // adjacency maps of the hubs (h* membership and T(h*, x) in one load), within a memory budget
    int32_t* hslot = A.alloc<int32_t>(n);
    int* hcnt = A.alloc<int>(1, true);
    const int max_maps = getenv("EVOKE_PAIR_NO_MAPS") ? 0  // (developer A/B: key search instead)
                         : (int)std::min<int64_t>(4096, std::max<int64_t>(0, (256ll << 20) / ((int64_t)n * 4)));
    int32_t* hubs = A.alloc<int32_t>(std::max(max_maps, 1));
    k_hub_slots<<<grid_for(n, B, SM), B, 0, C.st>>>(g, max_maps, hslot, hubs, hcnt);
    int hcs[1] = {0};
    CK(cudaMemcpyAsync(&hcs[0], hcnt, sizeof(int), cudaMemcpyDeviceToHost, C.st));
    CK(cudaStreamSynchronize(C.st));
    const int nmaps = std::min(hcs[0], max_maps);
    int32_t* hpos = A.alloc<int32_t>((size_t)std::max(nmaps, 1) * n);
    if (nmaps > 0) {
      CK(cudaMemsetAsync(hpos, 0xff, sizeof(int32_t) * (size_t)nmaps * n, C.st));
      k_hub_maps<<<std::min(nmaps, 4 * SM), 256, 0, C.st>>>(g, Te, hubs, nmaps, hpos);
    }
    C.launches += 2;
    pair_pa = A.alloc<u64>((size_t)n * PO_STRIDE);
    CK(cudaMemsetAsync(pair_pa, 0, sizeof(u64) * (size_t)n * PO_STRIDE, C.st));
    PairOut po{pair_pa, C4e, hstar, hstar_s, hslot, hpos};
    const size_t freeb = avail_bytes(C.dev) + lease.room();
    // heavy tiers: dense per-CTA tables, as many CTAs as keep the tables L2-resident
    const char* phg_env = getenv("EVOKE_PAIR_HG");  // developer knob: heavy-source CTAs
    // heavy tiers: one CTA (a whole SM: 1024 threads x 64 registers) per source at a time.
    // While the CTAs' dense tables fit L2 (small n) the heavy sources are not the long pole
    // and half the SMs leave room for the other passes (config 2: 0.1-0.3 ms better step);
    // past L2 the tables are DRAM-bound and the heavy sources dominate: every SM (config 5:
    // 173 s instead of 199 s).
    // The three heavy tiers share one memory budget (half the free estimate); each CTA
    // needs its dense table (word bytes per vertex), its touched list (4 per vertex) and its
    // engine queue, and each tier's share is taken off the budget before the next is sized.
    int64_t heavy_budget = (int64_t)(freeb / 2);
    const int heavy_qcap = 2 * g.max_deg + 65536;
    auto heavy_grid = [&](int nsrc, size_t word, int cap) {
      const int64_t l2_ctas = std::max<int64_t>(1, (56ll << 20) / ((int64_t)n * (int64_t)word));
      int64_t pg = std::min<int64_t>((l2_ctas >= SM / 2 && !whole_gpu_passes) ? SM / 2 : SM, cap);
      if (phg_env) pg = std::max(1, atoi(phg_env));  // developer knob: the grid itself
      pg = std::min<int64_t>(pg, nsrc);
      const int64_t per_cta = (int64_t)n * (int64_t)(word + 4) + (int64_t)eng_queue_bytes(heavy_qcap);
      pg = std::max<int64_t>(1, std::min<int64_t>(pg, heavy_budget / per_cta));
      heavy_budget -= pg * per_cta;
      return (int)pg;
    };
    // hot entries of the heavy tables: the top ranks in shared memory (EVOKE_PAIR_HOT: count cap)
    auto pair_hot_k = [&](int word) {
      return (int)std::min<int64_t>({(int64_t)env_cap("EVOKE_PAIR_HOT", PAIR_HOT_BYTES / word), (int64_t)n,
                                     (int64_t)(PAIR_HOT_BYTES / word)});
    };
    // the tables, touched lists and queues of pg heavy CTAs; on an allocation failure (the
    // free estimate is a reading from earlier in the process) half as many CTAs, down to one
    auto heavy_alloc = [&](int& pg, size_t word, bool with_list, void*& tabs, int32_t*& lists, char*& qmem) {
      for (;;) {
        const size_t per = (size_t)((n + 3) / 4 * 4) * word;
        tabs = A.try_zalloc<char>((size_t)pg * per);
        lists = (tabs && with_list) ? A.try_alloc<int32_t>((size_t)pg * n) : nullptr;
        qmem = (tabs && (lists || !with_list)) ? A.try_alloc<char>((size_t)pg * eng_queue_bytes(heavy_qcap)) : nullptr;
        if (qmem) return;
        if (tabs) A.release(tabs);
        if (lists) A.release(lists);
        if (pg == 1) throw EvokeError{EVOKE_ENOMEM};
        pg = std::max(1, pg / 2);
      }
    };
    if (ht[PT_G64] > 0) {
      // sources beyond the packed 16-bit counters (d(u) or T(u) >= 2^16): u64 tables
      int pg = heavy_grid(ht[PT_G64], 8, SM);
      void* tabs_v;
      int32_t* lists;
      char* qmem;
      heavy_alloc(pg, 8, true, tabs_v, lists, qmem);
      u64* tabs = (u64*)tabs_v;
      int* counter = A.alloc<int>(1, true);
      const int32_t* pl = plist(PT_G64);
      const int cnt = ht[PT_G64];
      const int qcap = heavy_qcap;
      const int hk = pair_hot_k(8);
      CK(cudaFuncSetAttribute(k_pairs_heavy<u64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, hk * 8));
      jobs.push_back({P_PAIR, 1, [=, &C](cudaStream_t st) {
        k_pairs_heavy<u64, false><<<pg, PAIR_HBT, hk * 8, st>>>(g, Te, pl, cnt, counter, tabs, lists, po, qmem, qcap,
                                                                hk);
        C.launches++;
      }});
    }
    for (int tier : {PT_G32S, PT_G32}) {
      if (ht[tier] == 0) continue;
      int pg = heavy_grid(ht[tier], 4, SM);
      void* tabs_v;
      int32_t* lists;
      char* qmem;
      heavy_alloc(pg, 4, tier == PT_G32, tabs_v, lists, qmem);
      u32* tabs = (u32*)tabs_v;
      int* counter = A.alloc<int>(1, true);
      const int32_t* pl = plist(tier);
      const int cnt = ht[tier];
      const int qcap = heavy_qcap;
      const int hk = pair_hot_k(4);
      CK(cudaFuncSetAttribute(k_pairs_heavy<u32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, hk * 4));
      CK(cudaFuncSetAttribute(k_pairs_heavy<u32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, hk * 4));
      jobs.push_back({P_PAIR, 1, [=, &C](cudaStream_t st) {
        if (tier == PT_G32S)
          k_pairs_heavy<u32, true><<<pg, PAIR_HBT, hk * 4, st>>>(g, Te, pl, cnt, counter, tabs, lists, po, qmem,
                                                                 qcap, hk);
        else
          k_pairs_heavy<u32, false><<<pg, PAIR_HBT, hk * 4, st>>>(g, Te, pl, cnt, counter, tabs, lists, po, qmem,
                                                                  qcap, hk);
        C.launches++;
      }});
    }
    // the small-mid kernel runs on the main tier's stream, ahead of it (one more concurrent
    // grid would take SMs from the other passes' persistent kernels)
    std::function<void(cudaStream_t)> mids_fn;
    if (ht[PT_MIDS] > 0) {
      const int smem = PAIR_MIDS_CAP * 8;
      CK(cudaFuncSetAttribute(k_pairs_mids, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      int bps = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_pairs_mids, PAIR_MIDS_BT, smem));
      int* counter = A.alloc<int>(1, true);
      const int32_t* pms = plist(PT_MIDS);
      const int nms = ht[PT_MIDS];
      const int grid = std::max(bps, 1) * SM;
      const int qcap = 2 * PAIR_MIDS_MAX + 16384;
      char* qmem = A.alloc<char>((size_t)grid * eng_queue_bytes(qcap));
      mids_fn = [=, &C](cudaStream_t st) {
        k_pairs_mids<<<grid, PAIR_MIDS_BT, smem, st>>>(g, Te, pms, nms, pest, counter, po, qmem, qcap);
        C.launches++;
      };
    }
    if (ht[PT_MID] + ht[PT_LIGHT] > 0) {
      CK(cudaFuncSetAttribute(k_pairs_main, cudaFuncAttributeMaxDynamicSharedMemorySize, PAIR_SMEM));
      int bps = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_pairs_main, PAIR_BT, PAIR_SMEM));
      int* counters = A.alloc<int>(2, true);
      const int32_t* pm = plist(PT_MID);
      const int32_t* pli = plist(PT_LIGHT);
      const int nmid = ht[PT_MID], nli = ht[PT_LIGHT];
      const int grid = std::max(bps, 1) * SM;
      const int qcap = 2 * PAIR_MID_MAX + 16384;
      char* qmem = A.alloc<char>((size_t)grid * eng_queue_bytes(qcap));
      jobs.push_back({P_PAIR, 3, [=, &C](cudaStream_t st) {
        if (mids_fn) mids_fn(st);
        k_pairs_main<<<grid, PAIR_BT, PAIR_SMEM, st>>>(g, Te, pm, nmid, pli, nli, pest, counters, po, qmem, qcap);
        C.launches++;
      }});
    } else if (mids_fn) {
      jobs.push_back({P_PAIR, 3, mids_fn});
    }
    if (ht[PT_TINY] > 0) {
      int bps = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_pairs_tiny<PAIR_TINY_CAP>, PAIR_BT, 0));
      int* counter = A.alloc<int>(1, true);
      const int32_t* pt = plist(PT_TINY);
      const int nt = ht[PT_TINY];
      const int grid = std::max(bps, 1) * SM;
      jobs.push_back({P_PAIR, 3, [=, &C](cudaStream_t st) {
        k_pairs_tiny<PAIR_TINY_CAP><<<grid, PAIR_BT, 0, st>>>(g, Te, pt, nt, pest, counter, po);
        C.launches++;
      }});
    }
  }

  // ------------------------------------------------------------------ a8: hub-local
  // (EVOKE_FLAG_FOUR: 4-vertex orbits only -- the 5-vertex passes a8, a10, theta66/70 and
  // the 5-vertex gathers are skipped, as in the paper's EVOKE-4, Table 1)
  const bool four = (o.flags & EVOKE_FLAG_FOUR) != 0;
  C.mark(P_HUB);
  C.tick("pair_rest");
  if (ntri > 0 && !four) {
    const int64_t m2s = 2 * m;
    int32_t* light = A.alloc<int32_t>(m2s);
    int32_t* heavy = A.alloc<int32_t>(m2s);
    u32* hest = A.alloc<u32>(m2s);
    int* hcnt = A.alloc<int>(8, true);  // n_light, n_heavy, counters [2], [3], [6], n_micro [4], n_giant [5]
    int32_t* micro = A.alloc<int32_t>(m2s);
    u64* hitem_est = A.alloc<u64>(m2s, true);
    if (ntri > 0)
      k_hub_est<<<grid_for(ntri, 256, SM), 256, 0, C.st>>>(g, Te, hitem_est);
    const uint8_t* hmine = shard_mask(A, C, hitem_est, m2s, si, ns, d_work + 2);
    const u64 hub_warp_max = env_cap("EVOKE_HUB_WARP_MAX", HUB_WARP_MAX);
    const u64 hub_micro_max = std::min(hub_warp_max, env_cap("EVOKE_HUB_MICRO_MAX", HUB_MICRO_MAX));
    const u64 hub_giant = env_cap("EVOKE_HUB_GIANT", HUB_GIANT);
    k_hub_bin<<<grid_for(m2s, 256, SM), 256, 0, C.st>>>(g, Te, hitem_est, hmine, hub_micro_max, hub_warp_max, micro,
                                                        hcnt + 4, light, hcnt, heavy, hest, hcnt + 1, hub_giant,
                                                        hcnt + 5);
    C.launches += 2;
    int hc[6];
    CK(cudaMemcpyAsync(hc, hcnt, sizeof(hc), cudaMemcpyDeviceToHost, C.st));
    CK(cudaStreamSynchronize(C.st));
    C.tick("hub_items+sync");
    const int n_light = hc[0], n_heavy = hc[1], n_micro = hc[4], n_giant = hc[5];
    if (getenv("EVOKE_DEBUG"))
      fprintf(stderr, "[evoke] hub items: micro %d light %d heavy %d (giant %d)\n", n_micro, n_light, n_heavy, n_giant);
    int32_t* heavy_sorted = heavy;
    u32* heavy_est_sorted = hest;
    if (n_heavy > 1) {
      int32_t* hs = A.alloc<int32_t>(n_heavy);
      u32* hk = A.alloc<u32>(n_heavy);
      size_t tb = 0;
      CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, hest, hk, heavy, hs, n_heavy, 0, 32, C.st));
      void* t = A.alloc<char>(tb);
      CK(cub::DeviceRadixSort::SortPairsDescending(t, tb, hest, hk, heavy, hs, n_heavy, 0, 32, C.st));
      C.lib_launches += 4;
      heavy_sorted = hs;
      heavy_est_sorted = hk;
    }
    if (n_light + n_heavy > 0) {
      // giant items (the est-sorted list's head): one 1024-thread CTA per SM with a large shared
      // table; the other heavy items: 256-thread CTAs, four per SM (a CTA per item, and most
      // items have too few middles to keep 32 warps busy)
      auto kgiant = k_hub_heavy<1024, HUB_GSMEM>;
      auto kheavy = k_hub_heavy<256, HUB_HSMEM>;
      int hb_per_sm = 0, lb_per_sm = 0;
      CK(cudaFuncSetAttribute(kgiant, cudaFuncAttributeMaxDynamicSharedMemorySize, HUB_GSMEM));
      CK(cudaFuncSetAttribute(kheavy, cudaFuncAttributeMaxDynamicSharedMemorySize, HUB_HSMEM));
      CK(cudaFuncSetAttribute(k_hub_light, cudaFuncAttributeMaxDynamicSharedMemorySize, HUB_SMEM));
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&hb_per_sm, kheavy, 256, HUB_HSMEM));
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&lb_per_sm, k_hub_light, HUB_BT, HUB_SMEM));
      const char* hhg_env = getenv("EVOKE_HUB_HG");  // developer knob: hub-local CTAs
      // a short hub-local pass (few items) gets one CTA per SM, not as many as fit: its CTAs
      // placed ahead of the heavy pair sources' whole-SM CTAs delay those (config 2: 0.1 ms
      // better); a long one (diamond-heavy graphs) keeps full occupancy
      const bool few = (int64_t)n_light + n_heavy <= HUB_FEW_ITEMS && !whole_gpu_passes;
      const int gg = std::max(1, std::min(n_giant, SM));
      const int hg = hhg_env ? std::max(1, atoi(hhg_env)) : (few ? 1 : std::max(1, hb_per_sm)) * SM;
      const int lg = hhg_env ? std::max(1, atoi(hhg_env)) : (few ? 1 : std::max(1, lb_per_sm)) * SM;
      u32* gt = nullptr;
      int32_t* gl = nullptr;
      const int sh_dense_max = (int)env_cap("EVOKE_HUB_SH_DENSE", HUB_SH_DENSE);
      const int hash_max = (int)env_cap("EVOKE_HUB_HASH_MAX", HUB_HASH_MAX);
      const int split = (int)std::max<u64>(1, env_cap("EVOKE_HUB_SPLIT", HUB_SPLIT));
      if (n_heavy > 0 && (g.max_deg > std::min(sh_dense_max, HUB_HSMEM / 2) || g.max_deg >= 65536)) {
        const int tg = std::max(gg, hg);
        gt = A.zalloc<u32>((size_t)tg * g.max_deg);
        gl = A.alloc<int32_t>((size_t)tg * g.max_deg);
      }
      u64* r68 = Fp(F_R68);
      u64* r69 = Fp(F_R69);
      const int n_rest = n_heavy - n_giant;
      jobs.push_back({P_HUB, 2, [=, &C](cudaStream_t st) {
        if (n_giant > 0)
          kgiant<<<gg, 1024, HUB_GSMEM, st>>>(g, heavy_sorted, heavy_est_sorted, n_giant, hcnt + 2, gt, gl, r68, r69,
                                              sh_dense_max, hash_max, split);
        if (n_rest > 0)
          kheavy<<<hg, 256, HUB_HSMEM, st>>>(g, heavy_sorted + n_giant, heavy_est_sorted + n_giant, n_rest, hcnt + 6,
                                             gt, gl, r68, r69, sh_dense_max, hash_max, split);
        if (n_light > 0) k_hub_light<<<lg, HUB_BT, HUB_SMEM, st>>>(g, Te, light, n_light, hcnt + 3, r68, r69);
        if (n_micro > 0) k_hub_micro<<<grid_for(n_micro, 128, SM), 128, 0, st>>>(g, micro, n_micro, r68, r69);
        C.launches += (n_giant > 0) + (n_rest > 0) + (n_light > 0) + (n_micro > 0);
      }});
    } else if (n_micro > 0) {
      u64* r68 = Fp(F_R68);
      u64* r69 = Fp(F_R69);
      jobs.push_back({P_HUB, 2, [=, &C](cudaStream_t st) {
        k_hub_micro<<<grid_for(n_micro, 128, SM), 128, 0, st>>>(g, micro, n_micro, r68, r69);
        C.launches++;
      }});
    }
  }

  // ------------------------------------------------------------------ a10: 5-cycles
  C.mark(P_C5);
  C.tick("hub_rest");
  if (n > 0 && m > 0 && !four) {
    // exact work W(l) and record bound R(l) of every endpoint (O(m)), this shard's endpoints
    // by position in the W-sorted list, tiers
    u32* splus = A.alloc<u32>(n);
    u64* c5W = A.alloc<u64>(n);
    u64* c5R = A.alloc<u64>(n);
    int4* c5s = A.alloc<int4>(m2 + 1);
    k_c5_slots<<<warp_grid, B, 0, C.st>>>(g, c5s);
    g.c5s = c5s;  // (the 5-cycle jobs capture g after this)
    C.launches++;
    k_c5_splus<<<grid_for(n, B, SM), B, 0, C.st>>>(g, splus);
    k_c5_work<<<warp_grid, B, 0, C.st>>>(g, splus, c5W, c5R);
    C.launches += 2;
    // giants (W(l) >= giant_w; W >= 2^32 always: their u64 records): the whole GPU per endpoint,
    // on every shard (step 3 split by j-key), so they take no part in the position split
    const u64 giant_w = env_cap("EVOKE_C5_GIANT_W", C5_GIANT_W);
    const uint8_t* c5mine = nullptr;
    if (ns > 1) {
      u64* c5Wm = A.alloc<u64>(n);
      k_c5_giant_mask<<<grid_for(n, B, SM), B, 0, C.st>>>(c5W, n, giant_w, ns, c5Wm, d_work + 4);
      C.launches++;
      c5mine = shard_mask(A, C, c5Wm, n, si, ns, d_work + 4);
    }
    int32_t* c5lists = A.alloc<int32_t>((size_t)4 * n);  // light, mid, big, giant
    u32* c5rb = A.alloc<u32>((size_t)2 * n);              // R(l) of the hashed tiers
    u64* c5bw = A.alloc<u64>(n);                          // W(l) of the big tier
    int* c5c = A.alloc<int>(8, true);  // tier sizes [0..3], persistent-kernel counters [4..6]
    u64* C5out = Fp(F_C5);
    // tier limits (lower only: env for tests); mid work < 2^16 keeps the packed records exact
    const u64 rec_light = env_cap("EVOKE_C5_LIGHT_REC", C5_WARP_MAX), work_light = env_cap("EVOKE_C5_LIGHT_WORK", C5_WARP_WORK);
    const u64 rec_mid = env_cap("EVOKE_C5_MID_REC", C5_MID_MAX), work_mid = env_cap("EVOKE_C5_MID_WORK", C5_MID_WORK);
    k_c5_bin<<<grid_for(n, B, SM), B, 0, C.st>>>(g, c5W, c5R, c5mine, rec_light, work_light, rec_mid, work_mid,
                                                 giant_w, c5lists, c5rb, c5bw, c5c);
    C.launches++;
    int hc5[4];
    CK(cudaMemcpyAsync(hc5, c5c, sizeof(hc5), cudaMemcpyDeviceToHost, C.st));
    CK(cudaStreamSynchronize(C.st));
    C.tick("c5_items+sync");
    const int n5l = hc5[0], n5m = hc5[1], n5b = hc5[2], n5g = hc5[3];
    int32_t* c5l = c5lists;
    u32* c5lr = c5rb;
    if (getenv("EVOKE_DEBUG"))
      fprintf(stderr, "[evoke] c5 endpoints: light %d mid %d big %d giant %d\n", n5l, n5m, n5b, n5g);
    if (getenv("EVOKE_C5_HIST")) {  // developer: W / R histogram of every endpoint
      std::vector<u64> hw(n), hr(n);
      CK(cudaMemcpyAsync(hw.data(), c5W, sizeof(u64) * n, cudaMemcpyDeviceToHost, C.st));
      CK(cudaMemcpyAsync(hr.data(), c5R, sizeof(u64) * n, cudaMemcpyDeviceToHost, C.st));
      CK(cudaStreamSynchronize(C.st));
      const u64 edges_[] = {256, 1024, 4096, 16384, 65536, 1ull << 20, ~0ull};
      u64 cw[7] = {}, sw[7] = {}, cr[7] = {};
      for (int32_t q = 0; q < n; q++)
        for (int b2 = 0; b2 < 7; b2++) {
          if (hw[q] <= edges_[b2]) { cw[b2]++; sw[b2] += hw[q]; break; }
        }
      for (int32_t q = 0; q < n; q++)
        for (int b2 = 0; b2 < 7; b2++)
          if (hr[q] <= edges_[b2]) { cr[b2]++; break; }
      for (int b2 = 0; b2 < 7; b2++)
        fprintf(stderr, "[evoke] c5 W <= %llu: %llu endpoints (work %llu); R <= it: %llu endpoints\n",
                (unsigned long long)edges_[b2], (unsigned long long)cw[b2], (unsigned long long)sw[b2],
                (unsigned long long)cr[b2]);
    }
    const size_t freeb = avail_bytes(C.dev) + lease.room();
    // W-descending order of a hashed tier's list (heaviest endpoints first)
    auto sort_tier = [&](int t, int cnt, int32_t*& ls, u32*& rs) {
      ls = c5lists + (size_t)t * n;
      rs = c5rb + (size_t)t * n;
      if (cnt <= 1) return;
      u64* mw = A.alloc<u64>(cnt);
      k_gather_u64<<<grid_for(cnt, B, SM), B, 0, C.st>>>(c5W, ls, cnt, mw);
      int32_t* idx = A.alloc<int32_t>(cnt);
      int32_t* sidx = A.alloc<int32_t>(cnt);
      u64* sk = A.alloc<u64>(cnt);
      k_iota_i32<<<grid_for(cnt, B, SM), B, 0, C.st>>>(idx, cnt);
      size_t tb = 0;
      CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, mw, sk, idx, sidx, cnt, 0, 64, C.st));
      void* t2 = A.alloc<char>(tb);
      CK(cub::DeviceRadixSort::SortPairsDescending(t2, tb, mw, sk, idx, sidx, cnt, 0, 64, C.st));
      int32_t* lo = A.alloc<int32_t>(cnt);
      u32* ro = A.alloc<u32>(cnt);
      k_permute_c5<<<grid_for(cnt, B, SM), B, 0, C.st>>>(sidx, cnt, ls, rs, lo, ro);
      C.launches += 3;
      C.lib_launches += 4;
      ls = lo;
      rs = ro;
    };
    std::vector<std::function<void(cudaStream_t)>> c5chain;  // big, then mid: one stream
    // big endpoints, W descending; returns W max
    auto sort_big = [&](int cnt, int32_t*& bs) -> u64 {
      int32_t* src = c5lists + (size_t)2 * n;
      bs = src;
      if (cnt <= 1) return d2h_scalar<u64>(c5bw, C.st);
      bs = A.alloc<int32_t>(cnt);
      u64* bk = A.alloc<u64>(cnt);
      size_t tb = 0;
      CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, c5bw, bk, src, bs, cnt, 0, 64, C.st));
      void* t2 = A.alloc<char>(tb);
      CK(cub::DeviceRadixSort::SortPairsDescending(t2, tb, c5bw, bk, src, bs, cnt, 0, 64, C.st));
      C.lib_launches += 4;
      return d2h_scalar<u64>(bk, C.st);
    };
    if (n5g > 0) {
      // one giant at a time on every SM: steps 0-2, step 3, steps 4-6, reset (four kernels each)
      const int32_t* gl = c5lists + (size_t)3 * n;
      C5Rec* gdense = A.zalloc<C5Rec>((size_t)n);
      int32_t* gdl = A.alloc<int32_t>((size_t)2 * n);
      int* gcnt = A.alloc<int>((size_t)2 * n5g, true);
      u64* gtot = A.alloc<u64>((size_t)n5g, true);
      int bpg = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpg, k_c5_giant, C5_HBT, 0));
      const int gg = std::max(1, bpg) * SM;
      int32_t* gq = A.alloc<int32_t>((size_t)gg * (2 * (size_t)g.max_deg + 1));
      c5chain.push_back([=, &C](cudaStream_t st) {
        for (int q = 0; q < n5g; q++)
          for (int part = 0; part < 4; part++) {
            k_c5_giant<<<gg, C5_HBT, 0, st>>>(part, g, Tmid, Thigh, gl, q, gdense, gdl, gcnt, gtot, C5out, gq, ns, si);
            C.launches++;
          }
      });
    }
    const char* hg_env = getenv("EVOKE_C5_HG");  // developer knob: big-endpoint CTAs
    // (passes running alone: two big-endpoint CTAs per SM when registers and shared memory
    // allow -- 64 warps hide more of the records' L2/DRAM round trips: config 4 47.9 -> 46.2 ms)
    const int64_t hg_want = hg_env ? std::max(1, atoi(hg_env)) : (whole_gpu_passes ? 2 * SM : SM);
    if (n5b > 0) {
      int32_t* bs = nullptr;
      const u64 wmax = sort_big(n5b, bs);
      // u32 record fields when every big endpoint's W < 2^32 (every field is <= W(l))
      const bool narrow = wmax < (1ull << 32) && !getenv("EVOKE_C5_WIDE");
      const size_t rec = narrow ? sizeof(C5RecT<u32>) : sizeof(C5Rec);
      const int64_t per = (int64_t)n * (int64_t)(rec + 8);
      // (whole-GPU passes run alone: half the free estimate; concurrent: a quarter)
      const int64_t budget = (int64_t)(whole_gpu_passes ? freeb / 2 : freeb / 4);
      const int hg0 = (int)std::min<int64_t>(std::min<int64_t>(hg_want, n5b), std::max<int64_t>(1, budget / per));
      // first-touch bitmaps (present, j-key) in shared memory when they fit
      const size_t bits_smem = (size_t)2 * ((n + 31) / 32) * sizeof(u32);
      const int use_bits = bits_smem <= C5_BITS_SMEM_MAX && !getenv("EVOKE_C5_NO_BITS") ? 1 : 0;
      // hot-vertex cache of the top ranks (u32 records): 12 bytes per cached vertex
      const size_t bits_b = use_bits ? bits_smem : 0;
      // (only when the big endpoints are large enough to repay the shared memory taken from L1)
      const int hot_k = (!narrow || wmax < env_cap("EVOKE_C5_HOT_MIN_W", C5_HOT_MIN_W)) ? 0
                        : (int)std::min<int64_t>({(int64_t)env_cap("EVOKE_C5_HOT", C5_HOT_MAX), (int64_t)n,
                                                  (int64_t)((C5_SMEM_MAX - bits_b) / 12)});
      const size_t bsm = bits_b + (size_t)12 * hot_k;
      if (bsm > 0) {
        CK(cudaFuncSetAttribute(k_c5_heavy<u32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
        CK(cudaFuncSetAttribute(k_c5_heavy<u64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
      }
      int hbps = 0;  // resident big-endpoint CTAs per SM: the grid never exceeds what is co-resident
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&hbps, narrow ? (const void*)k_c5_heavy<u32>
                                                                     : (const void*)k_c5_heavy<u64>, C5_HBT, bsm));
      const int hg = std::min(hg0, std::max(1, hbps) * SM);
      if (getenv("EVOKE_DEBUG"))
        fprintf(stderr, "[evoke] c5 big: %d endpoints, W max %llu, %d CTAs (%s records, free estimate %.1f GB)\n",
                n5b, (unsigned long long)wmax, hg, narrow ? "u32" : "u64", freeb / 1e9);
      char* dense = A.zalloc<char>((size_t)hg * n * rec);
      int32_t* dl = A.alloc<int32_t>((size_t)hg * 2 * n);
      int32_t* lq = A.alloc<int32_t>((size_t)hg * (2 * (size_t)g.max_deg + 1));
      c5chain.push_back([=, &C](cudaStream_t st) {
        if (narrow)
          k_c5_heavy<u32><<<hg, C5_HBT, bsm, st>>>(g, Tlow, Tmid, Thigh, bs, n5b, c5c + 6,
                                                   reinterpret_cast<C5RecT<u32>*>(dense), dl, C5out, lq, use_bits,
                                                   hot_k);
        else
          k_c5_heavy<u64><<<hg, C5_HBT, bsm, st>>>(g, Tlow, Tmid, Thigh, bs, n5b, c5c + 6,
                                                   reinterpret_cast<C5Rec*>(dense), dl, C5out, lq, use_bits, 0);
        C.launches++;
      });
    }
    if (n5m > 0) {
      // mid endpoints, W descending: several 4-warp CTAs per SM, hashed records in per-CTA
      // global regions
      int32_t* ms;
      u32* mr;
      sort_tier(1, n5m, ms, mr);
      int bpm = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpm, k_c5_mid, C5_MBT, 0));
      const char* mb_env = getenv("EVOKE_C5_MBPS");  // developer knob: mid CTAs per SM
      const int mbps = mb_env ? atoi(mb_env) : (whole_gpu_passes ? 16 : 4);
      const int gm = (int)std::min<int64_t>(std::max(1, std::min(bpm, mbps)) * SM, n5m);
      C5RecP* mreg = A.zalloc<C5RecP>((size_t)gm * C5_MID_CAP);
      int32_t* mlists = A.alloc<int32_t>((size_t)gm * 2 * C5_MID_CAP);
      int32_t* mq = A.alloc<int32_t>((size_t)gm * (2 * (size_t)g.max_deg + 1));
      c5chain.push_back([=, &C](cudaStream_t st) {
        k_c5_mid<<<gm, C5_MBT, 0, st>>>(g, Tlow, Tmid, Thigh, ms, mr, n5m, c5c + 5, mreg, mlists, C5out, mq);
        C.launches++;
      });
    }
    if (!c5chain.empty())
      jobs.push_back({P_C5, 0, [c5chain](cudaStream_t st) { for (auto& f : c5chain) f(st); }});
    if (n5l > 0) {
      int bps = 0;
      const char* shc_env = getenv("EVOKE_C5_SHCAP");  // developer knob: shared records per warp
      // (whole-GPU passes: smaller shared regions, more warps resident)
      const int sh_cap = shc_env ? std::max(64, std::min(C5_SH_CAP, atoi(shc_env))) : (whole_gpu_passes ? 64 : C5_SH_CAP_DEFAULT);
      const size_t sh_bytes = C5_SH_BYTES(sh_cap);
      CK(cudaFuncSetAttribute(k_c5_light, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh_bytes));
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_c5_light, C5_BT, sh_bytes));
      const char* lb_env = getenv("EVOKE_C5_LBPS");  // developer knob: light CTAs per SM
      const int lg = std::max(1, std::min(bps, lb_env ? atoi(lb_env) : (whole_gpu_passes ? 8 : 4))) * SM;
      const size_t nw = (size_t)lg * (C5_BT / 32);
      C5RecL* reg = A.zalloc<C5RecL>(nw * C5_WARP_CAP);
      int32_t* wl = A.alloc<int32_t>(nw * 2 * C5_WARP_CAP);
      jobs.push_back({P_C5, 4, [=, &C](cudaStream_t st) {
        k_c5_light<<<lg, C5_BT, sh_bytes, st>>>(g, Tlow, Tmid, Thigh, c5l, c5lr, n5l, c5c + 4, reg, wl, C5out,
                                                sh_cap);
        C.launches++;
      }});
    }
  }

  // ------------------------------------------------------------------ theta66 / theta70
  if (ntri > 0 && !four) jobs.push_back({P_CLIQ2, 5, [&](cudaStream_t st) { launch_cliques(1, st); }});

  // ------------------------------------------------------------------ concurrent launch
  C.mark(P_CLIQ2);
  C.tick("c5_rest");
  // one stream per job (jobs of one pass stay in order on a shared stream when they must:
  // the heavy and main pair kernels write different sources, so all jobs are independent)
  std::stable_sort(jobs.begin(), jobs.end(), [](const Job& x, const Job& y) { return x.rank < y.rank; });
  // kept streams 0..MAXJOBS-4 are the jobs'; the last three: main (no caller stream), tail
  // gathers, side
  if (jobs.size() > (size_t)Ctx::MAXJOBS - 3) { set_error("too many concurrent jobs"); throw EvokeError{EVOKE_EINTERNAL}; }
  const bool serial = (o.flags & EVOKE_FLAG_SERIAL) != 0 || whole_gpu_passes;
  C.serial_run = serial;
  if (C.side_used) CK(cudaStreamWaitEvent(C.st, C.ev_side, 0));
  CK(cudaEventRecord(C.ev_fork, C.st));
  for (size_t i = 0; i < jobs.size(); i++) {
    cudaStream_t st = serial ? C.st : C.stream(i, jobs[i].rank);
    CK(cudaStreamWaitEvent(st, C.ev_fork, 0));
    CK(cudaEventRecord(C.pev[i][0], st));
    jobs[i].fn(st);
    CK(cudaEventRecord(C.pev[i][1], st));
  }
  // gathers 2/3 and the triangle gather read, of the concurrent passes' outputs, only the
  // pair pass's (R8, C4e): they start on a stream of their own when the pair jobs end and run
  // beside the 5-cycle / hub-local / theta66-70 tails
  auto gathers23 = [&](cudaStream_t gs) {
    if (pair_pa) {  // the pair pass's credits, interleaved by vertex, into their fields
      const PairFields fl{{Fp(F_R8), Fp(F_R36), Fp(F_R50), Fp(F_R63), Fp(F_R51), Fp(F_R49), Fp(F_R62), Fp(F_R64)}};
      k_pair_fields<<<grid_for((int64_t)n * PO_STRIDE, B, SM), B, 0, gs>>>(pair_pa, n, fl);
      C.launches++;
    }
    if (n > 0) {  // rows of the values the late gathers read at random places
      k_pack_rows<<<grid_for(std::max<int64_t>(n, m), B, SM), B, 0, gs>>>(g, ev, F, V2rows, EVrows);
      C.launches++;
      ev.V2 = V2rows;
      ev.EV = EVrows;
    }
    if (n > 0) {
      gather_on(gs, k_nbr<2>, k_nbr_mid<2>, k_nbr_heavy<2>, 1);
      if (!four) gather_on(gs, k_nbr<3>, k_nbr_mid<3>, k_nbr_heavy<3>, 2);
    }
  };
  auto trigather = [&](cudaStream_t gs) {
    if (ntri > 0 && !four) {
      // rows while the graph averages few triangles per vertex (config 4: 4.2 -> 2.5 ms);
      // straight into the fields on triangle-heavy graphs (config 3: 48 ms vs 62 ms in rows)
      if (3 * ntri <= TG_ROWS_MAX_TPV * (int64_t)n) {
        CK(cudaMemsetAsync(TGrows, 0, sizeof(u64) * (size_t)n * TG_W, gs));
        k_trigather<true><<<grid_for(ntri, B, SM), B, 0, gs>>>(g, ev, TGrows);
        k_tg_fields<<<grid_for((int64_t)n * TG_W, B, SM), B, 0, gs>>>(TGrows, n, F);
        C.launches += 2;
      } else {
        k_trigather<false><<<grid_for(ntri, B, SM), B, 0, gs>>>(g, ev, F);
        C.launches++;
      }
    }
  };
  if (!serial && n > 0 && !getenv("EVOKE_NO_EARLY_GATHERS")) {
    C.gathers_early = true;
    cudaStream_t gs = C.stream(Ctx::MAXJOBS - 2, 0);
    CK(cudaStreamWaitEvent(gs, C.ev_fork, 0));
    for (size_t i = 0; i < jobs.size(); i++)
      if (jobs[i].pass == P_PAIR) CK(cudaStreamWaitEvent(gs, C.pev[i][1], 0));
    CK(cudaEventRecord(C.gev[0], gs));
    gathers23(gs);
    CK(cudaEventRecord(C.gev[1], gs));
    trigather(gs);
    CK(cudaEventRecord(C.gev[2], gs));
    CK(cudaStreamWaitEvent(C.st, C.gev[2], 0));
  }
  for (size_t i = 0; i < jobs.size(); i++) CK(cudaStreamWaitEvent(C.st, C.pev[i][1], 0));
  if (getenv("EVOKE_DEBUG")) {
    unsigned long long ph[2][8];
    CK(cudaStreamSynchronize(C.st));
    CK(cudaMemcpyFromSymbol(ph, g_pair_phase, sizeof(ph)));
    for (int t = 0; t < 2; t++)
      fprintf(stderr, "[evoke] pair %s phases (Mcycles): pass1 %.1f hstar %.1f terms %.1f pass2 %.1f tail %.1f"
              " | sweeps %.1f queue-rounds %.1f\n",
              t ? "dense" : "mid", ph[t][0] / 1e6, ph[t][1] / 1e6, ph[t][2] / 1e6, ph[t][3] / 1e6, ph[t][4] / 1e6,
              ph[t][5] / 1e6, ph[t][6] / 1e6);
    unsigned long long z[2][8] = {};
    CK(cudaMemcpyToSymbol(g_pair_phase, z, sizeof(z)));
    unsigned long long c5p[3][8];
    CK(cudaMemcpyFromSymbol(c5p, g_c5_phase, sizeof(c5p)));
    for (int t = 0; t < 3; t++)
      fprintf(stderr, "[evoke] c5 %s steps (Mcycles): s0 %.1f s1 %.1f s2 %.1f s3 %.1f s4 %.1f s5 %.1f s6 %.1f\n",
              t == 2 ? "light" : t ? "mid" : "heavy", c5p[t][0] / 1e6, c5p[t][1] / 1e6, c5p[t][2] / 1e6,
              c5p[t][3] / 1e6, c5p[t][4] / 1e6, c5p[t][5] / 1e6, c5p[t][6] / 1e6);
    fprintf(stderr, "[evoke] c5 light records used %llu of %llu region slots\n", c5p[2][7], c5p[1][7]);
    unsigned long long z3[3][8] = {};
    CK(cudaMemcpyToSymbol(g_c5_phase, z3, sizeof(z3)));
    unsigned long long umax[4], usum[4], uz[4] = {};
    int uarg[4];
    CK(cudaMemcpyFromSymbol(umax, g_unit_max, sizeof(umax)));
    CK(cudaMemcpyFromSymbol(usum, g_unit_sum, sizeof(usum)));
    CK(cudaMemcpyFromSymbol(uarg, g_unit_arg, sizeof(uarg)));
    const char* un[3] = {"pair heavy", "hub heavy", "c5 big"};
    for (int t = 0; t < 3; t++)
      fprintf(stderr, "[evoke] %s units: longest %.3f ms (list index %d), sum %.3f ms (SM clock %.0f MHz)\n", un[t],
              umax[t] / (C.sm_mhz * 1e3), uarg[t], usum[t] / (C.sm_mhz * 1e3), C.sm_mhz);
    CK(cudaMemcpyToSymbol(g_unit_max, uz, sizeof(uz)));
    CK(cudaMemcpyToSymbol(g_unit_sum, uz, sizeof(uz)));
  }
  C.njobs = (int)jobs.size();
  for (size_t i = 0; i < jobs.size(); i++) { C.job_pass[i] = jobs[i].pass; C.job_rank[i] = jobs[i].rank; }

  // ------------------------------------------------------------------ nbr gathers 2,3
  C.mark(P_NBR2);
  if (!C.gathers_early) gathers23(C.st);  // (serial mode: here, in order)
  // ------------------------------------------------------------------ triangle gather
  C.mark(P_TRIG);
  if (!C.gathers_early) trigather(C.st);

  // ------------------------------------------------------------------ a12: combine
  C.mark(P_COMB);
  u64* dout = nullptr;
  if (n > 0) {
    dout = A.alloc<u64>((size_t)n * 73);  // staged: `out` is written only after every check passed
    const size_t csm = (size_t)COMBINE_BT * EVOKE_NUM_ORBITS_DEV * sizeof(u64);
    CK(cudaFuncSetAttribute(k_combine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm));
    k_combine<<<grid_for(n, COMBINE_BT, SM), COMBINE_BT, csm, C.st>>>(g, F, perm, o.induced, si == 0 ? 1 : 0,
                                                                      four ? 15 : 73, dout);
    C.launches++;
  }
  // every check before `out` is touched: kernel faults (sync), and in the developer mode
  // the zero invariant of the kept scratch
  CK(cudaStreamSynchronize(C.st));
  CK(cudaGetLastError());
  lease.ok = true;  // every pass has reset its tables
  if (lease.zp && lease.used > 0 && getenv("EVOKE_CHECK_ZERO")) {
    int* flag = A.alloc<int>(1, true);
    k_check_zero<<<4 * SM, 256, 0, C.st>>>((const uint4*)lease.zp->p, lease.used / 16, flag);
    if (d2h_scalar<int>(flag, C.st)) {
      lease.ok = false;
      set_error("a pass left its scratch table nonzero (EVOKE_CHECK_ZERO)");
      throw EvokeError{EVOKE_EINTERNAL};
    }
  }
  C.mark(P_D2H);
  if (n > 0)
    CK(cudaMemcpyAsync(out, dout, sizeof(u64) * (size_t)n * 73,
                       o.device_pointers ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, C.st));
  C.mark(P_COUNT);
  CK(cudaStreamSynchronize(C.st));
  C.print_ticks();
  if (getenv("EVOKE_DEBUG")) {  // main-stream preparation time of the concurrent passes
    float a = 0, b = 0, c = 0, d = 0;
    CK(cudaEventElapsedTime(&a, C.ev[P_PAIR], C.ev[P_HUB]));
    CK(cudaEventElapsedTime(&b, C.ev[P_HUB], C.ev[P_C5]));
    CK(cudaEventElapsedTime(&c, C.ev[P_C5], C.ev[P_CLIQ2]));
    CK(cudaEventElapsedTime(&d, C.ev[0], C.ev[P_PAIR]));
    fprintf(stderr, "[evoke] preparations: pair %.3f hub %.3f c5 %.3f ms (stages before them %.3f ms)\n", a, b, c, d);
  }
  if (hostprof()) {
    float gms = 0;
    CK(cudaEventElapsedTime(&gms, C.ev[0], C.ev[P_COUNT]));
    const double hms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - C.hts[0]).count();
    if (hms > std::max(0.0, atof(getenv("EVOKE_HOSTPROF")))) {  // EVOKE_HOSTPROF=<ms>: report calls slower than this
      fprintf(stderr, "[evoke hostprof] call host %.1f ms gpu %.1f ms\n", hms, gms);
      C.host_report();
    }
  }

  if (o.stats) {
    evoke_stats* s = o.stats;
    std::memset(s, 0, sizeof(*s));
    s->n = n; s->m = m; s->triangles = ntri; s->max_degree = max_deg; s->degeneracy = max_out;
    s->num_passes = P_COUNT;
    for (int i = 0; i < P_COUNT; i++) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, C.ev[i], C.ev[i + 1]));
      s->ms_pass[i] = ms;
    }
    if (C.gathers_early) {  // gathers 2/3 and the triangle gather ran beside the 5-cycle tail
      float a = 0, b = 0;
      CK(cudaEventElapsedTime(&a, C.gev[0], C.gev[1]));
      CK(cudaEventElapsedTime(&b, C.gev[1], C.gev[2]));
      s->ms_pass[P_NBR2] = a;
      s->ms_pass[P_TRIG] = b;
    }
    if (C.side_used) {  // a5/a9 and gather 1 ran on the side stream, beside the preparations
      float a = 0, b = 0;
      CK(cudaEventElapsedTime(&a, C.sev[0], C.sev[1]));
      CK(cudaEventElapsedTime(&b, C.sev[1], C.sev[2]));
      s->ms_pass[P_CLIQ] = a;
      s->ms_pass[P_NBR1] = b;
    }
    // the pair, hub-local, 5-cycle and theta66/70 kernels run concurrently: each of these
    // passes reports its preparation (main stream) plus the span of its own kernels; the
    // overlap makes the per-pass times add up to more than ms_total
    s->ms_pass[P_CLIQ2] = 0;
    const bool serial = C.serial_run;
    for (int pass : {P_PAIR, P_HUB, P_C5, P_CLIQ2}) {
      float lo = 1e30f, hi = -1e30f, sum = 0;
      for (int j = 0; j < C.njobs; j++) {
        if (C.job_pass[j] != pass) continue;
        float a = 0, b = 0;
        CK(cudaEventElapsedTime(&a, C.ev[0], C.pev[j][0]));
        CK(cudaEventElapsedTime(&b, C.ev[0], C.pev[j][1]));
        lo = std::min(lo, a);
        hi = std::max(hi, b);
        sum += b - a;
      }
      // serial: the pass's own kernels (its jobs are interleaved with other passes' jobs);
      // concurrent: the span of its kernels
      if (hi > lo) s->ms_pass[pass] += serial ? sum : hi - lo;
    }
    if (getenv("EVOKE_JOBS")) {  // developer trace: start / end of every concurrent job
      std::string line;
      for (int j = 0; j < C.njobs; j++) {
        float a = 0, b = 0;
        CK(cudaEventElapsedTime(&a, C.ev[0], C.pev[j][0]));
        CK(cudaEventElapsedTime(&b, C.ev[0], C.pev[j][1]));
        char buf[96];
        snprintf(buf, sizeof(buf), " %s/r%d %.2f-%.2f", kPassNames[C.job_pass[j]], C.job_rank[j], a, b);
        line += buf;
      }
      fprintf(stderr, "[evoke jobs]%s\n", line.c_str());
    }
    float tot = 0;
    CK(cudaEventElapsedTime(&tot, C.ev[0], C.ev[P_COUNT]));
    s->ms_total = tot;
    {
      u64 hw[8];
      CK(cudaMemcpyAsync(hw, d_work, sizeof(hw), cudaMemcpyDeviceToHost, C.st));
      CK(cudaStreamSynchronize(C.st));
      for (int q = 0; q < 4; q++) { s->work_shard[q] = hw[2 * q]; s->work_total[q] = hw[2 * q + 1]; }
    }
    s->kernel_launches = C.launches;
    s->library_launches = C.lib_launches;
    u64* dw = A.alloc<u64>(1, true);
    if (n > 0) k_wedges<<<grid_for(n, B, SM), B, 0, C.st>>>(rp, n, dw);
    s->wedges = (int64_t)d2h_scalar<u64>(dw, C.st);
    if ((o.flags & EVOKE_FLAG_WORKMODEL) && n > 0) {
      WorkUnits* du = A.alloc<WorkUnits>(1, true);
      k_units_vertex<<<grid_for((int64_t)n * 32, B, SM), B, 0, C.st>>>(g, du);
      if (m > 0) k_units_edge<<<grid_for(m, B, SM), B, 0, C.st>>>(g, Te, du);
      if (ntri > 0) k_units_hub<<<grid_for(m2, B, SM), B, 0, C.st>>>(g, Te, du);
      WorkUnits hu = d2h_scalar<WorkUnits>(du, C.st);
      s->units[0] = (int64_t)hu.sum_d2; s->units[1] = (int64_t)hu.sum_te2; s->units[2] = (int64_t)hu.hub;
      s->units[3] = (int64_t)hu.c5_wedge; s->units[4] = (int64_t)hu.c5_q; s->units[5] = (int64_t)hu.tri_stream;
      s->units[6] = (int64_t)hu.pair_rwedge; s->units[7] = (int64_t)hu.pair_hwalk;
      // algorithmic bytes per pass = units x the bytes of graph data each unit must read
      // (DESIGN.md section 5.2); per-source / per-endpoint tables are on-chip or L2 scratch
      s->alg_bytes[P_TRI] = 8.0 * (double)hu.tri_stream + 16.0 * (double)ntri;
      s->alg_bytes[P_PAIR] = 16.0 * (double)hu.pair_rwedge + 8.0 * (double)hu.pair_hwalk + 8.0 * (double)hu.sum_te2;
      s->alg_bytes[P_HUB] = 28.0 * (double)hu.hub;
      s->alg_bytes[P_C5] = 12.0 * (double)hu.c5_wedge + 12.0 * (double)hu.c5_q;
      s->alg_bytes[P_TRIG] = 16.0 * (double)ntri + 3.0 * 14.0 * 16.0 * (double)ntri;
    }
  }
}

int guarded(const Input& in, uint64_t* out, const evoke_options* opt) {
  g_last_error.clear();
  evoke_options o;
  evoke_default_options(&o);
  if (opt) {
    if (opt->struct_size != 0 && opt->struct_size < sizeof(evoke_options)) {
      std::memcpy(&o, opt, opt->struct_size);
    } else {
      o = *opt;
    }
  }
  if (o.num_shards < 1 || o.shard_index < 0 || o.shard_index >= o.num_shards) {
    set_error("bad shard %d of %d", o.shard_index, o.num_shards);
    return EVOKE_EINVAL;
  }
  if (in.n < 0 || in.n >= (1ll << 31) - 1) { set_error("bad n = %lld", (long long)in.n); return EVOKE_EINVAL; }
  if (in.kind == 0) {
    if (in.m < 0) { set_error("bad m"); return EVOKE_EINVAL; }
    if (in.m > 0 && !in.edges) { set_error("edges is NULL"); return EVOKE_EINVAL; }
  } else {
    if (!in.rowptr) { set_error("rowptr is NULL"); return EVOKE_EINVAL; }
    if (!o.device_pointers) {
      if (in.rowptr[0] != 0) { set_error("rowptr[0] != 0"); return EVOKE_EINVAL; }
      for (int64_t v = 0; v < in.n; v++)
        if (in.rowptr[v + 1] < in.rowptr[v]) { set_error("rowptr not monotone at %lld", (long long)v); return EVOKE_EINVAL; }
      if (in.rowptr[in.n] > 0 && !in.col) { set_error("col is NULL"); return EVOKE_EINVAL; }
    }
  }
  if (in.n > 0 && !out) { set_error("out is NULL"); return EVOKE_EINVAL; }
  if (in.n == 0) {
    if (o.stats) { std::memset(o.stats, 0, sizeof(*o.stats)); o.stats->num_passes = P_COUNT; }
    return EVOKE_OK;
  }
  try {
    run(in, out, o);
  } catch (const EvokeError& e) {
    return e.code;
  } catch (const std::exception& e) {
    set_error("%s", e.what());
    return EVOKE_EINTERNAL;
  }
  return EVOKE_OK;
}

// ---- several GPUs from one process (SURVEY 8(b) num_gpus) ----------
// acc[i] += src[i] modulo 2^64.  src is a partial matrix on this device or on a peer device
// (then every load crosses NVLink: the reduction reads the peer's memory directly, there is
// no staging copy).  Buffers from cudaMalloc, so 16-byte aligned.
__global__ void k_add_partial(u64* __restrict__ acc, const u64* __restrict__ src, int64_t cnt) {
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  ulonglong2* a2 = reinterpret_cast<ulonglong2*>(acc);
  const ulonglong2* s2 = reinterpret_cast<const ulonglong2*>(src);
  for (int64_t i = t0; i < cnt / 2; i += nt) {
    ulonglong2 a = a2[i];
    const ulonglong2 b = s2[i];
    a.x += b.x;
    a.y += b.y;
    a2[i] = a;
  }
  if (t0 == 0 && (cnt & 1)) acc[cnt - 1] += src[cnt - 1];
}

// Shard d of num_devices runs on devices[d] (one host thread per distinct device; shards
// that name the same device run one after the other on it), every device with its own copy
// of the edge list (the graph is replicated), each shard's partial n x 73
// matrix in that device's memory.  devices[0] then sums the partials (k_add_partial over
// peer memory, or staged chunks when peer access is unavailable) and the sum is copied to
// out only after every shard and the reduction succeeded.
int multi_edges(int64_t n, int64_t m, const int32_t* edges, uint64_t* out, const int* devices, int nd,
                const evoke_options* opt) {
  g_last_error.clear();
  evoke_options o;
  evoke_default_options(&o);
  if (opt) {
    if (opt->struct_size != 0 && opt->struct_size < sizeof(evoke_options)) std::memcpy(&o, opt, opt->struct_size);
    else o = *opt;
  }
  if (!devices || nd < 1 || nd > 64) { set_error("need 1..64 devices, got %d", nd); return EVOKE_EINVAL; }
  if (o.num_shards < 1 || o.shard_index < 0 || o.shard_index >= o.num_shards ||
      (int64_t)o.num_shards * nd > (int64_t)INT32_MAX) {
    set_error("bad shard %d of %d (x %d devices)", o.shard_index, o.num_shards, nd);
    return EVOKE_EINVAL;
  }
  if (n < 0 || n >= (1ll << 31) - 1) { set_error("bad n = %lld", (long long)n); return EVOKE_EINVAL; }
  if (m < 0 || (m > 0 && !edges)) { set_error("bad m or NULL edges"); return EVOKE_EINVAL; }
  if (n > 0 && !out) { set_error("out is NULL"); return EVOKE_EINVAL; }
  if (n == 0) {
    if (o.stats) { std::memset(o.stats, 0, sizeof(*o.stats)); o.stats->num_passes = P_COUNT; }
    return EVOKE_OK;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess) {
    set_error("cudaGetDeviceCount: %s", cudaGetErrorString(cudaGetLastError()));
    return EVOKE_ECUDA;
  }
  for (int d = 0; d < nd; d++)
    if (devices[d] < 0 || devices[d] >= ndev) { set_error("device %d not in [0, %d)", devices[d], ndev); return EVOKE_EINVAL; }
  int cur = 0;
  (void)cudaGetDevice(&cur);
  const int dev0 = devices[0];
  std::vector<int> uniq;
  std::vector<std::vector<int>> shards_of;
  for (int d = 0; d < nd; d++) {
    const size_t u = std::find(uniq.begin(), uniq.end(), devices[d]) - uniq.begin();
    if (u == uniq.size()) { uniq.push_back(devices[d]); shards_of.emplace_back(); }
    shards_of[u].push_back(d);
  }
  const size_t cells = (size_t)n * EVOKE_NUM_ORBITS, ebytes = sizeof(int32_t) * 2 * (size_t)m;
  std::vector<u64*> part(nd, nullptr);
  std::vector<int> rc(uniq.size(), EVOKE_OK);
  std::vector<std::string> msg(uniq.size());
  auto worker = [&](size_t ui) {
    const int dev = uniq[ui];
    int32_t* dedges = nullptr;
    bool own_edges = false;
    auto fail = [&](int code, const std::string& what) { rc[ui] = code; msg[ui] = what; };
    auto cuda_ok = [&](cudaError_t e, const char* what) {
      if (e == cudaSuccess) return true;
      (void)cudaGetLastError();
      fail(e == cudaErrorMemoryAllocation ? EVOKE_ENOMEM : EVOKE_ECUDA,
           std::string(what) + ": " + cudaGetErrorString(e) + " (device " + std::to_string(dev) + ")");
      return false;
    };
    if (!cuda_ok(cudaSetDevice(dev), "cudaSetDevice")) return;
    if (m > 0) {
      if (o.device_pointers && dev == dev0) {
        dedges = const_cast<int32_t*>(edges);  // the caller's copy, on devices[0]
      } else if (cuda_ok(cudaMalloc(&dedges, ebytes), "edge list copy")) {
        own_edges = true;
        if (o.device_pointers) cuda_ok(cudaMemcpyPeer(dedges, dev, edges, dev0, ebytes), "edge list peer copy");
        else cuda_ok(cudaMemcpy(dedges, edges, ebytes, cudaMemcpyHostToDevice), "edge list H2D");
      }
    }
    for (int d : shards_of[ui]) {
      if (rc[ui] != EVOKE_OK) break;
      if (!cuda_ok(cudaMalloc(&part[d], sizeof(u64) * cells), "partial matrix")) break;
      evoke_options od = o;
      od.device = dev;
      od.device_pointers = 1;
      od.stream = nullptr;
      od.num_shards = o.num_shards * nd;
      od.shard_index = o.shard_index * nd + d;
      od.stats = d == 0 ? o.stats : nullptr;
      const int r = evoke_orbits_edges(n, m, dedges, reinterpret_cast<uint64_t*>(part[d]), &od);
      if (r != EVOKE_OK) fail(r, std::string("shard ") + std::to_string(d) + ": " + evoke_last_error());
      else cuda_ok(cudaDeviceSynchronize(), "shard synchronise");
    }
    if (own_edges) (void)cudaFree(dedges);
  };
  std::vector<std::thread> th;
  for (size_t ui = 1; ui < uniq.size(); ui++) th.emplace_back(worker, ui);
  worker(0);
  for (auto& t : th) t.join();
  int code = EVOKE_OK;
  std::string why;
  for (size_t ui = 0; ui < uniq.size(); ui++)
    if (rc[ui] != EVOKE_OK && code == EVOKE_OK) { code = rc[ui]; why = msg[ui]; }
  // the reduction on devices[0]: acc = partial of shard 0 (which runs there)
  u64* stage = nullptr;
  if (code == EVOKE_OK) {
    auto step = [&](cudaError_t e, const char* what) {
      if (e == cudaSuccess || code != EVOKE_OK) return code == EVOKE_OK;
      (void)cudaGetLastError();
      code = e == cudaErrorMemoryAllocation ? EVOKE_ENOMEM : EVOKE_ECUDA;
      why = std::string(what) + ": " + cudaGetErrorString(e);
      return false;
    };
    step(cudaSetDevice(dev0), "cudaSetDevice");
    int SM = 148;
    step(cudaDeviceGetAttribute(&SM, cudaDevAttrMultiProcessorCount, dev0), "SM count");
    u64* acc = part[0];
    const size_t chunk = std::min<size_t>(cells, (size_t)1 << 25);  // 256 MB staging chunks
    for (int d = 1; d < nd && code == EVOKE_OK; d++) {
      int peer = devices[d] == dev0;
      if (!peer) {
        (void)cudaDeviceCanAccessPeer(&peer, dev0, devices[d]);
        if (peer) {
          const cudaError_t e = cudaDeviceEnablePeerAccess(devices[d], 0);
          if (e != cudaSuccess) {
            (void)cudaGetLastError();
            if (e != cudaErrorPeerAccessAlreadyEnabled) peer = 0;
          }
        }
      }
      if (peer) {
        k_add_partial<<<SM * 4, 256>>>(acc, part[d], (int64_t)cells);
        step(cudaGetLastError(), "k_add_partial");
      } else {
        if (!stage && !step(cudaMalloc(&stage, sizeof(u64) * chunk), "staging buffer")) break;
        for (size_t off = 0; off < cells && code == EVOKE_OK; off += chunk) {
          const size_t c = std::min(chunk, cells - off);
          if (!step(cudaMemcpyPeer(stage, dev0, part[d] + off, devices[d], sizeof(u64) * c), "partial peer copy")) break;
          k_add_partial<<<SM * 4, 256>>>(acc + off, stage, (int64_t)c);
          step(cudaGetLastError(), "k_add_partial");
        }
      }
    }
    step(cudaDeviceSynchronize(), "reduction");
    if (code == EVOKE_OK)  // out is written only now, after every shard and the sum succeeded
      step(cudaMemcpy(out, acc, sizeof(u64) * cells, o.device_pointers ? cudaMemcpyDeviceToDevice
                                                                        : cudaMemcpyDeviceToHost), "result copy");
  }
  for (int d = 0; d < nd; d++)
    if (part[d]) { (void)cudaSetDevice(devices[d]); (void)cudaFree(part[d]); }
  if (stage) { (void)cudaSetDevice(dev0); (void)cudaFree(stage); }
  (void)cudaGetLastError();
  (void)cudaSetDevice(cur);
  if (code != EVOKE_OK) set_error("%s", why.c_str());
  return code;
}

}  // namespace

extern "C" {

void evoke_default_options(evoke_options* opt) {
  if (!opt) return;
  std::memset(opt, 0, sizeof(*opt));
  opt->struct_size = sizeof(evoke_options);
  opt->induced = 1;
  opt->device_pointers = 0;
  opt->shard_index = 0;
  opt->num_shards = 1;
  opt->device = -1;
  opt->stream = nullptr;
  opt->stats = nullptr;
  opt->flags = 0;
}

int evoke_orbits_edges(int64_t n, int64_t m, const int32_t* edges, uint64_t* out, const evoke_options* opt) {
  Input in{0, n, m, edges, nullptr, nullptr};
  return guarded(in, out, opt);
}

int evoke_orbits_csr(int64_t n, const int64_t* rowptr, const int32_t* col, uint64_t* out,
                     const evoke_options* opt) {
  Input in{1, n, 0, nullptr, rowptr, col};
  return guarded(in, out, opt);
}

int evoke_orbits_edges_multi(int64_t n, int64_t m, const int32_t* edges, uint64_t* out, const int* devices,
                             int num_devices, const evoke_options* opt) {
  try {
    return multi_edges(n, m, edges, out, devices, num_devices, opt);
  } catch (const std::exception& e) {
    set_error("%s", e.what());
    return EVOKE_EINTERNAL;
  }
}

int evoke_ccd(int64_t n, const uint64_t* dim, int orbit, uint64_t* values, uint64_t* counts, int64_t* nvals,
              const evoke_options* opt) {
  g_last_error.clear();
  evoke_options o;
  evoke_default_options(&o);
  if (opt) {
    if (opt->struct_size != 0 && opt->struct_size < sizeof(evoke_options)) std::memcpy(&o, opt, opt->struct_size);
    else o = *opt;
  }
  if (n < 0 || orbit < 0 || orbit >= EVOKE_NUM_ORBITS || !nvals || (n > 0 && (!dim || !values || !counts))) {
    set_error("evoke_ccd: bad arguments");
    return EVOKE_EINVAL;
  }
  *nvals = 0;
  if (n == 0) return EVOKE_OK;
  try {
    int dev = o.device;
    if (dev < 0) CK(cudaGetDevice(&dev));
    CK(cudaSetDevice(dev));
    int SM = 0;
    CK(cudaDeviceGetAttribute(&SM, cudaDevAttrMultiProcessorCount, dev));
    cudaStream_t st = (cudaStream_t)o.stream;
    cudaStream_t own = nullptr;
    if (!st) { CK(cudaStreamCreateWithFlags(&own, cudaStreamNonBlocking)); st = own; }
    struct Own { cudaStream_t s; ~Own() { if (s) { cudaStreamSynchronize(s); cudaStreamDestroy(s); } } } own_guard{own};
    Arena A(st, dev);
    Ctx C;
    C.st = st;
    const u64* ddim = reinterpret_cast<const u64*>(dim);
    if (!o.device_pointers) {
      u64* t = A.alloc<u64>((size_t)n * EVOKE_NUM_ORBITS);
      CK(cudaMemcpyAsync(t, dim, sizeof(u64) * (size_t)n * EVOKE_NUM_ORBITS, cudaMemcpyHostToDevice, st));
      ddim = t;
    }
    u64* col = A.alloc<u64>(n);
    u64* sorted = A.alloc<u64>(n);
    k_ccd_gather<<<grid_for(n, 256, SM), 256, 0, st>>>(ddim, n, orbit, col);
    sort_keys_u64(A, C, col, sorted, n, 64);
    u64* uniq = A.alloc<u64>(n);
    u64* run = A.alloc<u64>(n);
    int64_t* nr = A.alloc<int64_t>(1);
    size_t tb = 0;
    CK(cub::DeviceRunLengthEncode::Encode(nullptr, tb, sorted, uniq, run, nr, n, st));
    void* t = A.alloc<char>(tb);
    CK(cub::DeviceRunLengthEncode::Encode(t, tb, sorted, uniq, run, nr, n, st));
    const int64_t k = d2h_scalar<int64_t>(nr, st);
    // suffix sums of the run lengths: reverse, inclusive scan, reverse
    u64* rev = A.alloc<u64>(k);
    u64* cum = A.alloc<u64>(k);
    u64* ccd = A.alloc<u64>(k);
    k_ccd_reverse<<<grid_for(k, 256, SM), 256, 0, st>>>(run, k, rev);
    inclusive_sum(A, C, rev, cum, k);
    k_ccd_reverse<<<grid_for(k, 256, SM), 256, 0, st>>>(cum, k, ccd);
    const cudaMemcpyKind kind = o.device_pointers ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    CK(cudaMemcpyAsync(values, uniq, sizeof(u64) * k, kind, st));
    CK(cudaMemcpyAsync(counts, ccd, sizeof(u64) * k, kind, st));
    CK(cudaStreamSynchronize(st));
    *nvals = k;
  } catch (const EvokeError& e) {
    return e.code;
  }
  return EVOKE_OK;
}

const char* evoke_pass_name(int i) {
  if (i < 0 || i >= (int)(sizeof(kPassNames) / sizeof(kPassNames[0]))) return nullptr;
  return kPassNames[i];
}

const char* evoke_strerror(int code) {
  switch (code) {
    case EVOKE_OK: return "ok";
    case EVOKE_EINVAL: return "invalid argument";
    case EVOKE_ENOMEM: return "out of device memory";
    case EVOKE_ECUDA: return "CUDA error";
    case EVOKE_EINTERNAL: return "internal error";
    default: return "unknown error";
  }
}

const char* evoke_last_error(void) { return g_last_error.c_str(); }

const char* evoke_version(void) { return EVOKE_VERSION; }

int evoke_release_scratch(int device) {
  if (device < -1 || device >= 64) {
    set_error("device ordinal %d outside [-1, 64)", device);
    return EVOKE_EINVAL;
  }
  int cur = 0;
  if (cudaGetDevice(&cur) != cudaSuccess) { (void)cudaGetLastError(); cur = 0; }
  for (int d = (device < 0 ? 0 : device); d < (device < 0 ? 64 : device + 1); d++) {
    ZeroPool& z = zero_pool(d);
    std::lock_guard<std::mutex> lk(z.mu);  // waits for a call that holds the lease
    if (!z.p) continue;
    if (cudaSetDevice(d) == cudaSuccess) {
      (void)cudaFree(z.p);  // stream-ordered allocation; cudaFree synchronises the device
    }
    (void)cudaGetLastError();
    z.p = nullptr;
    z.bytes = 0;
    z.target = 0;
    z.dirty = false;
  }
  // hand the pools' cached memory back to the device (other allocators, NCCL)
  for (int d = (device < 0 ? 0 : device); d < (device < 0 ? 64 : device + 1); d++) {
    cudaMemPool_t pool = evoke_pool_if_any(d);
    if (!pool || cudaSetDevice(d) != cudaSuccess) continue;
    (void)cudaDeviceSynchronize();
    (void)cudaMemPoolTrimTo(pool, 0);
    (void)cudaGetLastError();
  }
  (void)cudaSetDevice(cur);
  return EVOKE_OK;
}

}  // extern "C"
