/*
 * evoke.h -- C ABI of the B200-native EVOKE vertex-orbit counter (arXiv 1911.10616).
 *
 * Operation (Sec. 1.1 "Problem Description"): for a simple
 * undirected graph G and every vertex v and every orbit theta of the
 * 30 connected patterns on 2..5 vertices (Fig. 2; numbering = DESIGN.md
 * reading R1), output the number of times v occurs in a copy of theta: 73 counts per
 * vertex.  Induced counts by default ("we ask for induced counts"); non-induced
 * DM (Def. "unlabeled-match") on request.  The induced vector is
 * obtained from the non-induced one per vertex by DIM = A^-1 DM (Appendix A,
 * P:1103-1112).
 *
 * Method: degeneracy orientation G-> (any total order gives
 * identical counts), directed enumerations (triangles, 4-/5-cliques by out-
 * neighbourhood bitmaps, wedge pair tables, diamonds, the 5-cycle theorem P:866-886)
 * feeding the equations of Lemma 4vertexorbit, Lemma 4edgeorbit
 * and Theorem B.1, all on the GPU.
 *
 * Integer semantics: every count is the exact count modulo 2^64 (R20).
 *
 * Threading: calls are independent; one call uses one CUDA device (the current one,
 * or opt->device) and the given stream.  No caller pointer is retained after return.
 * The library keeps, per device, a few CUDA streams and a zeroed scratch buffer for its
 * per-CTA tables between calls (a call running concurrently with another on the same
 * device allocates its own); evoke_release_scratch frees the buffer.
 */
#ifndef EVOKE_H_
#define EVOKE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EVOKE_NUM_ORBITS 73

enum {
  EVOKE_OK = 0,
  EVOKE_EINVAL = -1,    /* bad argument: n<0, m<0, n >= 2^31, null pointer with a
                           non-zero size, vertex id outside [0,n), malformed CSR,
                           shard_index outside [0,num_shards)                      */
  EVOKE_ENOMEM = -2,    /* device allocation failed                                */
  EVOKE_ECUDA = -3,     /* any other CUDA runtime error (message: evoke_last_error) */
  EVOKE_EINTERNAL = -5, /* an internal invariant failed (e.g. graph too large:
                           m >= 2^31 undirected edges)                             */
};

/* Optional per-call statistics (filled if opt->stats != NULL). Times in ms measured
 * with CUDA events on the call's stream. */
typedef struct evoke_stats {
  int64_t n, m;                 /* vertices, undirected edges after cleaning        */
  int64_t triangles;            /* #triangles                                        */
  int64_t max_degree;           /* d_max                                             */
  int64_t degeneracy;           /* max out-degree of the degeneracy orientation      */
  int64_t wedges;               /* W(G) = sum_v C(d(v),2)                            */
  double ms_total;              /* whole call (device work, incl. H2D/D2H copies)    */
  double ms_pass[16];           /* per pass, see evoke_pass_name()                   */
  int32_t num_passes;
  int32_t kernel_launches;      /* kernels of this library launched in the call      */
  int32_t library_launches;     /* CUB sort/scan/select launches in the call         */
  int32_t reserved0;
  /* work model (only with EVOKE_FLAG_WORKMODEL): algorithmic bytes per pass, i.e. units
   * the pass must visit x bytes each visit must touch; 0 = not modelled */
  double alg_bytes[16];
  int64_t units[8];             /* sum d^2, sum T(e)^2, hub visits, c5 wedge visits,
                                   c5 out-out + path visits, triangle-pass stream,
                                   pair wedges walked (without h*), sum d(h*)         */
  /* work-balanced sharding (num_shards > 1): the work estimates of the sharded passes
   * [pair, hub-local, 5-cycle, 4/5-clique] summed over this shard's units and over all
   * units; max over shards / (total / num_shards) is the imbalance */
  uint64_t work_shard[4];
  uint64_t work_total[4];
} evoke_stats;

#define EVOKE_FLAG_WORKMODEL 1  /* fill evoke_stats.alg_bytes / units (extra kernels)  */
#define EVOKE_FLAG_SERIAL 2     /* run the pair, hub-local, 5-cycle and theta66/70 passes one
                                   after the other on the caller's stream (isolated per-pass
                                   timings) instead of concurrently on internal streams     */
#define EVOKE_FLAG_FOUR 4       /* 4-vertex orbits only (columns 0..14; 15..72 written as 0):
                                   the paper's EVOKE-4 (Table 1): the 5-vertex
                                   passes (hub-local, 5-cycles, theta66/70, 5-vertex
                                   gathers) are skipped                                     */

typedef struct evoke_options {
  uint32_t struct_size;   /* sizeof(evoke_options): ABI versioning; 0 = defaults   */
  int32_t induced;        /* 1 (default): induced counts DIM; 0: non-induced DM      */
  int32_t device_pointers;/* 1: edges / rowptr / col / out are device pointers on the
                             call's device; 0 (default): host pointers              */
  int32_t shard_index;    /* 0..num_shards-1                                         */
  int32_t num_shards;     /* 1 (default): whole result.  >1: this call returns the
                             shard's partial matrix; the element-wise sum mod 2^64 of
                             the partials of all shards equals the full result bit
                             for bit (multi-GPU data parallelism)         */
  int32_t device;         /* CUDA device ordinal; -1 (default) = current device      */
  int32_t flags;          /* EVOKE_FLAG_* bits; 0 default                            */
  void* stream;           /* cudaStream_t to run on; NULL = a library-owned stream,
                             ordered after the work already queued on the legacy
                             default stream (so device-pointer inputs produced there,
                             e.g. by torch's default stream, are complete)            */
  evoke_stats* stats;     /* optional output                                         */
} evoke_options;

/* Fill *opt with defaults (induced, host pointers, one shard, current device). */
void evoke_default_options(evoke_options* opt);

/*
 * evoke_orbits_edges -- orbit counts from an edge list.
 *   n      number of vertices; row v of the output is vertex v (ids are not compacted;
 *          ids never mentioned get an all-zero row) (R21)
 *   m      number of input pairs
 *   edges  int32[2*m], pair e = (edges[2e], edges[2e+1]); any order; reverse and exact
 *          duplicates collapse, self-loops are dropped
 *   out    uint64[n*73], row-major: out[v*73 + j] = count of orbit j at vertex v;
 *          caller-owned; written only on success (EVOKE_OK)
 *   opt    NULL for defaults
 * Host pointers are copied to the device inside the call (the copies are part of the
 * call); with device_pointers=1 no host transfer happens.  Returns EVOKE_OK or a
 * negative code; on error `out` is untouched and evoke_last_error() has a message (the
 * result is staged in library scratch and copied to `out` only after the final checks,
 * for host and device pointers alike).
 */
int evoke_orbits_edges(int64_t n, int64_t m, const int32_t* edges, uint64_t* out,
                       const evoke_options* opt);

/*
 * evoke_orbits_csr -- same, from a CSR: rowptr int64[n+1] (non-decreasing, rowptr[0]=0),
 * col int32[rowptr[n]].  The CSR need not be symmetric or sorted: every (v, col[k]) is an
 * undirected edge, cleaned as above.
 */
int evoke_orbits_csr(int64_t n, const int64_t* rowptr, const int32_t* col, uint64_t* out,
                     const evoke_options* opt);

/*
 * evoke_orbits_edges_multi -- the same result computed on several GPUs of one process
 * (SURVEY 8(b)'s num_gpus; the north star's data-parallel layout: the graph replicated on
 * every GPU, the work units of the sharded passes split by balanced work estimate,
 * DESIGN.md section 7; the paper's parallel orbit groups).
 *   devices      int[num_devices], CUDA ordinals; shard d of num_devices runs on devices[d]
 *                (one host thread per distinct device; shards naming the same device run
 *                one after the other on it, which tests the decomposition on one GPU)
 *   num_devices  1..64
 *   opt          as for evoke_orbits_edges, except: opt->device and opt->stream are
 *                ignored (each shard runs on its device's library stream); with
 *                device_pointers=1, edges and out live on devices[0] (the other devices
 *                copy the edge list over peer memory); opt->num_shards / shard_index compose
 *                (this call computes shards shard_index*num_devices + d of
 *                num_shards*num_devices, so several processes or nodes can split further);
 *                opt->stats, if set, receives shard 0's statistics.
 * Each device computes its shard's partial n x 73 matrix (exact modulo 2^64); devices[0]
 * sums them element-wise modulo 2^64, reading peer partials directly over NVLink when peer
 * access is available (staged copies otherwise).  Memory: every device holds the edge list,
 * its call's scratch and one n x 73 uint64 partial.  Returns EVOKE_OK or the first failing
 * shard's code (message via evoke_last_error(), naming the shard and device); out is written
 * only on success.
 */
int evoke_orbits_edges_multi(int64_t n, int64_t m, const int32_t* edges, uint64_t* out,
                             const int* devices, int num_devices, const evoke_options* opt);

/*
 * evoke_ccd -- complementary cumulative distribution of one orbit (the paper's VOC
 * distributions: "for x, ... the fraction of vertices whose orbit count is at
 * least x").
 *   n       number of rows of dim
 *   dim     uint64[n*73], an output of evoke_orbits_* (row-major)
 *   orbit   column 0..72
 *   values  uint64[n] output: the distinct counts of the column, ascending
 *   counts  uint64[n] output: counts[i] = number of vertices whose count is >= values[i]
 *           (divide by n for the fraction)
 *   nvals   output: number of entries written to values / counts
 * Pointers are host pointers, or device pointers with opt->device_pointers = 1 (opt may be
 * NULL: defaults).  Scratch is allocated on the device and freed before returning.
 * Errors: EVOKE_EINVAL for a bad orbit / null pointers; outputs untouched on error.
 */
int evoke_ccd(int64_t n, const uint64_t* dim, int orbit, uint64_t* values, uint64_t* counts, int64_t* nvals,
              const evoke_options* opt);

/*
 * evoke_release_scratch -- free the per-device scratch kept between calls.
 * The per-CTA tables of the pair, hub-local and 5-cycle passes are zero before and after
 * every successful call, so the library keeps one zeroed buffer per device (about 1 GB at
 * n = 1e5) and reuses it, which saves re-zeroing it on every call.  This frees it:
 * device = a CUDA device ordinal, or -1 for every device.  It waits for a call in progress
 * on that device, and also trims the library's private stream-ordered memory pool (the
 * scratch of earlier calls it keeps mapped for reuse) back to zero bytes, so the memory is
 * available to other allocators again.  Returns EVOKE_OK, or EVOKE_EINVAL for an ordinal
 * outside [-1, 64).
 */
int evoke_release_scratch(int device);

/* Static name of pass i of evoke_stats.ms_pass (NULL if out of range). */
const char* evoke_pass_name(int i);

/* Static text of an error code. */
const char* evoke_strerror(int code);

/* Thread-local detail of the last failure in this thread ("" if none). */
const char* evoke_last_error(void);

/* Library version string. */
const char* evoke_version(void);

#ifdef __cplusplus
}
#endif

#endif /* EVOKE_H_ */
