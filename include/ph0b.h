/* ph0b — B200-native (sm_100a) H0 persistent-homology barcode pipeline, C ABI.
 *
 * Drop-in for the reference library's hot path (namespace ph0, /root/reference/proj):
 *
 *     pairwise_distances        proj/include/ph0/filtration.hpp:35   (proj/src/filtration.cpp:8-18)
 *   ∘ build_filtration          proj/include/ph0/filtration.hpp:40   (proj/src/filtration.cpp:20-35)
 *   ∘ build_boundary_matrix     proj/include/ph0/boundary_matrix.hpp:30 (proj/src/boundary_matrix.cpp:15-28)
 *   ∘ reduce / reduce_parallel  proj/include/ph0/reduction.hpp:33,39 (proj/src/reduction.cpp:129-138)
 *   ∘ extract_barcode           proj/include/ph0/reduction.hpp:43   (proj/src/reduction.cpp:140-150)
 *
 * composed exactly as in proj/src/bench.cpp:45-59, proj/tools/ph0_cli.cpp:58-71 and
 * proj/tests/acceptance.cpp:56-68.  Input: point cloud X (N x d, f64).  Output: the finite
 * bars (0, b) in filtration order — death grade (1-based index into D) and death length —
 * the essential count, and the deduplicated, strictly increasing distance list D
 * (Filtration::scale, proj/include/ph0/filtration.hpp:28-31).  Results are bit-identical
 * to the reference on the same X.
 *
 * Plain C types only; no CUDA or torch types in any signature (`stream` is a cudaStream_t
 * passed as void*).  Every call is synchronous from the caller's view unless stated.
 */
#ifndef PH0B_H
#define PH0B_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 3: + peer-memory exchange (ph0b_shard_partition_count/recv_peer/scatter_peers, ph0b_ipc_*),
 *    ph0b_scale_to_host, ph0b_decode_packed
 * 4: + ph0b_options.n_gpus/devices (in-process multi-GPU), ph0b_scale_release,
 *    ph0b_host_cache_trim, ph0b_reduced_supports; ph0b_h0_barcode streams D like
 *    ph0b_run_host */
#define PH0B_ABI_VERSION 4u

/* Return codes.  The message of ph0b_last_error() repeats the reference's exception text
 * where the reference has one. */
#define PH0B_OK 0
#define PH0B_ERR_INVALID_ARGUMENT 1 /* std::invalid_argument in the reference */
#define PH0B_ERR_NONFINITE 2        /* "point cloud contains non-finite coordinates" (point_cloud.cpp:17) */
#define PH0B_ERR_TOO_LARGE 3        /* N above this build's limit (PH0B_MAX_POINTS) or N > 2^32-1 */
#define PH0B_ERR_CUDA 4             /* CUDA runtime / launch failure */
#define PH0B_ERR_OUT_OF_MEMORY 5    /* device or pinned-host allocation failed */
#define PH0B_ERR_NO_DEVICE 6        /* no sm_100 device visible */
#define PH0B_ERR_CAPACITY 7         /* caller-provided output buffer too small */

/* Each edge column travels through the sort as one u32: u << 16 | v for N <= 65536, the
 * u-major edge index above (K = N(N-1)/2 < 2^32 up to N = 92682).  The reference allows
 * N <= 2^32-1 (filtration.cpp:10-11) but its K x N-bit matrix cannot go past N ~ 10^4 in
 * practice; one B200 holds the whole pipeline to N = 92682 (K = 4.3e9 edges,
 * ~110 GB of keys, columns and ping-pong buffers).  PH0B_FLAG_KRUSKAL: N <= 65536. */
#define PH0B_MAX_POINTS 92682u

/* Layout of X. */
#define PH0B_COL_MAJOR 0u /* Eigen::MatrixXd storage (point_cloud.hpp:30): x(i,j) at j*N + i */
#define PH0B_ROW_MAJOR 1u /* one point per contiguous row: x(i,j) at i*d + j */

/* ph0b_options.flags */
#define PH0B_FLAG_NO_SCALE 0x1u   /* do not copy D back (n_scale is still reported) */
#define PH0B_FLAG_KRUSKAL 0x2u    /* barcode by union-find over the filtration (the reference's
                                     kruskal_barcode, oracle.cpp:32-46) instead of the column
                                     reduction; same result (acceptance.cpp:79-90) */

typedef struct ph0b_options {
    uint32_t struct_size; /* sizeof(ph0b_options); 0 = all defaults */
    int32_t device;       /* CUDA device ordinal; default 0 */
    uint32_t flags;       /* PH0B_FLAG_* */
    /* ReductionOptions (reduction.hpp:11-17): accepted for drop-in compatibility and
     * result-neutral, exactly as in the reference (pivot on/off and any worker count give
     * identical reduced matrices, reduction.hpp:35-39).  workers == 0 is rejected with the
     * reference's message "worker count must be at least 1" (reduction.cpp:134). */
    uint32_t pivoting;
    uint32_t workers;
    /* ABI 4 — multi-GPU; struct_size of an ABI-3 caller (20 bytes) still
     * works and means one GPU.  n_gpus > 1: ph0b_h0_barcode / ph0b_h0_barcode_into split the
     * cloud over that many GPUs of this node in this process — row blocks for the distances,
     * a splitter partition whose kernel stores every part straight into its destination
     * GPU's receive buffer (NVLink P2P), local sort/unique (D sharded), the column reduction
     * continuing the forest from key range to key range, D slices to the host in parallel.
     * Same results bit for bit.  PH0B_FLAG_KRUSKAL runs on one GPU. */
    uint32_t n_gpus;          /* 0 or 1: one GPU (`device`) */
    const int32_t* devices;   /* n_gpus ordinals, or NULL for device, device+1, ...; an
                                 ordinal may repeat (ranks sharing a GPU: tests) */
} ph0b_options;

/* Per-stage device milliseconds of the last run (CUDA events on the pipeline stream). */
typedef struct ph0b_stage_times {
    float distance_ms;  /* K1 tiled distance kernel                     */
    float sort_ms;      /* K2 radix sort (all passes)                   */
    float unique_ms;    /* K2c/K3 flag-and-scan unique -> D, M          */
    float reduce_ms;    /* K4 column reduction                          */
    float collect_ms;   /* K5 barcode collect                           */
    float total_ms;     /* first kernel start -> last kernel end        */
    uint32_t sort_passes;
    uint32_t reduce_rounds;
    uint64_t columns_scanned; /* edge columns streamed by the reduction */
    float sort_passes_ms;     /* the radix passes alone (sort_ms minus the digit histogram) */
    uint32_t reduce_iterations; /* parallel resolution rounds of the reduction (hook + jump) */
    uint64_t d2h_bytes;       /* host-output calls: bytes actually moved device -> host
                                 (D is shipped delta-encoded: 3-4 B per distinct length) */
} ph0b_stage_times;

/* Host-side result of ph0b_h0_barcode; arrays are owned by the library. */
typedef struct ph0b_result {
    uint64_t n_finite;        /* = Barcode::finite.size()                      */
    uint64_t* death_grade;    /* [n_finite], Interval::death_grade (1-based)   */
    double* death_length;     /* [n_finite], Interval::death_length            */
    uint64_t essential_count; /* Barcode::essential_count                      */
    uint64_t n_scale;         /* |D|                                           */
    double* scale;            /* [n_scale] D, or NULL with PH0B_FLAG_NO_SCALE  */
    ph0b_stage_times times;
} ph0b_result;

/* ---- drop-in entry point --------------------------------------------------------------
 * X (host memory) -> barcode + D (host memory, allocated by the library; free with
 * ph0b_result_free).  Replaces the five-call composition above. */
int ph0b_h0_barcode(const double* X, uint64_t n, uint64_t d, uint32_t layout,
                    const ph0b_options* opt, ph0b_result* out);

/* Replaces kruskal_barcode(build_filtration(pairwise_distances(cloud)), n)
 * (oracle.cpp:32-46, the `oracle` subcommand of ph0_cli.cpp:73-80): the same filtration on
 * the GPU, then a GPU union-find in filtration order with early stop at n-1 merges.  Equal
 * to ph0b_h0_barcode with PH0B_FLAG_KRUSKAL. */
int ph0b_kruskal_barcode(const double* X, uint64_t n, uint64_t d, uint32_t layout,
                         const ph0b_options* opt, ph0b_result* out);
void ph0b_result_free(ph0b_result* r);
/* Takes D out of a result: the caller keeps r->scale (and sets it to NULL before
 * ph0b_result_free), then hands it back here when done.  Result buffers of large D are
 * cached by the library (a freed one is reused by the next call without new page faults);
 * ph0b_host_cache_trim() returns the idle ones to the system. */
void ph0b_scale_release(double* scale);
void ph0b_host_cache_trim(void);
/* Frees what the library keeps between calls for speed: the multi-GPU runners (their
 * per-GPU contexts and buffers) and the idle result buffers.  The next call re-creates
 * what it needs. */
void ph0b_release_resources(void);

/* Same, writing into caller-provided host buffers (no allocation inside the call; pinned
 * buffers from ph0b_host_alloc give full PCIe bandwidth).  death_* need n-1 entries,
 * scale needs scale_capacity >= |D| (|D| <= n(n-1)/2) or may be NULL. */
int ph0b_h0_barcode_into(const double* X, uint64_t n, uint64_t d, uint32_t layout,
                         const ph0b_options* opt, uint64_t* death_grade, double* death_length,
                         uint64_t* n_finite, uint64_t* essential_count, double* scale,
                         uint64_t scale_capacity, uint64_t* n_scale, ph0b_stage_times* times);

/* ---- stage-level mirrors (parity surfaces for the reference's own tests) ---------------
 * pairwise_distances (filtration.cpp:8-18): lengths of all pairs u < v in u-major order. */
int ph0b_pairwise_distances(const double* X, uint64_t n, uint64_t d, uint32_t layout,
                            const ph0b_options* opt, double* lengths);

/* pairwise_distances ∘ build_filtration ∘ build_boundary_matrix (filtration.cpp:20-35,
 * boundary_matrix.cpp:15-28): column j of M in filtration order is {u[j], v[j]} at grade
 * grade[j]; scale receives D. Arrays have K = n(n-1)/2 entries (scale: >= |D|). */
int ph0b_build_filtration(const double* X, uint64_t n, uint64_t d, uint32_t layout,
                          const ph0b_options* opt, uint32_t* u, uint32_t* v, uint64_t* grade,
                          double* scale, uint64_t* n_scale);

/* Claimed low of every surviving column after reduce() — the row the reference's
 * claimed_by_ table (reduction.cpp:44-45,121) maps to it — in filtration order (n-1
 * entries).  Stronger-than-barcode parity surface. */
int ph0b_claimed_lows(const double* X, uint64_t n, uint64_t d, uint32_t layout,
                      const ph0b_options* opt, uint32_t* lows, uint64_t* n_lows);

/* The whole reduced matrix of reduce() (reduction.cpp:33-49): every column of M ends empty
 * (a cycle) or as a 2-element support {rows_lo[i], rows_hi[i]} (rows_lo < rows_hi =
 * its claimed low, reduction.cpp:44-45).  Lists the n_columns = n-1 surviving columns in
 * filtration order: columns[i] is the column index j (0-based position in the filtration);
 * all other columns are empty.  The reference compares whole reduced matrices across its
 * options (acceptance.cpp:106-133); so can a caller, against this. Arrays need n-1 entries. */
int ph0b_reduced_supports(const double* X, uint64_t n, uint64_t d, uint32_t layout,
                          const ph0b_options* opt, uint64_t* columns, uint32_t* rows_lo,
                          uint32_t* rows_hi, uint64_t* n_columns);

/* ---- device-resident path (benchmarks, multi-GPU orchestration) ----------------------- */
typedef struct ph0b_context ph0b_context;

int ph0b_context_create(int device, ph0b_context** ctx);
void ph0b_context_destroy(ph0b_context* ctx);
/* Pre-size the device workspace for clouds up to (n, d); optional. */
int ph0b_context_reserve(ph0b_context* ctx, uint64_t n, uint64_t d);
uint64_t ph0b_context_workspace_bytes(const ph0b_context* ctx);

typedef struct ph0b_device_result {
    uint64_t n_finite;
    uint64_t essential_count;
    uint64_t n_scale;
    const double* d_scale;         /* device pointer into the context workspace [n_scale] */
    const uint64_t* d_death_grade; /* device [n_finite] */
    const double* d_death_length;  /* device [n_finite] */
    ph0b_stage_times times;
} ph0b_device_result;

/* X is a DEVICE pointer (layout as above).  Outputs stay on the device, valid until the
 * next call on this context.  Blocks until done (reads back n_scale). */
int ph0b_run_device(ph0b_context* ctx, const double* dX, uint64_t n, uint64_t d,
                    uint32_t layout, void* stream, ph0b_device_result* out);

/* Host X -> host outputs through the context (reuses workspace and pinned staging). */
int ph0b_run_host(ph0b_context* ctx, const double* X, uint64_t n, uint64_t d, uint32_t layout,
                  void* stream, uint64_t* death_grade, double* death_length,
                  uint64_t* n_finite, uint64_t* essential_count, double* scale,
                  uint64_t scale_capacity, uint64_t* n_scale, ph0b_stage_times* times);

/* A device-resident D (e.g. a sharded rank's slice, or ph0b_device_result::d_scale) -> host,
 * shipped like ph0b_run_host ships it: 3/4-byte deltas per 1024-value chunk through the
 * pinned ring and decoded by the context's host threads (plain copy for small n or where
 * stream memory operations are unavailable).  Blocks until host_scale holds the exact bit
 * patterns.  *bytes_moved (optional): bytes that crossed PCIe. */
int ph0b_scale_to_host(ph0b_context* ctx, const double* d_scale, uint64_t n, double* host_scale,
                       uint64_t capacity, void* stream, uint64_t* bytes_moved);

/* ---- sharded (multi-GPU) stages: one context per rank; the caller exchanges data between
 * ranks (NCCL).  SURVEY.md §8(e); orchestration in paper_2203_02527_b200/sharded.py. ----- */
/* K1 over rows [u_lo, u_hi): their edges in u-major order, into the context workspace. */
int ph0b_shard_distances(ph0b_context* ctx, const double* dX, uint64_t n, uint64_t d,
                         uint32_t layout, uint64_t u_lo, uint64_t u_hi, void* stream,
                         uint64_t* count, uint64_t* kmin, uint64_t* kmax);
/* s evenly spaced length keys of the local edges (host), for splitter selection. */
int ph0b_shard_sample(ph0b_context* ctx, uint64_t s, uint64_t* out_host);
/* Stable partition of the local edges by parts-1 ascending splitter keys: segment j
 * (contiguous in the returned device send buffers) goes to rank j.  counts/part_min/
 * part_max: host arrays of `parts` entries; part_min/part_max bound the keys of segment j
 * ([splitter j-1, splitter j) clipped to the local key range). */
int ph0b_shard_partition(ph0b_context* ctx, const uint64_t* splitters, uint32_t parts,
                         void* stream, uint64_t** d_keys_send, uint32_t** d_vals_send,
                         uint64_t* counts, uint64_t* part_min, uint64_t* part_max);
/* Device receive buffers for `count` edges (keys u64, columns u32). */
int ph0b_shard_recv(ph0b_context* ctx, uint64_t count, uint64_t** d_keys, uint32_t** d_vals);
/* ---- exchange over peer memory (replaces partition + NCCL all-to-all-v): the partition's
 * counts only, then ONE kernel that scatters every part straight into its destination
 * rank's receive buffer (NVLink P2P stores through CUDA IPC mappings), in the same stable
 * order the all-to-all-v would deliver.  Sequence per rank: partition_count -> all-gather
 * counts -> recv_peer -> all-gather IPC handles -> open peers' handles -> scatter_peers
 * -> barrier -> sort_unique. */
/* Counts and key bounds of the stable partition (as ph0b_shard_partition, no scatter). */
int ph0b_shard_partition_count(ph0b_context* ctx, const uint64_t* splitters, uint32_t parts,
                               void* stream, uint64_t* counts, uint64_t* part_min,
                               uint64_t* part_max);
/* Receive buffers for `count` edges that peers write into (cudaMalloc bases: IPC-exportable;
 * the local edges stay intact). Synchronizes the device. */
int ph0b_shard_recv_peer(ph0b_context* ctx, uint64_t count, uint64_t** d_keys,
                         uint32_t** d_vals);
/* Scatter of the local edges: part b -> device byte addresses dst_keys[b]/dst_vals[b] (the
 * receive buffers of rank b, mapped into this process) starting at element dst_offsets[b]
 * (= edges of part b held by lower ranks).  Returns when the stores are complete. */
int ph0b_shard_scatter_peers(ph0b_context* ctx, uint32_t parts, const uint64_t* dst_keys,
                             const uint64_t* dst_vals, const uint64_t* dst_offsets,
                             void* stream);
/* CUDA IPC of receive buffers between rank processes (64-byte opaque handles). */
int ph0b_ipc_get_handle(const void* d_ptr, void* handle_out);
int ph0b_ipc_open_handle(const void* handle, void** d_ptr);
int ph0b_ipc_close(void* d_ptr);
/* Sort + unique of the received slice: local |D| and the device pointer of the D slice. */
int ph0b_shard_sort_unique(ph0b_context* ctx, uint64_t count, uint64_t kmin, uint64_t kmax,
                           void* stream, uint64_t* n_distinct, const double** d_scale,
                           uint32_t* passes);
/* Column reduction of the local slice + collect: m surviving columns in slice order, their
 * supports (u << 16 | v), grades (+ grade_offset) and lengths, as device pointers. */
int ph0b_shard_reduce(ph0b_context* ctx, uint64_t n, uint64_t count, uint64_t grade_offset,
                      void* stream, uint64_t* m, const uint32_t** d_uv,
                      const uint64_t** d_grade, const double** d_length);
/* The same, continuing the forest left by the key ranges before this one (the reference's
 * left-to-right reduction cut at range boundaries): init_labels (host, n entries; NULL:
 * singletons) are the preceding ranges' final tree labels, the reduction stops after
 * `target` surviving columns (0: n - 1), and final_labels (host, optional) receives this
 * range's final labels for the next range.  Survivors' outputs as ph0b_shard_reduce. */
int ph0b_shard_reduce_continue(ph0b_context* ctx, uint64_t n, uint64_t count,
                               uint64_t grade_offset, const uint32_t* init_labels,
                               uint32_t target, void* stream, uint64_t* m,
                               const uint32_t** d_uv, const uint64_t** d_grade,
                               const double** d_length, uint32_t* final_labels);
/* Column reduction of `count` columns given in filtration order (device supports): host
 * indices of the surviving columns, ascending. */
int ph0b_reduce_columns(ph0b_context* ctx, const uint32_t* d_uv, uint64_t count, uint64_t n,
                        void* stream, uint32_t* idx_host, uint64_t* n_out);

/* ---- utilities ------------------------------------------------------------------------ */
const char* ph0b_last_error(void);
uint32_t ph0b_abi_version(void);
/* Pinned host memory (cudaHostAlloc) for zero-staging D2H of D. */
void* ph0b_host_alloc(uint64_t bytes);
void ph0b_host_free(void* p);
/* Number of kernel launches issued by the last run on this thread (evidence counter). */
uint64_t ph0b_last_launch_count(void);

/* Synthetic clouds of the BASELINE.json configs; column-major output.
 * kind: 0 = generate_uniform_cloud(n, d, seed) exactly (point_cloud.cpp:20-29);
 *       1 = Gaussian mixture: `clusters` centres U[lo,hi]^d, isotropic sigma;
 *       2 = noisy unit circle (z=0 plane) + n_background uniform points in [lo,hi]^d (C2);
 *       3 = two equal Gaussian clusters centred at (lo,..,lo) and (hi,..,hi) (config C1).
 * All randomness is SplitMix64 (splitmix64.hpp:20-43). */
/* Replaces generate_uniform_cloud(n, dim, seed) (point_cloud.cpp:20-29) on the device: the
 * identical SplitMix64 stream (jumpable, zero draws rejected exactly as next_unit_open does),
 * written column-major into d_out (n*dim doubles, device memory) on `stream` (NULL: the
 * context's stream).  n > 0 with dim < 1 -> PH0B_ERR_INVALID_ARGUMENT, "point dimension
 * must be at least 1" (point_cloud.cpp:21-22). */
int ph0b_generate_uniform_cloud_device(ph0b_context* ctx, uint64_t n, uint64_t dim,
                                       uint64_t seed, double* d_out, void* stream);

/* Host-side decoder of a delta-encoded D stream with fixed 32-bit deltas: chunks of `chunk`
 * values, chunk j = bases[j] followed by 32-bit deltas
 * (deltas[j*chunk] unused); chunks with raw[j] != 0 are skipped (shipped uncompressed).
 * Writes out[0..n).  Exposed for callers that move D between processes the same way. */
int ph0b_decode_deltas(const uint32_t* deltas, const uint64_t* bases, const uint8_t* raw,
                       uint64_t n, uint32_t chunk, uint64_t* out);
/* The packed stream ph0b_run_host ships D in (d2h_codec.cu): chunks of `chunk` values (1024
 * on the host path), chunk j = bases[j] followed by deltas of widths[j] bytes each (3 or 4,
 * little-endian, the first one unused) at packed + offs[j]; widths[j] == 0: the chunk was
 * shipped raw and is skipped.  `packed` must have 8 readable bytes past the last chunk's
 * data.  Writes out[0..n). */
int ph0b_decode_packed(const uint8_t* packed, const uint64_t* bases, const uint8_t* widths,
                       const uint32_t* offs, uint64_t n, uint32_t chunk, uint64_t* out);

int ph0b_generate_cloud(uint32_t kind, uint64_t n, uint64_t d, uint64_t seed, uint32_t clusters,
                        double sigma, double lo, double hi, uint64_t n_background,
                        double* out_colmajor);

#ifdef __cplusplus
}
#endif

#endif /* PH0B_H */
