// Host-side launchers for the sm_100a kernels (one .cu per subsystem).  Internal header.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "colcodec.h"

namespace ph0b {

// ---- per-device launch attributes (launch_attr.cpp) -----------------------------------
// Opts `kern` into `smem` bytes of dynamic shared memory on the current device and returns
// its resident blocks per SM at `threads` threads (0 on failure).  Cached per (device,
// kernel, smem, threads); thread-safe.
int kernel_blocks_per_sm(const void* kern, int threads, size_t smem);
int device_sm_count();

// ---- K1: tiled upper-triangle distance kernel (distance.cu) ----------------------------
struct DistanceArgs {
    const double* xpad;   // device, coordinate-major [d][ldx], zero padded (ldx % 128 == 0)
    uint64_t ldx;
    uint32_t n, d;
    uint64_t* keys;       // [K] f64 length bits, u-major edge order
    uint32_t* vals;       // [K] u << 16 | v
    uint64_t* minmax;     // [2] running min / max key (init ~0 / 0)
    uint32_t* hist0;      // [256] histogram of raw key bits 0..7
    uint32_t u_lo = 0;    // rows [u_lo, u_hi) only (sharded runs); u_hi = n for all rows
    uint32_t u_hi = 0;
    uint64_t e_off = 0;   // edge index of (u_lo, u_lo+1): outputs are written at e - e_off
};
// Returns number of kernel launches issued (0 on error; check cudaGetLastError).
int launch_distance(const DistanceArgs& a, cudaStream_t s, int num_sms);

// TMA descriptor of the padded coordinate-major cloud, box {128 points, d coords}.
bool make_point_tmap(const double* xpad, uint64_t ldx, uint32_t d, CUtensorMap* map);

// Reorders a host-provided cloud into the padded coordinate-major layout.
int launch_pack_points(const double* x, uint32_t layout, uint32_t n, uint32_t d, double* xpad,
                       uint64_t ldx, uint32_t* nonfinite_flag, cudaStream_t s);

// ---- K2: onesweep LSD radix sort (radix_sort.cu) ---------------------------------------
struct SortPlan {
    uint32_t passes;      // digit passes actually executed
    uint32_t shift[8];    // bit position of each executed digit
};
struct SortArgs {
    uint64_t count;
    uint64_t kmin;              // keys are ordered by (key - kmin)
    uint64_t* keys[2];          // ping-pong
    uint32_t* vals[2];          // ping-pong (may be null: keys only)
    uint64_t* status;           // look-back status [tiles][256]
    uint32_t* hist;             // [8][256] global digit histograms (device)
    uint32_t* tile_counter;     // [8] dynamic tile ids per pass
    uint32_t epoch_base;        // look-back epoch of pass 0 (unique per pass, per call)
    uint32_t hist0_rot;         // hist row 0 is indexed (digit + rot) & 255 (raw low byte)
};
uint64_t sort_tiles(uint64_t count);
// Device check of the ATOMS lane-ordering property used by the atomic ranking; selects the
// ranking variant (atomic if it holds, bit-sliced ballots otherwise).
bool sort_self_test(cudaStream_t s);
// Runs the passes listed in plan; returns the buffer index (0/1) holding the result.
// hist[p][*] must already hold the digit-p histogram of (key-kmin) for p = 0 (the
// remaining histograms are produced by the passes themselves).
int launch_sort_passes(const SortArgs& a, const SortPlan& plan, cudaStream_t s, int num_sms,
                       int* launches);
// Histogram of digit `shift` of (key - kmin) over all keys (used when hist0 is unusable).
int launch_digit_histogram(const uint64_t* keys, uint64_t count, uint64_t kmin, uint32_t shift,
                           uint32_t* hist, cudaStream_t s, int num_sms);

// ---- K2c/K3: flag-and-scan unique -> D, and boundary matrix grades (unique.cu) ----------
struct UniqueArgs {
    uint64_t* keys;         // sorted raw keys (f64 length bits); runs fixed up in place
    uint32_t* vals;         // columns (u << 16 | v), permuted with the keys
    uint64_t count;
    uint64_t kmin;
    uint32_t low_bits;      // keys are sorted by (key - kmin) >> low_bits only (0 = fully)
    double* scale;          // out: D
    uint32_t* grade;        // out (optional): 1-based grade per column
    uint64_t* n_scale;      // out: |D| (device)
    uint32_t* redo;         // out: set when a run exceeded the in-place fix-up limit
    uint64_t* scratch;      // unique_scratch_words(count) words
    const uint64_t* d_base = nullptr;  // device: D index of this range's first distinct length
};
// Returns launches, or -1 when the kernels cannot be configured on this device.
int launch_unique(const UniqueArgs& a, cudaStream_t s);
uint64_t unique_scratch_words(uint64_t count);

// ---- K4: GPU column reduction (reduce.cu) ----------------------------------------------
struct ReduceState {
    uint32_t n;
    uint64_t k;
    const uint32_t* uv;      // sorted columns (u << 16 | v), filtration order
    uint32_t* comp;          // [n] component label (root)
    uint32_t* best;          // [2n]: per-root minimum candidate column | hook parent
    uint32_t* cand[2];       // candidate column ids (capacity cap)
    uint64_t cap;
    uint32_t* surv;          // [n] survivor column ids (unordered)
    uint32_t* counters;      // [8] device counters (see reduce.cu)
    uint64_t* scan_status;   // look-back status for ordered compaction
    uint32_t* scan_tile_counter;
    uint32_t* pair_min;      // [kPairMax] sparse phase
    uint8_t* cid;            // [n] compact component ids (sparse phase)
    uint32_t* host_counters;   // zero-copy host mirror [8] ...
    uint32_t* mapped_counters; // ... and its device alias (written by k4_publish)
};
struct ReduceStats {
    uint32_t rounds = 0;
    uint32_t iterations = 0;
    uint64_t scanned = 0;     // columns streamed
    uint32_t survivors = 0;
    int launches = 0;
};
// Runs the full reduction; leaves survivor column ids (unordered) in st.surv and the final
// tree labels in st.comp.  init_comp (device, optional): labels left by the reduction of the
// preceding part of the filtration (a continued forest); target: stop after this many
// survivors (0: n - 1).
int run_reduction(ReduceState& st, cudaStream_t s, int num_sms, uint32_t& epoch,
                  ReduceStats* stats, const uint32_t* init_comp = nullptr,
                  uint32_t target = 0);

// ---- K9: compressed D for the host path (d2h_codec.cu) ----------------------------------
// Packed stream of the slice [lohi[0], lohi[1]) of d (device words; n_upper >= its length):
// kPackChunk-value chunks of 3- or 4-byte deltas (width 0 = raw: not in the stream), the
// chunks' bases, widths, absolute byte offsets (device) and offsets within their piece of
// piece_chunks chunks; piece_off[p] = byte offset of piece p, piece_off[#pieces] = total
// (mapped host memory: the host sizes the copies from it).  Returns launches.
constexpr int kPackChunk = 1024;
int launch_d2h_pack_bucket(const double* d, const uint64_t* lohi, uint64_t n_upper,
                           uint64_t* bases, uint8_t* widths, uint64_t* offs, uint32_t* poff,
                           uint64_t* piece_off, uint32_t piece_chunks, uint8_t* out,
                           cudaStream_t s);

// ---- K8: on-device generate_uniform_cloud (generate.cu) --------------------------------
// returns launches (>0), -1 on a CUDA error, -2 if more than 64 zero draws were met
int launch_uniform_cloud(uint64_t n, uint64_t dim, uint64_t seed, double* d_out,
                         unsigned long long* d_zeros, unsigned long long* h_zeros,
                         cudaStream_t s, int num_sms);

// ---- K6: GPU Kruskal oracle (kruskal.cu) ----------------------------------------------
size_t kruskal_smem_bytes();
int launch_kruskal(const uint32_t* uv, const uint64_t* sorted_keys, uint64_t count, uint32_t n,
                   const double* D, const uint64_t* n_scale, uint32_t* accepted,
                   uint32_t* n_accepted, uint64_t* death_grade, double* death_length,
                   cudaStream_t s);

// ---- K5: barcode collect (collect.cu) --------------------------------------------------
// cols_sorted: survivor column ids in filtration order (u64, from the keys-only sort).
// Writes surv_sorted (u32), death_grade = 1 + lower_bound(D, length), death_length.
int launch_collect_map(const uint64_t* cols_sorted, uint32_t m, const uint64_t* sorted_keys,
                       const double* scale, const uint64_t* n_scale, uint64_t grade_offset,
                       uint32_t* surv_sorted, uint64_t* death_grade, double* death_length,
                       cudaStream_t s);
int launch_widen(const uint32_t* in, uint32_t m, uint64_t* out, cudaStream_t s);
int launch_narrow(const uint64_t* in, uint32_t m, uint32_t* out, cudaStream_t s);

// Reduced supports {xs[i], lows[i]} of the survivors in filtration order (reduction.cpp:33-49)
// and their claimed lows (reduction.cpp:44-45), replaying the reference's column additions
// over the survivors; xs may be null; *err = 1 if a survivor emptied (internal error);
// scratch: n u32 of device memory (used above N = 65536).
int launch_reduced_supports(const uint32_t* surv_sorted, uint32_t m, const uint32_t* uv,
                            uint32_t n, uint32_t* xs, uint32_t* lows, uint32_t* err,
                            uint32_t* scratch, cudaStream_t s);

// ---- multi-GPU splitter partition (shard.cu) ---------------------------------------------
int launch_partition(const uint64_t* keys, const uint32_t* vals, uint64_t count,
                     const uint64_t* d_splitters, uint32_t parts, uint32_t* d_counts_scratch,
                     uint64_t* d_totals, uint64_t* d_bminmax, uint64_t* keys_out,
                     uint32_t* vals_out, cudaStream_t s, uint32_t align, uint64_t kmin,
                     uint64_t kmax, const uint64_t* h_splitters, uint16_t* d_table);
size_t partition_table_bytes();  // device scratch for the bucket lookup table
// The same in phases: counts + scan + layout (segment starts, padding, key bounds); optional
// early extraction of one segment; the scatter of every other segment.
int launch_partition_count(const uint64_t* keys, uint64_t count, const uint64_t* d_splitters,
                           uint32_t parts, uint32_t* d_counts_scratch, uint64_t* d_totals,
                           uint64_t* d_bminmax, uint64_t* keys_out, uint32_t* vals_out,
                           cudaStream_t s, uint32_t align, uint64_t kmin, uint64_t kmax,
                           const uint64_t* h_splitters, uint16_t* d_table,
                           uint32_t pad_val = 0);
int launch_partition_select(const uint64_t* keys, const uint32_t* vals, uint64_t count,
                            uint32_t parts, uint32_t bucket, const uint32_t* d_counts_scratch,
                            const uint64_t* d_totals, const uint64_t* d_bminmax,
                            uint64_t* keys_out, uint32_t* vals_out, cudaStream_t s);
// pad_val: the cycle column of this N (col_cycle, colcodec.h) in the padding slots
int launch_partition_pad(const uint64_t* d_totals, uint32_t parts, uint32_t align,
                         uint64_t* keys, uint32_t* vals, cudaStream_t s, uint32_t pad_val = 0);
int launch_partition_scatter(const uint64_t* keys, const uint32_t* vals, uint64_t count,
                             const uint64_t* d_splitters, uint32_t parts,
                             const uint32_t* d_counts_scratch, const uint64_t* d_totals,
                             uint64_t* keys_out, uint32_t* vals_out, cudaStream_t s,
                             uint64_t kmin, uint64_t kmax, const uint16_t* d_table,
                             uint32_t skip_bucket, const uint64_t* d_peer_k = nullptr,
                             const uint64_t* d_peer_v = nullptr);
uint64_t partition_scratch_words(uint64_t count, uint32_t parts);
int launch_sample(const uint64_t* keys, uint64_t count, uint64_t s, uint64_t* out, cudaStream_t st);
int launch_gather_u32(const uint32_t* src, const uint32_t* idx, uint64_t m, uint32_t* out,
                      cudaStream_t st);

}  // namespace ph0b
