// Host-side pipeline context (device workspace, streams, orchestration).  Internal header.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ph0b.h"
#include "host_decode.h"
#include "kernels.h"

namespace ph0b {

// NVTX range over a host-side stage (visible in Nsight Systems / ncu --nvtx; no-op unless a
// tool is attached).
struct NvtxRange {
    explicit NvtxRange(const char* name);
    ~NvtxRange();
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

struct Status {
    int code = PH0B_OK;
    std::string msg;
    static Status ok() { return {}; }
    bool good() const { return code == PH0B_OK; }
};

enum class StopAfter { Distance, Filtration, Barcode };

struct RunOutputs {
    // device pointers into the workspace after a run
    const uint64_t* d_lengths_umajor = nullptr;  // StopAfter::Distance (bits)
    const uint32_t* d_uv_sorted = nullptr;       // >= Filtration
    const uint32_t* d_grade = nullptr;           // Filtration with want_grade
    const double* d_scale = nullptr;             // >= Filtration
    const uint64_t* d_death_grade = nullptr;     // Barcode
    const double* d_death_length = nullptr;
    const uint32_t* d_surv_sorted = nullptr;
    uint64_t k = 0;
    uint64_t n_scale = 0;
    uint64_t n_finite = 0;
    uint64_t essential = 0;
    ph0b_stage_times times{};
};

class Context {
public:
    explicit Context(int device);
    ~Context();
    Status init();
    Status reserve(uint64_t n, uint64_t d);
    uint64_t workspace_bytes() const { return bytes_; }

    // Runs the pipeline on a device-resident cloud.
    Status run(const double* dX, uint64_t n, uint64_t d, uint32_t layout, cudaStream_t stream,
               StopAfter stop, bool want_grade, RunOutputs* out);
    // Host cloud -> device staging buffer, then run().
    Status run_host_input(const double* X, uint64_t n, uint64_t d, uint32_t layout,
                          cudaStream_t stream, StopAfter stop, bool want_grade, RunOutputs* out);
    // Reduced supports {xs, lows} of the survivors (filtration order) into lows_buffer():
    // lows at [0, n), xs at [n, 2n) when want_x.
    Status reduced_supports(const RunOutputs& r, uint32_t n, bool want_x, cudaStream_t stream);

    // ---- pipeline stages (single-GPU run() composes them; sharded runs call them) ------
    Status stage_distances(const double* dX, uint64_t n, uint64_t d, uint32_t layout,
                           uint64_t u_lo, uint64_t u_hi, cudaStream_t st, uint64_t* count,
                           uint64_t* kmin, uint64_t* kmax);
    Status stage_sort_unique(uint64_t count, uint64_t kmin, uint64_t kmax, bool raw_hist,
                             bool want_grade, cudaStream_t st, uint32_t* passes, int src = 0);
    // init_comp/target: continue the forest of a preceding part of the filtration (device
    // labels, this device) and stop after `target` survivors (see run_reduction)
    Status stage_reduce(const uint32_t* uv, uint64_t count, uint32_t n, cudaStream_t st,
                        ReduceStats* rst, const uint32_t* init_comp = nullptr,
                        uint32_t target = 0);
    uint32_t* comp() { return comp_; }
    // Sort (kb0, vb0) of k edges (ping-pong with kb1/vb1) and write its distinct lengths to
    // scale_out (null: the free key buffer) starting at *d_base (null: 0); *d_count receives
    // base + |D|.  *res: 0/1 = buffer holding the sorted data.
    Status sort_unique_range(uint64_t* kb0, uint32_t* vb0, uint64_t* kb1, uint32_t* vb1,
                             uint64_t k, uint64_t kmin, uint64_t kmax, bool raw_hist,
                             double* scale_out, const uint64_t* d_base, uint64_t* d_count,
                             uint32_t* grade_out, cudaStream_t st, int* res, uint32_t* passes,
                             const std::function<Status()>* after_enqueue = nullptr);
    // Host-output run with the D2H of D overlapped with the sort: edges are split into
    // key-range buckets (one stable partition pass), each bucket is sorted + deduplicated
    // in turn and its slice of D streams to the host while the next bucket sorts.
    Status run_host_overlapped_impl(const double* X, uint64_t n, uint64_t d, uint32_t layout,
                                    cudaStream_t stream, double* host_scale,
                                    uint64_t scale_capacity, RunOutputs* out);
    Status run_host_overlapped(const double* X, uint64_t n, uint64_t d, uint32_t layout,
                               cudaStream_t st, double* host_scale, uint64_t scale_capacity,
                               RunOutputs* out);
    Status stage_collect(uint32_t m, uint64_t count, uint64_t grade_offset, cudaStream_t st);
    // Barcode by the GPU union-find (Kruskal) over the sorted columns instead of K4 + K5.
    Status stage_kruskal(uint64_t count, uint32_t n, cudaStream_t st, uint32_t* merges);
    bool kruskal_mode = false;  // set by the C entry points (under mu) for one run
    Status reserve_edges(uint64_t count);  // ping-pong key/column buffers for count edges
    Status reserve_points(uint64_t n, uint64_t d);
    // sharded receive side: one ping-pong buffer only (0: NCCL path, whose send data sits in
    // buffer 1; 1: peer-memory exchange, while the local scatter still reads buffer 0)
    Status reserve_recv(uint64_t count, int buffer = 0);
    Status sort_survivors(uint32_t m, uint64_t count, cudaStream_t st);
    // workspace accessors for the sharded C entry points
    uint64_t* keys(int i) { return keys_[i]; }
    uint32_t* vals(int i) { return vals_[i]; }
    int cur() const { return cur_; }
    double* scale() { return scale_; }
    uint64_t* small_dev() { return small_; }
    uint64_t* small_host() { return h_small_; }
    uint32_t* surv() { return surv_; }
    uint32_t* surv_sorted() { return surv_sorted_; }
    uint64_t* death_grade() { return death_grade_; }
    double* death_length() { return death_length_; }
    uint32_t* hist() { return hist_; }
    uint64_t* status() { return status_; }
    uint32_t* counters() { return counters_; }
    int num_sms() const { return num_sms_; }
    uint32_t epochs(uint32_t count, cudaStream_t s) { return next_epochs(count, s); }
    uint32_t* lows_buffer() { return lows_; }

    // host threads decoding this context's D stream (0: cores - 1); set before the first
    // host-output call (several contexts of one process share the cores)
    void set_decode_threads(unsigned t) { decode_threads_ = t; }
    // or share one pool between contexts (the multi-GPU path: the ranks' D slices stream at
    // the same time; each rank's pieces stay in submission order, so no piece waits on a
    // piece queued behind it)
    void set_decode_pool(std::shared_ptr<DecodePool> p) { pool_ = std::move(p); }

    std::mutex mu;
    int device() const { return device_; }
    cudaStream_t own_stream() const { return stream_; }
    uint64_t launches = 0;

private:
    Status grow(void** p, uint64_t* cap_bytes, uint64_t need_bytes);
    unsigned decode_threads_ = 0;
    uint32_t next_epochs(uint32_t count, cudaStream_t s);

    int device_;
    int num_sms_ = 148;
    cudaStream_t stream_ = nullptr;
    cudaEvent_t ev_[9] = {};  // [6]: per-bucket completion, [7]: redo check, [8]: passes start
    uint64_t bytes_ = 0;

    // workspace (capacities in bytes)
    double* xin_ = nullptr;        uint64_t xin_cap_ = 0;
    double* xpad_ = nullptr;       uint64_t xpad_cap_ = 0;
    uint64_t* keys_[2] = {};       uint64_t keys_cap_[2] = {};
    uint32_t* vals_[2] = {};       uint64_t vals_cap_[2] = {};
    uint64_t* status_ = nullptr;   uint64_t status_cap_ = 0;
    uint32_t* grade_ = nullptr;    uint64_t grade_cap_ = 0;
    uint32_t* comp_ = nullptr;     uint64_t comp_cap_ = 0;
    uint32_t* best_ = nullptr;     uint64_t best_cap_ = 0;
    uint32_t* surv_ = nullptr;     uint64_t surv_cap_ = 0;
    uint32_t* surv_sorted_ = nullptr; uint64_t surv_sorted_cap_ = 0;
    uint32_t* lows_ = nullptr;     uint64_t lows_cap_ = 0;
    uint32_t* cand_[2] = {};       uint64_t cand_cap_[2] = {};
    uint64_t* survkeys_[2] = {};   uint64_t survkeys_cap_[2] = {};
    uint64_t* death_grade_ = nullptr; uint64_t death_grade_cap_ = 0;
    double* death_length_ = nullptr;  uint64_t death_length_cap_ = 0;
    uint64_t* uscratch_ = nullptr; uint64_t uscratch_cap_ = 0;
    double* dbuf_ = nullptr;       uint64_t dbuf_cap_ = 0;        // D (overlapped host path)
    // compressed D for the host path: device deltas/chunk bases/raw flags, pinned mirrors
    uint32_t* d_delta_ = nullptr;  uint64_t d_delta_cap_ = 0;
    uint64_t* d_cbase_ = nullptr;  uint64_t d_cbase_cap_ = 0;
    uint8_t* d_craw_ = nullptr;    uint64_t d_craw_cap_ = 0;
    // streamed D2H ring: pinned slots the copy engine fills and the decode pool drains; ring
    // flags in mapped host memory ([0,256) ready, [256,512) freed, by slot)
    uint32_t* h_ring_ = nullptr;   uint64_t h_ring_cap_ = 0;
    uint32_t* h_ringflags_ = nullptr;
    uint32_t* d_ringflags_ = nullptr;
    uint64_t ring_seq_ = 0;
    std::atomic<uint64_t> ring_done_[256] = {};  // per slot: decode tasks completed (monotone)
    // ring geometry (1024-value chunks per piece, slots) of this call, and its per-context
    // choice between the two measured geometries (ring_geometry(), pipeline.cpp)
    uint32_t ring_g_ = 0, ring_r_ = 0;
    int ring_calls_ = 0, ring_pick_ = -1;
    uint64_t ring_tune_k_ = 0, ring_tune_d_ = 0;
    double ring_ms_[2] = {0.0, 0.0};
    void set_ring_geometry(uint32_t g, uint32_t r);
    int ring_choice(uint64_t k);
    void ring_record(uint64_t k, uint64_t n_scale, double ms);
    cudaEvent_t enc_ev_ = nullptr;
    std::vector<cudaStream_t> ring_streams_;  // [0] = copy_stream_
    Status ensure_ring();
    Status prepare_stream(uint64_t k, uint32_t buckets);
    Status enqueue_stream(uint64_t cbase, uint64_t nch, const std::vector<uint64_t>& poffs,
                          const uint8_t* d_src, const volatile uint64_t* bounds,
                          cudaEvent_t meta_ev, double* host_scale, uint64_t capacity,
                          volatile int* overflow, uint64_t* moved, uint64_t* enq_ns);
  public:
    // D (device, n values) -> host_scale through the compressed ring (one slice); *moved =
    // bytes that crossed PCIe.  Requires stream_memops_ok().
    Status stream_scale(const double* d_scale, uint64_t n, double* host_scale, uint64_t capacity,
                        cudaStream_t st, uint64_t* moved);
    // the compressed D stream is available (PH0B_D2H_COMPRESS != 0 and stream memory
    // operations on mapped host memory work here; probed once)
    bool compressed_d2h_ok();
  private:
    bool stream_memops_ok();
    int memops_probe_ = 0;    // 0 = not probed, 1 = ok, -1 = unavailable
    uint64_t* h_cbase_ = nullptr;  uint64_t h_cbase_cap_ = 0;
    uint64_t* d_coff_ = nullptr;   uint64_t d_coff_cap_ = 0;    // packed: chunk byte offsets
    uint32_t* d_cpoff_ = nullptr;  uint64_t d_cpoff_cap_ = 0;   // packed: offsets in the piece
    uint32_t* h_cpoff_ = nullptr;  uint64_t h_cpoff_cap_ = 0;
    uint64_t* h_pieceoff_ = nullptr;  uint64_t* d_pieceoff_ = nullptr;  // mapped
    uint64_t h_pieceoff_cap_ = 0;
    uint8_t* h_craw_ = nullptr;    uint64_t h_craw_cap_ = 0;
    std::shared_ptr<DecodePool> pool_;
    std::vector<cudaEvent_t> bucket_ev_;
    Status grow_host(void** p, uint64_t* cap, uint64_t need);
    uint32_t* part_counts_ = nullptr; uint64_t part_counts_cap_ = 0;
    uint64_t* part_small_ = nullptr;  uint64_t part_small_cap_ = 0;
    cudaStream_t copy_stream_ = nullptr;
    // fixed small buffers
    uint32_t* hist_ = nullptr;     // [8][256]
    uint32_t* counters_ = nullptr; // [64]
    uint64_t* small_ = nullptr;    // [0..1] minmax, [2] n_scale, [3] nonfinite flag (u32)
    uint64_t* h_small_ = nullptr;  // pinned mirror of small_
    uint32_t* h_counters_ = nullptr;  // pinned [64]
    uint64_t* h_mapped_ = nullptr;    // mapped pinned [256] (zero-copy flags / offsets)
    uint64_t* d_mapped_ = nullptr;    // device alias of h_mapped_
    uint32_t epoch_ = 1;
    bool status_zeroed_ = false;
    bool atomic_rank_ok_ = false;
    int cur_ = 0;              // ping-pong index holding the sorted keys/columns
    int surv_sorted_idx_ = 0;  // survkeys_ index holding the sorted survivor ids
    double* scale_ = nullptr;  // D of the last sort_unique stage
    uint64_t xpad_ld_ = 128, xpad_d_ = 0;
    bool hist_valid_ = false;  // hist_ row 0 holds the raw low-byte histogram of keys_[0]
};

void shard_scratch_release(Context* c);  // shard_capi.cpp

// Default per-device contexts used by the stateless C entry points.
Context* default_context(int device, Status* st);

}  // namespace ph0b
