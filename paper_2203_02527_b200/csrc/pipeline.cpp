// Host orchestration of the B200 H0 pipeline: workspace management and the stage order of
// proj/src/bench.cpp:45-59 (distances -> filtration -> matrix -> reduce -> barcode).
#include "pipeline.h"

#include <cuda.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <thread>
#include <vector>

#include "kernels.h"

namespace ph0b {
namespace {

constexpr uint64_t kCandCap = 1ull << 25;  // reduction candidate buffer (columns)

Status cuda_fail(cudaError_t e, const char* what) {
    Status s;
    s.code = (e == cudaErrorMemoryAllocation) ? PH0B_ERR_OUT_OF_MEMORY : PH0B_ERR_CUDA;
    s.msg = std::string(what) + ": " + cudaGetErrorString(e);
    return s;
}

#define PH0B_TRY(expr, what)                                         \
    do {                                                             \
        const cudaError_t e_ = (expr);                               \
        if (e_ != cudaSuccess) return cuda_fail(e_, what);           \
    } while (0)

#define PH0B_CHECK_LAUNCH(what)                                      \
    do {                                                             \
        const cudaError_t e_ = cudaGetLastError();                   \
        if (e_ != cudaSuccess) return cuda_fail(e_, what);           \
    } while (0)

inline uint32_t span_passes(uint64_t span, SortPlan* plan) {
    const uint32_t bits = span ? 64u - (uint32_t)__builtin_clzll(span) : 0u;
    plan->passes = (bits + 7) / 8;
    for (uint32_t p = 0; p < plan->passes; ++p) plan->shift[p] = 8 * p;
    return plan->passes;
}

// Radix plan over the top 8*max_passes bits of the key span; returns the number of low
// bits left unsorted (fixed up per equal-prefix run by the unique kernel).
inline uint32_t truncated_plan(uint64_t span, uint32_t max_passes, SortPlan* plan) {
    const uint32_t bits = span ? 64u - (uint32_t)__builtin_clzll(span) : 0u;
    uint32_t passes = (bits + 7) / 8, low = 0;
    if (passes > max_passes) {
        passes = max_passes;
        low = bits - 8 * passes;
    }
    plan->passes = passes;
    for (uint32_t p = 0; p < passes; ++p) plan->shift[p] = low + 8 * p;
    return low;
}

// PH0B_TRACE=1: host-side timeline of the overlapped host path on stderr (diagnostics only).
struct Trace {
    bool on;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    Trace() {
        const char* e = getenv("PH0B_TRACE");
        on = e && e[0] == '1';
    }
    void mark(const char* what, long a = -1) {
        if (!on) return;
        const double ms = std::chrono::duration<double, std::milli>(
                              std::chrono::steady_clock::now() - t0).count();
        if (a >= 0)
            fprintf(stderr, "[ph0b trace] %8.2f ms %s %ld\n", ms, what, a);
        else
            fprintf(stderr, "[ph0b trace] %8.2f ms %s\n", ms, what);
    }
};

bool d2h_compress() {
    static const bool v = [] {
        const char* e = getenv("PH0B_D2H_COMPRESS");
        return !(e && e[0] == '0');
    }();
    return v;
}

uint64_t d2h_chunk_elems() {
    static const uint64_t v = [] {
        const char* e = getenv("PH0B_D2H_CHUNK_MB");
        const uint64_t mb = e ? (uint64_t)atoll(e) : 32;
        return (mb ? mb : 32) << 17;  // MiB -> f64 elements
    }();
    return v;
}

// Streamed D2H ring of the compressed host path: slots of packed 1024-value chunks, filled on
// PH0B_RING_STREAMS copy streams (default 2) and decoded by PH0B_RING_SUBTASKS pool tasks per
// piece (default 32); a ring of tens of MiB replaces a k*4-byte pinned staging buffer (8.6 GB
// at C5).  Two geometries, chosen per context by measurement (ring_choice()): 10 slots of
// 8 MiB pieces (2048 chunks) and 16 slots of 2 MiB pieces (512 chunks).  Which one is faster
// depends on the box (C5 e2e, tools/box_probe.sh, same CPU model, L3 and host-memory
// bandwidth everywhere): on most boxes of the pool 16 x 2 MiB gives 224-228 ms against
// 237-267 ms, on others 10 x 8 MiB gives 184-194 ms against 225-227.  PH0B_RING_CHUNKS /
// PH0B_RING_SLOTS fix a geometry (tools/ring_sweep.sh), PH0B_RING_TUNE=0 fixes the first.
constexpr uint32_t kRingGeom[2][2] = {{2048, 10}, {512, 16}};  // {chunks per piece, slots}

int env_ring(const char* name, int lo, int hi) {  // 0 = unset
    const char* e = getenv(name);
    if (!e) return 0;
    const int x = atoi(e);
    return x < lo ? lo : (x > hi ? hi : x);
}

bool ring_fixed() {
    static const bool v = env_ring("PH0B_RING_CHUNKS", 1, 16384) ||
                          env_ring("PH0B_RING_SLOTS", 2, 256) ||
                          (getenv("PH0B_RING_TUNE") && getenv("PH0B_RING_TUNE")[0] == '0');
    return v;
}

uint64_t ring_slot_bytes(uint32_t g) {  // a piece at 4 bytes per value + slack for the decoder
    return (uint64_t)g * kPackChunk * 4 + 128;
}

uint32_t ring_subtasks() {
    static const uint32_t v = [] {
        const char* e = getenv("PH0B_RING_SUBTASKS");
        const int x = e ? atoi(e) : 32;
        return (uint32_t)(x < 1 ? 1 : (x > 256 ? 256 : x));
    }();
    return v;
}

// Stream memory operations (driver API, resolved through the runtime): the copy stream
// waits for a slot to be released by the host decoder, and flags a slot as filled, without
// any CUDA call from the decoder threads.
using StreamValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
StreamValueFn stream_fn(const char* name) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return reinterpret_cast<StreamValueFn>(fn);
}

bool stream_wait_u32(cudaStream_t s, uint64_t dptr, uint32_t value) {
    static const StreamValueFn fn = stream_fn("cuStreamWaitValue32");
    return fn && fn(reinterpret_cast<CUstream>(s), (CUdeviceptr)dptr, value,
                    CU_STREAM_WAIT_VALUE_EQ) == CUDA_SUCCESS;
}

bool stream_write_u32(cudaStream_t s, uint64_t dptr, uint32_t value) {
    static const StreamValueFn fn = stream_fn("cuStreamWriteValue32");
    return fn && fn(reinterpret_cast<CUstream>(s), (CUdeviceptr)dptr, value,
                    CU_STREAM_WRITE_VALUE_DEFAULT) == CUDA_SUCCESS;
}

uint32_t max_sort_passes() {
    static const uint32_t v = [] {
        const char* e = getenv("PH0B_MAX_PASSES");
        const int x = e ? atoi(e) : 5;
        return (uint32_t)(x < 1 ? 1 : (x > 8 ? 8 : x));
    }();
    return v;
}

}  // namespace

NvtxRange::NvtxRange(const char* name) { nvtxRangePushA(name); }
NvtxRange::~NvtxRange() { nvtxRangePop(); }

Context::Context(int device) : device_(device) {}

Context::~Context() {
    // (a context whose init() failed may name an invalid device: leave no error behind for
    // the next, unrelated CUDA call of this thread to report)
    if (cudaSetDevice(device_) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    void* ps[] = {xin_,  xpad_, keys_[0], keys_[1], vals_[0], vals_[1], status_,
                  grade_, comp_, best_, surv_, surv_sorted_, lows_, cand_[0], cand_[1],
                  survkeys_[0], survkeys_[1], death_grade_, death_length_, hist_, counters_,
                  small_, uscratch_, dbuf_, part_counts_, part_small_, d_delta_, d_cbase_,
                  d_craw_};
    for (void* p : ps)
        if (p) cudaFree(p);
    pool_.reset();
    for (void* p : {(void*)h_ring_, (void*)h_ringflags_, (void*)h_cbase_, (void*)h_craw_,
                    (void*)h_cpoff_, (void*)h_pieceoff_})
        if (p) cudaFreeHost(p);
    for (void* p : {(void*)d_coff_, (void*)d_cpoff_})
        if (p) cudaFree(p);
    if (enc_ev_) cudaEventDestroy(enc_ev_);
    for (auto& e : bucket_ev_)
        if (e) cudaEventDestroy(e);
    if (h_small_) cudaFreeHost(h_small_);
    if (h_counters_) cudaFreeHost(h_counters_);
    if (h_mapped_) cudaFreeHost(h_mapped_);
    for (size_t i = 1; i < ring_streams_.size(); ++i) cudaStreamDestroy(ring_streams_[i]);
    if (copy_stream_) cudaStreamDestroy(copy_stream_);
    for (auto& e : ev_)
        if (e) cudaEventDestroy(e);
    if (stream_) cudaStreamDestroy(stream_);
    cudaGetLastError();
}

Status Context::init() {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count <= device_ || device_ < 0) {
        cudaGetLastError();
        return {PH0B_ERR_NO_DEVICE, "no CUDA device " + std::to_string(device_) + " visible"};
    }
    PH0B_TRY(cudaSetDevice(device_), "cudaSetDevice");
    cudaDeviceProp prop;
    PH0B_TRY(cudaGetDeviceProperties(&prop, device_), "cudaGetDeviceProperties");
    if (prop.major != 10) {
        return {PH0B_ERR_NO_DEVICE, std::string("device ") + prop.name +
                                        " is not sm_100 (this build targets sm_100a only)"};
    }
    num_sms_ = prop.multiProcessorCount;
    PH0B_TRY(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    for (auto& e : ev_) PH0B_TRY(cudaEventCreate(&e), "cudaEventCreate");
    PH0B_TRY(cudaMalloc(&hist_, sizeof(uint32_t) * 8 * 256), "cudaMalloc hist");
    PH0B_TRY(cudaMalloc(&counters_, sizeof(uint32_t) * 64), "cudaMalloc counters");
    PH0B_TRY(cudaMalloc(&small_, sizeof(uint64_t) * 8), "cudaMalloc small");
    PH0B_TRY(cudaHostAlloc(&h_small_, sizeof(uint64_t) * 8, cudaHostAllocDefault), "cudaHostAlloc");
    PH0B_TRY(cudaHostAlloc(&h_counters_, sizeof(uint32_t) * 64, cudaHostAllocDefault),
             "cudaHostAlloc");
    // Zero-copy host words for per-bucket results (D offsets, redo flag): kernels write them
    // over PCIe directly, so the host never queues a small D2H behind a large one.
    PH0B_TRY(cudaHostAlloc(&h_mapped_, sizeof(uint64_t) * 256, cudaHostAllocMapped),
             "cudaHostAlloc mapped");
    PH0B_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_mapped_), h_mapped_, 0),
             "cudaHostGetDevicePointer");
    bytes_ += 8 * 256 * 4 + 64 * 4 + 64;
    atomic_rank_ok_ = sort_self_test(stream_);
    return Status::ok();
}

Status Context::ensure_ring() {
    const uint64_t need = (uint64_t)ring_r_ * ring_slot_bytes(ring_g_);
    Status s = grow_host(reinterpret_cast<void**>(&h_ring_), &h_ring_cap_, need);
    if (!s.good()) return s;
    if (!h_ringflags_) {
        // [0, 256) ready, [256, 512) freed; slot generations start at 1, so 0 = never used
        PH0B_TRY(cudaHostAlloc(&h_ringflags_, 512 * 4, cudaHostAllocMapped), "cudaHostAlloc mapped");
        std::memset(h_ringflags_, 0, 512 * 4);
        PH0B_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_ringflags_), h_ringflags_, 0),
                 "cudaHostGetDevicePointer");
        ring_seq_ = 0;
    }
    return Status::ok();
}

bool Context::compressed_d2h_ok() { return d2h_compress() && stream_memops_ok(); }

bool Context::stream_memops_ok() {
    if (memops_probe_ == 0) {
        memops_probe_ = -1;
        uint32_t* h = nullptr;
        uint32_t* dp = nullptr;
        cudaStream_t s = nullptr;
        if (cudaHostAlloc(reinterpret_cast<void**>(&h), 8, cudaHostAllocMapped) == cudaSuccess &&
            cudaHostGetDevicePointer(reinterpret_cast<void**>(&dp), h, 0) == cudaSuccess &&
            cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess) {
            h[0] = 7;
            h[1] = 0;
            const uint64_t d0 = reinterpret_cast<uint64_t>(dp);
            if (stream_wait_u32(s, d0, 7) && stream_write_u32(s, d0 + 4, 42) &&
                cudaStreamSynchronize(s) == cudaSuccess &&
                __atomic_load_n(&h[1], __ATOMIC_ACQUIRE) == 42)
                memops_probe_ = 1;
        }
        if (s) cudaStreamDestroy(s);
        if (h) cudaFreeHost(h);
        cudaGetLastError();
    }
    return memops_probe_ == 1;
}

Status Context::grow_host(void** p, uint64_t* cap, uint64_t need) {
    if (need <= *cap) return Status::ok();
    if (*p) cudaFreeHost(*p);
    *p = nullptr;
    *cap = 0;
    need = (need + 4095) & ~4095ull;
    const cudaError_t e = cudaHostAlloc(p, need, cudaHostAllocDefault);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return {PH0B_ERR_OUT_OF_MEMORY, "pinned host allocation of " + std::to_string(need) +
                                            " bytes failed (" + cudaGetErrorString(e) + ")"};
    }
    *cap = need;
    return Status::ok();
}

Status Context::grow(void** p, uint64_t* cap, uint64_t need) {
    if (need <= *cap) return Status::ok();
    if (*p) {
        cudaFree(*p);
        bytes_ -= *cap;
        *p = nullptr;
        *cap = 0;
    }
    need = (need + 255) & ~255ull;
    const cudaError_t e = cudaMalloc(p, need);
    if (e != cudaSuccess) {
        cudaGetLastError();
        Status s;
        s.code = PH0B_ERR_OUT_OF_MEMORY;
        s.msg = "device allocation of " + std::to_string(need) + " bytes failed (" +
                cudaGetErrorString(e) + ")";
        return s;
    }
    *cap = need;
    bytes_ += need;
    return Status::ok();
}

Status Context::reserve_points(uint64_t n, uint64_t d) {
    PH0B_TRY(cudaSetDevice(device_), "cudaSetDevice");
    const uint64_t ldx = std::max<uint64_t>(128, (n + 127) / 128 * 128);
    const uint64_t status_words = sort_tiles(n + 1) * 256;
    Status s;
#define G(ptr, cap, bytes)                                                    \
    if (!(s = grow(reinterpret_cast<void**>(&(ptr)), &(cap), (bytes))).good()) return s;
    G(xin_, xin_cap_, std::max<uint64_t>(8, n * d * 8));
    G(xpad_, xpad_cap_, std::max<uint64_t>(8, d * ldx * 8));
    for (int i = 0; i < 2; ++i) G(survkeys_[i], survkeys_cap_[i], std::max<uint64_t>(8, n * 8));
    if (status_words * 8 > status_cap_) status_zeroed_ = false;
    G(status_, status_cap_, status_words * 8);
    G(comp_, comp_cap_, std::max<uint64_t>(4, n * 4));
    G(best_, best_cap_, std::max<uint64_t>(16, 2 * n * 4 + n * 2 + 48));
    G(surv_, surv_cap_, std::max<uint64_t>(4, n * 4));
    G(surv_sorted_, surv_sorted_cap_, std::max<uint64_t>(4, n * 4));
    G(lows_, lows_cap_, std::max<uint64_t>(8, n * 8));  // lows | xs
    G(death_grade_, death_grade_cap_, std::max<uint64_t>(8, n * 8));
    G(death_length_, death_length_cap_, std::max<uint64_t>(8, n * 8));
#undef G
    if (!status_zeroed_) {
        PH0B_TRY(cudaMemset(status_, 0, status_cap_), "cudaMemset status");
        epoch_ = 1;
        status_zeroed_ = true;
    }
    return Status::ok();
}

Status Context::reserve(uint64_t n, uint64_t d) {
    Status s = reserve_points(n, d);
    if (!s.good()) return s;
    return reserve_edges(n * (n - (n > 0)) / 2);
}

Status Context::reserve_recv(uint64_t k, int buffer) {
    Status s;
    if (!(s = grow(reinterpret_cast<void**>(&keys_[buffer]), &keys_cap_[buffer], k * 8 + 4096))
             .good())
        return s;
    return grow(reinterpret_cast<void**>(&vals_[buffer]), &vals_cap_[buffer], k * 4 + 4096);
}

Status Context::sort_survivors(uint32_t m, uint64_t count, cudaStream_t st) {
    if (m == 0) return Status::ok();
    launches += launch_widen(surv_, m, survkeys_[0], st);
    SortPlan sp{};
    span_passes(count > 1 ? count - 1 : 1, &sp);
    PH0B_TRY(cudaMemsetAsync(hist_, 0, 256 * 4, st), "memset");
    launches += launch_digit_histogram(survkeys_[0], m, 0, 0, hist_, st, num_sms_);
    SortArgs sv{};
    sv.count = m;
    sv.kmin = 0;
    sv.keys[0] = survkeys_[0];
    sv.keys[1] = survkeys_[1];
    sv.status = status_;
    sv.hist = hist_;
    sv.tile_counter = counters_ + 48;
    sv.epoch_base = next_epochs(sp.passes + 1, st);
    sv.hist0_rot = 0;
    int l2 = 0;
    surv_sorted_idx_ = launch_sort_passes(sv, sp, st, num_sms_, &l2);
    launches += l2;
    launches += launch_narrow(survkeys_[surv_sorted_idx_], m, surv_sorted_, st);
    PH0B_CHECK_LAUNCH("survivor sort");
    return Status::ok();
}

Status Context::reserve_edges(uint64_t k) {
    PH0B_TRY(cudaSetDevice(device_), "cudaSetDevice");
    const uint64_t status_words = sort_tiles(std::max<uint64_t>(k, 1)) * 256;
    Status s;
#define G(ptr, cap, bytes)                                                    \
    if (!(s = grow(reinterpret_cast<void**>(&(ptr)), &(cap), (bytes))).good()) return s;
    const uint64_t cand = std::max<uint64_t>(1, std::min<uint64_t>(k, kCandCap));
    for (int i = 0; i < 2; ++i) {
        // +256 B: the TMA bulk prefetch of the last sort tile rounds its size up to 16 B
        G(keys_[i], keys_cap_[i], k * 8 + 4096);  // + bucket padding, TMA size rounding
        G(vals_[i], vals_cap_[i], k * 4 + 4096);
        G(cand_[i], cand_cap_[i], cand * 4);
    }
    if (status_words * 8 > status_cap_) status_zeroed_ = false;
    G(status_, status_cap_, status_words * 8);
#undef G
    if (!status_zeroed_) {
        PH0B_TRY(cudaMemset(status_, 0, status_cap_), "cudaMemset status");
        epoch_ = 1;
        status_zeroed_ = true;
    }
    return Status::ok();
}

uint32_t Context::next_epochs(uint32_t count, cudaStream_t s) {
    if (epoch_ + count >= (1u << 30) - 1) {
        cudaMemsetAsync(status_, 0, status_cap_, s);
        epoch_ = 1;
    }
    const uint32_t e = epoch_;
    epoch_ += count;
    return e;
}

Status Context::run_host_input(const double* X, uint64_t n, uint64_t d, uint32_t layout,
                               cudaStream_t stream, StopAfter stop, bool want_grade,
                               RunOutputs* out) {
    Status s = reserve(n, d);
    if (!s.good()) return s;
    if (n * d)
        PH0B_TRY(cudaMemcpyAsync(xin_, X, n * d * 8, cudaMemcpyHostToDevice, stream),
                 "H2D point cloud");
    return run(xin_, n, d, layout, stream, stop, want_grade, out);
}

Status Context::stage_distances(const double* dX, uint64_t n, uint64_t d, uint32_t layout,
                                uint64_t u_lo, uint64_t u_hi, cudaStream_t st, uint64_t* count,
                                uint64_t* kmin, uint64_t* kmax) {
    NvtxRange nvtx_("K1 distances");
    const uint64_t ldx = std::max<uint64_t>(128, (n + 127) / 128 * 128);
    PH0B_TRY(cudaMemsetAsync(small_, 0xFF, 8, st), "memset");        // min = ~0
    PH0B_TRY(cudaMemsetAsync(small_ + 1, 0, 3 * 8, st), "memset");   // max, n_scale, flag
    PH0B_TRY(cudaMemsetAsync(hist_, 0, 256 * 4, st), "memset");
    launches += launch_pack_points(dX, layout, (uint32_t)n, (uint32_t)d, xpad_, ldx,
                                   reinterpret_cast<uint32_t*>(small_ + 3), st);
    PH0B_CHECK_LAUNCH("pack_points");
    // The raw low-byte histogram only serves the first radix pass when the key span fits in
    // the 5-pass plan (shift 0): small problems.  Large ones count their first (truncated)
    // digit in a separate pass anyway, so the per-edge shared atomic is skipped there.
    const uint64_t kedges = row_base(std::min<uint64_t>(u_hi, n), n) - row_base(u_lo, n);
    hist_valid_ = kedges < (1ull << 24);
    DistanceArgs da{xpad_, ldx, (uint32_t)n, (uint32_t)d, keys_[0], vals_[0], small_,
                    hist_valid_ ? hist_ : nullptr};
    da.u_lo = (uint32_t)u_lo;
    da.u_hi = (uint32_t)u_hi;
    da.e_off = u_lo < n ? row_base(u_lo, n) : 0;
    const int dl = launch_distance(da, st, num_sms_);
    PH0B_CHECK_LAUNCH("distance kernel");
    if (dl == 0 && kedges > 0)
        return {PH0B_ERR_CUDA, "distance kernel: launch configuration failed"};
    launches += dl;
    PH0B_TRY(cudaMemcpyAsync(h_small_, small_, 4 * 8, cudaMemcpyDeviceToHost, st), "D2H");
    PH0B_TRY(cudaStreamSynchronize(st), "distance stage");
    if (static_cast<uint32_t>(h_small_[3]) != 0)
        return {PH0B_ERR_NONFINITE, "point cloud contains non-finite coordinates"};
    const uint64_t hi = std::min<uint64_t>(u_hi, n);
    *count = (u_lo < hi) ? row_base(hi, n) - row_base(u_lo, n) : 0;
    *kmin = h_small_[0];
    *kmax = h_small_[1];
    xpad_ld_ = ldx;
    xpad_d_ = d;
    return Status::ok();
}

Status Context::sort_unique_range(uint64_t* kb0, uint32_t* vb0, uint64_t* kb1, uint32_t* vb1,
                                  uint64_t k, uint64_t kmin, uint64_t kmax, bool raw_hist,
                                  double* scale_out, const uint64_t* d_base, uint64_t* d_count,
                                  uint32_t* grade_out, cudaStream_t st, int* res,
                                  uint32_t* passes, const std::function<Status()>* after_enqueue) {
    NvtxRange nvtx_("K2 sort + K3 unique");
    uint64_t* kb[2] = {kb0, kb1};
    uint32_t* vb[2] = {vb0, vb1};
    int src = 0;
    *res = 0;
    if (k == 0) {
        if (d_base)
            PH0B_TRY(cudaMemcpyAsync(d_count, d_base, 8, cudaMemcpyDeviceToDevice, st), "copy");
        else
            PH0B_TRY(cudaMemsetAsync(d_count, 0, 8, st), "memset");
        return after_enqueue ? (*after_enqueue)() : Status::ok();
    }
    for (int attempt = 0;; ++attempt) {
        SortPlan plan{};
        const uint32_t low_bits =
            truncated_plan(kmax - kmin, attempt == 0 ? max_sort_passes() : 8u, &plan);
        // attempt > 0: an equal-prefix run was too long to fix up in place; every radix pass
        // and every run fix-up so far was stable, so re-sorting the current order over all
        // digits restores the exact (length, u, v) order.
        SortArgs sa{};
        sa.count = k;
        sa.kmin = kmin;
        sa.keys[0] = kb[src];
        sa.keys[1] = kb[src ^ 1];
        sa.vals[0] = vb[src];
        sa.vals[1] = vb[src ^ 1];
        sa.status = status_;
        sa.hist = hist_;
        sa.tile_counter = counters_ + 32;
        sa.epoch_base = next_epochs(plan.passes + 1, st);
        if (plan.passes > 0 && (plan.shift[0] != 0 || !raw_hist || !hist_valid_ || attempt > 0)) {
            PH0B_TRY(cudaMemsetAsync(hist_, 0, 256 * 4, st), "memset");
            launches += launch_digit_histogram(kb[src], k, kmin, plan.shift[0], hist_, st,
                                               num_sms_);
            sa.hist0_rot = 0;
        } else {
            sa.hist0_rot = (uint32_t)(kmin & 0xFFu);  // distance kernel's raw low-byte histogram
        }
        int sl = 0;
        PH0B_TRY(cudaEventRecord(ev_[8], st), "event");
        const int out = launch_sort_passes(sa, plan, st, num_sms_, &sl);
        *res = src ^ out;
        launches += sl;
        PH0B_CHECK_LAUNCH("radix sort");
        PH0B_TRY(cudaEventRecord(ev_[2], st), "event");
        *passes += plan.passes;

        double* scale = scale_out ? scale_out : reinterpret_cast<double*>(kb[*res ^ 1]);
        volatile uint64_t* h_redo = h_mapped_;
        *h_redo = 0;  // (no kernel of this context is running: the previous check synced)
        uint32_t* redo = reinterpret_cast<uint32_t*>(d_mapped_);
        Status gs = grow(reinterpret_cast<void**>(&uscratch_), &uscratch_cap_,
                         unique_scratch_words(k) * 8);
        if (!gs.good()) return gs;
        UniqueArgs ua{kb[*res], vb[*res], k, kmin, low_bits, scale, grade_out, d_count, redo,
                      uscratch_, d_base};
        const int ul = launch_unique(ua, st);
        if (ul < 0) return {PH0B_ERR_CUDA, "unique kernels: launch configuration failed"};
        launches += ul;
        PH0B_CHECK_LAUNCH("unique kernel");
        if (attempt == 0 && after_enqueue) {  // host work that overlaps this range's kernels
            const Status hs = (*after_enqueue)();
            if (!hs.good()) return hs;
        }
        if (low_bits == 0) break;
        PH0B_TRY(cudaEventRecord(ev_[7], st), "event");
        PH0B_TRY(cudaEventSynchronize(ev_[7]), "unique");
        if (static_cast<uint32_t>(*h_redo) == 0) break;
        src = *res;
    }
    return Status::ok();
}

Status Context::stage_sort_unique(uint64_t k, uint64_t kmin, uint64_t kmax, bool raw_hist,
                                  bool want_grade, cudaStream_t st, uint32_t* passes, int src) {
    if (want_grade) {
        Status s = grow(reinterpret_cast<void**>(&grade_), &grade_cap_, std::max<uint64_t>(4, k * 4));
        if (!s.good()) return s;
    }
    cur_ = src;
    *passes = 0;
    int res = 0;
    Status s = sort_unique_range(keys_[src], vals_[src], keys_[src ^ 1], vals_[src ^ 1], k, kmin,
                                 kmax, raw_hist && src == 0, nullptr, nullptr, small_ + 2,
                                 want_grade ? grade_ : nullptr, st, &res, passes);
    if (!s.good()) return s;
    cur_ = src ^ res;
    scale_ = reinterpret_cast<double*>(keys_[cur_ ^ 1]);
    return Status::ok();
}

Status Context::stage_reduce(const uint32_t* uv, uint64_t count, uint32_t n, cudaStream_t st,
                             ReduceStats* rst, const uint32_t* init_comp, uint32_t target) {
    NvtxRange nvtx_("K4 column reduction");
    ReduceState rs{};
    rs.n = n;
    rs.k = count;
    rs.uv = uv;
    rs.comp = comp_;
    rs.best = best_;
    rs.cand[0] = cand_[0];
    rs.cand[1] = cand_[1];
    rs.cap = cand_cap_[0] / 4;
    rs.surv = surv_;
    rs.counters = counters_;
    rs.host_counters = reinterpret_cast<uint32_t*>(h_mapped_ + 128);
    rs.mapped_counters = reinterpret_cast<uint32_t*>(d_mapped_ + 128);
    uint32_t ep = 0;
    run_reduction(rs, st, num_sms_, ep, rst, init_comp, target);
    launches += rst->launches;
    PH0B_CHECK_LAUNCH("reduction");
    return Status::ok();
}

Status Context::stage_collect(uint32_t m, uint64_t count, uint64_t grade_offset, cudaStream_t st) {
    NvtxRange nvtx_("K5 collect");
    if (m == 0) return Status::ok();
    Status s = sort_survivors(m, count, st);
    if (!s.good()) return s;
    launches += launch_collect_map(survkeys_[surv_sorted_idx_], m, keys_[cur_], scale_, small_ + 2,
                                   grade_offset, surv_sorted_, death_grade_, death_length_, st);
    PH0B_CHECK_LAUNCH("collect");
    return Status::ok();
}

Status Context::run(const double* dX, uint64_t n, uint64_t d, uint32_t layout,
                    cudaStream_t stream, StopAfter stop, bool want_grade, RunOutputs* out) {
    NvtxRange nvtx_("ph0b pipeline (device)");
    Status s = reserve(n, d);
    if (!s.good()) return s;
    cudaStream_t st = stream ? stream : stream_;
    launches = 0;
    const uint64_t k = n * (n - (n > 0)) / 2;
    RunOutputs r;
    r.k = k;
    std::memset(&r.times, 0, sizeof(r.times));

    PH0B_TRY(cudaEventRecord(ev_[0], st), "event");
    // ---- K1: pack + distances ------------------------------------------------------------
    uint64_t cnt = 0, kmin = 0, kmax = 0;
    s = stage_distances(dX, n, d, layout, 0, n, st, &cnt, &kmin, &kmax);
    if (!s.good()) return s;
    PH0B_TRY(cudaEventRecord(ev_[1], st), "event");
    r.d_lengths_umajor = keys_[0];
    if (stop == StopAfter::Distance || k == 0) {
        r.essential = n;
        PH0B_TRY(cudaEventRecord(ev_[5], st), "event");
        PH0B_TRY(cudaEventSynchronize(ev_[5]), "sync");
        cudaEventElapsedTime(&r.times.distance_ms, ev_[0], ev_[1]);
        cudaEventElapsedTime(&r.times.total_ms, ev_[0], ev_[5]);
        r.d_scale = reinterpret_cast<const double*>(keys_[1]);
        r.d_uv_sorted = vals_[0];
        r.d_grade = grade_;
        if (out) *out = r;
        return Status::ok();
    }

    // ---- K2 + K2c/K3: radix sort over the top bits of the span, unique -> D, M -------------
    s = stage_sort_unique(k, kmin, kmax, true, want_grade, st, &r.times.sort_passes);
    if (!s.good()) return s;
    PH0B_TRY(cudaEventRecord(ev_[3], st), "event");
    r.d_uv_sorted = vals_[cur_];
    r.d_grade = want_grade ? grade_ : nullptr;
    r.d_scale = scale_;

    if (stop == StopAfter::Barcode && kruskal_mode) {
        uint32_t m = 0;
        s = stage_kruskal(k, (uint32_t)n, st, &m);
        if (!s.good()) return s;
        PH0B_TRY(cudaEventRecord(ev_[4], st), "event");
        r.d_death_grade = death_grade_;
        r.d_death_length = death_length_;
        r.n_finite = m;
        r.essential = n - m;
    } else if (stop == StopAfter::Barcode) {
        // ---- K4: column reduction ----------------------------------------------------------
        ReduceStats rst;
        s = stage_reduce(vals_[cur_], k, (uint32_t)n, st, &rst);
        if (!s.good()) return s;
        PH0B_TRY(cudaEventRecord(ev_[4], st), "event");
        r.times.reduce_rounds = rst.rounds;
        r.times.reduce_iterations = rst.iterations;
        r.times.columns_scanned = rst.scanned;
        const uint32_t m = rst.survivors;
        if (m != n - 1)
            return {PH0B_ERR_CUDA, "internal error: reduction produced " + std::to_string(m) +
                                       " surviving columns, expected " + std::to_string(n - 1)};
        // ---- K5: collect: survivors in filtration order -> intervals ----------------------
        s = stage_collect(m, k, 0, st);
        if (!s.good()) return s;
        r.d_death_grade = death_grade_;
        r.d_death_length = death_length_;
        r.d_surv_sorted = surv_sorted_;
        r.n_finite = m;
        r.essential = n - m;
    }
    PH0B_TRY(cudaEventRecord(ev_[5], st), "event");
    PH0B_TRY(cudaMemcpyAsync(h_small_ + 2, small_ + 2, 8, cudaMemcpyDeviceToHost, st), "D2H");
    PH0B_TRY(cudaStreamSynchronize(st), "pipeline");
    r.n_scale = h_small_[2];
    cudaEventElapsedTime(&r.times.distance_ms, ev_[0], ev_[1]);
    cudaEventElapsedTime(&r.times.sort_ms, ev_[1], ev_[2]);
    cudaEventElapsedTime(&r.times.sort_passes_ms, ev_[8], ev_[2]);
    cudaEventElapsedTime(&r.times.unique_ms, ev_[2], ev_[3]);
    if (stop == StopAfter::Barcode) {
        cudaEventElapsedTime(&r.times.reduce_ms, ev_[3], ev_[4]);
        cudaEventElapsedTime(&r.times.collect_ms, ev_[4], ev_[5]);
    }
    cudaEventElapsedTime(&r.times.total_ms, ev_[0], ev_[5]);
    if (out) *out = r;
    return Status::ok();
}

// Device/pinned buffers, ring, events, copy streams and decode pool of the compressed D
// stream, for k values split over B buckets.
Status Context::prepare_stream(uint64_t k, uint32_t B) {
    Status s;
    // per bucket, a chunk-aligned area sized by its edge count (>= its |D|): packed bytes
    // (<= 4 per value + slack), chunk bases, widths, offsets (device) and offsets within
    // a piece; pinned mirrors of the per-chunk metadata; mapped piece boundaries
    const uint64_t chunks = k / kPackChunk + B + 64;
    const uint64_t pieces = chunks / ring_g_ + B + 2;
    if (!(s = grow(reinterpret_cast<void**>(&d_delta_), &d_delta_cap_,
                   chunks * kPackChunk * 4 + 64 * B)).good() ||
        !(s = grow(reinterpret_cast<void**>(&d_cbase_), &d_cbase_cap_, chunks * 8)).good() ||
        !(s = grow(reinterpret_cast<void**>(&d_craw_), &d_craw_cap_, chunks)).good() ||
        !(s = grow(reinterpret_cast<void**>(&d_coff_), &d_coff_cap_, chunks * 8)).good() ||
        !(s = grow(reinterpret_cast<void**>(&d_cpoff_), &d_cpoff_cap_, chunks * 4)).good() ||
        !(s = grow_host(reinterpret_cast<void**>(&h_cbase_), &h_cbase_cap_, chunks * 8)).good() ||
        !(s = grow_host(reinterpret_cast<void**>(&h_craw_), &h_craw_cap_, chunks)).good() ||
        !(s = grow_host(reinterpret_cast<void**>(&h_cpoff_), &h_cpoff_cap_, chunks * 4)).good() ||
        !(s = ensure_ring()).good())
        return s;
    if (pieces > h_pieceoff_cap_) {
        if (h_pieceoff_) cudaFreeHost(h_pieceoff_);
        h_pieceoff_ = nullptr;
        h_pieceoff_cap_ = 0;
        PH0B_TRY(cudaHostAlloc(&h_pieceoff_, pieces * 8, cudaHostAllocMapped),
                 "cudaHostAlloc mapped");
        PH0B_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_pieceoff_), h_pieceoff_,
                                          0), "cudaHostGetDevicePointer");
        h_pieceoff_cap_ = pieces;
    }
    if (bucket_ev_.size() < B) {
        bucket_ev_.resize(B, nullptr);
        for (auto& e : bucket_ev_)
            if (!e) PH0B_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    }
    if (!enc_ev_) PH0B_TRY(cudaEventCreateWithFlags(&enc_ev_, cudaEventDisableTiming), "event");
    if (ring_streams_.empty()) {
        static const int ns = [] {
            const char* e = getenv("PH0B_RING_STREAMS");
            const int x = e ? atoi(e) : 2;
            return x < 1 ? 1 : (x > 8 ? 8 : x);
        }();
        ring_streams_.push_back(copy_stream_);
        for (int i = 1; i < ns; ++i) {
            cudaStream_t x;
            PH0B_TRY(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking), "cudaStreamCreate");
            ring_streams_.push_back(x);
        }
    }
    if (!pool_) {
        static const int env_threads = [] {
            const char* e = getenv("PH0B_DECODE_THREADS");
            return e ? atoi(e) : 0;
        }();
        const unsigned hw = std::thread::hardware_concurrency();
        const unsigned dflt = decode_threads_ ? decode_threads_ : (hw > 2 ? hw - 1 : 1);
        pool_ = std::make_shared<DecodePool>(env_threads > 0 ? (unsigned)env_threads : dflt);
    }
    return Status::ok();
}

// One packed slice -> host: its chunk metadata [cbase, cbase + nch) (pinned mirrors; meta_ev
// recorded after it), then its pieces (byte ranges poffs[p] .. poffs[p+1] of d_src) through
// the ring, each handed to the pool as ring_subtasks() decode tasks right after its copy is
// enqueued (when a copy stream's queue is full the enqueue blocks until earlier pieces are
// decoded).  Must follow the slice's encode (enc_ev_) in stream order.
Status Context::enqueue_stream(uint64_t cbase, uint64_t nch, const std::vector<uint64_t>& poffs,
                               const uint8_t* d_src, const volatile uint64_t* bounds,
                               cudaEvent_t meta_ev, double* host_scale, uint64_t capacity,
                               volatile int* overflow, uint64_t* moved, uint64_t* enq_ns) {
    const uint32_t G = ring_g_, R = ring_r_, NS = ring_subtasks();
    const uint64_t npieces = poffs.size() - 1;
    cudaStream_t cs = copy_stream_;
    PH0B_TRY(cudaStreamWaitEvent(cs, enc_ev_, 0), "wait");
    PH0B_TRY(cudaMemcpyAsync(h_cbase_ + cbase, d_cbase_ + cbase, nch * 8, cudaMemcpyDeviceToHost,
                             cs), "D2H bases");
    PH0B_TRY(cudaMemcpyAsync(h_craw_ + cbase, d_craw_ + cbase, nch, cudaMemcpyDeviceToHost, cs),
             "D2H widths");
    PH0B_TRY(cudaMemcpyAsync(h_cpoff_ + cbase, d_cpoff_ + cbase, nch * 4, cudaMemcpyDeviceToHost,
                             cs), "D2H offsets");
    PH0B_TRY(cudaEventRecord(meta_ev, cs), "event");
    // extra ring streams: their pieces must not land before the chunk metadata
    for (size_t i = 1; i < ring_streams_.size(); ++i)
        PH0B_TRY(cudaStreamWaitEvent(ring_streams_[i], meta_ev, 0), "wait");
    *moved += nch * 13;
    std::vector<DecodeTask> task;
    for (uint64_t p = 0; p < npieces; ++p) {
        const uint64_t j0 = p * G;
        const uint64_t pc = std::min<uint64_t>(G, nch - j0);
        const uint64_t bytes = poffs[p + 1] - poffs[p];
        cs = ring_streams_[ring_seq_ % ring_streams_.size()];
        const uint32_t slot = (uint32_t)(ring_seq_ % R);
        const uint32_t gen = (uint32_t)(ring_seq_ / R + 1);
        ++ring_seq_;
        uint8_t* ring = reinterpret_cast<uint8_t*>(h_ring_) + (uint64_t)slot * ring_slot_bytes(G);
        const auto e0 = std::chrono::steady_clock::now();
        if (!stream_wait_u32(cs, reinterpret_cast<uint64_t>(d_ringflags_ + R + slot), gen - 1))
            return {PH0B_ERR_CUDA, "D2H ring: stream wait failed"};
        if (bytes)
            PH0B_TRY(cudaMemcpyAsync(ring, d_src + poffs[p], bytes, cudaMemcpyDeviceToHost, cs),
                     "D2H packed D");
        if (!stream_write_u32(cs, reinterpret_cast<uint64_t>(d_ringflags_ + slot), gen))
            return {PH0B_ERR_CUDA, "D2H ring: stream write failed"};
        *enq_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(
                       std::chrono::steady_clock::now() - e0).count();
        *moved += bytes;
        // the piece is decoded by NS tasks of G/NS chunks (empty past the piece's end)
        task.clear();
        const uint64_t per = (G + NS - 1) / NS;
        for (uint32_t i = 0; i < NS; ++i) {
            const uint64_t c0 = std::min<uint64_t>(pc, i * per);
            const uint64_t c1 = std::min<uint64_t>(pc, c0 + per);
            const uint64_t c = cbase + j0 + c0;
            DecodeTask t{nullptr, h_cbase_ + c, nullptr, reinterpret_cast<uint64_t*>(host_scale),
                         (c1 - c0) * kPackChunk, (uint32_t)kPackChunk};
            t.widths = h_craw_ + c;
            t.poff = h_cpoff_ + c;
            t.packed = ring;
            t.ready = h_ringflags_ + slot;
            t.freed = h_ringflags_ + R + slot;
            t.gen = gen;
            t.bounds = bounds;
            t.v0 = (j0 + c0) * kPackChunk;
            t.capacity = capacity;
            t.overflow = overflow;
            t.done = &ring_done_[slot];
            t.nsub = NS;
            task.push_back(t);
        }
        pool_->submit(task);
    }
    return Status::ok();
}

Status Context::stream_scale(const double* d_scale, uint64_t n, double* host_scale,
                             uint64_t capacity, cudaStream_t st, uint64_t* moved) {
    NvtxRange nvtx_("D to host (packed ring)");
    *moved = 0;
    if (n == 0) return Status::ok();
    if (n > capacity)
        return {PH0B_ERR_CAPACITY, "scale buffer too small: need " + std::to_string(n) +
                                       " entries"};
    if (!copy_stream_) PH0B_TRY(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking),
                                "cudaStreamCreate");
    Trace tr;
    if (!ring_g_) ring_choice(0);  // (a geometry is set before the first prepare_stream)
    Status s = prepare_stream(n, 1);
    if (!s.good()) return s;
    tr.mark("stream_scale: prepared");
    const uint32_t G = ring_g_;
    volatile int overflow = 0;
    struct PoolGuard {
        DecodePool* p;
        ~PoolGuard() { p->wait(); }
    } pool_guard{pool_.get()};
    // the slice's bounds: device words for the encoder, pinned host words for the decoders
    h_small_[4] = 0;
    h_small_[5] = n;
    volatile uint64_t* bounds = h_small_ + 4;
    PH0B_TRY(cudaMemcpyAsync(small_ + 4, h_small_ + 4, 16, cudaMemcpyHostToDevice, st), "H2D");
    uint8_t* d_pack = reinterpret_cast<uint8_t*>(d_delta_);
    launches += launch_d2h_pack_bucket(d_scale, small_ + 4, n, d_cbase_, d_craw_, d_coff_,
                                       d_cpoff_, d_pieceoff_, G, d_pack, st);
    PH0B_CHECK_LAUNCH("D2H encode");
    PH0B_TRY(cudaEventRecord(enc_ev_, st), "event");
    PH0B_TRY(cudaEventSynchronize(enc_ev_), "D2H encode");
    tr.mark("stream_scale: encoded");
    const uint64_t nch = (n + kPackChunk - 1) / kPackChunk;
    const uint64_t npieces = (nch + G - 1) / G;
    std::vector<uint64_t> poffs(npieces + 1);
    for (uint64_t p = 0; p <= npieces; ++p) poffs[p] = h_pieceoff_[p];
    uint64_t enq = 0;
    s = enqueue_stream(0, nch, poffs, d_pack, bounds, bucket_ev_[0], host_scale, capacity,
                       &overflow, moved, &enq);
    if (!s.good()) return s;
    tr.mark("stream_scale: enqueued");
    // raw chunks (a gap >= 2^32) straight from the device D
    PH0B_TRY(cudaEventSynchronize(bucket_ev_[0]), "D2H metadata");
    for (uint64_t j = 0; j < nch;) {  // runs of consecutive raw chunks: one copy each
        if (h_craw_[j]) {
            ++j;
            continue;
        }
        uint64_t j1 = j + 1;
        while (j1 < nch && !h_craw_[j1]) ++j1;
        const uint64_t s0 = j * kPackChunk, s1 = std::min<uint64_t>(j1 * kPackChunk, n);
        PH0B_TRY(cudaMemcpyAsync(host_scale + s0, d_scale + s0, (s1 - s0) * 8,
                                 cudaMemcpyDeviceToHost, copy_stream_), "D2H raw");
        *moved += (s1 - s0) * 8;
        j = j1;
    }
    pool_->wait();
    tr.mark("stream_scale: decoded");
    for (cudaStream_t x : ring_streams_) PH0B_TRY(cudaStreamSynchronize(x), "D2H scale");
    if (overflow) return {PH0B_ERR_CUDA, "D2H of D stalled (the copy stream made no progress)"};
    return Status::ok();
}

void Context::set_ring_geometry(uint32_t g, uint32_t r) {
    if (g == ring_g_ && r == ring_r_) return;
    ring_g_ = g;
    ring_r_ = r;
    // no copy or decode of an earlier call is outstanding here: restart the slot generations
    if (h_ringflags_) std::memset(h_ringflags_, 0, 512 * 4);
    ring_seq_ = 0;
    for (auto& x : ring_done_) x.store(0);
}

// The ring geometry for a host-path call over k edges (and sets it).  Calls of one size: the
// first runs geometry 0 unmeasured (allocation and first-touch costs), the 2nd and 4th are
// timed with geometry 0, the 3rd with geometry 1 — compared only when all three moved the
// same D (same edge count and |D|; otherwise the timing restarts) — and every later call keeps
// the faster (geometry 0's better time against geometry 1's: one slow call does not decide).
int Context::ring_choice(uint64_t k) {
    if (ring_fixed()) {
        const int g = env_ring("PH0B_RING_CHUNKS", 1, 16384);
        const int r = env_ring("PH0B_RING_SLOTS", 2, 256);
        set_ring_geometry(g ? (uint32_t)g : kRingGeom[0][0], r ? (uint32_t)r : kRingGeom[0][1]);
        return -1;
    }
    int c = ring_pick_;
    if (c < 0) {
        if (k && k != ring_tune_k_) {
            ring_tune_k_ = k;
            ring_calls_ = 0;
        }
        c = (k && ring_calls_ == 2) ? 1 : 0;
    }
    set_ring_geometry(kRingGeom[c][0], kRingGeom[c][1]);
    return k ? c : -1;
}

void Context::ring_record(uint64_t k, uint64_t n_scale, double ms) {
    if (ring_pick_ >= 0 || k != ring_tune_k_) return;
    if (ring_calls_ == 1) {
        ring_ms_[0] = ms;
        ring_tune_d_ = n_scale;
    } else if (n_scale != ring_tune_d_) {  // another cloud: this call counts as a first one
        ring_calls_ = 0;
    } else if (ring_calls_ == 2) {
        ring_ms_[1] = ms;
    } else if (ring_calls_ == 3) {
        ring_ms_[0] = std::min(ring_ms_[0], ms);
        ring_pick_ = ring_ms_[1] < ring_ms_[0] ? 1 : 0;
        if (getenv("PH0B_TRACE"))
            fprintf(stderr, "[ph0b trace] D2H ring: %u x %u chunks %.1f ms, %u x %u chunks %.1f ms"
                    " -> %u x %u\n", kRingGeom[0][1], kRingGeom[0][0], ring_ms_[0],
                    kRingGeom[1][1], kRingGeom[1][0], ring_ms_[1], kRingGeom[ring_pick_][1],
                    kRingGeom[ring_pick_][0]);
    }
    ++ring_calls_;
}

Status Context::run_host_overlapped(const double* X, uint64_t n, uint64_t d, uint32_t layout,
                                    cudaStream_t st, double* host_scale,
                                    uint64_t scale_capacity, RunOutputs* out) {
    const uint64_t k = n * (n - (n > 0)) / 2;
    const int c = ring_choice(k);
    const auto t0 = std::chrono::steady_clock::now();
    Status s = run_host_overlapped_impl(X, n, d, layout, st, host_scale, scale_capacity, out);
    if (s.good() && c >= 0)
        ring_record(k, out ? out->n_scale : 0, std::chrono::duration<double, std::milli>(
                                         std::chrono::steady_clock::now() - t0).count());
    return s;
}

Status Context::run_host_overlapped_impl(const double* X, uint64_t n, uint64_t d, uint32_t layout,
                                    cudaStream_t st, double* host_scale, uint64_t scale_capacity,
                                    RunOutputs* out) {
    NvtxRange nvtx_("ph0b pipeline (host, bucketed D stream)");
    Status s = reserve(n, d);
    if (!s.good()) return s;
    const uint64_t k = n * (n - (n > 0)) / 2;
    // key-range buckets (cumulative edge fractions, /256): bucket 0 (1/16) is extracted and
    // sorted before the rest is partitioned, so its D slice (~19 ms on PCIe) covers the
    // partition; then small buckets (1/256 .. 1/32) so the copy engine never starves, then
    // buckets of 1/16
    // (PH0B_BUCKETS="c1,c2,...": another schedule, strictly increasing values in (0, 256),
    // c1 <= 64)
    static const std::vector<uint32_t> kCum = [] {
        std::vector<uint32_t> v = {16, 17, 19, 23, 31, 47, 63, 79, 95, 111, 127,
                                   143, 159, 175, 191, 207, 223, 239};
        if (const char* e = getenv("PH0B_BUCKETS")) {
            std::vector<uint32_t> w;
            for (const char* q = e; *q;) {
                char* end = nullptr;
                const long x = strtol(q, &end, 10);
                if (end == q) break;
                if (x > 0 && x < 256 && (w.empty() || (uint32_t)x > w.back()))
                    w.push_back((uint32_t)x);
                q = *end ? end + 1 : end;
            }
            // the first bucket is sorted inside buffer 1 before the partition: <= 1/4
            if (!w.empty() && w.size() < 100 && w[0] <= 64) v = w;
        }
        return v;
    }();
    const uint32_t B = (uint32_t)kCum.size() + 1;
    if (!(s = grow(reinterpret_cast<void**>(&dbuf_), &dbuf_cap_, k * 8 + 256)).good()) return s;
    const uint64_t part_words = partition_scratch_words(k, B);
    if (!(s = grow(reinterpret_cast<void**>(&part_counts_), &part_counts_cap_, part_words * 4 + 16))
             .good())
        return s;
    if (!(s = grow(reinterpret_cast<void**>(&part_small_), &part_small_cap_, 4096 * 8)).good())
        return s;
    if (!copy_stream_) PH0B_TRY(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking),
                                "cudaStreamCreate");
    // the compressed stream needs stream memory operations on mapped host memory (probed
    // once per context); without them D goes back uncompressed
    const bool compress = host_scale && d2h_compress() && stream_memops_ok();
    if (compress) {
        if (!(s = prepare_stream(k, B)).good()) return s;
    }
    volatile int overflow = 0;  // decode tasks: 1 = scale buffer too small, 2 = stream stalled
    // whatever the exit path, no decode task may still be writing the caller's buffer
    struct PoolGuard {
        DecodePool* p;
        ~PoolGuard() {
            if (p) p->wait();
        }
    } pool_guard{compress ? pool_.get() : nullptr};
    uint64_t* d_spl = part_small_;           // [256]
    uint64_t* d_tot = part_small_ + 256;     // [512]: totals | segment starts
    uint64_t* d_mm = part_small_ + 768;      // [512]: key bounds
    uint64_t* d_base = d_mapped_ + 8;        // [B + 1], zero-copy host words
    volatile uint64_t* h_base = h_mapped_ + 8;
    launches = 0;
    Trace tr;
    RunOutputs r;
    r.k = k;
    std::memset(&r.times, 0, sizeof(r.times));
    PH0B_TRY(cudaEventRecord(ev_[0], st), "event");
    if (n * d)
        PH0B_TRY(cudaMemcpyAsync(xin_, X, n * d * 8, cudaMemcpyHostToDevice, st), "H2D cloud");
    uint64_t cnt = 0, kmin = 0, kmax = 0;
    if (!(s = stage_distances(xin_, n, d, layout, 0, n, st, &cnt, &kmin, &kmax)).good()) return s;
    PH0B_TRY(cudaEventRecord(ev_[1], st), "event");
    tr.mark("distances done");

    // ---- splitters from an evenly spaced sample, stable partition into B key ranges -------
    const uint64_t S = std::min<uint64_t>(k, std::min<uint64_t>(n, 16384));
    std::vector<uint64_t> sample(S);
    launches += launch_sample(keys_[0], k, S, survkeys_[0], st);
    PH0B_TRY(cudaMemcpyAsync(sample.data(), survkeys_[0], S * 8, cudaMemcpyDeviceToHost, st), "D2H");
    PH0B_TRY(cudaStreamSynchronize(st), "sample");
    std::sort(sample.begin(), sample.end());
    std::vector<uint64_t> spl(B - 1);
    for (uint32_t j = 0; j + 1 < B; ++j)
        spl[j] = sample[std::min<uint64_t>(S - 1, (uint64_t)kCum[j] * S / 256)];
    PH0B_TRY(cudaMemcpyAsync(d_spl, spl.data(), (B - 1) * 8, cudaMemcpyHostToDevice, st), "H2D");
    // segments start on 4-element boundaries (16-byte aligned TMA bulk copies in the sort
    // and unique kernels); the <= 3 padding slots per segment hold the cycle column {0, 0}
    constexpr uint32_t kAlign = 4;
    uint16_t* d_table = reinterpret_cast<uint16_t*>(part_small_ + 1280);
    const int lc = launch_partition_count(keys_[0], k, d_spl, B, part_counts_, d_tot, d_mm,
                                          keys_[1], vals_[1], st, kAlign, kmin, kmax, spl.data(),
                                          d_table, col_cycle(n));
    if (lc < 0) return {PH0B_ERR_INVALID_ARGUMENT, "partition: bad bucket count"};
    launches += lc;
    PH0B_CHECK_LAUNCH("partition counts");
    std::vector<uint64_t> tot(B), mm(2 * B);
    PH0B_TRY(cudaMemcpyAsync(tot.data(), d_tot, B * 8, cudaMemcpyDeviceToHost, st), "D2H");
    PH0B_TRY(cudaMemcpyAsync(mm.data(), d_mm, 2 * B * 8, cudaMemcpyDeviceToHost, st), "D2H");
    PH0B_TRY(cudaStreamSynchronize(st), "partition");
    tr.mark("partition counts done");
    h_base[0] = 0;
    uint64_t start = 0;
    int target = -1;
    auto pad = [&](uint64_t c) { return (c + kAlign - 1) / kAlign * kAlign; };
    // D slices of finished buckets -> host.
    //  * compressed (default): the encoder turns the slice into a u64 base + u32 deltas per
    //    4096-value chunk (half the PCIe bytes); the copy engine streams the deltas through a
    //    small pinned ring (LLC-resident: the DMA writes land in the last-level cache and the
    //    decode reads them from there) and the pool decodes each piece as soon as its ready
    //    flag flips.  Nothing about a bucket is waited for on the host: the encode reads the
    //    slice bounds from device words and the copies are sized by the bucket's edge count
    //    (an upper bound of its |D|), so bucket b's copies are enqueued while bucket b+1 sorts.
    //  * uncompressed: plain D2H of the slice in medium chunks once the bucket is sorted.
    const uint32_t G = ring_g_;
    std::vector<uint64_t> nch_ub(B), cb(B + 1, 0), rb(B + 1, 0);
    for (uint32_t b = 0; b < B; ++b) {
        nch_ub[b] = (tot[b] + kPackChunk - 1) / kPackChunk;
        cb[b + 1] = cb[b] + nch_ub[b];
        rb[b + 1] = rb[b] + nch_ub[b] * kPackChunk * 4 + 64;  // packed bytes + store slack
    }
    uint64_t d2h_total = 0;  // bytes moved device -> host by this call
    uint64_t enq_ns = 0;     // host time spent enqueuing the pieces (trace)
    std::vector<uint32_t> pending;  // buckets whose raw chunks are not shipped yet
    uint64_t* d_lohi = part_small_ + 2304;  // [2B] device copy of each bucket's D bounds
    uint8_t* d_pack = reinterpret_cast<uint8_t*>(d_delta_);
    auto encode = [&](uint32_t b) -> Status {
        if (!compress || tot[b] == 0) return Status::ok();
        PH0B_TRY(cudaMemcpyAsync(d_lohi + 2 * b, d_base + b, 16, cudaMemcpyDefault, st), "copy");
        launches += launch_d2h_pack_bucket(dbuf_, d_lohi + 2 * b, tot[b], d_cbase_ + cb[b],
                                           d_craw_ + cb[b], d_coff_ + cb[b], d_cpoff_ + cb[b],
                                           d_pieceoff_, G, d_pack + rb[b], st);
        PH0B_CHECK_LAUNCH("D2H encode");
        PH0B_TRY(cudaEventRecord(enc_ev_, st), "event");
        return Status::ok();
    };
    // after encode(b) (the last one enqueued): per-chunk metadata, then the packed pieces
    // through the ring, each copy sized by the piece boundaries the encoder published
    auto stream_out = [&](uint32_t b) -> Status {
        if (!compress || tot[b] == 0) return Status::ok();
        PH0B_TRY(cudaEventSynchronize(enc_ev_), "D2H encode");
        const uint64_t nb = h_base[b + 1] - h_base[b];
        const uint64_t nch = (nb + kPackChunk - 1) / kPackChunk;
        if (nch == 0) return Status::ok();
        const uint64_t npieces = (nch + G - 1) / G;
        std::vector<uint64_t> poffs(npieces + 1);
        for (uint64_t p = 0; p <= npieces; ++p) poffs[p] = h_pieceoff_[p];
        uint64_t moved = 0;
        const Status es = enqueue_stream(cb[b], nch, poffs, d_pack + rb[b], h_base + b,
                                         bucket_ev_[b], host_scale, scale_capacity, &overflow,
                                         &moved, &enq_ns);
        if (!es.good()) return es;
        d2h_total += moved;
        pending.push_back(b);
        return Status::ok();
    };
    // raw chunks (a delta did not fit in 32 bits) of buckets whose metadata has landed
    auto drain = [&](bool wait) -> Status {
        while (!pending.empty()) {
            const uint32_t b = pending.front();
            if (!wait && cudaEventQuery(bucket_ev_[b]) == cudaErrorNotReady) {
                cudaGetLastError();
                break;
            }
            PH0B_TRY(cudaEventSynchronize(bucket_ev_[b]), "D2H bucket");
            const uint64_t lo = h_base[b], nb = h_base[b + 1] - lo;
            const uint64_t nchb = (nb + kPackChunk - 1) / kPackChunk;
            for (uint64_t j = 0; j < nchb;) {  // runs of consecutive raw chunks: one copy each
                if (h_craw_[cb[b] + j]) {
                    ++j;
                    continue;
                }
                uint64_t j1 = j + 1;
                while (j1 < nchb && !h_craw_[cb[b] + j1]) ++j1;
                const uint64_t s0 = lo + j * kPackChunk;
                const uint64_t s1 = lo + std::min<uint64_t>(j1 * kPackChunk, nb);
                j = j1;
                if (s1 > scale_capacity) {
                    overflow = 1;
                    continue;
                }
                PH0B_TRY(cudaMemcpyAsync(host_scale + s0, dbuf_ + s0, (s1 - s0) * 8,
                                         cudaMemcpyDeviceToHost, copy_stream_), "D2H raw");
                d2h_total += (s1 - s0) * 8;
            }
            pending.erase(pending.begin());
        }
        return Status::ok();
    };
    uint64_t host_base = 0;
    auto ship_plain = [&](uint32_t b) -> Status {
        PH0B_TRY(cudaEventRecord(ev_[6], st), "event");
        PH0B_TRY(cudaEventSynchronize(ev_[6]), "bucket");
        tr.mark("bucket sorted", (long)b);
        const uint64_t next_base = h_base[b + 1];
        if (host_scale && next_base > host_base) {
            if (next_base > scale_capacity)
                return {PH0B_ERR_CAPACITY, "scale buffer too small: need >= " +
                                               std::to_string(next_base) + " entries"};
            PH0B_TRY(cudaStreamWaitEvent(copy_stream_, ev_[6], 0), "wait");
            for (uint64_t q = host_base; q < next_base; q += d2h_chunk_elems()) {
                const uint64_t e = std::min<uint64_t>(next_base, q + d2h_chunk_elems());
                PH0B_TRY(cudaMemcpyAsync(host_scale + q, dbuf_ + q, (e - q) * 8,
                                         cudaMemcpyDeviceToHost, copy_stream_), "D2H scale");
            }
            d2h_total += (next_base - host_base) * 8;
        }
        host_base = next_base;
        return Status::ok();
    };

    // ---- bucket 0 ahead of the partition: extract it (stable) into its segment, sort it
    // there (ping-pong with the free space after it), and start its D2H ---------------------
    {
        const uint64_t c0 = tot[0];
        launches += launch_partition_select(keys_[0], vals_[0], k, B, 0, part_counts_, d_tot,
                                            d_mm, keys_[1], vals_[1], st);
        int res = 0;
        uint32_t passes = 0;
        const uint64_t c0p = pad(c0);
        // bucket 0 ping-pongs with the space right after it in buffer 1: it must fit twice
        // (<= 1/16 of the edges by construction: keys strictly below the 1/16 sample quantile)
        if ((2 * c0p + 4) * 8 > keys_cap_[1] || (2 * c0p + 4) * 4 > vals_cap_[1])
            return {PH0B_ERR_CUDA, "internal error: first key-range bucket holds " +
                                       std::to_string(c0) + " of " + std::to_string(k) +
                                       " edges (more than half)"};
        s = sort_unique_range(keys_[1], vals_[1], keys_[1] + c0p, vals_[1] + c0p, c0,
                              c0 ? mm[0] : 0, c0 ? mm[B] : 0, false, dbuf_, d_base,
                              d_base + 1, nullptr, st, &res, &passes);
        if (!s.good()) return s;
        tr.mark("bucket sorted", 0);
        r.times.sort_passes = passes;
        if (c0 && res == 1) {  // sorted data ended in the scratch half, which the scatter
                               // below overwrites: back into segment 0 first
            PH0B_TRY(cudaMemcpyAsync(keys_[1], keys_[1] + c0p, c0 * 8, cudaMemcpyDeviceToDevice,
                                     st), "D2D");
            PH0B_TRY(cudaMemcpyAsync(vals_[1], vals_[1] + c0p, c0 * 4, cudaMemcpyDeviceToDevice,
                                     st), "D2D");
        }
        if (compress) {
            if (!(s = encode(0)).good()) return s;
        } else if (!(s = ship_plain(0)).good()) {
            return s;
        }
        // ---- the rest of the partition (segment 0 is already in place) --------------------
        const int ls = launch_partition_scatter(keys_[0], vals_[0], k, d_spl, B, part_counts_,
                                                d_tot, keys_[1], vals_[1], st, kmin, kmax,
                                                d_table, 0u);
        PH0B_CHECK_LAUNCH("partition");
        if (ls < 0) return {PH0B_ERR_CUDA, "partition: launch configuration failed"};
        launches += ls;
        // M is assembled in buffer 0 (the 5-pass buckets end there): once the scatter has
        // consumed the u-major input, move sorted bucket 0 into its segment of buffer 0
        if (c0) {
            PH0B_TRY(cudaMemcpyAsync(keys_[0], keys_[1], c0 * 8, cudaMemcpyDeviceToDevice, st),
                     "D2D");
            PH0B_TRY(cudaMemcpyAsync(vals_[0], vals_[1], c0 * 4, cudaMemcpyDeviceToDevice, st),
                     "D2D");
            target = 0;
        }
        start = c0p;
        // bucket 0's pieces are enqueued while the scatter runs
        if (!(s = stream_out(0)).good()) return s;
    }

    // ---- per bucket: sort + unique into D, then stream that slice of D to the host ---------
    for (uint32_t b = 1; b < B; ++b) {
        const uint64_t c = tot[b];
        int res = 0;
        uint32_t passes = 0;
        // the previous bucket's copies are enqueued once this bucket's kernels are queued
        const std::function<Status()> after = [&]() -> Status { return stream_out(b - 1); };
        const bool hook = compress && b > 1;
        s = sort_unique_range(keys_[1] + start, vals_[1] + start, keys_[0] + start,
                              vals_[0] + start, c, c ? mm[b] : 0, c ? mm[B + b] : 0, false,
                              dbuf_, d_base + b, d_base + b + 1, nullptr, st, &res, &passes,
                              hook ? &after : nullptr);
        if (!s.good()) return s;
        if (compress && !hook && b > 1 && !(s = stream_out(b - 1)).good()) return s;
        r.times.sort_passes = std::max(r.times.sort_passes, passes);
        const int buf = res == 0 ? 1 : 0;  // global buffer holding this bucket's sorted data
        if (c && target < 0) target = buf;
        if (c && buf != target) {  // keep M contiguous in one buffer
            PH0B_TRY(cudaMemcpyAsync(keys_[target] + start, keys_[buf] + start, c * 8,
                                     cudaMemcpyDeviceToDevice, st), "D2D");
            PH0B_TRY(cudaMemcpyAsync(vals_[target] + start, vals_[buf] + start, c * 4,
                                     cudaMemcpyDeviceToDevice, st), "D2D");
        }
        if (compress) {
            tr.mark("bucket sorted", (long)b);
            if (!(s = encode(b)).good()) return s;
            if (!(s = drain(false)).good()) return s;
        } else if (!(s = ship_plain(b)).good()) {
            return s;
        }
        start += pad(c);
    }
    if (compress && B > 1 && !(s = stream_out(B - 1)).good()) return s;
    const uint64_t kpad = start;  // columns incl. the sentinel padding
    if (target < 0) target = 0;
    // padding slots of M hold the cycle column {0, 0} in whichever buffer M ended up
    launches += launch_partition_pad(d_tot, B, kAlign, keys_[target], vals_[target], st,
                                     col_cycle(n));
    PH0B_TRY(cudaEventRecord(ev_[2], st), "event");
    PH0B_TRY(cudaEventRecord(ev_[3], st), "event");
    cur_ = target;
    scale_ = dbuf_;
    PH0B_TRY(cudaMemcpyAsync(small_ + 2, d_base + B, 8, cudaMemcpyDefault, st), "copy");

    // ---- K4 + K5 (or the union-find oracle) on the whole (now sorted) matrix -------------
    ReduceStats rst;
    uint32_t m = 0;
    if (kruskal_mode) {
        if (!(s = stage_kruskal(kpad, (uint32_t)n, st, &m)).good()) return s;
        PH0B_TRY(cudaEventRecord(ev_[4], st), "event");
    } else {
        if (!(s = stage_reduce(vals_[cur_], kpad, (uint32_t)n, st, &rst)).good()) return s;
        PH0B_TRY(cudaEventRecord(ev_[4], st), "event");
        m = rst.survivors;
        if (m != n - 1)
            return {PH0B_ERR_CUDA, "internal error: reduction produced " + std::to_string(m) +
                                       " surviving columns, expected " + std::to_string(n - 1)};
        if (!(s = stage_collect(m, kpad, 0, st)).good()) return s;
    }
    PH0B_TRY(cudaEventRecord(ev_[5], st), "event");
    PH0B_TRY(cudaStreamSynchronize(st), "pipeline");
    tr.mark("reduce+collect done");
    if (compress) {
        if (!(s = drain(true)).good()) return s;
        pool_->wait();
        tr.mark("decode done");
        if (tr.on) {
            uint64_t w, dn, np;
            decode_stats(&w, &dn, &np, true);
            fprintf(stderr, "[ph0b trace] pieces %lu: wait %.1f ms, decode %.1f ms (summed over "
                    "%u threads), enqueue blocked %.1f ms\n", (unsigned long)np, w * 1e-6,
                    dn * 1e-6, pool_->threads(), enq_ns * 1e-6);
        }
    }
    PH0B_TRY(cudaStreamSynchronize(copy_stream_), "D2H scale");
    for (size_t i = 1; i < ring_streams_.size(); ++i)
        PH0B_TRY(cudaStreamSynchronize(ring_streams_[i]), "D2H scale");
    tr.mark("D2H done");
    const uint64_t n_scale = h_base[B];
    if (overflow == 1 || (host_scale && n_scale > scale_capacity))
        return {PH0B_ERR_CAPACITY,
                "scale buffer too small: need >= " + std::to_string(n_scale) + " entries"};
    if (overflow)
        return {PH0B_ERR_CUDA, "D2H of D stalled (the copy stream made no progress)"};
    r.times.d2h_bytes = d2h_total;
    r.n_scale = n_scale;
    r.d_uv_sorted = vals_[cur_];
    r.d_scale = dbuf_;
    r.d_death_grade = death_grade_;
    r.d_death_length = death_length_;
    r.d_surv_sorted = surv_sorted_;
    r.n_finite = m;
    r.essential = n - m;
    r.times.reduce_rounds = rst.rounds;
    r.times.reduce_iterations = rst.iterations;
    r.times.columns_scanned = rst.scanned;
    cudaEventElapsedTime(&r.times.distance_ms, ev_[0], ev_[1]);
    cudaEventElapsedTime(&r.times.sort_ms, ev_[1], ev_[2]);
    cudaEventElapsedTime(&r.times.reduce_ms, ev_[3], ev_[4]);
    cudaEventElapsedTime(&r.times.collect_ms, ev_[4], ev_[5]);
    cudaEventElapsedTime(&r.times.total_ms, ev_[0], ev_[5]);
    if (out) *out = r;
    return Status::ok();
}

Status Context::stage_kruskal(uint64_t count, uint32_t n, cudaStream_t st, uint32_t* merges) {
    NvtxRange nvtx_("K6 GPU Kruskal");
    if (n > 65536) return {PH0B_ERR_TOO_LARGE, "union-find forest is limited to 65536 points"};
    uint32_t* d_count = reinterpret_cast<uint32_t*>(d_mapped_ + 250);
    volatile uint32_t* h_count = reinterpret_cast<volatile uint32_t*>(h_mapped_ + 250);
    *h_count = 0;
    const int kl = launch_kruskal(vals_[cur_], keys_[cur_], count, n, scale_, small_ + 2, surv_,
                                  d_count, death_grade_, death_length_, st);
    PH0B_CHECK_LAUNCH("kruskal");
    if (kl < 0) return {PH0B_ERR_CUDA, "kruskal: launch configuration failed"};
    launches += kl;
    PH0B_TRY(cudaStreamSynchronize(st), "kruskal");
    *merges = *h_count;
    return Status::ok();
}

Status Context::reduced_supports(const RunOutputs& r, uint32_t n, bool want_x,
                                 cudaStream_t stream) {
    NvtxRange nvtx_("reduced supports");
    cudaStream_t st = stream ? stream : stream_;
    uint32_t* d_err = reinterpret_cast<uint32_t*>(d_mapped_ + 251);
    volatile uint32_t* h_err = reinterpret_cast<volatile uint32_t*>(h_mapped_ + 251);
    *h_err = 0;
    const int l = launch_reduced_supports(r.d_surv_sorted, (uint32_t)r.n_finite, r.d_uv_sorted,
                                          n, want_x ? lows_ + n : nullptr, lows_, d_err, comp_,
                                          st);
    PH0B_CHECK_LAUNCH("reduced supports");
    if (l < 0) return {PH0B_ERR_CUDA, "reduced supports: launch configuration failed"};
    launches += l;
    PH0B_TRY(cudaStreamSynchronize(st), "reduced supports");
    if (*h_err) return {PH0B_ERR_CUDA, "internal error: a surviving column reduced to zero"};
    return Status::ok();
}

Context* default_context(int device, Status* st) {
    static std::mutex mu;
    static std::map<int, std::unique_ptr<Context>> ctxs;
    std::lock_guard<std::mutex> lk(mu);
    auto it = ctxs.find(device);
    if (it != ctxs.end()) return it->second.get();
    auto c = std::make_unique<Context>(device);
    Status s = c->init();
    if (!s.good()) {
        if (st) *st = s;
        return nullptr;
    }
    Context* p = c.get();
    ctxs[device] = std::move(c);
    return p;
}

}  // namespace ph0b
