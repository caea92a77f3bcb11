// C ABI (include/ph0b.h): validation with the reference's error behaviour, result marshalling.
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/ph0b.h"
#include "colcodec.h"
#include "host_decode.h"
#include "pipeline.h"

using ph0b::Context;
using ph0b::RunOutputs;
using ph0b::Status;
using ph0b::StopAfter;

namespace {

thread_local std::string g_last_error;
thread_local uint64_t g_last_launches = 0;

int fail(const Status& s) {
    g_last_error = s.msg;
    return s.code;
}
int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

// below the bucketed path, a D of at least this many values is still shipped compressed
constexpr uint64_t kStreamMinValues = 1ull << 21;

// smallest edge count taking the bucketed, D-streaming host path (PH0B_OVERLAP_MIN_EDGES)
uint64_t overlap_min_edges() {
    static const uint64_t v = [] {
        const char* e = getenv("PH0B_OVERLAP_MIN_EDGES");
        return e ? (uint64_t)strtoull(e, nullptr, 10) : (1ull << 26);
    }();
    return v;
}

bool overlap_disabled() {
    static const bool v = [] {
        const char* e = getenv("PH0B_OVERLAP");
        return e && e[0] == '0';
    }();
    return v;
}

struct Opts {
    int device = 0;
    uint32_t flags = 0;
    uint32_t workers = 1;
    std::vector<int> devices;  // > 1 entries: the multi-GPU path (multi.cpp)
};

// ph0b_options before ABI 4 ended at `workers`
constexpr uint32_t kOptionsV3Size = 5 * sizeof(uint32_t);

// Validation mirrors the reference's throws: filtration.cpp:10-11 (N > 2^32-1),
// reduction.cpp:134 (workers < 1); PH0B_MAX_POINTS is this build's packing limit.
int parse(const ph0b_options* opt, uint64_t n, uint32_t layout, Opts* o) {
    if (opt && opt->struct_size != 0) {
        if (opt->struct_size < kOptionsV3Size)
            return fail(PH0B_ERR_INVALID_ARGUMENT, "ph0b_options.struct_size too small");
        o->device = opt->device;
        o->flags = opt->flags;
        o->workers = opt->workers;
        if (opt->workers < 1)
            return fail(PH0B_ERR_INVALID_ARGUMENT, "worker count must be at least 1");
        if (opt->struct_size >= sizeof(ph0b_options) && opt->n_gpus > 1) {
            if (opt->n_gpus > 64)
                return fail(PH0B_ERR_INVALID_ARGUMENT, "n_gpus must be at most 64");
            for (uint32_t i = 0; i < opt->n_gpus; ++i)
                o->devices.push_back(opt->devices ? opt->devices[i] : opt->device + (int)i);
        }
    }
    if (layout != PH0B_COL_MAJOR && layout != PH0B_ROW_MAJOR)
        return fail(PH0B_ERR_INVALID_ARGUMENT, "layout must be PH0B_COL_MAJOR or PH0B_ROW_MAJOR");
    if (n > 0xFFFFFFFFull)
        return fail(PH0B_ERR_TOO_LARGE, "point cloud too large for 32-bit vertex indices");
    if ((o->flags & PH0B_FLAG_KRUSKAL) && n > ph0b::kPackedMaxN)
        return fail(PH0B_ERR_TOO_LARGE, "union-find forest is limited to 65536 points");
    if (n > PH0B_MAX_POINTS)
        return fail(PH0B_ERR_TOO_LARGE,
                    "point cloud too large for this build (N <= " +
                        std::to_string(PH0B_MAX_POINTS) + ")");
    return PH0B_OK;
}

// Host buffers of library-allocated results (ph0b_result.scale holds D: up to 8*K bytes, 17 GB
// at C5).  Fresh memory costs one page fault per page on first touch (the kernel zeroes it),
// seconds at C5, so a freed D buffer is kept (at most kIdleMax, LRU) and handed to the next
// call that fits in it; large buffers are anonymous mappings with transparent huge pages
// requested.  ph0b_host_cache_trim() returns the idle ones to the system.
class ResultCache {
public:
    static constexpr size_t kMapMin = size_t(64) << 20;  // below: plain malloc
    static constexpr size_t kIdleMax = 2;

    void* take(size_t bytes) {
        bytes = std::max<size_t>(bytes, 8);
        if (bytes < kMapMin) return std::malloc(bytes);
        {
            std::lock_guard<std::mutex> lk(mu_);
            size_t best = idle_.size();
            for (size_t i = 0; i < idle_.size(); ++i)
                if (idle_[i].second.len >= bytes &&
                    (best == idle_.size() || idle_[i].second.len < idle_[best].second.len))
                    best = i;
            if (best != idle_.size()) {
                const auto e = idle_[best];
                idle_.erase(idle_.begin() + (long)best);
                live_[e.first] = e.second;
                return e.first;
            }
        }
        const size_t len = (bytes + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1);
        void* p = nullptr;
        if (pinned_results()) {  // page-locked: the decoders write it as fast as a caller's
                                 // pinned buffer (an anonymous mapping measured slower)
            if (cudaHostAlloc(&p, len, cudaHostAllocDefault) != cudaSuccess) {
                cudaGetLastError();
                p = nullptr;
            }
        }
        const bool pinned = p != nullptr;
        if (!p) {
            p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
            if (p == MAP_FAILED) return nullptr;
            madvise(p, len, MADV_HUGEPAGE);
        }
        std::lock_guard<std::mutex> lk(mu_);
        live_[p] = Buf{len, pinned};
        return p;
    }
    void give(void* p) {
        if (!p) return;
        std::vector<std::pair<void*, Buf>> drop;
        {
            std::lock_guard<std::mutex> lk(mu_);
            const auto it = live_.find(p);
            if (it == live_.end()) {
                std::free(p);  // a small (malloc) buffer
                return;
            }
            idle_.push_back(*it);
            live_.erase(it);
            while (idle_.size() > kIdleMax) {
                drop.push_back(idle_.front());
                idle_.erase(idle_.begin());
            }
        }
        for (auto& e : drop) release(e);
    }
    void trim() {
        std::vector<std::pair<void*, Buf>> drop;
        {
            std::lock_guard<std::mutex> lk(mu_);
            drop.swap(idle_);
        }
        for (auto& e : drop) release(e);
    }

private:
    struct Buf {
        size_t len;
        bool pinned;  // cudaHostAlloc (else an anonymous mapping)
    };
    static bool pinned_results() {  // PH0B_PINNED_RESULTS=0: anonymous mappings only
        static const bool v = [] {
            const char* e = getenv("PH0B_PINNED_RESULTS");
            return !(e && e[0] == '0');
        }();
        return v;
    }
    static void release(const std::pair<void*, Buf>& e) {
        if (e.second.pinned)
            cudaFreeHost(e.first);
        else
            munmap(e.first, e.second.len);
    }
    std::mutex mu_;
    std::map<void*, Buf> live_;
    std::vector<std::pair<void*, Buf>> idle_;
};

ResultCache& result_cache() {
    static ResultCache* c = new ResultCache();  // never destroyed: results may outlive statics
    return *c;
}

// The multi-GPU path: several devices requested, a cloud big enough to split (the per-rank
// stages cost fixed latency), and not the union-find variant (single GPU by definition).
bool use_multi(const Opts& o, uint64_t n) {
    return o.devices.size() > 1 && !(o.flags & PH0B_FLAG_KRUSKAL) &&
           n * (n - (n > 0)) / 2 >= (uint64_t)o.devices.size() * 4096;
}

// Host-side finiteness check (PointCloud ctor, point_cloud.cpp:15-18) before any device work.
bool all_finite(const double* x, uint64_t count) {
    for (uint64_t i = 0; i < count; ++i)
        if (!std::isfinite(x[i])) return false;
    return true;
}

Context* ctx_for(int device, int* rc) {
    Status st;
    Context* c = ph0b::default_context(device, &st);
    if (!c) *rc = fail(st);
    return c;
}

int copy_out(Context* c, const RunOutputs& r, cudaStream_t s, uint64_t* death_grade,
             double* death_length, double* scale, uint64_t scale_capacity, bool want_scale) {
    if (r.n_finite) {
        if (cudaMemcpyAsync(death_grade, r.d_death_grade, r.n_finite * 8, cudaMemcpyDeviceToHost,
                            s) != cudaSuccess ||
            cudaMemcpyAsync(death_length, r.d_death_length, r.n_finite * 8,
                            cudaMemcpyDeviceToHost, s) != cudaSuccess)
            return fail(PH0B_ERR_CUDA, std::string("D2H bars: ") +
                                           cudaGetErrorString(cudaGetLastError()));
    }
    if (want_scale && r.n_scale) {
        if (!scale || scale_capacity < r.n_scale)
            return fail(PH0B_ERR_CAPACITY, "scale buffer too small: need " +
                                               std::to_string(r.n_scale) + " entries");
        if (cudaMemcpyAsync(scale, r.d_scale, r.n_scale * 8, cudaMemcpyDeviceToHost, s) !=
            cudaSuccess)
            return fail(PH0B_ERR_CUDA, std::string("D2H scale: ") +
                                           cudaGetErrorString(cudaGetLastError()));
    }
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fail(PH0B_ERR_CUDA, std::string("D2H: ") + cudaGetErrorString(e));
    (void)c;
    return PH0B_OK;
}

}  // namespace

namespace ph0b {
int run_multi_gpu(const std::vector<int>& devices, const double* X, uint64_t n, uint64_t d,
                  uint32_t layout, uint64_t* death_grade, double* death_length,
                  uint64_t* n_finite, uint64_t* essential, double* scale,
                  uint64_t scale_capacity, uint64_t* n_scale, ph0b_stage_times* times);
void release_multi_gpu();
int capi_fail(const Status& s) { return fail(s); }
int capi_fail(int code, const std::string& msg) { return fail(code, msg); }
void capi_set_launches(uint64_t n) { g_last_launches = n; }
}  // namespace ph0b

extern "C" {

const char* ph0b_last_error(void) { return g_last_error.c_str(); }
uint32_t ph0b_abi_version(void) { return PH0B_ABI_VERSION; }
uint64_t ph0b_last_launch_count(void) { return g_last_launches; }

void* ph0b_host_alloc(uint64_t bytes) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}
void ph0b_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

int ph0b_context_create(int device, ph0b_context** out) {
    if (!out) return fail(PH0B_ERR_INVALID_ARGUMENT, "null context pointer");
    auto* c = new (std::nothrow) Context(device);
    if (!c) return fail(PH0B_ERR_OUT_OF_MEMORY, "host allocation failed");
    Status s = c->init();
    if (!s.good()) {
        delete c;
        return fail(s);
    }
    *out = reinterpret_cast<ph0b_context*>(c);
    return PH0B_OK;
}

void ph0b_context_destroy(ph0b_context* ctx) {
    if (!ctx) return;
    ph0b::shard_scratch_release(reinterpret_cast<Context*>(ctx));
    delete reinterpret_cast<Context*>(ctx);
}

int ph0b_context_reserve(ph0b_context* ctx, uint64_t n, uint64_t d) {
    if (!ctx) return fail(PH0B_ERR_INVALID_ARGUMENT, "null context");
    Context* c = reinterpret_cast<Context*>(ctx);
    std::lock_guard<std::mutex> lk(c->mu);
    Status s = c->reserve(n, d);
    return s.good() ? PH0B_OK : fail(s);
}

uint64_t ph0b_context_workspace_bytes(const ph0b_context* ctx) {
    if (!ctx) return 0;
    return reinterpret_cast<const Context*>(ctx)->workspace_bytes();
}

int ph0b_run_device(ph0b_context* ctx, const double* dX, uint64_t n, uint64_t d, uint32_t layout,
                    void* stream, ph0b_device_result* out) {
    if (!ctx) return fail(PH0B_ERR_INVALID_ARGUMENT, "null context");
    Opts o;
    int rc = parse(nullptr, n, layout, &o);
    if (rc) return rc;
    if (n * d && !dX) return fail(PH0B_ERR_INVALID_ARGUMENT, "null point cloud");
    Context* c = reinterpret_cast<Context*>(ctx);
    std::lock_guard<std::mutex> lk(c->mu);
    RunOutputs r;
    Status s = c->run(dX, n, d, layout, static_cast<cudaStream_t>(stream), StopAfter::Barcode,
                      false, &r);
    g_last_launches = c->launches;
    if (!s.good()) return fail(s);
    if (out) {
        out->n_finite = r.n_finite;
        out->essential_count = r.essential;
        out->n_scale = r.n_scale;
        out->d_scale = r.d_scale;
        out->d_death_grade = r.d_death_grade;
        out->d_death_length = r.d_death_length;
        out->times = r.times;
    }
    return PH0B_OK;
}

int ph0b_generate_uniform_cloud_device(ph0b_context* ctx, uint64_t n, uint64_t dim,
                                       uint64_t seed, double* d_out, void* stream) {
    if (!ctx) return fail(PH0B_ERR_INVALID_ARGUMENT, "null context");
    if (n > 0 && dim < 1)
        return fail(PH0B_ERR_INVALID_ARGUMENT, "point dimension must be at least 1");
    if (n * dim == 0) return PH0B_OK;
    if (!d_out) return fail(PH0B_ERR_INVALID_ARGUMENT, "null output");
    Context* c = reinterpret_cast<Context*>(ctx);
    std::lock_guard<std::mutex> lk(c->mu);
    cudaSetDevice(c->device());
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c->own_stream();
    unsigned long long *dz = nullptr, *hz = nullptr;
    if (cudaMalloc(&dz, 65 * 8) != cudaSuccess || cudaMallocHost(&hz, 65 * 8) != cudaSuccess) {
        if (dz) cudaFree(dz);
        cudaGetLastError();
        return fail(PH0B_ERR_OUT_OF_MEMORY, "generator scratch");
    }
    const int l = ph0b::launch_uniform_cloud(n, dim, seed, d_out, dz, hz, s, c->num_sms());
    cudaFree(dz);
    cudaFreeHost(hz);
    g_last_launches = l > 0 ? (uint64_t)l : 0;
    if (l == -2) return fail(PH0B_ERR_INVALID_ARGUMENT, "more than 64 zero draws (impossible in practice)");
    if (l < 0 || cudaGetLastError() != cudaSuccess) return fail(PH0B_ERR_CUDA, "generator kernel");
    return PH0B_OK;
}

int ph0b_decode_deltas(const uint32_t* deltas, const uint64_t* bases, const uint8_t* raw,
                       uint64_t n, uint32_t chunk, uint64_t* out) {
    if (n == 0) return PH0B_OK;
    if (!deltas || !bases || !raw || !out || chunk == 0)
        return fail(PH0B_ERR_INVALID_ARGUMENT, "null argument or zero chunk");
    ph0b::decode_chunk(ph0b::DecodeTask{deltas, bases, raw, out, n, chunk});
    return PH0B_OK;
}

int ph0b_decode_packed(const uint8_t* packed, const uint64_t* bases, const uint8_t* widths,
                       const uint32_t* offs, uint64_t n, uint32_t chunk, uint64_t* out) {
    if (n == 0) return PH0B_OK;
    if (!packed || !bases || !widths || !offs || !out || chunk == 0)
        return fail(PH0B_ERR_INVALID_ARGUMENT, "null argument or zero chunk");
    const uint64_t nch = (n + chunk - 1) / chunk;
    for (uint64_t j = 0; j < nch; ++j)
        if (widths[j] != 0 && widths[j] != 3 && widths[j] != 4)
            return fail(PH0B_ERR_INVALID_ARGUMENT, "chunk width must be 0, 3 or 4");
    ph0b::DecodeTask t{nullptr, bases, nullptr, out, n, chunk};
    t.widths = widths;
    t.poff = offs;
    t.packed = packed;
    ph0b::decode_chunk(t);
    return PH0B_OK;
}

int ph0b_scale_to_host(ph0b_context* ctx, const double* d_scale, uint64_t n, double* host_scale,
                       uint64_t capacity, void* stream, uint64_t* bytes_moved) {
    if (bytes_moved) *bytes_moved = 0;
    if (n == 0) return PH0B_OK;
    if (!ctx || !d_scale || !host_scale)
        return fail(PH0B_ERR_INVALID_ARGUMENT, "null context or buffer");
    if (capacity < n)
        return fail(PH0B_ERR_CAPACITY, "scale buffer too small: need " + std::to_string(n) +
                                           " entries");
    Context* c = reinterpret_cast<Context*>(ctx);
    std::lock_guard<std::mutex> lk(c->mu);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c->own_stream();
    uint64_t moved = n * 8;
    if (n >= kStreamMinValues && c->compressed_d2h_ok()) {
        const Status st = c->stream_scale(d_scale, n, host_scale, capacity, s, &moved);
        if (!st.good()) return fail(st);
    } else {
        if (cudaMemcpyAsync(host_scale, d_scale, n * 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return fail(PH0B_ERR_CUDA, std::string("D2H scale: ") +
                                           cudaGetErrorString(cudaGetLastError()));
    }
    if (bytes_moved) *bytes_moved = moved;
    return PH0B_OK;
}

}  // extern "C"

namespace {

// Host X -> host outputs on a context whose lock the caller holds (ph0b_run_host,
// ph0b_h0_barcode_into); kruskal: the union-find barcode instead of the column reduction.
int run_host_locked(Context* c, const double* X, uint64_t n, uint64_t d, uint32_t layout,
                    void* stream, uint64_t* death_grade, double* death_length,
                    uint64_t* n_finite, uint64_t* essential_count, double* scale,
                    uint64_t scale_capacity, uint64_t* n_scale, ph0b_stage_times* times,
                    bool kruskal) {
    int rc = PH0B_OK;
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c->own_stream();
    RunOutputs r;
    struct ModeGuard {
        Context* c;
        ~ModeGuard() { c->kruskal_mode = false; }
    } mode_guard{c};
    c->kruskal_mode = kruskal;
    const uint64_t k = n * (n - (n > 0)) / 2;
    // Large clouds returning D: overlap the D2H of D with the sort (key-range buckets).
    const bool overlap = scale && k >= overlap_min_edges() && !overlap_disabled();
    Status st = overlap ? c->run_host_overlapped(X, n, d, layout, s, scale, scale_capacity, &r)
                        : c->run_host_input(X, n, d, layout, s, StopAfter::Barcode, false, &r);
    g_last_launches = c->launches;
    if (!st.good()) return fail(st);
    // mid-size D (not bucketed): still shipped compressed through the ring when possible
    const bool streamed = scale && !overlap && r.n_scale >= kStreamMinValues &&
                          c->compressed_d2h_ok();
    rc = copy_out(c, r, s, death_grade, death_length, scale, scale_capacity,
                  scale != nullptr && !overlap && !streamed);
    if (rc) return rc;
    uint64_t moved = 0;
    if (streamed) {
        st = c->stream_scale(r.d_scale, r.n_scale, scale, scale_capacity, s, &moved);
        if (!st.good()) return fail(st);
    }
    r.times.d2h_bytes = (overlap ? r.times.d2h_bytes
                                 : (streamed ? moved : (scale ? r.n_scale * 8 : 0))) +
                        r.n_finite * 16;  // + the bars
    if (n_finite) *n_finite = r.n_finite;
    if (essential_count) *essential_count = r.essential;
    if (n_scale) *n_scale = r.n_scale;
    if (times) *times = r.times;
    return PH0B_OK;
}

}  // namespace

extern "C" {

int ph0b_run_host(ph0b_context* ctx, const double* X, uint64_t n, uint64_t d, uint32_t layout,
                  void* stream, uint64_t* death_grade, double* death_length, uint64_t* n_finite,
                  uint64_t* essential_count, double* scale, uint64_t scale_capacity,
                  uint64_t* n_scale, ph0b_stage_times* times) {
    if (!ctx) return fail(PH0B_ERR_INVALID_ARGUMENT, "null context");
    Opts o;
    int rc = parse(nullptr, n, layout, &o);
    if (rc) return rc;
    if (n * d && !X) return fail(PH0B_ERR_INVALID_ARGUMENT, "null point cloud");
    if (!all_finite(X, n * d))
        return fail(PH0B_ERR_NONFINITE, "point cloud contains non-finite coordinates");
    Context* c = reinterpret_cast<Context*>(ctx);
    std::lock_guard<std::mutex> lk(c->mu);
    return run_host_locked(c, X, n, d, layout, stream, death_grade, death_length, n_finite,
                           essential_count, scale, scale_capacity, n_scale, times, false);
}

int ph0b_h0_barcode_into(const double* X, uint64_t n, uint64_t d, uint32_t layout,
                         const ph0b_options* opt, uint64_t* death_grade, double* death_length,
                         uint64_t* n_finite, uint64_t* essential_count, double* scale,
                         uint64_t scale_capacity, uint64_t* n_scale, ph0b_stage_times* times) {
    Opts o;
    int rc = parse(opt, n, layout, &o);
    if (rc) return rc;
    if (n * d && !X) return fail(PH0B_ERR_INVALID_ARGUMENT, "null point cloud");
    if (!all_finite(X, n * d))
        return fail(PH0B_ERR_NONFINITE, "point cloud contains non-finite coordinates");
    if (o.flags & PH0B_FLAG_NO_SCALE) scale = nullptr;
    if (use_multi(o, n))
        return ph0b::run_multi_gpu(o.devices, X, n, d, layout, death_grade, death_length,
                                   n_finite, essential_count, scale, scale_capacity, n_scale,
                                   times);
    Context* c = ctx_for(o.device, &rc);
    if (!c) return rc;
    std::lock_guard<std::mutex> lk(c->mu);
    return run_host_locked(c, X, n, d, layout, nullptr, death_grade, death_length, n_finite,
                           essential_count, scale, scale_capacity, n_scale, times,
                           (o.flags & PH0B_FLAG_KRUSKAL) != 0);
}

int ph0b_h0_barcode(const double* X, uint64_t n, uint64_t d, uint32_t layout,
                    const ph0b_options* opt, ph0b_result* out) {
    if (!out) return fail(PH0B_ERR_INVALID_ARGUMENT, "null result");
    std::memset(out, 0, sizeof(*out));
    Opts o;
    int rc = parse(opt, n, layout, &o);
    if (rc) return rc;
    if (n * d && !X) return fail(PH0B_ERR_INVALID_ARGUMENT, "null point cloud");
    if (!all_finite(X, n * d))
        return fail(PH0B_ERR_NONFINITE, "point cloud contains non-finite coordinates");
    const bool want_scale = !(o.flags & PH0B_FLAG_NO_SCALE);
    const uint64_t k = n * (n - (n > 0)) / 2;
    if (use_multi(o, n)) {
        out->death_grade = static_cast<uint64_t*>(std::malloc(std::max<uint64_t>(1, n) * 8));
        out->death_length = static_cast<double*>(std::malloc(std::max<uint64_t>(1, n) * 8));
        if (want_scale) out->scale = static_cast<double*>(result_cache().take(k * 8));
        if (!out->death_grade || !out->death_length || (want_scale && !out->scale)) {
            ph0b_result_free(out);
            return fail(PH0B_ERR_OUT_OF_MEMORY, "host allocation of the result failed");
        }
        rc = ph0b::run_multi_gpu(o.devices, X, n, d, layout, out->death_grade,
                                 out->death_length, &out->n_finite, &out->essential_count,
                                 out->scale, want_scale ? k : 0, &out->n_scale, &out->times);
        if (rc) {
            const std::string msg = g_last_error;
            ph0b_result_free(out);
            std::memset(out, 0, sizeof(*out));
            return fail(rc, msg);
        }
        return PH0B_OK;
    }
    Context* c = ctx_for(o.device, &rc);
    if (!c) return rc;
    std::lock_guard<std::mutex> lk(c->mu);
    cudaStream_t s = c->own_stream();
    RunOutputs r;
    // Large clouds returning D take the same bucketed path as ph0b_run_host: D streams to the
    // host while the sort is still running, decoded straight into the result buffer (sized by
    // K >= |D|; a reused buffer from the result cache has no page faults left to take).
    const bool overlap = want_scale && k >= overlap_min_edges() && !overlap_disabled();
    if (overlap) {
        out->scale = static_cast<double*>(result_cache().take(k * 8));
        if (!out->scale) return fail(PH0B_ERR_OUT_OF_MEMORY, "host allocation of D failed");
    }
    c->kruskal_mode = (o.flags & PH0B_FLAG_KRUSKAL) != 0;
    Status st = overlap ? c->run_host_overlapped(X, n, d, layout, s, out->scale, k, &r)
                        : c->run_host_input(X, n, d, layout, s, StopAfter::Barcode, false, &r);
    c->kruskal_mode = false;
    g_last_launches = c->launches;
    if (!st.good()) {
        ph0b_result_free(out);
        return fail(st);
    }
    out->death_grade = static_cast<uint64_t*>(std::malloc(std::max<uint64_t>(1, r.n_finite) * 8));
    out->death_length = static_cast<double*>(std::malloc(std::max<uint64_t>(1, r.n_finite) * 8));
    if (want_scale && !overlap)
        out->scale = static_cast<double*>(result_cache().take(r.n_scale * 8));
    if (!out->death_grade || !out->death_length || (want_scale && !out->scale)) {
        ph0b_result_free(out);
        return fail(PH0B_ERR_OUT_OF_MEMORY, "host allocation of the result failed");
    }
    if (overlap) {  // D is on the host already; the bars follow
        rc = copy_out(c, r, s, out->death_grade, out->death_length, nullptr, 0, false);
        if (rc) {
            ph0b_result_free(out);
            return rc;
        }
        r.times.d2h_bytes += r.n_finite * 16;
        out->n_finite = r.n_finite;
        out->essential_count = r.essential;
        out->n_scale = r.n_scale;
        out->times = r.times;
        return PH0B_OK;
    }
    // a large D goes compressed through the pinned ring and is decoded by host threads into
    // the (pageable) result, instead of one pageable-memory DMA
    const bool streamed = want_scale && r.n_scale >= kStreamMinValues && c->compressed_d2h_ok();
    rc = copy_out(c, r, s, out->death_grade, out->death_length, out->scale, r.n_scale,
                  want_scale && !streamed);
    if (!rc && streamed) {
        uint64_t moved = 0;
        const Status ss = c->stream_scale(r.d_scale, r.n_scale, out->scale, r.n_scale, s, &moved);
        if (!ss.good()) rc = fail(ss);
    }
    if (rc) {
        ph0b_result_free(out);
        return rc;
    }
    out->n_finite = r.n_finite;
    out->essential_count = r.essential;
    out->n_scale = r.n_scale;
    out->times = r.times;
    return PH0B_OK;
}

int ph0b_kruskal_barcode(const double* X, uint64_t n, uint64_t d, uint32_t layout,
                         const ph0b_options* opt, ph0b_result* out) {
    ph0b_options o{};
    if (opt && opt->struct_size != 0) {
        o = *opt;
    } else {  // all defaults (struct_size 0 means defaults, as in parse())
        o.struct_size = sizeof(o);
        o.workers = 1;
        o.pivoting = 1;
    }
    o.flags |= PH0B_FLAG_KRUSKAL;
    return ph0b_h0_barcode(X, n, d, layout, &o, out);
}

void ph0b_scale_release(double* scale) { result_cache().give(scale); }

void ph0b_host_cache_trim(void) { result_cache().trim(); }

void ph0b_release_resources(void) {
    ph0b::release_multi_gpu();
    result_cache().trim();
}

void ph0b_result_free(ph0b_result* r) {
    if (!r) return;
    std::free(r->death_grade);
    std::free(r->death_length);
    result_cache().give(r->scale);
    r->death_grade = nullptr;
    r->death_length = nullptr;
    r->scale = nullptr;
}

int ph0b_pairwise_distances(const double* X, uint64_t n, uint64_t d, uint32_t layout,
                            const ph0b_options* opt, double* lengths) {
    Opts o;
    int rc = parse(opt, n, layout, &o);
    if (rc) return rc;
    if (n >= 2 && !lengths) return fail(PH0B_ERR_INVALID_ARGUMENT, "null output");
    if (n * d && !X) return fail(PH0B_ERR_INVALID_ARGUMENT, "null point cloud");
    if (!all_finite(X, n * d))
        return fail(PH0B_ERR_NONFINITE, "point cloud contains non-finite coordinates");
    Context* c = ctx_for(o.device, &rc);
    if (!c) return rc;
    std::lock_guard<std::mutex> lk(c->mu);
    cudaStream_t s = c->own_stream();
    RunOutputs r;
    Status st = c->run_host_input(X, n, d, layout, s, StopAfter::Distance, false, &r);
    g_last_launches = c->launches;
    if (!st.good()) return fail(st);
    if (r.k && cudaMemcpyAsync(lengths, r.d_lengths_umajor, r.k * 8, cudaMemcpyDeviceToHost, s) !=
                   cudaSuccess)
        return fail(PH0B_ERR_CUDA, "D2H lengths");
    if (cudaStreamSynchronize(s) != cudaSuccess) return fail(PH0B_ERR_CUDA, "D2H lengths");
    return PH0B_OK;
}

int ph0b_build_filtration(const double* X, uint64_t n, uint64_t d, uint32_t layout,
                          const ph0b_options* opt, uint32_t* u, uint32_t* v, uint64_t* grade,
                          double* scale, uint64_t* n_scale) {
    Opts o;
    int rc = parse(opt, n, layout, &o);
    if (rc) return rc;
    if (n * d && !X) return fail(PH0B_ERR_INVALID_ARGUMENT, "null point cloud");
    if (!all_finite(X, n * d))
        return fail(PH0B_ERR_NONFINITE, "point cloud contains non-finite coordinates");
    Context* c = ctx_for(o.device, &rc);
    if (!c) return rc;
    std::lock_guard<std::mutex> lk(c->mu);
    cudaStream_t s = c->own_stream();
    RunOutputs r;
    Status st = c->run_host_input(X, n, d, layout, s, StopAfter::Filtration, true, &r);
    g_last_launches = c->launches;
    if (!st.good()) return fail(st);
    if (n_scale) *n_scale = r.n_scale;
    if (r.k == 0) return PH0B_OK;
    std::vector<uint32_t> uv(r.k), g(r.k);
    if (cudaMemcpyAsync(uv.data(), r.d_uv_sorted, r.k * 4, cudaMemcpyDeviceToHost, s) ||
        cudaMemcpyAsync(g.data(), r.d_grade, r.k * 4, cudaMemcpyDeviceToHost, s) ||
        (scale && cudaMemcpyAsync(scale, r.d_scale, r.n_scale * 8, cudaMemcpyDeviceToHost, s)) ||
        cudaStreamSynchronize(s))
        return fail(PH0B_ERR_CUDA, "D2H filtration");
    for (uint64_t i = 0; i < r.k; ++i) {
        uint32_t a, b;
        ph0b::col_rows(uv[i], n, a, b);
        if (u) u[i] = a;
        if (v) v[i] = b;
        if (grade) grade[i] = g[i];
    }
    return PH0B_OK;
}

}  // extern "C"

namespace {

// The pipeline, then the survivors' reduced supports (claimed lows, and the other row when
// xs != nullptr) in filtration order; cols (optional) receives each survivor's column index.
int supports_impl(const double* X, uint64_t n, uint64_t d, uint32_t layout,
                  const ph0b_options* opt, uint64_t* cols, uint32_t* xs, uint32_t* lows,
                  uint64_t* m_out) {
    Opts o;
    int rc = parse(opt, n, layout, &o);
    if (rc) return rc;
    if (n * d && !X) return fail(PH0B_ERR_INVALID_ARGUMENT, "null point cloud");
    if (!all_finite(X, n * d))
        return fail(PH0B_ERR_NONFINITE, "point cloud contains non-finite coordinates");
    Context* c = ctx_for(o.device, &rc);
    if (!c) return rc;
    std::lock_guard<std::mutex> lk(c->mu);
    cudaStream_t s = c->own_stream();
    RunOutputs r;
    Status st = c->run_host_input(X, n, d, layout, s, StopAfter::Barcode, false, &r);
    if (!st.good()) return fail(st);
    if (m_out) *m_out = r.n_finite;
    if (r.n_finite == 0) return PH0B_OK;
    st = c->reduced_supports(r, (uint32_t)n, xs != nullptr, s);
    g_last_launches = c->launches;
    if (!st.good()) return fail(st);
    const uint64_t m = r.n_finite;
    std::vector<uint32_t> surv(cols ? m : 0);
    if ((lows && cudaMemcpy(lows, c->lows_buffer(), m * 4, cudaMemcpyDeviceToHost)) ||
        (xs && cudaMemcpy(xs, c->lows_buffer() + n, m * 4, cudaMemcpyDeviceToHost)) ||
        (cols && cudaMemcpy(surv.data(), r.d_surv_sorted, m * 4, cudaMemcpyDeviceToHost)))
        return fail(PH0B_ERR_CUDA, "D2H reduced supports");
    for (uint64_t i = 0; cols && i < m; ++i) cols[i] = surv[i];
    return PH0B_OK;
}

}  // namespace

extern "C" {

int ph0b_claimed_lows(const double* X, uint64_t n, uint64_t d, uint32_t layout,
                      const ph0b_options* opt, uint32_t* lows, uint64_t* n_lows) {
    if (n >= 2 && !lows) return fail(PH0B_ERR_INVALID_ARGUMENT, "null output");
    return supports_impl(X, n, d, layout, opt, nullptr, nullptr, lows, n_lows);
}

int ph0b_reduced_supports(const double* X, uint64_t n, uint64_t d, uint32_t layout,
                          const ph0b_options* opt, uint64_t* columns, uint32_t* rows_lo,
                          uint32_t* rows_hi, uint64_t* n_columns) {
    if (n >= 2 && (!columns || !rows_lo || !rows_hi))
        return fail(PH0B_ERR_INVALID_ARGUMENT, "null output");
    return supports_impl(X, n, d, layout, opt, columns, rows_lo, rows_hi, n_columns);
}

}  // extern "C"
