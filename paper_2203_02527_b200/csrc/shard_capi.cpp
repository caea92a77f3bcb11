// C ABI of the sharded (multi-GPU) pipeline stages — one ph0b_context per rank; the caller
// (paper_2203_02527_b200/sharded.py) moves data between ranks with NCCL (torch.distributed).
// K1 row blocks per rank (no communication), splitter partition + one
// all-to-all-v exchange, local sort/unique (D sharded, contiguous in global order), local
// column reduction per key range, then a final reduction over the gathered survivors (exact
// by the cycle property: a column that is a cycle within its own range is a cycle globally).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <string>
#include <mutex>
#include <vector>

#include "../../include/ph0b.h"
#include "kernels.h"
#include "pipeline.h"

using ph0b::Context;
using ph0b::Status;

namespace ph0b {
// defined in capi.cpp
int capi_fail(const Status& s);
int capi_fail(int code, const std::string& msg);
void capi_set_launches(uint64_t n);
}  // namespace ph0b

namespace {

struct ShardScratch {
    uint64_t* d_spl = nullptr;      // splitters (<= 255)
    uint64_t* d_totals = nullptr;   // per-part totals
    uint64_t* d_bminmax = nullptr;  // per-part [min | max]
    uint16_t* d_table = nullptr;    // partition bucket lookup table
    uint32_t* d_counts = nullptr;   // per (tile, part)
    uint64_t counts_cap = 0;
    uint64_t* d_sample = nullptr;
    uint64_t sample_cap = 0;
    uint32_t* d_cand_uv = nullptr;  // candidate columns of this rank
    uint64_t cand_cap = 0;
    uint64_t local_count = 0;       // edges produced by shard_distances
    uint64_t local_kmin = 0, local_kmax = 0;
    // peer-memory exchange: per-part local layout starts and the received slice's buffer
    std::vector<uint64_t> starts;   // [parts] from ph0b_shard_partition_count
    uint64_t* d_peer = nullptr;     // [2][256] adjusted destination byte addresses
    int recv_buffer = 0;            // ping-pong buffer holding the received slice
};

// One scratch per context.  A std::map: its elements never move, so the reference a rank
// thread holds stays valid while other threads add their contexts' scratch (the in-process
// multi-GPU path runs one thread per context).
std::mutex g_scratch_mu;
std::map<Context*, ShardScratch>& all_scratch() {
    static auto* all = new std::map<Context*, ShardScratch>();  // outlives static teardown
    return *all;
}

ShardScratch& scratch(Context* c) {
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    return all_scratch()[c];
}

cudaStream_t pick(Context* c, void* stream) {
    return stream ? static_cast<cudaStream_t>(stream) : c->own_stream();
}

int ensure(void** p, uint64_t* cap, uint64_t bytes) {
    if (bytes <= *cap && *p) return PH0B_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    if (cudaMalloc(p, std::max<uint64_t>(bytes, 256)) != cudaSuccess) {
        cudaGetLastError();
        *cap = 0;
        return ph0b::capi_fail(PH0B_ERR_OUT_OF_MEMORY, "device allocation failed (shard)");
    }
    *cap = std::max<uint64_t>(bytes, 256);
    return PH0B_OK;
}

// Device scratch of the partition stages and the splitters on the device.
int partition_setup(Context* c, ShardScratch& sc, const uint64_t* splitters, uint32_t parts,
                    cudaStream_t st) {
    uint64_t cap = 0;
    int rc = 0;
    if (!sc.d_spl) {
        if ((rc = ensure(reinterpret_cast<void**>(&sc.d_spl), &cap, 256 * 8))) return rc;
        cap = 0;
        if ((rc = ensure(reinterpret_cast<void**>(&sc.d_totals), &cap, 512 * 8))) return rc;
        cap = 0;
        if ((rc = ensure(reinterpret_cast<void**>(&sc.d_bminmax), &cap, 512 * 8))) return rc;
        cap = 0;
        if ((rc = ensure(reinterpret_cast<void**>(&sc.d_table), &cap,
                         ph0b::partition_table_bytes())))
            return rc;
    }
    const uint64_t words = ph0b::partition_scratch_words(sc.local_count, parts);
    if ((rc = ensure(reinterpret_cast<void**>(&sc.d_counts), &sc.counts_cap, words * 4 + 4)))
        return rc;
    (void)c;
    if (parts > 1 && cudaMemcpyAsync(sc.d_spl, splitters, (parts - 1) * 8,
                                     cudaMemcpyHostToDevice, st))
        return ph0b::capi_fail(PH0B_ERR_CUDA, "H2D splitters");
    return PH0B_OK;
}

// Per-part counts and key bounds back to the host; the local layout starts (align 1).
int read_partition(ShardScratch& sc, uint32_t parts, cudaStream_t st, uint64_t* counts,
                   uint64_t* part_min, uint64_t* part_max) {
    std::vector<uint64_t> tot(parts), mm(2 * parts);
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpyAsync(tot.data(), sc.d_totals, parts * 8, cudaMemcpyDeviceToHost, st) ||
        cudaMemcpyAsync(mm.data(), sc.d_bminmax, 2 * parts * 8, cudaMemcpyDeviceToHost, st) ||
        cudaStreamSynchronize(st))
        return ph0b::capi_fail(PH0B_ERR_CUDA, "shard partition");
    sc.starts.assign(parts, 0);
    for (uint32_t b = 1; b < parts; ++b) sc.starts[b] = sc.starts[b - 1] + tot[b - 1];
    if (counts) std::memcpy(counts, tot.data(), parts * 8);
    if (part_min) std::memcpy(part_min, mm.data(), parts * 8);
    if (part_max) std::memcpy(part_max, mm.data() + parts, parts * 8);
    return PH0B_OK;
}


}  // namespace

namespace ph0b {
// Frees the shard scratch of a context being destroyed (called by ph0b_context_destroy).
void shard_scratch_release(Context* c) {
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    auto& all = all_scratch();
    const auto it = all.find(c);
    if (it == all.end()) return;
    ShardScratch& sc = it->second;
    cudaSetDevice(c->device());
    void* ps[] = {sc.d_spl, sc.d_totals, sc.d_bminmax, sc.d_table, sc.d_counts,
                  sc.d_sample, sc.d_cand_uv, sc.d_peer};
    for (void* p : ps)
        if (p) cudaFree(p);
    all.erase(it);
}
}  // namespace ph0b

extern "C" {

int ph0b_shard_distances(ph0b_context* ctx, const double* dX, uint64_t n, uint64_t d,
                         uint32_t layout, uint64_t u_lo, uint64_t u_hi, void* stream,
                         uint64_t* count, uint64_t* kmin, uint64_t* kmax) {
    if (!ctx) return ph0b::capi_fail(PH0B_ERR_INVALID_ARGUMENT, "null context");
    Context* c = reinterpret_cast<Context*>(ctx);
    std::lock_guard<std::mutex> lk(c->mu);
    if (n > PH0B_MAX_POINTS) return ph0b::capi_fail(PH0B_ERR_TOO_LARGE, "point cloud too large");
    if (u_hi > n) u_hi = n;
    if (u_lo > u_hi) u_lo = u_hi;
    const uint64_t local = ph0b::row_base(u_hi, n) - ph0b::row_base(u_lo, n);
    Status s = c->reserve_points(n, d);
    if (s.good()) s = c->reserve_edges(local);
    if (!s.good()) return ph0b::capi_fail(s);
    c->launches = 0;
    uint64_t cnt = 0, lo = ~0ull, hi = 0;
    s = c->stage_distances(dX, n, d, layout, u_lo, u_hi, pick(c, stream), &cnt, &lo, &hi);
    ph0b::capi_set_launches(c->launches);
    if (!s.good()) return ph0b::capi_fail(s);
    scratch(c).local_count = cnt;
    scratch(c).local_kmin = lo;
    scratch(c).local_kmax = hi;
    if (count) *count = cnt;
    if (kmin) *kmin = lo;
    if (kmax) *kmax = hi;
    return PH0B_OK;
}

int ph0b_shard_sample(ph0b_context* ctx, uint64_t s, uint64_t* out_host) {
    if (!ctx) return ph0b::capi_fail(PH0B_ERR_INVALID_ARGUMENT, "null context");
    Context* c = reinterpret_cast<Context*>(ctx);
    std::lock_guard<std::mutex> lk(c->mu);
    ShardScratch& sc = scratch(c);
    if (s == 0 || sc.local_count == 0) return PH0B_OK;
    s = std::min<uint64_t>(s, sc.local_count);
    int rc = ensure(reinterpret_cast<void**>(&sc.d_sample), &sc.sample_cap, s * 8);
    if (rc) return rc;
    cudaStream_t st = c->own_stream();
    ph0b::launch_sample(c->keys(0), sc.local_count, s, sc.d_sample, st);
    if (cudaMemcpyAsync(out_host, sc.d_sample, s * 8, cudaMemcpyDeviceToHost, st) ||
        cudaStreamSynchronize(st))
        return ph0b::capi_fail(PH0B_ERR_CUDA, "shard sample");
    return PH0B_OK;
}

int ph0b_shard_partition(ph0b_context* ctx, const uint64_t* splitters, uint32_t parts,
                         void* stream, uint64_t** d_keys_send, uint32_t** d_vals_send,
                         uint64_t* counts, uint64_t* part_min, uint64_t* part_max) {
    if (!ctx) return ph0b::capi_fail(PH0B_ERR_INVALID_ARGUMENT, "null context");
    Context* c = reinterpret_cast<Context*>(ctx);
    std::lock_guard<std::mutex> lk(c->mu);
    if (parts < 1 || parts > 256)
        return ph0b::capi_fail(PH0B_ERR_INVALID_ARGUMENT, "parts must be in [1, 256]");
    ShardScratch& sc = scratch(c);
    cudaStream_t st = pick(c, stream);
    int rc = partition_setup(c, sc, splitters, parts, st);
    if (rc) return rc;
    c->launches = ph0b::launch_partition(c->keys(0), c->vals(0), sc.local_count, sc.d_spl, parts,
                                         sc.d_counts, sc.d_totals, sc.d_bminmax, c->keys(1),
                                         c->vals(1), st, 1, sc.local_kmin, sc.local_kmax,
                                         splitters, sc.d_table);
    if (c->launches < 0) return ph0b::capi_fail(PH0B_ERR_CUDA, "shard partition: launch failed");
    ph0b::capi_set_launches(c->launches);
    if ((rc = read_partition(sc, parts, st, counts, part_min, part_max))) return rc;
    if (d_keys_send) *d_keys_send = c->keys(1);
    if (d_vals_send) *d_vals_send = c->vals(1);
    return PH0B_OK;
}

int ph0b_shard_partition_count(ph0b_context* ctx, const uint64_t* splitters, uint32_t parts,
                               void* stream, uint64_t* counts, uint64_t* part_min,
                               uint64_t* part_max) {
    if (!ctx) return ph0b::capi_fail(PH0B_ERR_INVALID_ARGUMENT, "null context");
    Context* c = reinterpret_cast<Context*>(ctx);
    std::lock_guard<std::mutex> lk(c->mu);
    if (parts < 1 || parts > 256)
        return ph0b::capi_fail(PH0B_ERR_INVALID_ARGUMENT, "parts must be in [1, 256]");
    ShardScratch& sc = scratch(c);
    cudaStream_t st = pick(c, stream);
    int rc = partition_setup(c, sc, splitters, parts, st);
    if (rc) return rc;
    c->launches = ph0b::launch_partition_count(c->keys(0), sc.local_count, sc.d_spl, parts,
                                               sc.d_counts, sc.d_totals, sc.d_bminmax,
                                               c->keys(1), c->vals(1), st, 1, sc.local_kmin,
                                               sc.local_kmax, splitters, sc.d_table);
    ph0b::capi_set_launches(c->launches);
    return read_partition(sc, parts, st, counts, part_min, part_max);
}

int ph0b_shard_recv_peer(ph0b_context* ctx, uint64_t count, uint64_t** d_keys,
                         uint32_t** d_vals) {
    if (!ctx) return ph0b::capi_fail(PH0B_ERR_INVALID_ARGUMENT, "null context");
    Context* c = reinterpret_cast<Context*>(ctx);
    std::lock_guard<std::mutex> lk(c->mu);
    Status s = c->reserve_recv(count, 1);  // buffer 0 still holds the local edges
    if (!s.good()) return ph0b::capi_fail(s);
    if (cudaDeviceSynchronize() != cudaSuccess)  // peers may write as soon as they see it
        return ph0b::capi_fail(PH0B_ERR_CUDA, "shard recv");
    scratch(c).recv_buffer = 1;
    if (d_keys) *d_keys = c->keys(1);
    if (d_vals) *d_vals = c->vals(1);
    return PH0B_OK;
}

int ph0b_shard_scatter_peers(ph0b_context* ctx, uint32_t parts, const uint64_t* dst_keys,
                             const uint64_t* dst_vals, const uint64_t* dst_offsets,
                             void* stream) {
    if (!ctx) return ph0b::capi_fail(PH0B_ERR_INVALID_ARGUMENT, "null context");
    Context* c = reinterpret_cast<Context*>(ctx);
    std::lock_guard<std::mutex> lk(c->mu);
    ShardScratch& sc = scratch(c);
    if (parts < 1 || parts > 256 || sc.starts.size() != parts)
        return ph0b::capi_fail(PH0B_ERR_INVALID_ARGUMENT,
                               "scatter_peers: call ph0b_shard_partition_count first");
    cudaStream_t st = pick(c, stream);
    uint64_t cap = 0;
    int rc = 0;
    if (!sc.d_peer && (rc = ensure(reinterpret_cast<void**>(&sc.d_peer), &cap, 512 * 8)))
        return rc;
    // part b's local layout position q goes to dst_keys[b] + 8 * (dst_offsets[b] + q - start_b)
    std::vector<uint64_t> adj(512, 0);
    for (uint32_t b = 0; b < parts; ++b) {
        adj[b] = dst_keys[b] + 8 * (dst_offsets[b] - sc.starts[b]);
        adj[256 + b] = dst_vals[b] + 4 * (dst_offsets[b] - sc.starts[b]);
    }
    if (cudaMemcpyAsync(sc.d_peer, adj.data(), 512 * 8, cudaMemcpyHostToDevice, st))
        return ph0b::capi_fail(PH0B_ERR_CUDA, "H2D peer table");
    c->launches = ph0b::launch_partition_scatter(
        c->keys(0), c->vals(0), sc.local_count, sc.d_spl, parts, sc.d_counts, sc.d_totals,
        nullptr, nullptr, st, sc.local_kmin, sc.local_kmax, sc.d_table, ~0u, sc.d_peer,
        sc.d_peer + 256);
    if (c->launches < 0) return ph0b::capi_fail(PH0B_ERR_CUDA, "shard scatter: launch configuration failed");
    ph0b::capi_set_launches(c->launches);
    // the stores into peer memory are complete when the kernel is; the caller's barrier
    // then publishes them to the receiving ranks
    if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(st))
        return ph0b::capi_fail(PH0B_ERR_CUDA, "shard scatter to peers");
    return PH0B_OK;
}

int ph0b_ipc_get_handle(const void* d_ptr, void* handle_out) {
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)) != cudaSuccess) {
        cudaGetLastError();
        return ph0b::capi_fail(PH0B_ERR_CUDA, "cudaIpcGetMemHandle");
    }
    std::memcpy(handle_out, &h, sizeof(h));
    return PH0B_OK;
}

int ph0b_ipc_open_handle(const void* handle, void** d_ptr) {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    if (cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        return ph0b::capi_fail(PH0B_ERR_CUDA, "cudaIpcOpenMemHandle");
    }
    return PH0B_OK;
}

int ph0b_ipc_close(void* d_ptr) {
    if (cudaIpcCloseMemHandle(d_ptr) != cudaSuccess) {
        cudaGetLastError();
        return ph0b::capi_fail(PH0B_ERR_CUDA, "cudaIpcCloseMemHandle");
    }
    return PH0B_OK;
}

int ph0b_shard_recv(ph0b_context* ctx, uint64_t count, uint64_t** d_keys, uint32_t** d_vals) {
    if (!ctx) return ph0b::capi_fail(PH0B_ERR_INVALID_ARGUMENT, "null context");
    Context* c = reinterpret_cast<Context*>(ctx);
    std::lock_guard<std::mutex> lk(c->mu);
    Status s = c->reserve_recv(count);  // grows buffer 0 only: buffer 1 holds the send data
    if (!s.good()) return ph0b::capi_fail(s);
    scratch(c).recv_buffer = 0;
    if (d_keys) *d_keys = c->keys(0);
    if (d_vals) *d_vals = c->vals(0);
    return PH0B_OK;
}

int ph0b_shard_sort_unique(ph0b_context* ctx, uint64_t count, uint64_t kmin, uint64_t kmax,
                           void* stream, uint64_t* n_distinct, const double** d_scale,
                           uint32_t* passes_out) {
    if (!ctx) return ph0b::capi_fail(PH0B_ERR_INVALID_ARGUMENT, "null context");
    Context* c = reinterpret_cast<Context*>(ctx);
    std::lock_guard<std::mutex> lk(c->mu);
    Status s = c->reserve_edges(count);  // the send buffer is free now: grow the ping-pong
    if (!s.good()) return ph0b::capi_fail(s);
    cudaStream_t st = pick(c, stream);
    c->launches = 0;
    uint32_t passes = 0;
    if (kmax < kmin) kmax = kmin;
    s = c->stage_sort_unique(count, kmin, kmax, false, false, st, &passes,
                             scratch(c).recv_buffer);
    scratch(c).recv_buffer = 0;
    ph0b::capi_set_launches(c->launches);
    if (!s.good()) return ph0b::capi_fail(s);
    if (cudaMemcpyAsync(c->small_host() + 2, c->small_dev() + 2, 8, cudaMemcpyDeviceToHost, st) ||
        cudaStreamSynchronize(st))
        return ph0b::capi_fail(PH0B_ERR_CUDA, "shard sort");
    if (n_distinct) *n_distinct = c->small_host()[2];
    if (d_scale) *d_scale = c->scale();
    if (passes_out) *passes_out = passes;
    return PH0B_OK;
}

int ph0b_shard_reduce(ph0b_context* ctx, uint64_t n, uint64_t count, uint64_t grade_offset,
                      void* stream, uint64_t* m, const uint32_t** d_uv, const uint64_t** d_grade,
                      const double** d_length) {
    if (!ctx) return ph0b::capi_fail(PH0B_ERR_INVALID_ARGUMENT, "null context");
    Context* c = reinterpret_cast<Context*>(ctx);
    std::lock_guard<std::mutex> lk(c->mu);
    cudaStream_t st = pick(c, stream);
    c->launches = 0;
    ph0b::ReduceStats rst;
    Status s = count ? c->stage_reduce(c->vals(c->cur()), count, (uint32_t)n, st, &rst)
                     : Status::ok();
    if (s.good() && rst.survivors) s = c->stage_collect(rst.survivors, count, grade_offset, st);
    if (!s.good()) return ph0b::capi_fail(s);
    ShardScratch& sc = scratch(c);
    int rc = ensure(reinterpret_cast<void**>(&sc.d_cand_uv), &sc.cand_cap, (n + 1) * 4);
    if (rc) return rc;
    c->launches += ph0b::launch_gather_u32(c->vals(c->cur()), c->surv_sorted(), rst.survivors,
                                           sc.d_cand_uv, st);
    ph0b::capi_set_launches(c->launches);
    if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(st))
        return ph0b::capi_fail(PH0B_ERR_CUDA, "shard reduce");
    if (m) *m = rst.survivors;
    if (d_uv) *d_uv = sc.d_cand_uv;
    if (d_grade) *d_grade = c->death_grade();
    if (d_length) *d_length = c->death_length();
    return PH0B_OK;
}

int ph0b_shard_reduce_continue(ph0b_context* ctx, uint64_t n, uint64_t count,
                               uint64_t grade_offset, const uint32_t* init_labels,
                               uint32_t target, void* stream, uint64_t* m,
                               const uint32_t** d_uv, const uint64_t** d_grade,
                               const double** d_length, uint32_t* final_labels) {
    if (!ctx) return ph0b::capi_fail(PH0B_ERR_INVALID_ARGUMENT, "null context");
    Context* c = reinterpret_cast<Context*>(ctx);
    std::lock_guard<std::mutex> lk(c->mu);
    cudaStream_t st = pick(c, stream);
    c->launches = 0;
    const uint32_t* d_init = nullptr;
    if (init_labels && n) {  // the forest left by the preceding key ranges (host labels)
        if (cudaMemcpyAsync(c->lows_buffer(), init_labels, n * 4, cudaMemcpyHostToDevice, st))
            return ph0b::capi_fail(PH0B_ERR_CUDA, "H2D forest labels");
        d_init = c->lows_buffer();
    }
    ph0b::ReduceStats rst;
    Status s = count ? c->stage_reduce(c->vals(c->cur()), count, (uint32_t)n, st, &rst, d_init,
                                       target)
                     : Status::ok();
    if (s.good() && rst.survivors) s = c->stage_collect(rst.survivors, count, grade_offset, st);
    if (!s.good()) return ph0b::capi_fail(s);
    ShardScratch& sc = scratch(c);
    int rc = ensure(reinterpret_cast<void**>(&sc.d_cand_uv), &sc.cand_cap, (n + 1) * 4);
    if (rc) return rc;
    c->launches += ph0b::launch_gather_u32(c->vals(c->cur()), c->surv_sorted(), rst.survivors,
                                           sc.d_cand_uv, st);
    ph0b::capi_set_launches(c->launches);
    if (final_labels && n) {
        const uint32_t* src = count ? c->comp() : d_init;  // nothing reduced: labels unchanged
        if (src && cudaMemcpyAsync(final_labels, src, n * 4, cudaMemcpyDeviceToHost, st))
            return ph0b::capi_fail(PH0B_ERR_CUDA, "D2H forest labels");
        if (!src)
            for (uint64_t v = 0; v < n; ++v) final_labels[v] = (uint32_t)v;
    }
    if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(st))
        return ph0b::capi_fail(PH0B_ERR_CUDA, "shard reduce");
    if (m) *m = rst.survivors;
    if (d_uv) *d_uv = sc.d_cand_uv;
    if (d_grade) *d_grade = c->death_grade();
    if (d_length) *d_length = c->death_length();
    return PH0B_OK;
}

int ph0b_reduce_columns(ph0b_context* ctx, const uint32_t* d_uv, uint64_t count, uint64_t n,
                        void* stream, uint32_t* idx_host, uint64_t* n_out) {
    if (!ctx) return ph0b::capi_fail(PH0B_ERR_INVALID_ARGUMENT, "null context");
    Context* c = reinterpret_cast<Context*>(ctx);
    std::lock_guard<std::mutex> lk(c->mu);
    Status s = c->reserve_points(n, 0);
    if (!s.good()) return ph0b::capi_fail(s);
    cudaStream_t st = pick(c, stream);
    c->launches = 0;
    ph0b::ReduceStats rst;
    s = count ? c->stage_reduce(d_uv, count, (uint32_t)n, st, &rst) : Status::ok();
    if (s.good()) s = c->sort_survivors(rst.survivors, count, st);
    ph0b::capi_set_launches(c->launches);
    if (!s.good()) return ph0b::capi_fail(s);
    const uint32_t m = rst.survivors;
    if (m && (cudaMemcpyAsync(idx_host, c->surv_sorted(), m * 4ull, cudaMemcpyDeviceToHost, st) ||
              cudaStreamSynchronize(st)))
        return ph0b::capi_fail(PH0B_ERR_CUDA, "reduce columns");
    if (n_out) *n_out = m;
    return PH0B_OK;
}

}  // extern "C"
