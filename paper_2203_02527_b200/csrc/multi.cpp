// In-process multi-GPU H0 pipeline behind the drop-in entry points (ph0b_options.n_gpus > 1;
// SURVEY.md §8(e)).  One context and one host thread per GPU; no torch, no NCCL, no IPC:
//
//   rank r: K1 over rows [U_r, U_r+1)  (balanced edge counts; X replicated, <= 4 MiB)
//           an evenly spaced key sample -> host -> P-1 splitters on the length key
//           stable partition counts by splitter -> host: every part's place in its
//             destination's receive buffer (source-rank order = u-major, as an all-to-all-v
//             delivers it)
//           ONE partition kernel stores every part straight into its destination GPU's
//             receive buffer (NVLink P2P stores; peer access enabled once per device pair)
//           local radix sort + unique of the received key range -> D slice r (D stays
//             sharded: the ranges are ordered and no length straddles two of them)
//   then    the column reduction walks the ranges in filtration order: rank 0 reduces its
//           range; only if its forest is not yet spanning does rank r+1 continue it, from
//           rank r's final labels (N u32 copied peer to peer) — exactly the reference's left-
//           to-right reduction (reduction.cpp:33-49) split at range boundaries, so no final
//           re-reduction is needed (the reduction stays on one GPU whenever the first range
//           holds the spanning tree, as at C5, where it ends within the first 5.4% of edges)
//           every rank's D slice and bars -> host in parallel, each over its own PCIe link
//           (D compressed through that context's pinned ring, as ph0b_run_host ships it).
//
// A device ordinal may repeat in the device list: the ranks then share that GPU (virtual
// ranks), which is how the single-GPU test box exercises this path.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ph0b.h"
#include "kernels.h"
#include "pipeline.h"

namespace ph0b {
int capi_fail(const Status& s);
int capi_fail(int code, const std::string& msg);
void capi_set_launches(uint64_t n);
}  // namespace ph0b

namespace ph0b {
namespace {

constexpr uint64_t kSamplesPerRank = 4096;

struct Rank {
    int device = 0;
    ph0b_context* h = nullptr;
    double* dX = nullptr;
    uint64_t dX_cap = 0;
    uint64_t u_lo = 0, u_hi = 0;
    uint64_t count = 0, kmin = 0, kmax = 0;
    std::vector<uint64_t> sample, counts, pmin, pmax;
    uint64_t* recv_k = nullptr;
    uint32_t* recv_v = nullptr;
    uint64_t total = 0, rkmin = 0, rkmax = 0;
    uint64_t nd = 0, d_off = 0, moved = 0;
    const double* d_scale = nullptr;
    uint32_t passes = 0;
    uint32_t m = 0;  // surviving columns found in this range
    uint64_t bar_off = 0;
    int rc = 0;
    std::string err;
    Context* ctx() const { return reinterpret_cast<Context*>(h); }
};

// Contiguous row ranges with ~K/P edges each (row u holds n-1-u edges).
std::vector<std::pair<uint64_t, uint64_t>> row_ranges(uint64_t n, uint32_t parts) {
    const uint64_t k = n * (n - 1) / 2;
    std::vector<uint64_t> b{0};
    uint64_t cum = 0, u = 0;
    for (uint32_t r = 1; r < parts; ++r) {
        const uint64_t target = k * r / parts;
        while (u < n && cum + (n - 1 - u) <= target) cum += n - 1 - u++;
        b.push_back(u);
    }
    b.push_back(n);
    std::vector<std::pair<uint64_t, uint64_t>> out;
    for (uint32_t r = 0; r < parts; ++r) out.emplace_back(b[r], b[r + 1]);
    return out;
}

class MultiRunner {
public:
    explicit MultiRunner(std::vector<int> devices) {
        for (int d : devices) {
            Rank r;
            r.device = d;
            ranks_.push_back(r);
        }
    }
    ~MultiRunner() {
        for (auto& r : ranks_) {
            if (r.dX && cudaSetDevice(r.device) == cudaSuccess) cudaFree(r.dX);
            if (r.h) ph0b_context_destroy(r.h);
        }
        cudaGetLastError();
    }

    int init() {
        const unsigned hw = std::thread::hardware_concurrency();
        if (!pool_) pool_ = std::make_shared<DecodePool>(hw > 2 ? hw - 1 : 1);
        for (auto& r : ranks_) {
            if (r.h) continue;
            const int rc = ph0b_context_create(r.device, &r.h);
            if (rc) return rc;
            r.ctx()->set_decode_pool(pool_);  // one host decoder pool for every rank's D slice
        }
        // NVLink P2P between every pair of distinct devices (the partition kernel stores into
        // its peers' receive buffers)
        for (auto& a : ranks_)
            for (auto& b : ranks_) {
                if (a.device == b.device) continue;
                int ok = 0;
                if (cudaDeviceCanAccessPeer(&ok, a.device, b.device) != cudaSuccess || !ok) {
                    cudaGetLastError();
                    return capi_fail(PH0B_ERR_CUDA, "no peer access from GPU " +
                                                        std::to_string(a.device) + " to GPU " +
                                                        std::to_string(b.device));
                }
                cudaSetDevice(a.device);
                const cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                    return capi_fail(PH0B_ERR_CUDA, std::string("cudaDeviceEnablePeerAccess: ") +
                                                        cudaGetErrorString(e));
                cudaGetLastError();
            }
        return PH0B_OK;
    }

    // Runs f(rank, index) on every rank, one host thread each (device set); the first
    // failure (lowest rank) is reported with its rank's message.
    template <class F>
    int each(F f) {
        std::vector<std::thread> th;
        for (size_t i = 0; i < ranks_.size(); ++i)
            th.emplace_back([&, i] {
                Rank& r = ranks_[i];
                r.rc = 0;
                cudaSetDevice(r.device);
                const int rc = f(r, i);
                if (rc) {
                    r.rc = rc;
                    r.err = ph0b_last_error();
                }
            });
        for (auto& t : th) t.join();
        for (size_t i = 0; i < ranks_.size(); ++i)
            if (ranks_[i].rc)
                return capi_fail(ranks_[i].rc, "rank " + std::to_string(i) + " (GPU " +
                                                   std::to_string(ranks_[i].device) + "): " +
                                                   ranks_[i].err);
        return PH0B_OK;
    }

    int run(const double* X, uint64_t n, uint64_t d, uint32_t layout, uint64_t* death_grade,
            double* death_length, uint64_t* n_finite, uint64_t* essential, double* scale,
            uint64_t scale_capacity, uint64_t* n_scale, ph0b_stage_times* times) {
        NvtxRange nvtx_("ph0b multi-GPU pipeline");
        const auto t0 = std::chrono::steady_clock::now();
        const uint32_t P = (uint32_t)ranks_.size();
        int rc = init();
        if (rc) return rc;
        const auto rows = row_ranges(n, P);
        uint64_t launches = 0;
        // ---- K1 per row range, key samples -------------------------------------------------
        rc = each([&](Rank& r, size_t i) -> int {
            r.u_lo = rows[i].first;
            r.u_hi = rows[i].second;
            const uint64_t bytes = std::max<uint64_t>(8, n * d * 8);
            if (bytes > r.dX_cap) {
                if (r.dX) cudaFree(r.dX);
                r.dX = nullptr;
                r.dX_cap = 0;
                if (cudaMalloc(&r.dX, bytes) != cudaSuccess) {
                    cudaGetLastError();
                    return capi_fail(PH0B_ERR_OUT_OF_MEMORY, "device allocation of X failed");
                }
                r.dX_cap = bytes;
            }
            if (n * d && cudaMemcpy(r.dX, X, n * d * 8, cudaMemcpyHostToDevice) != cudaSuccess)
                return capi_fail(PH0B_ERR_CUDA, "H2D point cloud");
            int e = ph0b_shard_distances(r.h, r.dX, n, d, layout, r.u_lo, r.u_hi, nullptr,
                                         &r.count, &r.kmin, &r.kmax);
            if (e) return e;
            r.sample.assign(std::min<uint64_t>(kSamplesPerRank, r.count), 0);
            return r.sample.empty() ? PH0B_OK
                                    : ph0b_shard_sample(r.h, r.sample.size(), r.sample.data());
        });
        if (rc) return rc;
        // ---- splitters on the length key (equal lengths never straddle two ranges) ------------
        std::vector<uint64_t> all;
        for (auto& r : ranks_) all.insert(all.end(), r.sample.begin(), r.sample.end());
        std::sort(all.begin(), all.end());
        std::vector<uint64_t> spl(P - 1, 0);
        for (uint32_t j = 0; j + 1 < P && !all.empty(); ++j)
            spl[j] = all[std::min<uint64_t>(all.size() - 1, (uint64_t)(j + 1) * all.size() / P)];
        // ---- partition counts, receive buffers, one scatter kernel per rank ----------------
        rc = each([&](Rank& r, size_t) -> int {
            r.counts.assign(P, 0);
            r.pmin.assign(P, 0);
            r.pmax.assign(P, 0);
            return ph0b_shard_partition_count(r.h, spl.data(), P, nullptr, r.counts.data(),
                                              r.pmin.data(), r.pmax.data());
        });
        if (rc) return rc;
        for (uint32_t b = 0; b < P; ++b) {
            Rank& dst = ranks_[b];
            dst.total = 0;
            dst.rkmin = ~0ull;
            dst.rkmax = 0;
            for (auto& src : ranks_) {
                if (!src.counts[b]) continue;
                dst.total += src.counts[b];
                dst.rkmin = std::min(dst.rkmin, src.pmin[b]);
                dst.rkmax = std::max(dst.rkmax, src.pmax[b]);
            }
            if (!dst.total) dst.rkmin = dst.rkmax = 0;
        }
        rc = each([&](Rank& r, size_t) -> int {
            return ph0b_shard_recv_peer(r.h, r.total, &r.recv_k, &r.recv_v);
        });
        if (rc) return rc;
        std::vector<uint64_t> dk(P), dv(P);
        for (uint32_t b = 0; b < P; ++b) {
            dk[b] = reinterpret_cast<uint64_t>(ranks_[b].recv_k);
            dv[b] = reinterpret_cast<uint64_t>(ranks_[b].recv_v);
        }
        rc = each([&](Rank& r, size_t i) -> int {
            std::vector<uint64_t> off(P, 0);
            for (uint32_t b = 0; b < P; ++b)
                for (size_t s = 0; s < i; ++s) off[b] += ranks_[s].counts[b];
            return ph0b_shard_scatter_peers(r.h, P, dk.data(), dv.data(), off.data(), nullptr);
        });
        if (rc) return rc;  // (every scatter kernel has completed: the receive buffers are whole)
        // ---- local sort + unique: D slice per rank -----------------------------------------
        rc = each([&](Rank& r, size_t) -> int {
            return ph0b_shard_sort_unique(r.h, r.total, r.rkmin, r.rkmax, nullptr, &r.nd,
                                          &r.d_scale, &r.passes);
        });
        if (rc) return rc;
        uint64_t nd_total = 0;
        for (auto& r : ranks_) {
            r.d_off = nd_total;
            nd_total += r.nd;
        }
        if (scale && nd_total > scale_capacity)
            return capi_fail(PH0B_ERR_CAPACITY, "scale buffer too small: need " +
                                                    std::to_string(nd_total) + " entries");
        // ---- the column reduction continues the forest from range to range ------------------
        uint32_t found = 0;
        const uint32_t need = n >= 1 ? (uint32_t)(n - 1) : 0;
        int last = -1;  // the last rank that reduced (ranks with an empty range are skipped)
        for (uint32_t i = 0; i < P; ++i) {
            Rank& r = ranks_[i];
            r.m = 0;
            r.bar_off = found;
            if (found >= need || r.total == 0) continue;
            Context* c = r.ctx();
            cudaSetDevice(r.device);
            cudaStream_t st = c->own_stream();
            const uint32_t* init = nullptr;
            if (last >= 0) {  // continue that rank's forest: its labels, copied peer to peer
                const Rank& p = ranks_[last];
                if (cudaMemcpyPeerAsync(c->lows_buffer(), r.device, p.ctx()->comp(), p.device,
                                        n * 4, st) != cudaSuccess)
                    return capi_fail(PH0B_ERR_CUDA, "peer copy of the forest labels");
                init = c->lows_buffer();
            }
            ReduceStats rst;
            c->launches = 0;
            Status s = c->stage_reduce(c->vals(c->cur()), r.total, (uint32_t)n, st, &rst, init,
                                       need - found);
            if (s.good() && rst.survivors)
                s = c->stage_collect(rst.survivors, r.total, r.d_off, st);
            if (s.good() && cudaStreamSynchronize(st) != cudaSuccess)
                s = {PH0B_ERR_CUDA, "reduction"};
            if (!s.good()) return capi_fail(s.code, "rank " + std::to_string(i) + ": " + s.msg);
            launches += c->launches;
            r.m = rst.survivors;
            found += rst.survivors;
            last = (int)i;
        }
        if (found != need)
            return capi_fail(PH0B_ERR_CUDA, "internal error: reduction produced " +
                                                std::to_string(found) + " surviving columns, " +
                                                "expected " + std::to_string(need));
        // ---- bars and D slices -> host, every rank over its own link ----------------------
        rc = each([&](Rank& r, size_t) -> int {
            Context* c = r.ctx();
            cudaStream_t st = c->own_stream();
            if (r.m && (cudaMemcpyAsync(death_grade + r.bar_off, c->death_grade(), r.m * 8ull,
                                        cudaMemcpyDeviceToHost, st) ||
                        cudaMemcpyAsync(death_length + r.bar_off, c->death_length(),
                                        r.m * 8ull, cudaMemcpyDeviceToHost, st) ||
                        cudaStreamSynchronize(st)))
                return capi_fail(PH0B_ERR_CUDA, "D2H bars");
            r.moved = 0;
            if (!scale || !r.nd) return PH0B_OK;
            return ph0b_scale_to_host(r.h, r.d_scale, r.nd, scale + r.d_off,
                                      scale_capacity - r.d_off, nullptr, &r.moved);
        });
        if (rc) return rc;
        uint64_t moved = 16ull * found;
        uint32_t passes = 0;
        for (auto& r : ranks_) {
            moved += r.moved;
            passes = std::max(passes, r.passes);
        }
        if (n_finite) *n_finite = found;
        if (essential) *essential = n - found;
        if (n_scale) *n_scale = nd_total;
        if (times) {
            *times = ph0b_stage_times{};
            times->total_ms = std::chrono::duration<float, std::milli>(
                                  std::chrono::steady_clock::now() - t0).count();
            times->sort_passes = passes;
            times->d2h_bytes = moved;
        }
        capi_set_launches(launches);
        return PH0B_OK;
    }

private:
    std::vector<Rank> ranks_;
    std::shared_ptr<DecodePool> pool_;
};

}  // namespace

std::mutex g_runners_mu;
std::map<std::vector<int>, std::unique_ptr<MultiRunner>>& runners() {
    static auto* r = new std::map<std::vector<int>, std::unique_ptr<MultiRunner>>();
    return *r;
}

// Frees every cached runner (their contexts and device buffers); ph0b_release_resources.
void release_multi_gpu() {
    std::lock_guard<std::mutex> lk(g_runners_mu);
    runners().clear();
}

// The multi-GPU run of ph0b_h0_barcode / ph0b_h0_barcode_into: one runner (contexts, receive
// buffers, decode pools) per device list, reused across calls.
int run_multi_gpu(const std::vector<int>& devices, const double* X, uint64_t n, uint64_t d,
                  uint32_t layout, uint64_t* death_grade, double* death_length,
                  uint64_t* n_finite, uint64_t* essential, double* scale,
                  uint64_t scale_capacity, uint64_t* n_scale, ph0b_stage_times* times) {
    std::lock_guard<std::mutex> lk(g_runners_mu);  // one multi-GPU run at a time
    struct DeviceGuard {  // the caller's current device is left as it was
        int dev = 0;
        DeviceGuard() {
            if (cudaGetDevice(&dev) != cudaSuccess) cudaGetLastError();
        }
        ~DeviceGuard() {
            if (cudaSetDevice(dev) != cudaSuccess) cudaGetLastError();
        }
    } device_guard;
    auto& slot = runners()[devices];
    if (!slot) slot = std::make_unique<MultiRunner>(devices);
    int rc = slot->run(X, n, d, layout, death_grade, death_length, n_finite, essential, scale,
                       scale_capacity, n_scale, times);
    if (rc != PH0B_ERR_OUT_OF_MEMORY || runners().size() == 1) return rc;
    // out of device memory while other device lists' runners hold theirs: free those, retry
    for (auto it = runners().begin(); it != runners().end();) {
        if (it->first != devices)
            it = runners().erase(it);
        else
            ++it;
    }
    return slot->run(X, n, d, layout, death_grade, death_length, n_finite, essential, scale,
                  scale_capacity, n_scale, times);
}

}  // namespace ph0b
