// K4 — GPU-parallel column reduction of the boundary matrix M over Z2 (replaces
// ReduceEngine::run, /root/reference/proj/src/reduction.cpp:31-51, and its pivot table
// claimed_by_, reduction.cpp:121).
//
// Why this is the reference's reduction, not an approximation of it:
//  * Every column of M starts as {u, v} (boundary_matrix.cpp:22-24) and every addition XORs
//    it with the unique earlier column owning its low (reduction.cpp:36-42), so supports stay
//    2-sparse.  The claimed columns form a "pivot forest" (claimed row r -> the other row of
//    its column, always < r), whose roots are the unclaimed rows = the minimum vertex of each
//    tree.  Reducing column {u, v} walks both endpoints up that forest, XOR by XOR: it empties
//    iff u and v are in the same tree, and otherwise claims max(root(u), root(v)).
//  * So a column is a cycle (reduces to 0) exactly when label[u] == label[v] — this is the
//    clearing filter below, applied in bulk and provably result-preserving — and the
//    surviving columns are exactly the columns that join two trees, in filtration order:
//    the minimum spanning forest under the strict column order (length, u, v).
//
// Parallel schedule (rounds over windows of the filtration):
//   (i)   filter: stream the window's columns, drop those whose endpoints share a label
//         (one 4-byte load + two label gathers per column), compact the rest;
//   (ii)  resolve the candidates in parallel rounds: every live tree takes the minimum-index
//         candidate column touching it (atomicMin into a per-tree pivot slot), each such
//         column is a surviving column (cut property: it is the first column in filtration
//         order leaving that tree), trees hook along it (mutual pairs keep the smaller root),
//         labels are re-pointed by pointer jumping, candidates are re-filtered; repeat until
//         no candidate joins two trees;
//   (iii) early exit as soon as N-1 columns survived — every later column is provably a
//         cycle (the reference still walks all K columns).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace ph0b {
namespace {

constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr int kThreads = 256;

// counters[] layout
constexpr int kCntCand = 0;      // candidates written by the last filter
constexpr int kCntSurv = 1;      // surviving columns found so far
constexpr int kCntHooks = 2;     // hooks made by the last resolve round
constexpr int kCntOverflow = 3;  // filter exceeded the candidate capacity

// Labels start as singletons, or (continuing an earlier range of the filtration, e.g. the
// previous rank's key range) as that range's final labels: every label is a tree root, and a
// root's hook parent is itself.
__global__ void k4_init(uint32_t* comp, uint32_t* best, uint32_t* par, uint32_t n,
                        uint16_t* comp16, const uint32_t* __restrict__ init) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const uint32_t c = init ? init[v] : v;
        comp[v] = c;
        comp16[v] = (uint16_t)c;
        par[v] = c;
        best[v] = kNone;
    }
}

// Clearing filter over columns [begin, end) (list == nullptr) or over a candidate list.
__global__ void __launch_bounds__(kThreads)
    k4_filter(const uint32_t* __restrict__ uv, uint64_t begin, uint64_t end,
              const uint32_t* __restrict__ list, uint32_t list_n,
              const uint32_t* __restrict__ comp, uint32_t* __restrict__ out, uint64_t cap,
              uint32_t* counters, uint32_t n) {
    const uint64_t total = list ? (uint64_t)list_n : end - begin;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < total; base += stride) {
        const uint64_t i = base + threadIdx.x;
        bool keep = false;
        uint32_t j = 0;
        if (i < total) {
            j = list ? list[i] : (uint32_t)(begin + i);
            uint32_t a, b;
            col_rows(__ldg(uv + j), n, a, b);
            keep = __ldg(comp + a) != __ldg(comp + b);
        }
        const uint32_t ballot = __ballot_sync(0xffffffffu, keep);
        if (ballot) {
            uint32_t slot = 0;
            if (lane == 0) slot = atomicAdd(&counters[kCntCand], (uint32_t)__popc(ballot));
            slot = __shfl_sync(0xffffffffu, slot, 0) + __popc(ballot & lanemask_lt());
            if (keep) {
                if (slot < cap)
                    out[slot] = j;
                else
                    counters[kCntOverflow] = 1;
            }
        }
    }
}

// Clearing filter over a window of the filtration with 8 columns per thread (two 16-byte
// loads, 16 independent label gathers from a 128 KB u16 label copy that stays in L1).
// kIds (N > 65536, edge-id columns, colcodec.h): the labels are the u32 ones.
template <bool kIds>
__global__ void __launch_bounds__(kThreads)
    k4_filter_range(const uint32_t* __restrict__ uv, uint64_t begin, uint64_t end,
                    const uint16_t* __restrict__ comp16, const uint32_t* __restrict__ comp,
                    uint32_t n, uint32_t* __restrict__ out, uint64_t cap, uint32_t* counters) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t a0 = begin & ~7ull;  // 8-column (32 B) aligned groups
    const uint64_t groups = (end - a0 + 7) / 8;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t g0 = (uint64_t)blockIdx.x * blockDim.x; g0 < groups; g0 += stride) {
        const uint64_t g = g0 + threadIdx.x;
        uint32_t e[8];
        uint32_t keep = 0;
        if (g < groups) {
            const uint64_t first = a0 + 8 * g;
            if (first + 8 <= end) {
                const uint4* p = reinterpret_cast<const uint4*>(uv + first);
                const uint4 x = __ldg(p), y = __ldg(p + 1);
                e[0] = x.x; e[1] = x.y; e[2] = x.z; e[3] = x.w;
                e[4] = y.x; e[5] = y.y; e[6] = y.z; e[7] = y.w;
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) e[i] = first + i < end ? __ldg(uv + first + i) : 0u;
            }
            uint32_t lu[8], lv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if constexpr (kIds) {
                    uint32_t a, b;
                    col_rows(e[i], n, a, b);
                    lu[i] = __ldg(comp + a);
                    lv[i] = __ldg(comp + b);
                } else {
                    lu[i] = __ldg(comp16 + (e[i] >> 16));
                    lv[i] = __ldg(comp16 + (e[i] & 0xFFFFu));
                }
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint64_t j = a0 + 8 * g + i;
                if (j >= begin && j < end && lu[i] != lv[i]) keep |= 1u << i;
            }
        }
        const uint32_t c = __popc(keep);
        uint32_t inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        const uint32_t wtot = __shfl_sync(0xffffffffu, inc, 31);
        if (wtot == 0) continue;
        uint32_t slot = 0;
        if (lane == 31) slot = atomicAdd(&counters[kCntCand], wtot);
        slot = __shfl_sync(0xffffffffu, slot, 31) + inc - c;
        if (slot + c > cap) {
            if (c) counters[kCntOverflow] = 1;
            continue;
        }
        for (int i = 0; i < 8; ++i)
            if (keep & (1u << i)) out[slot++] = (uint32_t)(a0 + 8 * g + i);
    }
}

// Same filter with the u16 label copy staged in shared memory (≤ 128 KB for N ≤ 65536): the
// 16 label gathers per thread are shared-memory reads instead of L1/L2 round trips.  One
// 1024-thread CTA per SM.
constexpr int kFThreads = 1024;
__global__ void __launch_bounds__(kFThreads)
    k4_filter_range_s(const uint32_t* __restrict__ uv, uint64_t begin, uint64_t end,
                      const uint16_t* __restrict__ comp16, uint32_t n, uint32_t* __restrict__ out,
                      uint64_t cap, uint32_t* counters) {
    extern __shared__ __align__(16) uint16_t s_comp[];
    {
        const uint32_t n8 = (n + 7) / 8;  // 16-byte pieces (the label copy is padded)
        const uint4* src = reinterpret_cast<const uint4*>(comp16);
        uint4* dst = reinterpret_cast<uint4*>(s_comp);
        for (uint32_t i = threadIdx.x; i < n8; i += kFThreads) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t a0 = begin & ~7ull;
    const uint64_t groups = (end - a0 + 7) / 8;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t g0 = (uint64_t)blockIdx.x * blockDim.x; g0 < groups; g0 += stride) {
        const uint64_t g = g0 + threadIdx.x;
        uint32_t e[8];
        uint32_t keep = 0;
        if (g < groups) {
            const uint64_t first = a0 + 8 * g;
            if (first + 8 <= end) {
                const uint4* p = reinterpret_cast<const uint4*>(uv + first);
                const uint4 x = __ldg(p), y = __ldg(p + 1);
                e[0] = x.x; e[1] = x.y; e[2] = x.z; e[3] = x.w;
                e[4] = y.x; e[5] = y.y; e[6] = y.z; e[7] = y.w;
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) e[i] = first + i < end ? __ldg(uv + first + i) : 0u;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint64_t j = a0 + 8 * g + i;
                if (j >= begin && j < end && s_comp[e[i] >> 16] != s_comp[e[i] & 0xFFFFu])
                    keep |= 1u << i;
            }
        }
        const uint32_t c = __popc(keep);
        uint32_t inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        const uint32_t wtot = __shfl_sync(0xffffffffu, inc, 31);
        if (wtot == 0) continue;
        uint32_t slot = 0;
        if (lane == 31) slot = atomicAdd(&counters[kCntCand], wtot);
        slot = __shfl_sync(0xffffffffu, slot, 31) + inc - c;
        if (slot + c > cap) {
            if (c) counters[kCntOverflow] = 1;
            continue;
        }
        for (int i = 0; i < 8; ++i)
            if (keep & (1u << i)) out[slot++] = (uint32_t)(a0 + 8 * g + i);
    }
}

// Each live tree's minimum candidate column (its pivot candidate for this round).
__global__ void __launch_bounds__(kThreads)
    k4_min_edge(const uint32_t* __restrict__ cand, uint32_t ncand, const uint32_t* __restrict__ uv,
                const uint32_t* __restrict__ comp, uint32_t* best, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ncand;
         i += gridDim.x * blockDim.x) {
        const uint32_t j = cand[i];
        uint32_t a, b;
        col_rows(uv[j], n, a, b);
        const uint32_t cu = comp[a], cv = comp[b];
        if (cu == cv) continue;
        if (j < ld_cg_u32(best + cu)) atomicMin(best + cu, j);
        if (j < ld_cg_u32(best + cv)) atomicMin(best + cv, j);
    }
}

// Hook every tree along its minimum candidate column; record the surviving column.
__global__ void k4_hook(uint32_t n, const uint32_t* __restrict__ uv,
                        const uint32_t* __restrict__ comp, const uint32_t* __restrict__ best,
                        uint32_t* par, uint32_t* surv, uint32_t* counters) {
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
        if (comp[x] != x) continue;  // not a tree label
        const uint32_t j = best[x];
        if (j == kNone) continue;
        uint32_t a, b;
        col_rows(uv[j], n, a, b);
        const uint32_t cu = comp[a], cv = comp[b];
        const uint32_t other = (cu == x) ? cv : cu;
        const bool mutual = best[other] == j;
        if (mutual && x < other) continue;  // the larger label of a mutual pair hooks
        par[x] = other;
        surv[atomicAdd(&counters[kCntSurv], 1u)] = j;
        counters[kCntHooks] = 1;
    }
}

// Pointer jumping on the hooked labels (each label ends at the root of its hook tree).
__global__ void k4_jump_roots(uint32_t n, const uint32_t* __restrict__ comp, uint32_t* par) {
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
        if (comp[x] != x) continue;
        uint32_t r = par[x];
        if (r == x) continue;
        uint32_t nx = par[r];
        while (nx != r) {
            r = nx;
            nx = par[r];
        }
        // path compression: every pointer written is to the true root
        uint32_t y = x;
        while (par[y] != r) {
            const uint32_t t = par[y];
            par[y] = r;
            y = t;
        }
    }
}

__global__ void k4_relabel(uint32_t n, uint32_t* comp, const uint32_t* __restrict__ par,
                           uint32_t* best, uint16_t* comp16) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const uint32_t c = par[comp[v]];
        comp[v] = c;
        comp16[v] = (uint16_t)c;
        best[v] = kNone;
    }
}

// Publish the round counters to zero-copy host memory with plain stores (no copy engine:
// a D2H of D may be streaming on another stream and would delay a queued small copy).
__global__ void k4_publish(const uint32_t* __restrict__ counters, uint32_t* mapped) {
    if (threadIdx.x < 8) mapped[threadIdx.x] = counters[threadIdx.x];
}

inline unsigned grid_for(uint64_t work, int num_sms, int per_sm = 8) {
    uint64_t b = (work + kThreads - 1) / kThreads;
    const uint64_t cap = (uint64_t)num_sms * per_sm;
    if (b > cap) b = cap;
    if (b == 0) b = 1;
    return (unsigned)b;
}

}  // namespace

int run_reduction(ReduceState& st, cudaStream_t s, int num_sms, uint32_t& epoch,
                  ReduceStats* stats, const uint32_t* init_comp, uint32_t target) {
    (void)epoch;
    ReduceStats local;
    ReduceStats& S = stats ? *stats : local;
    const uint32_t n = st.n;
    if (n < 2 || st.k == 0) {
        cudaMemsetAsync(st.counters, 0, sizeof(uint32_t) * 8, s);
        return 0;
    }
    uint32_t* par = st.best + n;  // best buffer holds [best | par | comp16]
    // (16-byte aligned: the shared-memory filter stages it with 16-byte loads)
    uint16_t* comp16 = reinterpret_cast<uint16_t*>(st.best + ((2ull * n + 3) & ~3ull));
    const unsigned gn = grid_for(n, num_sms, 4);
    cudaMemsetAsync(st.counters, 0, sizeof(uint32_t) * 8, s);
    k4_init<<<gn, kThreads, 0, s>>>(st.comp, st.best, par, n, comp16, init_comp);
    if (target == 0 || target > n - 1) target = n - 1;
    S.launches += 1;

    volatile uint32_t* h = st.host_counters;
    auto pull = [&]() {
        k4_publish<<<1, 32, 0, s>>>(st.counters, st.mapped_counters);
        cudaStreamSynchronize(s);
    };

    // labels in shared memory for the window filter (N <= 65536; C5 reduce 2.65 -> 2.53 ms
    // vs gathering them through L1)
    const size_t fsmem = ((size_t)n * 2 + 15) & ~(size_t)15;
    bool smem_filter = fsmem <= 200 * 1024 && !col_ids(n);
    if (smem_filter && kernel_blocks_per_sm((const void*)k4_filter_range_s, kFThreads, fsmem) < 1)
        smem_filter = false;
    uint64_t pos = 0;
    uint64_t window = std::min<uint64_t>(st.k, std::max<uint64_t>(8ull * n, 1u << 16));
    uint32_t survivors = 0;
    while (survivors < target && pos < st.k) {
        uint64_t end = std::min<uint64_t>(st.k, pos + window);
        // (i) clearing filter over the window
        cudaMemsetAsync(st.counters + kCntCand, 0, sizeof(uint32_t), s);
        cudaMemsetAsync(st.counters + kCntOverflow, 0, sizeof(uint32_t), s);
        if (smem_filter) {
            uint64_t blocks = ((end - pos + 7) / 8 + kFThreads - 1) / kFThreads;
            if (blocks > (uint64_t)num_sms) blocks = num_sms;
            k4_filter_range_s<<<(unsigned)(blocks ? blocks : 1), kFThreads, fsmem, s>>>(
                st.uv, pos, end, comp16, n, st.cand[0], st.cap, st.counters);
        } else if (col_ids(n)) {
            k4_filter_range<true><<<grid_for((end - pos + 7) / 8, num_sms), kThreads, 0, s>>>(
                st.uv, pos, end, comp16, st.comp, n, st.cand[0], st.cap, st.counters);
        } else {
            k4_filter_range<false><<<grid_for((end - pos + 7) / 8, num_sms), kThreads, 0, s>>>(
                st.uv, pos, end, comp16, st.comp, n, st.cand[0], st.cap, st.counters);
        }
        S.launches += 1;
        pull();
        if (h[kCntOverflow]) {  // too many live columns in this window: shrink and retry
            window = std::max<uint64_t>(window / 4, 1024);
            continue;
        }
        S.rounds += 1;
        S.scanned += end - pos;
        uint32_t ncand = h[kCntCand];
        int cur = 0;
        // (ii) parallel resolution rounds
        while (ncand > 0) {
            S.iterations += 1;
            k4_min_edge<<<grid_for(ncand, num_sms), kThreads, 0, s>>>(st.cand[cur], ncand, st.uv,
                                                                       st.comp, st.best, n);
            cudaMemsetAsync(st.counters + kCntHooks, 0, sizeof(uint32_t), s);
            k4_hook<<<gn, kThreads, 0, s>>>(n, st.uv, st.comp, st.best, par, st.surv,
                                            st.counters);
            k4_jump_roots<<<gn, kThreads, 0, s>>>(n, st.comp, par);
            k4_relabel<<<gn, kThreads, 0, s>>>(n, st.comp, par, st.best, comp16);
            cudaMemsetAsync(st.counters + kCntCand, 0, sizeof(uint32_t), s);
            k4_filter<<<grid_for(ncand, num_sms), kThreads, 0, s>>>(
                st.uv, 0, 0, st.cand[cur], ncand, st.comp, st.cand[cur ^ 1], st.cap,
                st.counters, n);
            S.launches += 5;
            pull();
            cur ^= 1;
            ncand = h[kCntCand];
            survivors = h[kCntSurv];
        }
        survivors = h[kCntSurv];
        pos = end;
        window = std::min<uint64_t>(window * 2, 1ull << 40);
    }
    S.survivors = survivors;
    return 0;
}

}  // namespace ph0b
