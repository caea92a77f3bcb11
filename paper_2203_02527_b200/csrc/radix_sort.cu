// K2 — onesweep-style LSD radix sort of (length bits, column) pairs (replaces the
// std::sort of build_filtration, /root/reference/proj/src/filtration.cpp:21-25).
//
// Keys are the f64 bit patterns of non-negative lengths, ordered as unsigned integers;
// only the digits of (key - kmin) that can differ are sorted (span = bits of kmax-kmin),
// 8 bits per pass.  Every pass is stable and the input is the reference's u-major order,
// so equal lengths end up ordered by (u, v) exactly as filtration.cpp:21-25 orders them.
//
// One kernel per digit (Adinets & Merrill's single-pass "onesweep"): each CTA takes the
// next 4096-key tile (dynamic tile id), ranks its keys with warp-level match_any ranking
// into per-warp histograms, publishes its per-digit counts and obtains the exclusive
// prefix over earlier tiles by decoupled look-back, scatters the tile into shared memory
// in digit order and writes it out so that each digit's run is a contiguous global run.
// The same pass counts the NEXT digit's histogram, so no separate upsweep over the keys
// is needed (pass 0's histogram comes from the distance kernel).
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace ph0b {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;
constexpr int kTileKeys = kThreads * kItems;  // 4096
constexpr int kBins = 256;
static_assert(kThreads == kBins, "one thread per digit value");

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t x, uint32_t* sh_warp,
                                                         uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) sh_warp[warp] = inc;
    __syncthreads();
    uint32_t wbase = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        const uint32_t t = sh_warp[w];
        wbase += (w < warp) ? t : 0u;
        tot += t;
    }
    if (total) *total = tot;
    return wbase + inc - x;
}

template <bool kVals, bool kCountNext>
__global__ void __launch_bounds__(kThreads)
    k2_onesweep(const uint64_t* __restrict__ keys_in, uint64_t* __restrict__ keys_out,
                const uint32_t* __restrict__ vals_in, uint32_t* __restrict__ vals_out,
                uint64_t count, uint64_t kmin, uint32_t shift, uint32_t next_shift,
                const uint32_t* __restrict__ hist, uint32_t hist_rot,
                uint64_t* __restrict__ status, uint32_t* tile_counter, uint32_t epoch,
                uint32_t* __restrict__ next_hist) {
    extern __shared__ __align__(16) uint64_t s_dyn[];
    uint64_t* s_keys = s_dyn;                                          // [kTileKeys]
    uint32_t* s_vals = reinterpret_cast<uint32_t*>(s_dyn + kTileKeys);  // [kTileKeys] if kVals
    __shared__ uint32_t s_whist[kWarps][kBins];
    __shared__ uint32_t s_tile_start[kBins];
    __shared__ uint32_t s_global[kBins];
    __shared__ uint32_t s_next[kCountNext ? kBins : 1];
    __shared__ uint32_t s_scan[kWarps];
    __shared__ uint32_t s_tile;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s_whist[w][tid] = 0;
    if (kCountNext) s_next[tid] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t base = (uint64_t)tile * kTileKeys;

    // ---- load (warp-striped, coalesced) and rank within the warp ------------------------
    uint64_t k[kItems];
    uint32_t v[kItems];
    uint32_t rank[kItems];
    const uint64_t wbase = base + (uint64_t)warp * (32 * kItems) + lane;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const uint64_t idx = wbase + 32 * i;
        const bool valid = idx < count;
        k[i] = valid ? keys_in[idx] : ~0ull;
        if (kVals) v[i] = valid ? vals_in[idx] : 0u;
    }
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const bool valid = wbase + 32 * i < count;
        const uint32_t d = valid ? (uint32_t)((k[i] - kmin) >> shift) & 0xFFu : 0x100u;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const int leader = __ffs(peers) - 1;
        uint32_t old = 0;
        if (valid && lane == leader) old = s_whist[warp][d];
        old = __shfl_sync(0xffffffffu, old, leader);
        rank[i] = old + __popc(peers & lt);
        if (valid && lane == leader) s_whist[warp][d] = old + __popc(peers);
        __syncwarp();
    }
    __syncthreads();

    // ---- per-digit counts, warp offsets, tile-local digit starts ------------------------
    const uint32_t t = tid;  // digit handled by this thread
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        const uint32_t c = s_whist[w][t];
        s_whist[w][t] = cnt;
        cnt += c;
    }
    uint64_t* my_status = status + (uint64_t)tile * kBins + t;
    if (tile == 0)
        st_relaxed_u64(my_status, pack_status(kStateInclusive, epoch, cnt));
    else
        st_relaxed_u64(my_status, pack_status(kStateAggregate, epoch, cnt));

    // global start of digit t: exclusive scan of the (rotated) digit histogram
    const uint32_t hcount = hist[(t + hist_rot) & 0xFFu];
    const uint32_t bin_start = block_exclusive_scan(hcount, s_scan, nullptr);
    __syncthreads();
    s_tile_start[t] = block_exclusive_scan(cnt, s_scan, nullptr);

    // ---- decoupled look-back over earlier tiles, per digit -------------------------------
    uint32_t excl = 0;
    if (tile > 0) {
        int64_t p = (int64_t)tile - 1;
        while (p >= 0) {
            const uint64_t s = ld_relaxed_u64(status + (uint64_t)p * kBins + t);
            const uint32_t st = status_state(s, epoch);
            if (st == 0) continue;  // predecessor not published yet
            excl += (uint32_t)s;
            if (st == kStateInclusive) break;
            --p;
        }
        st_relaxed_u64(my_status, pack_status(kStateInclusive, epoch, excl + cnt));
    }
    s_global[t] = bin_start + excl;
    __syncthreads();

    // ---- scatter into shared memory in (digit, input order) order -----------------------
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        if (wbase + 32 * i < count) {
            const uint32_t d = (uint32_t)((k[i] - kmin) >> shift) & 0xFFu;
            const uint32_t pos = s_tile_start[d] + s_whist[warp][d] + rank[i];
            s_keys[pos] = k[i];
            if (kVals) s_vals[pos] = v[i];
        }
    }
    __syncthreads();

    // ---- write out: consecutive threads -> consecutive positions within each digit run --
    const uint64_t rem = count - base;
    const uint32_t tile_n = rem < (uint64_t)kTileKeys ? (uint32_t)rem : (uint32_t)kTileKeys;
#pragma unroll 4
    for (int j = 0; j < kItems; ++j) {
        const uint32_t p = j * kThreads + tid;
        if (p < tile_n) {
            const uint64_t key = s_keys[p];
            const uint64_t rel = key - kmin;
            const uint32_t d = (uint32_t)(rel >> shift) & 0xFFu;
            const uint64_t out = (uint64_t)s_global[d] + (p - s_tile_start[d]);
            keys_out[out] = key;
            if (kVals) vals_out[out] = s_vals[p];
            if (kCountNext) atomicAdd(&s_next[(uint32_t)(rel >> next_shift) & 0xFFu], 1u);
        }
    }
    if (kCountNext) {
        __syncthreads();
        const uint32_t c = s_next[tid];
        if (c) atomicAdd(&next_hist[tid], c);
    }
}

// Histogram of one digit of (key - kmin) (used only when the distance kernel's raw
// low-byte histogram does not apply, e.g. for the survivor sort).
__global__ void k2_digit_histogram(const uint64_t* __restrict__ keys, uint64_t count,
                                   uint64_t kmin, uint32_t shift, uint32_t* hist) {
    __shared__ uint32_t h[kBins];
    h[threadIdx.x] = 0;
    __syncthreads();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(&h[(uint32_t)((keys[i] - kmin) >> shift) & 0xFFu], 1u);
    __syncthreads();
    if (h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], h[threadIdx.x]);
}

template <bool kVals, bool kCountNext>
void launch_pass(const SortArgs& a, int cur, uint32_t p, const SortPlan& plan, uint32_t rot,
                 uint32_t* next_hist, uint64_t tiles, cudaStream_t s) {
    auto kern = k2_onesweep<kVals, kCountNext>;
    const size_t smem = kTileKeys * (sizeof(uint64_t) + (kVals ? sizeof(uint32_t) : 0));
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    const uint32_t next_shift = kCountNext ? plan.shift[p + 1] : 0u;
    kern<<<(unsigned)tiles, kThreads, smem, s>>>(
        a.keys[cur], a.keys[cur ^ 1], kVals ? a.vals[cur] : nullptr,
        kVals ? a.vals[cur ^ 1] : nullptr, a.count, a.kmin, plan.shift[p], next_shift,
        a.hist + kBins * p, rot, a.status, a.tile_counter + p, a.epoch_base + p, next_hist);
}

}  // namespace

uint64_t sort_tiles(uint64_t count) { return (count + kTileKeys - 1) / kTileKeys; }

int launch_digit_histogram(const uint64_t* keys, uint64_t count, uint64_t kmin, uint32_t shift,
                           uint32_t* hist, cudaStream_t s, int num_sms) {
    if (count == 0) return 0;
    uint64_t blocks = (count + kBins - 1) / kBins;
    const uint64_t cap = (uint64_t)num_sms * 8;
    if (blocks > cap) blocks = cap;
    k2_digit_histogram<<<(unsigned)blocks, kBins, 0, s>>>(keys, count, kmin, shift, hist);
    return 1;
}

int launch_sort_passes(const SortArgs& a, const SortPlan& plan, cudaStream_t s, int num_sms,
                       int* launches) {
    (void)num_sms;
    int cur = 0;
    const uint64_t tiles = sort_tiles(a.count);
    if (a.count == 0 || plan.passes == 0) return 0;
    cudaMemsetAsync(a.tile_counter, 0, sizeof(uint32_t) * 8, s);
    // hist rows 1..passes-1 are produced by the passes themselves
    if (plan.passes > 1)
        cudaMemsetAsync(a.hist + kBins, 0, sizeof(uint32_t) * kBins * (plan.passes - 1), s);
    for (uint32_t p = 0; p < plan.passes; ++p) {
        const bool last = p + 1 == plan.passes;
        uint32_t* next_hist = last ? nullptr : a.hist + kBins * (p + 1);
        const uint32_t rot = (p == 0) ? a.hist0_rot : 0u;
        if (a.vals[0]) {
            if (last)
                launch_pass<true, false>(a, cur, p, plan, rot, next_hist, tiles, s);
            else
                launch_pass<true, true>(a, cur, p, plan, rot, next_hist, tiles, s);
        } else {
            if (last)
                launch_pass<false, false>(a, cur, p, plan, rot, next_hist, tiles, s);
            else
                launch_pass<false, true>(a, cur, p, plan, rot, next_hist, tiles, s);
        }
        if (launches) ++*launches;
        cur ^= 1;
    }
    return cur;
}

}  // namespace ph0b
