// K2 — onesweep-style LSD radix sort of (length bits, column) pairs (replaces the
// std::sort of build_filtration, /root/reference/proj/src/filtration.cpp:21-25).
//
// Keys are the f64 bit patterns of non-negative lengths, ordered as unsigned integers;
// only the digits of (key - kmin) that can differ are sorted (span = bits of kmax-kmin),
// 8 bits per pass.  Every pass is stable and the input is the reference's u-major order,
// so equal lengths end up ordered by (u, v) exactly as filtration.cpp:21-25 orders them.
//
// One kernel per digit (Adinets & Merrill's single-pass "onesweep"), persistent: each CTA
// claims 4096-key tiles in increasing order with an atomic ticket (the next one while the
// current one is still being written, its keys and columns prefetched into shared memory
// with TMA bulk copies), ranks the tile's keys in-warp with shared-memory atomics on
// per-warp digit counters (B200 resolves the same-address lanes of one ATOMS in lane
// order — checked on the device at context creation; bit-sliced ballots otherwise),
// publishes its per-digit counts, obtains the exclusive prefix over earlier tiles by
// decoupled look-back on epoch-tagged status words, scatters the tile into shared memory in
// digit order and writes it out so that each digit's run is a contiguous global run.  The
// same pass counts the NEXT digit's histogram, so no separate upsweep over the keys is
// needed.  Tickets make the look-back deadlock-free whatever else shares the GPU: every
// tile a CTA waits on was claimed earlier by a CTA that is already running.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace ph0b {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
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

// Stable in-warp rank of one digit per lane by bit-sliced ballots (pure ALU): the mask of
// the lanes holding the same digit.  Used when the ATOMS lane-order self-test fails.
__device__ __forceinline__ uint32_t ballot_peers(uint32_t d, uint32_t valid_mask) {
    uint32_t peers = valid_mask;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const uint32_t bit = (d >> b) & 1u;
        const uint32_t bal = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? bal : ~bal;
    }
    return peers;
}

constexpr int kPTile = 4096;
constexpr int kPItems = kPTile / kThreads;  // 16

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITP_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITP_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

// Look-back after the early probe of tile - 1: its aggregate is kept and the walk continues
// at tile - 2 in windows of 4 predecessors per round trip (C5: 14.85 -> 14.26 ms per pass vs
// restarting at tile - 1 in windows of 8; windows of 3 / 6 measured slower).
constexpr int kLookbackWin = 4;

template <bool kVals, bool kCountNext, bool kBallot>
__global__ void __launch_bounds__(kThreads, 2)
    k2_onesweep_p(const uint64_t* __restrict__ keys_in, uint64_t* __restrict__ keys_out,
                  const uint32_t* __restrict__ vals_in, uint32_t* __restrict__ vals_out,
                  uint64_t count, uint64_t kmin, uint32_t shift, uint32_t next_shift,
                  const uint32_t* __restrict__ hist, uint32_t hist_rot,
                  uint64_t* __restrict__ status, uint32_t epoch,
                  uint32_t* __restrict__ next_hist, uint32_t num_tiles,
                  uint32_t* __restrict__ ticket) {
    extern __shared__ __align__(128) uint64_t p_dyn[];
    uint64_t* st_k = p_dyn;                                                    // stage keys
    uint32_t* st_v = reinterpret_cast<uint32_t*>(p_dyn + kPTile);              // stage vals
    uint64_t* so_k = p_dyn + kPTile + kPTile / 2;                              // sorted keys
    uint32_t* so_v = reinterpret_cast<uint32_t*>(so_k + kPTile);               // sorted vals
    // per-warp digit counters; after the scan: tile-local start of (warp, digit)
    __shared__ uint32_t s_whist[kWarps][kBins];
    __shared__ uint32_t s_global[kBins];
    __shared__ uint32_t s_bin_start[kBins];
    __shared__ uint32_t s_next[kCountNext ? kBins : 1];
    __shared__ uint32_t s_scan[kWarps];
    __shared__ uint32_t s_tile[2];
    __shared__ __align__(8) uint64_t s_bar;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t t = tid;  // digit handled by this thread in the per-digit phases
    auto issue = [&](uint32_t tl) {
        const uint64_t b0 = (uint64_t)tl * kPTile;
        const uint64_t n = count - b0 < (uint64_t)kPTile ? count - b0 : (uint64_t)kPTile;
        const uint32_t bk = (uint32_t)((n * 8 + 15) & ~15ull);
        const uint32_t bv = kVals ? (uint32_t)((n * 4 + 15) & ~15ull) : 0u;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_tx(&s_bar, bk + bv);
        bulk_g2s(st_k, keys_in + b0, bk, &s_bar);
        if (kVals) bulk_g2s(st_v, vals_in + b0, bv, &s_bar);
    };
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&s_bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const uint32_t first = atomicAdd(ticket, 1u);
        s_tile[0] = first;
        if (first < num_tiles) issue(first);
    }
    if (kCountNext) s_next[tid] = 0;
    {
        const uint32_t hcount = hist[(t + hist_rot) & 0xFFu];
        s_bin_start[t] = block_exclusive_scan(hcount, s_scan, nullptr);
    }
    __syncthreads();
    uint32_t tile = s_tile[0];
    uint32_t parity = 0;
    const uint32_t lt = lanemask_lt();

    while (tile < num_tiles) {
        const uint64_t base = (uint64_t)tile * kPTile;
        const uint64_t rem = count - base;
        const uint32_t tile_n = rem < (uint64_t)kPTile ? (uint32_t)rem : (uint32_t)kPTile;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s_whist[w][tid] = 0;
        __syncthreads();
        // the look-back's probe of tile - 1 goes out before this tile is even ranked: its
        // latency hides behind the rank, scan and scatter phases (C5: 14.51 -> 13.83 ms per
        // pass vs issuing it after this tile's aggregate is published)
        const uint64_t probe =
            tile > 0 ? ld_relaxed_u64(status + (uint64_t)(tile - 1) * kBins + t) : 0ull;
        mbar_wait_parity(&s_bar, parity);
        parity ^= 1u;

        // ---- rank within the warp (keys from the staged tile) --------------------------
        uint64_t k[kPItems];
        uint32_t rank2[kPItems / 2];
        const uint32_t wofs = warp * (32 * kPItems) + lane;
#pragma unroll
        for (int i = 0; i < kPItems; ++i) {
            const uint32_t pos = wofs + 32 * i;
            const bool valid = pos < tile_n;
            k[i] = valid ? st_k[pos] : ~0ull;
            const uint32_t d = valid ? (uint32_t)((k[i] - kmin) >> shift) & 0xFFu : 0x100u;
            uint32_t r;
            if constexpr (kBallot) {
                const uint32_t peers = ballot_peers(d, __ballot_sync(0xffffffffu, valid));
                const uint32_t leader = __ffs(peers) - 1;
                const uint32_t o = (valid && lane == (int)leader)
                                       ? atomicAdd(&s_whist[warp][d], __popc(peers))
                                       : 0u;
                r = __shfl_sync(0xffffffffu, o, leader & 31u) + __popc(peers & lt);
            } else {
                // ATOMS resolves same-address lanes of one instruction in ascending lane
                // order, and instructions of one warp in program order: the returned count
                // IS the stable in-warp rank
                r = valid ? atomicAdd(&s_whist[warp][d], 1u) : 0u;
            }
            if (i & 1)
                rank2[i / 2] |= r << 16;
            else
                rank2[i / 2] = r;
        }
        __syncthreads();

        // ---- per-digit counts; publish this tile's aggregate; tile-local starts ----------
        uint32_t wpre[kWarps];
        uint32_t cnt = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            wpre[w] = cnt;
            cnt += s_whist[w][t];
        }
        uint64_t* my_status = status + (uint64_t)tile * kBins + t;
        st_relaxed_u64(my_status,
                       pack_status(tile == 0 ? kStateInclusive : kStateAggregate, epoch, cnt));
        const uint32_t tstart = block_exclusive_scan(cnt, s_scan, nullptr);
        // one lookup per key in the scatter: tile start of the digit + the warp's offset in it
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s_whist[w][t] = tstart + wpre[w];
        __syncthreads();

        // ---- scatter the staged tile into the sorted buffer (shared -> shared) ----------
#pragma unroll
        for (int i = 0; i < kPItems; ++i) {
            const uint32_t pos = wofs + 32 * i;
            if (pos < tile_n) {
                const uint32_t d = (uint32_t)((k[i] - kmin) >> shift) & 0xFFu;
                const uint32_t dst = s_whist[warp][d] +
                                     ((i & 1) ? (rank2[i / 2] >> 16) : (rank2[i / 2] & 0xFFFFu));
                so_k[dst] = k[i];
                if (kVals) so_v[dst] = st_v[pos];
            }
        }
        __syncthreads();  // the stage buffer is free: claim and prefetch the next tile now
        if (tid == 0) {
            const uint32_t nx = atomicAdd(ticket, 1u);
            s_tile[1] = nx;
            if (nx < num_tiles) issue(nx);
        }

        // ---- decoupled look-back, per digit ----------------------------------------------
        uint32_t excl = 0;
        if (tile > 0) {
            const uint32_t st0 = status_state(probe, epoch);
            if (st0 == kStateInclusive) {
                excl = (uint32_t)probe;  // the early probe already has it
            } else if (st0 == 0) {
                excl = lookback_window<kLookbackWin>(status + t, kBins, tile, epoch);
            } else {
                excl = (uint32_t)probe +
                       lookback_window<kLookbackWin>(status + t, kBins, tile - 1, epoch);
            }
            st_relaxed_u64(my_status, pack_status(kStateInclusive, epoch, excl + cnt));
        }
        s_global[t] = s_bin_start[t] + excl - tstart;
        __syncthreads();
        const uint32_t next_tile = s_tile[1];

        // ---- write out: consecutive threads -> consecutive positions of each digit run ---
#pragma unroll 4
        for (int j = 0; j < kPItems; ++j) {
            const uint32_t p = j * kThreads + tid;
            if (p < tile_n) {
                const uint64_t key = so_k[p];
                const uint64_t rel = key - kmin;
                const uint32_t d = (uint32_t)(rel >> shift) & 0xFFu;
                const uint64_t out = (uint64_t)(uint32_t)(s_global[d] + p);
                keys_out[out] = key;
                if (kVals) vals_out[out] = so_v[p];
                if (kCountNext) atomicAdd(&s_next[(uint32_t)(rel >> next_shift) & 0xFFu], 1u);
            }
        }
        tile = next_tile;
    }
    if (kCountNext) {
        __syncthreads();
        const uint32_t c = s_next[tid];
        if (c) atomicAdd(&next_hist[tid], c);
    }
}

// Histogram of one digit of (key - kmin) (used only when the distance kernel's raw
// low-byte histogram does not apply, e.g. for the survivor sort).
// 8 independent 16-byte loads (16 keys) in flight per thread per step, per-warp shared
// histograms (no cross-warp contention), one global add per bin per block.
__global__ void __launch_bounds__(kBins)
    k2_digit_histogram(const uint64_t* __restrict__ keys, uint64_t count, uint64_t kmin,
                       uint32_t shift, uint32_t* hist) {
    __shared__ uint32_t h[kBins / 32][kBins];
    const int warp = threadIdx.x >> 5;
#pragma unroll
    for (int w = 0; w < kBins / 32; ++w) h[w][threadIdx.x] = 0;
    __syncthreads();
    auto add = [&](uint64_t k) { atomicAdd(&h[warp][(uint32_t)((k - kmin) >> shift) & 0xFFu], 1u); };
    constexpr int kU = 8;  // ulonglong2 loads per thread per step
    const uint64_t pairs = count / 2;
    const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(keys);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    for (; i + (kU - 1) * stride < pairs; i += kU * stride) {
        ulonglong2 v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) v[u] = k2[i + u * stride];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            add(v[u].x);
            add(v[u].y);
        }
    }
    for (; i < pairs; i += stride) {
        const ulonglong2 v = k2[i];
        add(v.x);
        add(v.y);
    }
    if ((count & 1) && blockIdx.x == 0 && threadIdx.x == 0) add(keys[count - 1]);
    __syncthreads();
    uint32_t c = 0;
#pragma unroll
    for (int w = 0; w < kBins / 32; ++w) c += h[w][threadIdx.x];
    if (c) atomicAdd(&hist[threadIdx.x], c);
}

int g_rank_variant = -1;  // 3 = ATOMS ranking, 2 = ballots; set by sort_self_test()

int rank_variant() {
    if (g_rank_variant < 0) {
        const char* e = getenv("PH0B_RANK");  // test hook: force the ballot ranking
        g_rank_variant = e ? atoi(e) : 2;
    }
    return g_rank_variant;
}

template <bool kVals, bool kCountNext, bool kBallot>
int launch_pass_t(const SortArgs& a, int cur, uint32_t p, const SortPlan& plan, uint32_t rot,
                  uint32_t* next_hist, cudaStream_t s, int num_sms) {
    auto kern = k2_onesweep_p<kVals, kCountNext, kBallot>;
    const size_t smem = (size_t)kPTile * 8 * 2 + (size_t)kPTile * 4 * 2;
    const int per_sm = kernel_blocks_per_sm((const void*)kern, kThreads, smem);
    if (per_sm < 1) return -1;
    const uint64_t tiles = (a.count + kPTile - 1) / kPTile;
    uint64_t grid = (uint64_t)num_sms * per_sm;
    if (grid > tiles) grid = tiles;
    const uint32_t next_shift = kCountNext ? plan.shift[p + 1] : 0u;
    kern<<<(unsigned)grid, kThreads, smem, s>>>(
        a.keys[cur], a.keys[cur ^ 1], kVals ? a.vals[cur] : nullptr,
        kVals ? a.vals[cur ^ 1] : nullptr, a.count, a.kmin, plan.shift[p], next_shift,
        a.hist + kBins * p, rot, a.status, a.epoch_base + p, next_hist, (uint32_t)tiles,
        a.tile_counter + p);
    return 1;
}

template <bool kVals, bool kCountNext>
int launch_pass(const SortArgs& a, int cur, uint32_t p, const SortPlan& plan, uint32_t rot,
                uint32_t* next_hist, cudaStream_t s, int num_sms) {
    return rank_variant() == 3
               ? launch_pass_t<kVals, kCountNext, false>(a, cur, p, plan, rot, next_hist, s, num_sms)
               : launch_pass_t<kVals, kCountNext, true>(a, cur, p, plan, rot, next_hist, s, num_sms);
}

// Self-test of the ordering property rank variant 3 relies on.  Returns true when every
// same-address lane pair of every ATOMS instruction was resolved in ascending lane order.
__global__ void k2_rank_self_test(unsigned long long* viol) {
    __shared__ uint32_t h[8][256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    uint32_t x = (blockIdx.x * 7919u + threadIdx.x * 104729u) ^ 0x9e3779b9u;
    unsigned long long v = 0;
    for (int it = 0; it < 64; ++it) {
        x = x * 1664525u + 1013904223u;
        const uint32_t d = (x >> 11) & ((it & 1) ? 7u : 255u);
        const uint32_t old = atomicAdd(&h[warp][d], 1u);
        for (int o = 0; o < 32; ++o) {  // uniform loop: every lane joins every shuffle
            const uint32_t od = __shfl_sync(0xffffffffu, d, o);
            const uint32_t oo = __shfl_sync(0xffffffffu, old, o);
            if (o < lane && od == d && !(oo < old)) ++v;
        }
    }
    if (v) atomicAdd(viol, v);
}

}  // namespace

bool sort_self_test(cudaStream_t s) {
    const char* e = getenv("PH0B_RANK");
    unsigned long long* d = nullptr;
    unsigned long long h = 1;
    if (cudaMalloc(&d, sizeof(h)) == cudaSuccess) {
        cudaMemsetAsync(d, 0, sizeof(h), s);
        k2_rank_self_test<<<64, 256, 0, s>>>(d);
        cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        cudaFree(d);
    }
    cudaGetLastError();
    g_rank_variant = e ? atoi(e) : (h == 0 ? 3 : 2);
    return h == 0;
}

uint64_t sort_tiles(uint64_t count) { return (count + kPTile - 1) / kPTile; }

int launch_digit_histogram(const uint64_t* keys, uint64_t count, uint64_t kmin, uint32_t shift,
                           uint32_t* hist, cudaStream_t s, int num_sms) {
    if (count == 0) return 0;
    uint64_t blocks = (count + kBins - 1) / kBins;
    const uint64_t cap = (uint64_t)num_sms * 8;
    if (blocks > cap) blocks = cap;
    if (reinterpret_cast<uintptr_t>(keys) & 15u) {  // 16-byte loads: peel one key
        k2_digit_histogram<<<1, kBins, 0, s>>>(keys, 1, kmin, shift, hist);
        ++keys;
        --count;
    }
    k2_digit_histogram<<<(unsigned)blocks, kBins, 0, s>>>(keys, count, kmin, shift, hist);
    return 1;
}

int launch_sort_passes(const SortArgs& a, const SortPlan& plan, cudaStream_t s, int num_sms,
                       int* launches) {
    int cur = 0;
    if (a.count == 0 || plan.passes == 0) return 0;
    cudaMemsetAsync(a.tile_counter, 0, sizeof(uint32_t) * 8, s);  // tile tickets per pass
    // hist rows 1..passes-1 are produced by the passes themselves
    if (plan.passes > 1)
        cudaMemsetAsync(a.hist + kBins, 0, sizeof(uint32_t) * kBins * (plan.passes - 1), s);
    for (uint32_t p = 0; p < plan.passes; ++p) {
        const bool last = p + 1 == plan.passes;
        uint32_t* next_hist = last ? nullptr : a.hist + kBins * (p + 1);
        const uint32_t rot = (p == 0) ? a.hist0_rot : 0u;
        int r;
        if (a.vals[0])
            r = last ? launch_pass<true, false>(a, cur, p, plan, rot, next_hist, s, num_sms)
                     : launch_pass<true, true>(a, cur, p, plan, rot, next_hist, s, num_sms);
        else
            r = last ? launch_pass<false, false>(a, cur, p, plan, rot, next_hist, s, num_sms)
                     : launch_pass<false, true>(a, cur, p, plan, rot, next_hist, s, num_sms);
        if (r < 0) return -1;
        if (launches) ++*launches;
        cur ^= 1;
    }
    return cur;
}

}  // namespace ph0b
