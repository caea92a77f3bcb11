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
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace ph0b {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 12;
constexpr int kTileKeys = kThreads * kItems;
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

// Stable warp-level multisplit of one digit per lane: the mask of lanes holding the same
// digit, by bit-sliced ballots (pure ALU, no MIO round trip) or by match.any.
template <int kRank>
__device__ __forceinline__ uint32_t peer_mask(uint32_t d, uint32_t valid_mask) {
    if constexpr (kRank == 2) {
        uint32_t peers = valid_mask;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const uint32_t bit = (d >> b) & 1u;
            const uint32_t bal = __ballot_sync(0xffffffffu, bit);
            peers &= bit ? bal : ~bal;
        }
        return peers;
    } else {
        return __match_any_sync(0xffffffffu, d);
    }
}

// kRank: 0 = match.any + leader LDS/STS chain, 1 = match.any + leader atomicAdd (pipelined),
//        2 = bit-sliced ballots + leader atomicAdd.
template <bool kVals, bool kCountNext, int kRank, int kMinBlocks>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
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

    // ---- load keys (warp-striped, coalesced) and rank within the warp ------------------
    uint64_t k[kItems];
    // per item: [4:0] leader lane, [9:5] peers before me, [31:10] leader's warp-counter value
    uint32_t pk[kItems];
    const uint64_t wbase = base + (uint64_t)warp * (32 * kItems) + lane;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const uint64_t idx = wbase + 32 * i;
        k[i] = idx < count ? keys_in[idx] : ~0ull;
    }
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const bool valid = wbase + 32 * i < count;
        const uint32_t d = valid ? (uint32_t)((k[i] - kmin) >> shift) & 0xFFu : 0x100u;
        if constexpr (kRank == 3) {
            // ATOMS resolves same-address lanes of one instruction in ascending lane order
            // (verified on the device at context creation, see rank_self_test), and
            // instructions of one warp in program order: the returned count IS the stable
            // in-warp rank.
            pk[i] = valid ? atomicAdd(&s_whist[warp][d], 1u) : 0u;
            continue;
        }
        const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
        const uint32_t peers = peer_mask<kRank>(d, vmask);
        const uint32_t leader = __ffs(peers) - 1;
        const uint32_t before = __popc(peers & lt);
        if constexpr (kRank == 0) {
            uint32_t o = 0;
            if (valid && lane == (int)leader) o = s_whist[warp][d];
            o = __shfl_sync(0xffffffffu, o, leader);
            pk[i] = o + before;
            if (valid && lane == (int)leader) s_whist[warp][d] = o + __popc(peers);
            __syncwarp();
        } else {
            const uint32_t o = (valid && lane == (int)leader)
                                   ? atomicAdd(&s_whist[warp][d], __popc(peers))
                                   : 0u;
            pk[i] = leader | (before << 5) | (o << 10);
        }
    }
    uint32_t rank2[kItems / 2];  // two 16-bit in-warp ranks per register
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        uint32_t r;
        if constexpr (kRank == 0 || kRank == 3) {
            r = pk[i];
        } else {
            r = (__shfl_sync(0xffffffffu, pk[i], pk[i] & 31u) >> 10) + ((pk[i] >> 5) & 31u);
        }
        if (i & 1)
            rank2[i / 2] |= r << 16;
        else
            rank2[i / 2] = r;
    }
    __syncthreads();

    // ---- per-digit counts, warp offsets; publish this tile's aggregate early -------------
    const uint32_t t = tid;  // digit handled by this thread
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        const uint32_t c = s_whist[w][t];
        s_whist[w][t] = cnt;
        cnt += c;
    }
    uint64_t* my_status = status + (uint64_t)tile * kBins + t;
    st_relaxed_u64(my_status, pack_status(tile == 0 ? kStateInclusive : kStateAggregate, epoch, cnt));
    // first look-back probe goes out now; its latency hides behind the scans and the scatter
    uint64_t probe = tile > 0 ? ld_relaxed_u64(status + (uint64_t)(tile - 1) * kBins + t) : 0ull;

    // global start of digit t (exclusive scan of the rotated digit histogram) and the
    // tile-local start of digit t (exclusive scan of this tile's counts)
    const uint32_t hcount = hist[(t + hist_rot) & 0xFFu];
    const uint32_t bin_start = block_exclusive_scan(hcount, s_scan, nullptr);
    __syncthreads();
    const uint32_t tstart = block_exclusive_scan(cnt, s_scan, nullptr);
    s_tile_start[t] = tstart;
    __syncthreads();

    // ---- scatter into shared memory in (digit, input order) order -----------------------
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const uint64_t idx = wbase + 32 * i;
        if (idx < count) {
            const uint32_t d = (uint32_t)((k[i] - kmin) >> shift) & 0xFFu;
            const uint32_t pos = s_tile_start[d] + s_whist[warp][d] +
                                 ((i & 1) ? (rank2[i / 2] >> 16) : (rank2[i / 2] & 0xFFFFu));
            s_keys[pos] = k[i];
            if (kVals) s_vals[pos] = vals_in[idx];
        }
    }

    // ---- decoupled look-back over earlier tiles, per digit -------------------------------
    uint32_t excl = 0;
    if (tile > 0) {
        int64_t p = (int64_t)tile - 1;
        for (;;) {
            const uint32_t st = status_state(probe, epoch);
            if (st != 0) {
                excl += (uint32_t)probe;
                if (st == kStateInclusive) break;
                --p;
            }
            probe = ld_relaxed_u64(status + (uint64_t)p * kBins + t);
        }
        st_relaxed_u64(my_status, pack_status(kStateInclusive, epoch, excl + cnt));
    }
    // output position of the element at tile-local position p with digit d: delta[d] + p
    s_global[t] = bin_start + excl - tstart;
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
            const uint64_t out = (uint64_t)(uint32_t)(s_global[d] + p);
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

// ---- persistent onesweep with TMA bulk prefetch -------------------------------------------
// Static tile assignment (tile = blockIdx.x + r * gridDim.x, all CTAs co-resident), so a
// CTA can prefetch its next tile with cp.async.bulk (TMA, mbarrier completion) while it is
// still in the look-back and write-out phases of the current one; the look-back chain only
// ever waits on tiles of the same or an earlier round, which are being processed by
// co-resident CTAs (deadlock-free).
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

// kRestart: if the early probe of tile - 1 is not inclusive, the look-back restarts at tile - 1
// (measured ablation: PH0B_LOOKBACK=restart); default: the early probe's aggregate is
// consumed and the look-back continues at tile - 2 in windows of kLookbackWin.
constexpr int kLookbackWin = 4;
template <bool kVals, bool kCountNext, bool kRestart, bool kTop = false>
__global__ void __launch_bounds__(kThreads, 2)
    k2_onesweep_p(const uint64_t* __restrict__ keys_in, uint64_t* __restrict__ keys_out,
                  const uint32_t* __restrict__ vals_in, uint32_t* __restrict__ vals_out,
                  uint64_t count, uint64_t kmin, uint32_t shift, uint32_t next_shift,
                  const uint32_t* __restrict__ hist, uint32_t hist_rot,
                  uint64_t* __restrict__ status, uint32_t epoch,
                  uint32_t* __restrict__ next_hist, uint32_t num_tiles) {
    extern __shared__ __align__(128) uint64_t p_dyn[];
    uint64_t* st_k = p_dyn;                                                    // stage keys
    uint32_t* st_v = reinterpret_cast<uint32_t*>(p_dyn + kPTile);              // stage vals
    uint64_t* so_k = p_dyn + kPTile + kPTile / 2;                              // sorted keys
    uint32_t* so_v = reinterpret_cast<uint32_t*>(so_k + kPTile);               // sorted vals
    __shared__ uint32_t s_whist[kWarps][kBins];
    __shared__ uint32_t s_tile_start[kBins];
    __shared__ uint32_t s_global[kBins];
    __shared__ uint32_t s_bin_start[kBins];
    __shared__ uint32_t s_next[kCountNext ? kBins : 1];
    __shared__ uint32_t s_scan[kWarps];
    __shared__ __align__(8) uint64_t s_bar;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t t = tid;  // digit handled by this thread in the per-digit phases
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&s_bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (kCountNext) s_next[tid] = 0;
    {
        const uint32_t hcount = hist[(t + hist_rot) & 0xFFu];
        s_bin_start[t] = block_exclusive_scan(hcount, s_scan, nullptr);
    }
    __syncthreads();

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
    uint32_t tile = blockIdx.x;
    if (tid == 0 && tile < num_tiles) issue(tile);
    uint32_t parity = 0;
    const uint32_t lt = lanemask_lt();

    for (; tile < num_tiles; tile += gridDim.x) {
        const uint64_t base = (uint64_t)tile * kPTile;
        const uint64_t rem = count - base;
        const uint32_t tile_n = rem < (uint64_t)kPTile ? (uint32_t)rem : (uint32_t)kPTile;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s_whist[w][tid] = 0;
        __syncthreads();
        // kTop: the look-back's probe of tile - 1 goes out here, before this tile is even
        // ranked: its latency hides behind the rank, scan and scatter phases (C5: 14.51 ->
        // 13.83 ms per pass vs issuing it after this tile's aggregate is published)
        uint64_t probe_top = 0;
        if (kTop && tile > 0) probe_top = ld_relaxed_u64(status + (uint64_t)(tile - 1) * kBins + t);
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
            const uint32_t r = valid ? atomicAdd(&s_whist[warp][d], 1u) : 0u;
            if (i & 1)
                rank2[i / 2] |= r << 16;
            else
                rank2[i / 2] = r;
        }
        (void)lt;
        __syncthreads();

        uint32_t cnt = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t c = s_whist[w][t];
            s_whist[w][t] = cnt;
            cnt += c;
        }
        uint64_t* my_status = status + (uint64_t)tile * kBins + t;
        st_relaxed_u64(my_status,
                       pack_status(tile == 0 ? kStateInclusive : kStateAggregate, epoch, cnt));
        // early probe of tile - 1 (its latency hides behind the scan and the scatter; an
        // aggregate read now is still valid after the scatter)
        const uint64_t probe =
            kTop ? probe_top
                 : (tile > 0 ? ld_relaxed_u64(status + (uint64_t)(tile - 1) * kBins + t) : 0ull);
        const uint32_t tstart = block_exclusive_scan(cnt, s_scan, nullptr);
        s_tile_start[t] = tstart;
        __syncthreads();

        // ---- scatter the staged tile into the sorted buffer (shared -> shared) ----------
#pragma unroll
        for (int i = 0; i < kPItems; ++i) {
            const uint32_t pos = wofs + 32 * i;
            if (pos < tile_n) {
                const uint32_t d = (uint32_t)((k[i] - kmin) >> shift) & 0xFFu;
                const uint32_t dst = s_tile_start[d] + s_whist[warp][d] +
                                     ((i & 1) ? (rank2[i / 2] >> 16) : (rank2[i / 2] & 0xFFFFu));
                so_k[dst] = k[i];
                if (kVals) so_v[dst] = st_v[pos];
            }
        }
        __syncthreads();  // the stage buffer is free: prefetch the next tile now
        const uint32_t next = tile + gridDim.x;
        if (tid == 0 && next < num_tiles) issue(next);

        // ---- decoupled look-back, per digit ----------------------------------------------
        uint32_t excl = 0;
        if (tile > 0) {
            const uint32_t st0 = status_state(probe, epoch);
            if (st0 == kStateInclusive) {
                excl = (uint32_t)probe;  // the early probe already has it
            } else if (kRestart || st0 == 0) {
                excl = lookback_window<kRestart ? 8 : kLookbackWin>(status + t, kBins, tile, epoch);
            } else {
                // tile - 1 had published its aggregate: keep it and continue at tile - 2
                // (older tiles are the ones likely inclusive by now); C5: 14.85 -> 14.26
                // ms per pass vs restarting at tile - 1 with windows of 8
                excl = (uint32_t)probe +
                       lookback_window<kLookbackWin>(status + t, kBins, tile - 1, epoch);
            }
            st_relaxed_u64(my_status, pack_status(kStateInclusive, epoch, excl + cnt));
        }
        s_global[t] = s_bin_start[t] + excl - tstart;
        __syncthreads();

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

template <bool kVals, bool kCountNext, int kRank, int kMinBlocks>
void launch_pass_r(const SortArgs& a, int cur, uint32_t p, const SortPlan& plan, uint32_t rot,
                   uint32_t* next_hist, uint64_t tiles, cudaStream_t s) {
    auto kern = k2_onesweep<kVals, kCountNext, kRank, kMinBlocks>;
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

int g_rank_variant = -1;  // set by sort_self_test(); env PH0B_RANK overrides

int rank_variant() {
    if (g_rank_variant < 0) {
        const char* e = getenv("PH0B_RANK");
        g_rank_variant = e ? atoi(e) : 2;
    }
    return g_rank_variant;
}

bool lookback_restart() {
    static const bool v = [] {
        const char* e = getenv("PH0B_LOOKBACK");
        return e && e[0] == 'r';  // "restart": the pre-continuation look-back (ablation)
    }();
    return v;
}

template <bool kVals, bool kCountNext>
void launch_pass_p(const SortArgs& a, int cur, uint32_t p, const SortPlan& plan, uint32_t rot,
                   uint32_t* next_hist, cudaStream_t s, int num_sms) {
    static const bool top = [] {  // PH0B_TOP_PROBE=0: probe after the publish (ablation)
        const char* e = getenv("PH0B_TOP_PROBE");
        return !(e && e[0] == '0');
    }();
    auto kern = lookback_restart() ? k2_onesweep_p<kVals, kCountNext, true>
                : top              ? k2_onesweep_p<kVals, kCountNext, false, true>
                                   : k2_onesweep_p<kVals, kCountNext, false>;
    const size_t smem = (size_t)kPTile * 8 * 2 + (size_t)kPTile * 4 * 2;
    static int grid_per_sm = 0;
    if (!grid_per_sm) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&grid_per_sm, kern, kThreads, smem);
        if (grid_per_sm < 1) grid_per_sm = 1;
    }
    const uint64_t tiles = (a.count + kPTile - 1) / kPTile;
    uint64_t grid = (uint64_t)num_sms * grid_per_sm;
    if (grid > tiles) grid = tiles;
    const uint32_t next_shift = kCountNext ? plan.shift[p + 1] : 0u;
    kern<<<(unsigned)grid, kThreads, smem, s>>>(
        a.keys[cur], a.keys[cur ^ 1], kVals ? a.vals[cur] : nullptr,
        kVals ? a.vals[cur ^ 1] : nullptr, a.count, a.kmin, plan.shift[p], next_shift,
        a.hist + kBins * p, rot, a.status, a.epoch_base + p, next_hist, (uint32_t)tiles);
}

bool use_persistent() {
    static const bool v = [] {
        const char* e = getenv("PH0B_SORT_KERNEL");
        return !(e && e[0] == 'o');  // 'o' = original dynamic-tile onesweep
    }();
    return v;
}

template <bool kVals, bool kCountNext>
void launch_pass(const SortArgs& a, int cur, uint32_t p, const SortPlan& plan, uint32_t rot,
                 uint32_t* next_hist, uint64_t tiles, cudaStream_t s) {
    static const int minb = [] {
        const char* e = getenv("PH0B_MINB");
        return e ? atoi(e) : 4;
    }();
    const int rv = rank_variant();
    if (rv == 3) {
        if (minb == 3)
            launch_pass_r<kVals, kCountNext, 3, 3>(a, cur, p, plan, rot, next_hist, tiles, s);
        else
            launch_pass_r<kVals, kCountNext, 3, 4>(a, cur, p, plan, rot, next_hist, tiles, s);
    } else {
        launch_pass_r<kVals, kCountNext, 2, 4>(a, cur, p, plan, rot, next_hist, tiles, s);
    }
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

uint64_t sort_tiles(uint64_t count) { return (count + kTileKeys - 1) / kTileKeys; }

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
        if (use_persistent() && rank_variant() == 3) {
            if (a.vals[0]) {
                if (last)
                    launch_pass_p<true, false>(a, cur, p, plan, rot, next_hist, s, num_sms);
                else
                    launch_pass_p<true, true>(a, cur, p, plan, rot, next_hist, s, num_sms);
            } else {
                if (last)
                    launch_pass_p<false, false>(a, cur, p, plan, rot, next_hist, s, num_sms);
                else
                    launch_pass_p<false, true>(a, cur, p, plan, rot, next_hist, s, num_sms);
            }
        } else if (a.vals[0]) {
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
