// K2 — onesweep-style LSD radix sort of (length bits, column) pairs (replaces the
// std::sort of build_filtration, /root/reference/proj/src/filtration.cpp:21-25).
//
// Keys are the f64 bit patterns of non-negative lengths, ordered as unsigned integers;
// only the digits of (key - kmin) that can differ are sorted (span = bits of kmax-kmin),
// 8 bits per pass.  Every pass is stable and the input is the reference's u-major order,
// so equal lengths end up ordered by (u, v) exactly as filtration.cpp:21-25 orders them.
//
// One kernel per digit (Adinets & Merrill's single-pass "onesweep"), persistent, launched as
// thread-block clusters of two CTAs.  A cluster claims two consecutive 4096-key tiles at a
// time with an atomic ticket (the next pair while the current one is still being written;
// keys and columns are prefetched into shared memory with TMA bulk copies).  Each CTA ranks
// its tile's keys in-warp with shared-memory atomics on per-warp digit counters (B200
// resolves the same-address lanes of one ATOMS in lane order — checked on the device at
// context creation; bit-sliced ballots otherwise) and pushes its per-digit counts into its
// partner's shared memory (DSMEM stores tracked by an mbarrier).  One look-back status per
// tile pair is published; the exclusive prefix over earlier pairs comes from a decoupled
// look-back on epoch-tagged status words.  Each CTA then scatters its tile into shared memory
// in digit order and writes it out so that each digit's run is a contiguous global run.  The
// same pass counts the NEXT digit's histogram, so no separate upsweep over the keys is
// needed.  Tickets make the look-back deadlock-free whatever else shares the GPU: every pair
// a CTA waits on was claimed earlier by a cluster that is already running.
#include <cuda_runtime.h>

#include <algorithm>
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

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `p` (this CTA's shared memory) in cluster CTA `rank`
__device__ __forceinline__ uint32_t dsmem_addr(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_dsmem(uint32_t addr, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
// Asynchronous store into a cluster peer's shared memory that completes 4 bytes of the
// transaction count of the peer's mbarrier (no cluster-wide barrier, no memory fence).
__device__ __forceinline__ void st_async_dsmem(uint32_t addr, uint32_t v, uint32_t bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u32 [%0], %1, [%2];" ::"r"(
                     addr),
                 "r"(v), "r"(bar)
                 : "memory");
}

// kC == 1: one CTA per tile, one look-back status per tile.
// kC > 1 (thread-block cluster of kC CTAs): the cluster claims a super-tile of kC consecutive
// tiles, CTA r sorts tile kC*s + r; every CTA pushes its per-digit counts into its peers'
// shared memory with mbarrier-tracked asynchronous stores (CTA 0 also pushes the next
// super-tile's ticket), CTA 0 publishes ONE look-back status per super-tile as soon as the
// counts are in, so the look-back walks kC times fewer links (each covering kC*4096 keys).
template <bool kVals, bool kCountNext, bool kBallot, int kC>
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
    __shared__ uint32_t s_tile[2];                       // (kC > 1: super-tile, by parity)
    // kC > 1: counts of every cluster CTA, by iteration parity, and their mbarriers
    __shared__ uint32_t s_cnt[kC > 1 ? 2 : 1][kC > 1 ? kC : 1][kC > 1 ? kBins : 1];
    __shared__ __align__(8) uint64_t s_cbar[2];
    __shared__ __align__(8) uint64_t s_bar;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t t = tid;  // digit handled by this thread in the per-digit phases
    const uint32_t cr = kC > 1 ? cluster_rank() : 0u;
    const uint32_t num_super = (num_tiles + kC - 1) / kC;
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
        if constexpr (kC == 1) {
            const uint32_t first = atomicAdd(ticket, 1u);
            s_tile[0] = first;
            if (first < num_tiles) issue(first);
        } else {
            for (int q = 0; q < 2; ++q)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&s_cbar[q])));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            if (cr == 0) {  // the cluster's first super-tile, to every CTA of the cluster
                const uint32_t first = atomicAdd(ticket, 1u);
                for (uint32_t q = 0; q < (uint32_t)kC; ++q)
                    st_dsmem(dsmem_addr(&s_tile[0], q), first);
            }
        }
    }
    if (kCountNext) s_next[tid] = 0;
    {
        const uint32_t hcount = hist[(t + hist_rot) & 0xFFu];
        s_bin_start[t] = block_exclusive_scan(hcount, s_scan, nullptr);
    }
    if constexpr (kC > 1) {
        cluster_arrive();
        cluster_wait();
        if (tid == 0 && kC * s_tile[0] + cr < num_tiles) issue(kC * s_tile[0] + cr);
    }
    __syncthreads();
    uint32_t sup = s_tile[0];  // (super-)tile being processed
    uint32_t parity = 0, it = 0, cpar = 0;  // cpar: phase bits of s_cbar[0..1]
    const uint32_t lt = lanemask_lt();

    while (sup < num_super) {
        const uint32_t tile = kC * sup + cr;
        const uint64_t base = (uint64_t)tile * kPTile;
        const uint64_t rem = tile < num_tiles ? count - base : 0;
        const uint32_t tile_n = rem < (uint64_t)kPTile ? (uint32_t)rem : (uint32_t)kPTile;
        const uint32_t par = it & 1u;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s_whist[w][tid] = 0;
        __syncthreads();
        // kC > 1: the next super-tile is claimed now; its latency hides behind this tile
        uint32_t claimed = 0;
        if (kC > 1 && cr == 0 && tid == 0) claimed = atomicAdd(ticket, 1u);
        // the look-back's probe of the previous (super-)tile goes out before this tile is
        // even ranked: its latency hides behind the rank, scan and scatter phases (C5: 14.51
        // -> 13.83 ms per pass vs issuing it after this tile's aggregate is published)
        const uint64_t probe =
            sup > 0 ? ld_relaxed_u64(status + (uint64_t)(sup - 1) * kBins + t) : 0ull;
        if (tile_n) {
            mbar_wait_parity(&s_bar, parity);
            parity ^= 1u;
        }

        // ---- rank within the warp (keys from the staged tile) --------------------------
        uint64_t k[kPItems];
        uint32_t vv[kVals ? kPItems : 1];  // columns, read with the keys (C5: 13.04 -> 12.92 ms
                                           // per pass vs reading them during the scatter)
        uint32_t rank2[kPItems / 2];
        const uint32_t wofs = warp * (32 * kPItems) + lane;
#pragma unroll
        for (int i = 0; i < kPItems; ++i) {
            const uint32_t pos = wofs + 32 * i;
            const bool valid = pos < tile_n;
            k[i] = valid ? st_k[pos] : ~0ull;
            if constexpr (kVals) vv[i] = valid ? st_v[pos] : 0u;
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

        // ---- per-digit counts; publish them; tile-local starts ----------------------------
        uint32_t wpre[kWarps];
        uint32_t cnt = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            wpre[w] = cnt;
            cnt += s_whist[w][t];
        }
        uint64_t* my_status = status + (uint64_t)sup * kBins + t;
        uint32_t before = 0, agg = cnt;  // kC > 1: counts of the earlier CTAs / whole cluster
        auto gather = [&]() {  // (kC > 1) after the counts of every peer have landed
            agg = 0;
#pragma unroll
            for (int q = 0; q < kC; ++q) {
                const uint32_t c = s_cnt[par][q][t];
                before += (uint32_t)q < cr ? c : 0u;
                agg += c;
            }
        };
        bool got = false;  // kC > 1: the cluster's counts for my digit are in
        auto publish_agg = [&]() {
            gather();
            st_relaxed_u64(my_status,
                           pack_status(sup == 0 ? kStateInclusive : kStateAggregate, epoch, agg));
        };
        if constexpr (kC == 1) {
            st_relaxed_u64(my_status,
                           pack_status(sup == 0 ? kStateInclusive : kStateAggregate, epoch, cnt));
        } else {
            // my counts into every CTA's slot [cr]; CTA 0 also hands out the next super-tile
            s_cnt[par][cr][t] = cnt;
            const uint32_t bytes = (kC - 1) * kBins * 4 + (cr != 0 ? 4u : 0u);
            if (tid == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                                 smem_addr(&s_cbar[par])),
                             "r"(bytes)
                             : "memory");
            for (uint32_t q = 0; q < (uint32_t)kC; ++q) {
                if (q == cr) continue;
                const uint32_t bar = dsmem_addr(&s_cbar[par], q);
                st_async_dsmem(dsmem_addr(&s_cnt[par][cr][t], q), cnt, bar);
                if (cr == 0 && tid == 0) st_async_dsmem(dsmem_addr(&s_tile[par ^ 1u], q), claimed, bar);
            }
            if (cr == 0 && tid == 0) s_tile[par ^ 1u] = claimed;
            // CTA 0 waits for its peers' counts right away and publishes the super-tile's
            // aggregate before its own scan; the others collect the counts after their
            // scatter.  (C5, per pass: 12.96 ms; 13.09 ms when a peer that already has all
            // counts publishes the aggregate too, 13.71 ms when every CTA publishes after its
            // scatter — late and duplicate status stores lengthen successors' look-backs.)
            // Each thread reads only its own digit's column.
            if (cr == 0) {
                mbar_wait_parity(&s_cbar[par], (cpar >> par) & 1u);
                got = true;
                publish_agg();
            }
        }
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
                if constexpr (kVals) so_v[dst] = vv[i];
            }
        }
        __syncthreads();  // the stage buffer is free: prefetch the next tile now
        uint32_t next_sup;
        if constexpr (kC == 1) {
            if (tid == 0) {
                const uint32_t nx = atomicAdd(ticket, 1u);
                s_tile[1] = nx;
                if (nx < num_tiles) issue(nx);
            }
        } else {
            if (!got) {  // (CTA r > 0 only) the counts of the earlier CTAs
                mbar_wait_parity(&s_cbar[par], (cpar >> par) & 1u);
                gather();
            }
            cpar ^= 1u << par;
            next_sup = s_tile[par ^ 1u];
            if (tid == 0 && kC * next_sup + cr < num_tiles) issue(kC * next_sup + cr);
        }

        // ---- decoupled look-back over earlier (super-)tiles, per digit --------------------
        uint32_t excl = 0;
        if (sup > 0) {
            const uint32_t st0 = status_state(probe, epoch);
            if (st0 == kStateInclusive) {
                excl = (uint32_t)probe;  // the early probe already has it
            } else if (st0 == 0) {
                excl = lookback_window<kLookbackWin>(status + t, kBins, sup, epoch);
            } else {
                excl = (uint32_t)probe +
                       lookback_window<kLookbackWin>(status + t, kBins, sup - 1, epoch);
            }
            if (cr == 0) st_relaxed_u64(my_status, pack_status(kStateInclusive, epoch, excl + agg));
        }
        s_global[t] = s_bin_start[t] + excl + before - tstart;
        __syncthreads();
        if constexpr (kC == 1) next_sup = s_tile[1];

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
        sup = next_sup;
        ++it;
    }
    if (kCountNext) {
        __syncthreads();
        const uint32_t c = s_next[tid];
        if (c) atomicAdd(&next_hist[tid], c);
    }
    if constexpr (kC > 1) {  // no CTA leaves while a peer may still read its counts
        cluster_arrive();
        cluster_wait();
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

// CTAs per look-back super-tile.  C5, per pass: 13.70 ms with one CTA per look-back status,
// 12.96-13.02 ms with clusters of 2, 21.3 ms with clusters of 4 (every super-tile waits for
// the slowest of four CTAs before its aggregate is out); look-back windows of 2 / 3 / 6
// super-tiles per round trip with clusters of 2: 13.42 / 13.06-13.09 / 13.07-13.08 ms.
constexpr int kSortCluster = 2;

template <bool kVals, bool kCountNext, bool kBallot, int kC>
int launch_pass_c(const SortArgs& a, int cur, uint32_t p, const SortPlan& plan, uint32_t rot,
                  uint32_t* next_hist, cudaStream_t s, int num_sms) {
    auto kern = k2_onesweep_p<kVals, kCountNext, kBallot, kC>;
    const size_t smem = (size_t)kPTile * 8 * 2 + (size_t)kPTile * 4 * 2;
    const int per_sm = kernel_blocks_per_sm((const void*)kern, kThreads, smem);
    if (per_sm < 1) return -1;
    const uint64_t tiles = (a.count + kPTile - 1) / kPTile;
    const uint32_t next_shift = kCountNext ? plan.shift[p + 1] : 0u;
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    uint64_t grid = (uint64_t)num_sms * per_sm;
    if (kC > 1) {
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = kC;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(kC);
        int clusters = 0;
        if (cudaOccupancyMaxActiveClusters(&clusters, (void*)kern, &cfg) != cudaSuccess ||
            clusters < 1) {
            cudaGetLastError();
            return -1;
        }
        // tickets keep a cluster that starts late from blocking anyone: size the grid by
        // the SM count, not by the (conservative) cluster occupancy estimate
        const uint64_t supers = (tiles + kC - 1) / kC;
        grid = std::min<uint64_t>(grid / kC, supers) * kC;
    } else if (grid > tiles) {
        grid = tiles;
    }
    cfg.gridDim = dim3((unsigned)grid);
    const cudaError_t e = cudaLaunchKernelEx(
        &cfg, kern, (const uint64_t*)a.keys[cur], a.keys[cur ^ 1],
        (const uint32_t*)(kVals ? a.vals[cur] : nullptr), kVals ? a.vals[cur ^ 1] : nullptr,
        a.count, a.kmin, plan.shift[p], next_shift, (const uint32_t*)(a.hist + kBins * p), rot,
        a.status, a.epoch_base + p, next_hist, (uint32_t)tiles, a.tile_counter + p);
    return e == cudaSuccess ? 1 : -1;
}

template <bool kVals, bool kCountNext>
int launch_pass(const SortArgs& a, int cur, uint32_t p, const SortPlan& plan, uint32_t rot,
                uint32_t* next_hist, cudaStream_t s, int num_sms) {
    return rank_variant() == 3
               ? launch_pass_c<kVals, kCountNext, false, kSortCluster>(a, cur, p, plan, rot,
                                                                       next_hist, s, num_sms)
               : launch_pass_c<kVals, kCountNext, true, kSortCluster>(a, cur, p, plan, rot,
                                                                      next_hist, s, num_sms);
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
