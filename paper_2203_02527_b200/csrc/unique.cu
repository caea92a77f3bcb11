// K2c/K3 — flag-and-scan unique and boundary-matrix grades (replaces the dedup/grade loop
// of build_filtration, /root/reference/proj/src/filtration.cpp:29-33, and the grade half
// of build_boundary_matrix, /root/reference/proj/src/boundary_matrix.cpp:19-26).
//
//   flag_i  = (i == 0) || key_i != key_{i-1}            (exact f64 `!=`, filtration.cpp:30)
//   grade_i = inclusive_scan(flag)_i                     (1-based, filtration.cpp:32)
//   D[grade_i - 1] = length_i  for flagged i             (Filtration::scale)
//
// A chain-free split over 4096-key tiles — (1) a persistent TMA-staged count pass (run
// fix-ups of truncated radix plans, per-tile distinct counts and owned ranges), (2) a scan of
// the tile counts, (3) a persistent TMA-staged pass writing D and the grades.  No tile waits
// on another tile (a single pass with decoupled look-back measured 15.4 ms at C5 against
// 12.1 ms for the split: its look-back serialised every tile behind one warp).  Column j of M
// is {u_j, v_j} at grade_j: the sorted (u << 16 | v) array already holds the supports, and
// the grades are written only when requested (parity surfaces); the barcode collect
// recovers a survivor's grade from D by binary search instead.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace ph0b {
namespace {

constexpr int kTileKeys = 4096;  // keys per tile (all unique kernels and the scratch sizing)

constexpr uint32_t kMaxRun = 64;  // longest equal-prefix run fixed up in place

constexpr int kExt = (int)kMaxRun + 1;  // extension past the tile end (runs crossing it)

// Exclusive scan of the per-tile distinct counts by one block of 32 warps: warp w owns a
// contiguous chunk and walks it 32 counts at a time (coalesced loads, warp scan, running
// carry); the 32 chunk totals are scanned in shared memory; a second walk writes offsets.
__global__ void __launch_bounds__(1024)
    k3_scan(const uint32_t* __restrict__ counts, uint32_t tiles, uint64_t* __restrict__ offsets,
            uint64_t* n_scale, const uint64_t* __restrict__ d_base) {
    __shared__ uint64_t s_tot[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t per = ((tiles + 31) / 32 + 31) / 32 * 32;  // chunk, multiple of 32
    const uint32_t b = warp * per;
    const uint32_t e = b + per < tiles ? b + per : tiles;
    uint64_t tot = 0;
    constexpr int kU = 8;  // independent loads in flight per lane
    for (uint32_t t0 = b; t0 < e; t0 += 32 * kU) {
        uint32_t x[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t t = t0 + 32 * u + lane;
            x[u] = t < e ? counts[t] : 0u;
        }
        uint32_t sum = 0;
#pragma unroll
        for (int u = 0; u < kU; ++u) sum += x[u];
        tot += __reduce_add_sync(0xffffffffu, sum);
    }
    if (lane == 0) s_tot[warp] = tot;
    __syncthreads();
    uint64_t carry = 0, all = 0;
    for (int w = 0; w < 32; ++w) {
        carry += w < warp ? s_tot[w] : 0u;
        all += s_tot[w];
    }
    for (uint32_t t0 = b; t0 < e; t0 += 32 * kU) {
        uint32_t x[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t t = t0 + 32 * u + lane;
            x[u] = t < e ? counts[t] : 0u;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t t = t0 + 32 * u + lane;
            uint32_t inc = x[u];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            if (t < e) offsets[t] = carry + inc - x[u];
            carry += __shfl_sync(0xffffffffu, inc, 31);
        }
    }
    if (threadIdx.x == 0) *n_scale = (d_base ? *d_base : 0ull) + all;
}

}  // namespace

// ---- persistent count / write passes ------------------------------------------------------
// Static tile order (no tile waits on another, so residency is not required); the next
// tile's keys (+ the kMaxRun extension) are prefetched with a TMA bulk copy while this tile
// is fixed up and counted (pass 1) or written (pass 2).
__device__ __forceinline__ uint32_t u_smem(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

constexpr int kUT = 4096;  // keys per tile
constexpr int kUThreads = 512;
constexpr int kUWarps = kUThreads / 32;
constexpr int kUItems = kUT / kUThreads;
constexpr int kUStage = kUT + 72;  // tile + extension (>= kExt), 16 B multiple

// kMode 1: fix-ups + per-tile counts and owned ranges only (no D).  kMode 2: D and grades
// from the per-tile offsets of a scan of those counts (no fix-ups).
template <int kMode>
__global__ void __launch_bounds__(kUThreads, 3)
    k3_unique_p(uint64_t* __restrict__ keys, uint32_t* __restrict__ vals, uint64_t count,
                uint64_t kmin, uint32_t low_bits, double* __restrict__ scale,
                uint32_t* __restrict__ grade, uint32_t* redo, uint32_t num_tiles,
                const uint64_t* __restrict__ d_base, uint32_t* __restrict__ tile_counts,
                int2* __restrict__ tile_own, const uint64_t* __restrict__ tile_offsets) {
    extern __shared__ __align__(128) uint64_t up_dyn[];
    __shared__ __align__(8) uint64_t s_bar[2];
    // by buffer parity: in the count pass a warp may start the next tile while slower warps
    // still read this tile's totals and owned range (no barrier at the loop top there)
    __shared__ uint32_t s_warp_tot[2][kUWarps];
    __shared__ int s_own[2][2];
    // kMode 1: run starts to fix, one per thread after the claims barrier (the claiming thread
    // keeps any beyond kRunList: a tile's runs then cost one run of latency, not several)
    constexpr uint32_t kRunList = kMode == 1 ? 512 : 1;
    __shared__ uint32_t s_runs[kRunList];
    __shared__ uint32_t s_nruns;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    auto pre = [&](uint64_t kk) { return (kk - kmin) >> low_bits; };
    if (tid == 0) {
        if (kMode == 1) s_nruns = 0;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(u_smem(&s_bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(u_smem(&s_bar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](uint32_t tl, int b) {
        const uint64_t b0 = (uint64_t)tl * kUT;
        const uint64_t n = count - b0 < (uint64_t)kUStage ? count - b0 : (uint64_t)kUStage;
        const uint32_t bytes = (uint32_t)((n * 8 + 15) & ~15ull);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                         u_smem(&s_bar[b])),
                     "r"(bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(u_smem(up_dyn + b * kUStage)),
            "l"(keys + b0), "r"(bytes), "r"(u_smem(&s_bar[b]))
            : "memory");
    };
    uint32_t tile = blockIdx.x;
    if (tid == 0 && tile < num_tiles) issue(tile, 0);
    // the key before each tile is loaded one tile ahead (its latency hides behind a tile)
    uint64_t k_before_next =
        tile < num_tiles && tile > 0 ? keys[(uint64_t)tile * kUT - 1] : 0ull;
    // kMode 2: the tile's owned range and D offset, also loaded one tile ahead (C5: their
    // exposed latency was ~30 % of the write pass's stall samples)
    int2 own_next = make_int2(0, 0);
    uint64_t off_next = 0;
    if (kMode == 2 && tile < num_tiles) {
        own_next = tile_own[tile];
        off_next = tile_offsets[tile];
    }
    const uint64_t base0 = d_base ? *d_base : 0ull;  // D index of this range's first length
    uint32_t phase[2] = {0, 0};
    int b = 0;
    for (; tile < num_tiles; tile += gridDim.x, b ^= 1) {
        uint64_t* s_k = up_dyn + b * kUStage;
        const uint64_t tile_start = (uint64_t)tile * kUT;
        const uint64_t tile_end = tile_start + kUT < count ? tile_start + kUT : count;
        const uint32_t tn = (uint32_t)(tile_end - tile_start);
        const uint64_t ext_end = tile_end + kExt < count ? tile_end + kExt : count;
        const uint32_t staged = (uint32_t)(ext_end - tile_start);
        {
            const uint32_t par = phase[b];
            asm volatile(
                "{\n\t.reg .pred p;\n"
                "UW_%=:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                "@!p bra UW_%=;\n}" ::"r"(u_smem(&s_bar[b])),
                "r"(par)
                : "memory");
            phase[b] ^= 1u;
        }
        // everyone is done with the other buffer: prefetch into it.  (The count pass needs no
        // barrier here: every read of the other buffer precedes the previous tile's last
        // barrier, which thread 0 — the one issuing the copy — has passed.)
        if (kMode == 2) __syncthreads();
        const uint32_t next = tile + gridDim.x;
        if (tid == 0 && next < num_tiles) issue(next, b ^ 1);
        const uint64_t k_before = k_before_next;
        // (run fix-ups of earlier tiles may rewrite keys[next*kUT - 1] — only in order
        // within an equal-prefix run, and only the prefix of k_before is used for run
        // bookkeeping; its exact value matters for the first flag only when the run
        // fix-ups are off, i.e. when nothing rewrites it)
        if (next < num_tiles) k_before_next = keys[(uint64_t)next * kUT - 1];
        const int2 ow = own_next;
        const uint64_t tile_off = off_next;
        if (kMode == 2 && next < num_tiles) {
            own_next = tile_own[next];
            off_next = tile_offsets[next];
        }

        uint32_t os = 0, oe = tn;
        uint32_t ext_tot = 0;  // (kMode 1, thread 0)
        if (kMode == 2) {
            os = (uint32_t)ow.x;
            oe = (uint32_t)ow.y;
        } else if (low_bits) {
            // ---- fix the equal-prefix runs that start in this tile (stable, in smem) -----
            const uint64_t p_before = pre(k_before);
            // Work is only needed where a run is out of order, and an out-of-order adjacent
            // pair can only lie inside an equal-prefix run (pre() is monotone, the array is
            // sorted by it): so the scan is one 64-bit compare per position (consecutive
            // lanes read consecutive keys).  Each out-of-order run is claimed by the thread
            // holding its first inversion, if the run starts in this tile; claims are made
            // read-only, before any thread reorders anything.
            // item j < kUItems: position wofs0 + 32 j of the tile; item kUItems: position
            // kUT + tid of the extension (a run starting here may be out of order only there)
            const uint32_t wofs0 = warp * (32 * kUItems) + lane;
            auto item_pos = [&](uint32_t j) {
                return j < (uint32_t)kUItems ? wofs0 + 32 * j : (uint32_t)kUT + tid;
            };
            uint32_t starts = 0;
            {
#pragma unroll
                for (int j = 0; j <= kUItems; ++j) {
                    const uint32_t i = item_pos(j);
                    const bool in = i > 0 && i < staged;
                    const bool inv = in && s_k[i] < s_k[i - 1];
                    starts |= inv ? (1u << j) : 0u;
                }
                uint32_t claims = 0;
                while (starts) {
                    const uint32_t j = (uint32_t)(__ffs(starts) - 1);
                    starts &= starts - 1;
                    const uint32_t i = item_pos(j);
                    const uint64_t p = pre(s_k[i]);
                    uint32_t st = i - 1;  // run start within the staged window
                    bool first = true;
                    while (st > 0 && pre(s_k[st - 1]) == p) {
                        first = first && !(s_k[st] < s_k[st - 1]);
                        --st;
                    }
                    const bool from_prev = st == 0 && tile_start > 0 && p == p_before;
                    if (first && !from_prev && st < tn) {
                        // the run's columns are loaded after the claims barrier: start
                        // bringing them into L1 now (their latency was ~35 % of this pass's
                        // stall samples, all threads waiting at the barrier behind it)
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(vals + tile_start + st));
                        const uint32_t slot = atomicAdd(&s_nruns, 1u);
                        if (slot < kRunList)
                            s_runs[slot] = st;
                        else
                            claims |= 1u << j;  // list full: this thread fixes it itself
                    }
                }
                starts = claims;
            }
            if (tid == kUThreads - 1) {
                // the owned range depends on prefixes only, which the fix-ups never change:
                // it is found here, beside the claims, not serially after the fix-ups
                uint32_t st = 0;
                if (tile_start > 0)
                    while (st < tn && pre(s_k[st]) == p_before) ++st;
                uint32_t e = tn;
                if (e > st && e < staged) {
                    const uint64_t pl = pre(s_k[e - 1]);
                    while (e < staged && pre(s_k[e]) == pl) ++e;
                }
                // this tile's last run runs past the staged window: its end (and the next
                // tile's first owned position) is not visible here — sorted or not, redo
                if (st < tn && e == staged && ext_end < count) atomicOr(redo, 1u);
                if (st >= tn) st = e = tn;
                s_own[b][0] = (int)st;
                s_own[b][1] = (int)e;
            }
            __syncthreads();  // every claim is made before any run is reordered
            const uint32_t listed = s_nruns < kRunList ? s_nruns : kRunList;
            bool mine = tid < listed;  // thread t fixes listed run t, then its own overflow
            while (mine || starts) {
                uint32_t i;
                uint64_t p;
                if (mine) {
                    mine = false;
                    i = s_runs[tid];
                    p = pre(s_k[i]);
                } else {
                    const uint32_t j = (uint32_t)(__ffs(starts) - 1);
                    starts &= starts - 1;
                    const uint32_t inv = item_pos(j);
                    p = pre(s_k[inv]);
                    i = inv - 1;  // prefixes never change: safe to re-walk while others fix
                    while (i > 0 && pre(s_k[i - 1]) == p) --i;
                }
                const uint64_t g = tile_start + i;
                uint32_t len = 2;
                while (i + len < staged && len <= kMaxRun && pre(s_k[i + len]) == p) ++len;
                if (len > kMaxRun || (i + len == staged && ext_end < count)) {
                    atomicOr(redo, 1u);
                    continue;
                }
                bool sorted = true;
                for (uint32_t a = 1; a < len; ++a) sorted = sorted && s_k[i + a - 1] <= s_k[i + a];
                if (sorted) continue;
                // the run's columns: all loads issued together (one memory latency), then a
                // stable insertion sort of (key, column) with the keys in shared memory
                uint32_t lv[kMaxRun + 1];
                for (uint32_t a = 0; a < len; ++a) lv[a] = vals[g + a];
                for (uint32_t a = 1; a < len; ++a) {
                    const uint64_t kk = s_k[i + a];
                    const uint32_t v = lv[a];
                    uint32_t j = a;
                    while (j > 0 && s_k[i + j - 1] > kk) {
                        s_k[i + j] = s_k[i + j - 1];
                        lv[j] = lv[j - 1];
                        --j;
                    }
                    s_k[i + j] = kk;
                    lv[j] = v;
                }
                for (uint32_t a = 0; a < len; ++a) {
                    keys[g + a] = s_k[i + a];
                    vals[g + a] = lv[a];
                }
            }
            __syncthreads();  // runs fixed; the owned range is in s_own
            os = (uint32_t)s_own[b][0];
            oe = (uint32_t)s_own[b][1];
            if (tid == 0) {
                s_nruns = 0;  // the run list is free again (next tile: after two barriers)
                // distinct lengths of this tile's last run past the tile end (fixed keys)
                for (uint32_t g = tn; g < oe; ++g) ext_tot += s_k[g] != s_k[g - 1] ? 1u : 0u;
            }
        }

        // ---- flags and counts (keys from shared memory) ------------------------------------
        uint32_t ball[kUItems];
        uint32_t total = 0;
        const uint32_t wofs = warp * (32 * kUItems) + lane;
#pragma unroll
        for (int i = 0; i < kUItems; ++i) {
            const uint32_t pos = wofs + 32 * i;
            const bool owned = pos < tn && pos >= os && pos < oe;
            const uint64_t prev = pos > 0 ? s_k[pos - 1] : k_before;
            const bool f = owned && (tile_start + pos == 0 || s_k[pos] != prev);
            ball[i] = __ballot_sync(0xffffffffu, f);
            total += __popc(ball[i]);
        }
        if (lane == 0) s_warp_tot[b][warp] = total;
        __syncthreads();
        uint32_t warp_base = 0, main_tot = 0;
#pragma unroll
        for (int w = 0; w < kUWarps; ++w) {
            warp_base += (w < warp) ? s_warp_tot[b][w] : 0u;
            main_tot += s_warp_tot[b][w];
        }
        if (kMode == 1) {  // counts and owned range of this tile for the scan
            if (tid == 0) {
                tile_counts[tile] = main_tot + ext_tot;
                tile_own[tile] = make_int2((int)os, (int)oe);
            }
            continue;  // (the loop-top barrier orders the buffer reuse)
        }
        const uint64_t base = base0 + tile_off;
        uint64_t run = base + warp_base;
        const uint32_t lt = lanemask_lt();
#pragma unroll
        for (int i = 0; i < kUItems; ++i) {
            const uint32_t pos = wofs + 32 * i;
            const bool flag = (ball[i] >> lane) & 1u;
            const uint64_t before = run + __popc(ball[i] & lt);
            if (flag) scale[before] = __longlong_as_double((long long)s_k[pos]);
            if (grade && pos < tn && pos >= os && pos < oe)
                grade[tile_start + pos] = (uint32_t)(before + (flag ? 1u : 0u));
            run += __popc(ball[i]);
        }
        if (tid == 0 && oe > tn) {  // the extension of this tile's last run
            uint64_t r = base + main_tot;
            for (uint32_t g = tn; g < oe; ++g) {
                const bool f = s_k[g] != s_k[g - 1];
                if (f) scale[r] = __longlong_as_double((long long)s_k[g]);
                r += f ? 1u : 0u;
                if (grade) grade[tile_start + g] = (uint32_t)r;
            }
        }
    }
}

uint64_t unique_scratch_words(uint64_t count) {
    const uint64_t tiles = (count + kTileKeys - 1) / kTileKeys;
    return (tiles + 1) / 2 + 1 + 2 * (tiles + 1) + 1;
}

int launch_unique(const UniqueArgs& a, cudaStream_t s) {
    if (a.count == 0) {
        cudaMemsetAsync(a.n_scale, 0, sizeof(uint64_t), s);
        return 0;
    }
    const uint64_t tiles = (a.count + kUT - 1) / kUT;
    static_assert(kUT == kTileKeys, "scratch sizing uses the same tiling");
    // scratch: counts (u32) | own (int2) | offsets (u64), unique_scratch_words(count) words
    uint32_t* counts = reinterpret_cast<uint32_t*>(a.scratch);
    int2* own = reinterpret_cast<int2*>(a.scratch + (tiles + 1) / 2 + 1);
    uint64_t* offsets = a.scratch + (tiles + 1) / 2 + 1 + tiles + 1;
    const size_t smem = (size_t)2 * kUStage * 8;
    const int per_sm1 = kernel_blocks_per_sm((const void*)k3_unique_p<1>, kUThreads, smem);
    const int per_sm2 = kernel_blocks_per_sm((const void*)k3_unique_p<2>, kUThreads, smem);
    if (per_sm1 < 1 || per_sm2 < 1) return -1;
    const uint64_t sms = (uint64_t)device_sm_count();
    const uint64_t g1 = std::min<uint64_t>(sms * per_sm1, tiles);
    const uint64_t g2 = std::min<uint64_t>(sms * per_sm2, tiles);
    k3_unique_p<1><<<(unsigned)g1, kUThreads, smem, s>>>(
        a.keys, a.vals, a.count, a.kmin, a.low_bits, a.scale, a.grade, a.redo, (uint32_t)tiles,
        a.d_base, counts, own, nullptr);
    k3_scan<<<1, 1024, 0, s>>>(counts, (uint32_t)tiles, offsets, a.n_scale, a.d_base);
    k3_unique_p<2><<<(unsigned)g2, kUThreads, smem, s>>>(
        a.keys, a.vals, a.count, a.kmin, a.low_bits, a.scale, a.grade, a.redo, (uint32_t)tiles,
        a.d_base, counts, own, offsets);
    return 3;
}

}  // namespace ph0b
