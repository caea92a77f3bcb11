// K2c/K3 — flag-and-scan unique and boundary-matrix grades (replaces the dedup/grade loop
// of build_filtration, /root/reference/proj/src/filtration.cpp:29-33, and the grade half
// of build_boundary_matrix, /root/reference/proj/src/boundary_matrix.cpp:19-26).
//
//   flag_i  = (i == 0) || key_i != key_{i-1}            (exact f64 `!=`, filtration.cpp:30)
//   grade_i = inclusive_scan(flag)_i                     (1-based, filtration.cpp:32)
//   D[grade_i - 1] = length_i  for flagged i             (Filtration::scale)
//
// Single pass: one 4096-key tile per CTA (dynamic tile ids), warp ballots for the
// in-tile scan, decoupled look-back for the prefix across tiles.  Column j of M is
// {u_j, v_j} at grade_j: the sorted (u << 16 | v) array already holds the supports, and
// the grades are written only when requested (parity surfaces); the barcode collect
// recovers a survivor's grade from D by binary search instead.
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace ph0b {
namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;
constexpr int kTileKeys = kThreads * kItems;

constexpr uint32_t kMaxRun = 64;  // longest equal-prefix run fixed up in place

// Stable insertion sort of the run [a, a+len) by full key, in global memory (runs are short:
// the radix passes ordered by the top 40 bits of the span, so a run is a handful of lengths
// within one 2^low_bits-ULP cell, already in (u, v) order among themselves).
__device__ void fix_run(uint64_t* keys, uint32_t* vals, uint64_t a, uint32_t len) {
    for (uint32_t i = 1; i < len; ++i) {
        const uint64_t k = keys[a + i];
        const uint32_t v = vals[a + i];
        uint32_t j = i;
        while (j > 0 && keys[a + j - 1] > k) {
            keys[a + j] = keys[a + j - 1];
            vals[a + j] = vals[a + j - 1];
            --j;
        }
        keys[a + j] = k;
        vals[a + j] = v;
    }
}

// low_bits == 0: keys are fully sorted; flag-and-scan unique over the tile.
// low_bits  > 0: keys are sorted by prefix = (key - kmin) >> low_bits only.  Every run of
// equal prefix is first sorted by full key (stably) by the tile in which it starts; a tile
// owns exactly the runs that start in it (its first elements may continue the previous
// tile's run; its last run may extend past its end).  Runs longer than kMaxRun raise
// *redo and the caller re-sorts with the full digit plan.
__global__ void __launch_bounds__(kThreads, 2)
    k3_unique(uint64_t* __restrict__ keys, uint32_t* __restrict__ vals, uint64_t count,
              uint64_t kmin, uint32_t low_bits, double* __restrict__ scale,
              uint32_t* __restrict__ grade, uint64_t* __restrict__ status,
              uint32_t* tile_counter, uint32_t epoch, uint64_t* n_scale, uint32_t* redo) {
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_warp_tot[kWarps];
    __shared__ uint32_t s_prefix;
    __shared__ uint64_t s_own[2];
    __shared__ uint32_t s_ext_tot;
    __shared__ int s_fixed;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        s_tile = atomicAdd(tile_counter, 1u);
        s_fixed = 0;
    }
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t tile_start = (uint64_t)tile * kTileKeys;
    const uint64_t tile_end = tile_start + kTileKeys < count ? tile_start + kTileKeys : count;
    const uint64_t wbase = tile_start + (uint64_t)warp * (32 * kItems) + lane;
    auto pre = [&](uint64_t kk) { return (kk - kmin) >> low_bits; };

    uint64_t k[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const uint64_t idx = wbase + 32 * i;
        k[i] = idx < tile_end ? keys[idx] : 0ull;
    }

    uint64_t own_start = tile_start, own_end = tile_end;
    if (low_bits) {
        // ---- phase A: sort the equal-prefix runs that start in this tile ----------------
        bool fixed = false;
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            const uint64_t idx = wbase + 32 * i;
            uint64_t prev = __shfl_up_sync(0xffffffffu, k[i], 1);
            uint64_t next = __shfl_down_sync(0xffffffffu, k[i], 1);
            if (lane == 0 && idx > 0 && idx < tile_end) prev = keys[idx - 1];
            if (lane == 31 && idx + 1 < count && idx < tile_end) next = keys[idx + 1];
            if (idx + 1 >= count || idx >= tile_end) continue;
            const uint64_t p = pre(k[i]);
            if (pre(next) != p || (idx > 0 && pre(prev) == p)) continue;  // not a run start
            uint32_t len = 2;
            while (idx + len < count && len <= kMaxRun && pre(keys[idx + len]) == p) ++len;
            if (len > kMaxRun) {
                atomicOr(redo, 1u);
                continue;
            }
            fix_run(keys, vals, idx, len);
            fixed = true;
        }
        if (__syncthreads_or(fixed)) {
#pragma unroll
            for (int i = 0; i < kItems; ++i) {  // re-read the (partly) re-ordered tile
                const uint64_t idx = wbase + 32 * i;
                k[i] = idx < tile_end ? keys[idx] : 0ull;
            }
        }
        if (tid == 0) {
            // skip the continuation of a run owned by an earlier tile
            uint64_t st = tile_start;
            if (st > 0) {
                const uint64_t p0 = pre(keys[st - 1]);
                while (st < tile_end && st < tile_start + kMaxRun + 1 && pre(keys[st]) == p0) ++st;
            }
            // extend through the run that crosses the tile end
            uint64_t e = tile_end;
            if (e < count && e > st) {
                const uint64_t pl = pre(keys[e - 1]);
                while (e < count && e < tile_end + kMaxRun + 1 && pre(keys[e]) == pl) ++e;
            }
            if (st >= tile_end) st = e = tile_end;  // the whole tile continues an earlier run
            s_own[0] = st;
            s_own[1] = e;
            uint32_t ext = 0;  // distinct values in the extension [tile_end, e)
            for (uint64_t g = tile_end; g < e; ++g) ext += keys[g] != keys[g - 1] ? 1u : 0u;
            s_ext_tot = ext;
        }
        __syncthreads();
        own_start = s_own[0];
        own_end = s_own[1];
    }

    // ---- phase B: flags, counts, look-back, D -------------------------------------------
    uint32_t ball[kItems];
    uint32_t total = 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const uint64_t idx = wbase + 32 * i;
        const bool valid = idx < tile_end;
        uint64_t prev = __shfl_up_sync(0xffffffffu, k[i], 1);
        if (lane == 0 && valid && idx > 0) prev = keys[idx - 1];
        const bool owned = valid && idx >= own_start && idx < own_end;
        const bool flag = owned && (idx == 0 || k[i] != prev);
        ball[i] = __ballot_sync(0xffffffffu, flag);
        total += __popc(ball[i]);
    }
    if (lane == 0) s_warp_tot[warp] = total;
    __syncthreads();
    uint32_t warp_base = 0, tile_tot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        warp_base += (w < warp) ? s_warp_tot[w] : 0u;
        tile_tot += s_warp_tot[w];
    }
    const uint32_t main_tot = tile_tot;
    if (low_bits) tile_tot += s_ext_tot;
    if (tid == 0) {
        uint64_t* my = status + tile;
        uint32_t excl = 0;
        if (tile == 0) {
            st_relaxed_u64(my, pack_status(kStateInclusive, epoch, tile_tot));
        } else {
            st_relaxed_u64(my, pack_status(kStateAggregate, epoch, tile_tot));
            excl = lookback_window<8>(status, 1, tile, epoch);
            st_relaxed_u64(my, pack_status(kStateInclusive, epoch, excl + tile_tot));
        }
        s_prefix = excl;
        const uint64_t tiles = (count + kTileKeys - 1) / kTileKeys;
        if (tile == tiles - 1) *n_scale = (uint64_t)excl + tile_tot;
        // the extension: elements past the tile end that belong to this tile's last run
        if (low_bits) {
            uint32_t r = excl + main_tot;
            for (uint64_t g = tile_end; g < own_end; ++g) {
                const bool f = keys[g] != keys[g - 1];
                if (f) scale[r] = __longlong_as_double((long long)keys[g]);
                r += f ? 1u : 0u;
                if (grade) grade[g] = r;
            }
        }
    }
    __syncthreads();
    uint32_t run = s_prefix + warp_base;
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const uint64_t idx = wbase + 32 * i;
        const bool flag = (ball[i] >> lane) & 1u;
        const uint32_t before = run + __popc(ball[i] & lt);  // flags strictly before idx
        if (flag) scale[before] = __longlong_as_double((long long)k[i]);
        if (grade && idx >= own_start && idx < own_end) grade[idx] = before + (flag ? 1u : 0u);
        run += __popc(ball[i]);
    }
}

}  // namespace

int launch_unique(const UniqueArgs& a, cudaStream_t s) {
    if (a.count == 0) {
        cudaMemsetAsync(a.n_scale, 0, sizeof(uint64_t), s);
        return 0;
    }
    const uint64_t tiles = (a.count + kTileKeys - 1) / kTileKeys;
    cudaMemsetAsync(a.tile_counter, 0, sizeof(uint32_t), s);
    k3_unique<<<(unsigned)tiles, kThreads, 0, s>>>(a.keys, a.vals, a.count, a.kmin, a.low_bits,
                                                   a.scale, a.grade, a.status, a.tile_counter,
                                                   a.epoch, a.n_scale, a.redo);
    return 1;
}

}  // namespace ph0b
