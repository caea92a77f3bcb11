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

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;
constexpr int kTileKeys = kThreads * kItems;

__global__ void __launch_bounds__(kThreads)
    k3_unique(const uint64_t* __restrict__ keys, uint64_t count, double* __restrict__ scale,
              uint32_t* __restrict__ grade, uint64_t* __restrict__ status,
              uint32_t* tile_counter, uint32_t epoch, uint64_t* n_scale) {
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_warp_tot[kWarps];
    __shared__ uint32_t s_prefix;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t wbase = (uint64_t)tile * kTileKeys + (uint64_t)warp * (32 * kItems) + lane;

    uint64_t k[kItems];
    uint32_t ball[kItems];
    uint32_t total = 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const uint64_t idx = wbase + 32 * i;
        const bool valid = idx < count;
        k[i] = valid ? keys[idx] : 0ull;
        uint64_t prev = __shfl_up_sync(0xffffffffu, k[i], 1);
        if (lane == 0 && valid && idx > 0) prev = keys[idx - 1];
        const bool flag = valid && (idx == 0 || k[i] != prev);
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
    if (tid == 0) {
        uint64_t* my = status + tile;
        uint32_t excl = 0;
        if (tile == 0) {
            st_relaxed_u64(my, pack_status(kStateInclusive, epoch, tile_tot));
        } else {
            st_relaxed_u64(my, pack_status(kStateAggregate, epoch, tile_tot));
            int64_t p = (int64_t)tile - 1;
            while (p >= 0) {
                const uint64_t s = ld_relaxed_u64(status + p);
                const uint32_t st = status_state(s, epoch);
                if (st == 0) continue;
                excl += (uint32_t)s;
                if (st == kStateInclusive) break;
                --p;
            }
            st_relaxed_u64(my, pack_status(kStateInclusive, epoch, excl + tile_tot));
        }
        s_prefix = excl;
        const uint64_t tiles = (count + kTileKeys - 1) / kTileKeys;
        if (tile == tiles - 1) *n_scale = (uint64_t)excl + tile_tot;
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
        if (grade && idx < count) grade[idx] = before + (flag ? 1u : 0u);
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
    k3_unique<<<(unsigned)tiles, kThreads, 0, s>>>(a.keys, a.count, a.scale, a.grade, a.status,
                                                   a.tile_counter, a.epoch, a.n_scale);
    return 1;
}

}  // namespace ph0b
