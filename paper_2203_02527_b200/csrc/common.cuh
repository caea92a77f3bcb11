// Shared device helpers for the sm_100a kernels (inline PTX wrappers, constants).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "colcodec.h"

namespace ph0b {

constexpr int kWarp = 32;

__device__ __forceinline__ uint32_t lane_id() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
    return r;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

// Relaxed gpu-scope 64-bit load/store for decoupled look-back status words: the payload
// (count) lives inside the same word as the flag, so no acquire/release pairing is needed.
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_cg_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// Streaming (evict-first) stores for write-once outputs.
__device__ __forceinline__ void st_cs_u64(uint64_t* p, uint64_t v) {
    asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_cs_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Look-back status word: [63:62] state, [61:32] epoch, [31:0] count.
constexpr uint64_t kStateAggregate = 1ull;
constexpr uint64_t kStateInclusive = 2ull;
__device__ __forceinline__ uint64_t pack_status(uint64_t state, uint32_t epoch, uint32_t count) {
    return (state << 62) | ((uint64_t)(epoch & 0x3FFFFFFFu) << 32) | count;
}
__device__ __forceinline__ uint32_t status_state(uint64_t s, uint32_t epoch) {
    return ((uint32_t)(s >> 32) & 0x3FFFFFFFu) == (epoch & 0x3FFFFFFFu) ? (uint32_t)(s >> 62) : 0u;
}

// Decoupled look-back for one prefix column: sums the counts of tiles tile-1, tile-2, ...
// down to the nearest INCLUSIVE entry.  `stride` is the distance in words between the
// status entries of consecutive tiles for this column.  Instead of one L2 round trip per
// predecessor, a window of W predecessors is read per round trip.
template <int W>
__device__ __forceinline__ uint32_t lookback_window(const uint64_t* status, uint64_t stride,
                                                    uint32_t tile, uint32_t epoch) {
    uint32_t excl = 0;
    int64_t p = (int64_t)tile - 1;
    while (p >= 0) {
        uint64_t s[W];
#pragma unroll
        for (int j = 0; j < W; ++j)
            s[j] = (p - j >= 0) ? ld_relaxed_u64(status + (uint64_t)(p - j) * stride) : 0ull;
        int consumed = 0;
        bool done = false;
#pragma unroll
        for (int j = 0; j < W; ++j) {
            if (done || consumed != j) break;
            if (p - j < 0) break;
            const uint32_t st = status_state(s[j], epoch);
            if (st == 0) break;  // not yet published: poll again from here
            excl += (uint32_t)s[j];
            ++consumed;
            if (st == kStateInclusive) done = true;
        }
        if (done) break;
        p -= consumed;
    }
    return excl;
}


}  // namespace ph0b
