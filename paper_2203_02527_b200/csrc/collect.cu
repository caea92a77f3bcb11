// K5 — barcode collect (replaces extract_barcode, /root/reference/proj/src/reduction.cpp:140-150).
//
// The reduction leaves the surviving column ids unordered; they are put in filtration order
// with the same onesweep radix sort (keys only), then each survivor j becomes the interval
// (0, grade_j, scale[grade_j - 1]) with grade_j = 1 + lower_bound(D, length_j) — D is strictly
// increasing and contains length_j, so this is exactly the grade build_filtration assigned
// (filtration.cpp:29-33).  essential_count = N - #finite (reduction.cpp:148) is done on host.
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace ph0b {
namespace {

__global__ void k5_widen(const uint32_t* __restrict__ in, uint32_t m, uint64_t* __restrict__ out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
        out[i] = in[i];
}

__global__ void k5_narrow(const uint64_t* __restrict__ in, uint32_t m, uint32_t* __restrict__ out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
        out[i] = (uint32_t)in[i];
}

__global__ void k5_map(const uint64_t* __restrict__ cols_sorted, uint32_t m,
                       const uint64_t* __restrict__ sorted_keys, const double* __restrict__ scale,
                       const uint64_t* __restrict__ n_scale, uint64_t grade_offset,
                       uint32_t* __restrict__ surv_sorted,
                       uint64_t* __restrict__ death_grade, double* __restrict__ death_length) {
    const uint64_t* dbits = reinterpret_cast<const uint64_t*>(scale);
    const uint64_t ns = *n_scale;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        const uint64_t j = cols_sorted[i];
        const uint64_t key = sorted_keys[j];
        uint64_t lo = 0, hi = ns;  // first index with D[idx] >= key
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (dbits[mid] < key)
                lo = mid + 1;
            else
                hi = mid;
        }
        death_grade[i] = grade_offset + lo + 1;
        death_length[i] = __longlong_as_double((long long)key);
        surv_sorted[i] = (uint32_t)j;
    }
}

// Claimed low of each surviving column, in filtration order (reduction.cpp:44-45): the larger
// of the two pivot-tree roots (= minimum vertex of each tree) it joins.  One thread walks the
// N-1 survivors with a union-find whose root is always the tree minimum; parity surface only.
__global__ void k5_claimed_lows(const uint32_t* __restrict__ surv_sorted, uint32_t m,
                                const uint32_t* __restrict__ uv, uint32_t n, uint32_t* lows) {
    extern __shared__ uint16_t parent[];
    for (uint32_t v = threadIdx.x; v < n; v += blockDim.x) parent[v] = (uint16_t)v;
    __syncthreads();
    if (threadIdx.x != 0) return;
    auto find = [&](uint32_t x) {
        while (parent[x] != x) {
            parent[x] = parent[parent[x]];
            x = parent[x];
        }
        return x;
    };
    for (uint32_t i = 0; i < m; ++i) {
        const uint32_t e = uv[surv_sorted[i]];
        const uint32_t ru = find(e >> 16), rv = find(e & 0xFFFFu);
        const uint32_t hi = ru > rv ? ru : rv, lo = ru > rv ? rv : ru;
        lows[i] = hi;
        parent[hi] = (uint16_t)lo;
    }
}

}  // namespace

// a.surv: unordered survivors; a.surv_scratch reinterpreted as 2 x m u64 ping-pong is not
// enough room, so the caller passes u64 scratch through SortArgs (see pipeline).
int launch_collect_map(const uint64_t* cols_sorted, uint32_t m, const uint64_t* sorted_keys,
                       const double* scale, const uint64_t* n_scale, uint64_t grade_offset,
                       uint32_t* surv_sorted, uint64_t* death_grade, double* death_length,
                       cudaStream_t s) {
    if (m == 0) return 0;
    const unsigned grid = (m + 255) / 256;
    k5_map<<<grid, 256, 0, s>>>(cols_sorted, m, sorted_keys, scale, n_scale, grade_offset,
                                surv_sorted, death_grade, death_length);
    return 1;
}

int launch_narrow(const uint64_t* in, uint32_t m, uint32_t* out, cudaStream_t s) {
    if (m == 0) return 0;
    k5_narrow<<<(m + 255) / 256, 256, 0, s>>>(in, m, out);
    return 1;
}

int launch_widen(const uint32_t* in, uint32_t m, uint64_t* out, cudaStream_t s) {
    if (m == 0) return 0;
    k5_widen<<<(m + 255) / 256, 256, 0, s>>>(in, m, out);
    return 1;
}

int launch_claimed_lows(const uint32_t* surv_sorted, uint32_t m, const uint32_t* uv, uint32_t n,
                        uint32_t* lows, cudaStream_t s) {
    if (m == 0) return 0;
    const size_t smem = sizeof(uint16_t) * ((n + 1) & ~1u);
    cudaFuncSetAttribute(k5_claimed_lows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k5_claimed_lows<<<1, 1024, smem, s>>>(surv_sorted, m, uv, n, lows);
    return 1;
}

}  // namespace ph0b
