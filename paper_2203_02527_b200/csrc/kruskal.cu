// GPU Kruskal barcode — an independent second computation of the H0 barcode over the same
// device filtration.  Restates the reference oracle
// kruskal_barcode (/root/reference/proj/src/oracle.cpp:32-46): edges in filtration order,
// union-find, a bar (0, grade, length) for every edge joining two components, early stop at
// n - 1 merges (oracle.cpp:41), essential = n - merges.
//
// Unlike K4 (windowed clearing filter + Borůvka hooking) this is the sequential algorithm
// itself, run by one CTA with the whole union-find forest in shared memory (u16 parents +
// u8 ranks for N <= 65536, 192 KiB): 1024 edges per step are tested in parallel against the
// current forest (read-only finds; an edge whose endpoints already share a root can never
// merge later), and the few survivors of that test are replayed in order by one thread with
// union by rank and path halving (the reference's UnionFind, oracle.cpp:8-30).
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace ph0b {
namespace {

constexpr int kKThreads = 1024;

__device__ __forceinline__ uint32_t find_ro(const uint16_t* parent, uint32_t x) {
    uint32_t p = parent[x];
    while (p != x) {
        x = p;
        p = parent[x];
    }
    return x;
}

__device__ __forceinline__ uint32_t find_halving(uint16_t* parent, uint32_t x) {
    while (parent[x] != x) {
        const uint32_t gp = parent[parent[x]];
        parent[x] = (uint16_t)gp;
        x = gp;
    }
    return x;
}

__global__ void __launch_bounds__(kKThreads, 1)
    k6_kruskal(const uint32_t* __restrict__ uv, uint64_t count, uint32_t n,
               uint32_t* __restrict__ accepted, uint32_t* __restrict__ n_accepted) {
    extern __shared__ __align__(16) uint8_t kr_dyn[];
    uint16_t* parent = reinterpret_cast<uint16_t*>(kr_dyn);              // [65536]
    uint8_t* rank = kr_dyn + 65536 * 2;                                   // [65536]
    uint32_t* cand = reinterpret_cast<uint32_t*>(rank + 65536);           // [kKThreads]
    __shared__ uint32_t s_warp[kKThreads / 32];
    __shared__ uint32_t s_merges;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (uint32_t i = tid; i < n; i += kKThreads) {
        parent[i] = (uint16_t)i;
        rank[i] = 0;
    }
    if (tid == 0) s_merges = 0;
    __syncthreads();
    const uint32_t target = n > 0 ? n - 1 : 0;
    for (uint64_t base = 0; base < count; base += kKThreads) {
        if (s_merges >= target) break;  // uniform: read after a barrier
        // ---- parallel test against the current forest ----------------------------------
        const uint64_t e = base + tid;
        bool c = false;
        if (e < count) {
            const uint32_t w = uv[e];
            c = find_ro(parent, w >> 16) != find_ro(parent, w & 0xFFFFu);
        }
        const uint32_t ball = __ballot_sync(0xffffffffu, c);
        if (lane == 0) s_warp[warp] = __popc(ball);
        __syncthreads();
        uint32_t before = 0, total = 0;
#pragma unroll
        for (int w = 0; w < kKThreads / 32; ++w) {
            const uint32_t x = s_warp[w];
            before += (w < warp) ? x : 0u;
            total += x;
        }
        if (c) cand[before + __popc(ball & lanemask_lt())] = (uint32_t)tid;
        __syncthreads();
        // ---- in-order replay of the candidates (one thread, the reference's union-find) -
        if (tid == 0) {
            uint32_t merges = s_merges;
            for (uint32_t j = 0; j < total && merges < target; ++j) {
                const uint64_t ej = base + cand[j];
                const uint32_t w = uv[ej];
                uint32_t a = find_halving(parent, w >> 16);
                uint32_t b = find_halving(parent, w & 0xFFFFu);
                if (a == b) continue;
                if (rank[a] < rank[b]) {
                    const uint32_t t = a;
                    a = b;
                    b = t;
                }
                parent[b] = (uint16_t)a;
                if (rank[a] == rank[b]) ++rank[a];
                accepted[merges++] = (uint32_t)ej;
            }
            s_merges = merges;
        }
        __syncthreads();
    }
    if (tid == 0) *n_accepted = s_merges;
}

// Bars of the accepted edges: length from the sorted key, grade = 1 + #distinct lengths
// below it (binary search in D; D[grade-1] == length, test_filtration.cpp:109).
__global__ void k6_bars(const uint32_t* __restrict__ accepted, const uint32_t* __restrict__ n_acc,
                        const uint64_t* __restrict__ sorted_keys, const double* __restrict__ D,
                        const uint64_t* __restrict__ n_scale, uint64_t* __restrict__ death_grade,
                        double* __restrict__ death_length) {
    const uint32_t m = *n_acc;
    const uint64_t nd = *n_scale;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        const double len = __longlong_as_double((long long)sorted_keys[accepted[i]]);
        uint64_t lo = 0, hi = nd;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (D[mid] < len)
                lo = mid + 1;
            else
                hi = mid;
        }
        death_grade[i] = lo + 1;
        death_length[i] = len;
    }
}

}  // namespace

size_t kruskal_smem_bytes() { return 65536 * 2 + 65536 + kKThreads * 4; }

int launch_kruskal(const uint32_t* uv, const uint64_t* sorted_keys, uint64_t count, uint32_t n,
                   const double* D, const uint64_t* n_scale, uint32_t* accepted,
                   uint32_t* n_accepted, uint64_t* death_grade, double* death_length,
                   cudaStream_t s) {
    if (kernel_blocks_per_sm((const void*)k6_kruskal, kKThreads, kruskal_smem_bytes()) < 1)
        return -1;
    k6_kruskal<<<1, kKThreads, kruskal_smem_bytes(), s>>>(uv, count, n, accepted, n_accepted);
    k6_bars<<<(n + 255) / 256 + 1, 256, 0, s>>>(accepted, n_accepted, sorted_keys, D, n_scale,
                                                death_grade, death_length);
    return 2;
}

}  // namespace ph0b
