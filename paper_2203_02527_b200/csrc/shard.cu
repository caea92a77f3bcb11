// Multi-GPU splitter partition: each rank computes the edges of its own
// row range (u-major), then stably partitions them into P contiguous segments by global
// splitters on the length key; segment j goes to rank j in the all-to-all exchange.
// Because rank r owns rows [U_r, U_{r+1}) with U increasing, and every segment keeps the
// u-major order, the data a rank receives (sources concatenated in rank order) is again in
// u-major order, so the local stable radix sort yields exactly the global (length, u, v)
// order restricted to that rank's key range — no merge step is needed.
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace ph0b {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;
constexpr int kMaxParts = 256;

__device__ __forceinline__ uint32_t bucket_of(uint64_t key, const uint64_t* spl, uint32_t nspl) {
    // number of splitters <= key (upper_bound): keys equal to a splitter go right, so equal
    // lengths always land in the same bucket
    uint32_t lo = 0, hi = nspl;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (spl[mid] <= key)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(kThreads)
    k7_count(const uint64_t* __restrict__ keys, uint64_t count, const uint64_t* __restrict__ splitters,
             uint32_t parts, uint32_t* __restrict__ counts, unsigned long long* bmin,
             unsigned long long* bmax) {
    __shared__ uint64_t s_spl[kMaxParts];
    __shared__ uint32_t s_cnt[kMaxParts];
    __shared__ unsigned long long s_min[kMaxParts], s_max[kMaxParts];
    for (uint32_t i = threadIdx.x; i < kMaxParts; i += kThreads) {
        s_spl[i] = i + 1 < parts ? splitters[i] : ~0ull;
        s_cnt[i] = 0;
        s_min[i] = ~0ull;
        s_max[i] = 0;
    }
    __syncthreads();
    const uint64_t base = (uint64_t)blockIdx.x * kTile;
    for (int i = 0; i < kItems; ++i) {
        const uint64_t idx = base + (uint64_t)i * kThreads + threadIdx.x;
        if (idx < count) {
            const uint64_t k = keys[idx];
            const uint32_t b = bucket_of(k, s_spl, parts - 1);
            atomicAdd(&s_cnt[b], 1u);
            atomicMin(&s_min[b], (unsigned long long)k);
            atomicMax(&s_max[b], (unsigned long long)k);
        }
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < parts; b += kThreads) {
        counts[(uint64_t)blockIdx.x * parts + b] = s_cnt[b];
        if (s_cnt[b]) {
            atomicMin(&bmin[b], s_min[b]);
            atomicMax(&bmax[b], s_max[b]);
        }
    }
}

// Evenly spaced sample of keys[0..count) (splitter selection).
__global__ void k7_sample(const uint64_t* __restrict__ keys, uint64_t count, uint64_t s,
                          uint64_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < s;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = keys[(i * count) / s + (count / s) / 2];
}

__global__ void k7_gather_u32(const uint32_t* __restrict__ src, const uint32_t* __restrict__ idx,
                              uint64_t m, uint32_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = src[idx[i]];
}

// One block per bucket: exclusive scan of that bucket's per-tile counts, and its total.
__global__ void k7_scan(uint32_t* __restrict__ counts, uint32_t tiles, uint32_t parts,
                        uint64_t* __restrict__ totals) {
    __shared__ uint64_t s_carry;
    __shared__ uint32_t s_warp[32];
    const uint32_t b = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (uint32_t t0 = 0; t0 < tiles; t0 += blockDim.x) {
        const uint32_t t = t0 + threadIdx.x;
        const uint32_t x = t < tiles ? counts[(uint64_t)t * parts + b] : 0u;
        uint32_t inc = x;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) s_warp[warp] = inc;
        __syncthreads();
        uint32_t wb = 0, tot = 0;
        for (int w = 0; w < nw; ++w) {
            wb += w < warp ? s_warp[w] : 0u;
            tot += s_warp[w];
        }
        const uint64_t carry = s_carry;
        if (t < tiles) counts[(uint64_t)t * parts + b] = (uint32_t)(carry + wb + inc - x);
        __syncthreads();
        if (threadIdx.x == 0) s_carry = carry + tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) totals[b] = s_carry;
}

// Stable scatter of one 4096-element tile into its segments: ranks from per-warp shared
// histograms (ATOMS lane order = stable), the tile staged in shared memory in segment order,
// then written out so consecutive threads write consecutive positions of each segment run.
__global__ void __launch_bounds__(kThreads)
    k7_scatter(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals, uint64_t count,
               const uint64_t* __restrict__ splitters, uint32_t parts,
               const uint32_t* __restrict__ offsets, const uint64_t* __restrict__ totals,
               uint64_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
               uint32_t align) {
    __shared__ uint64_t s_spl[kMaxParts];
    __shared__ uint32_t s_whist[kWarps][kMaxParts];
    __shared__ uint32_t s_tstart[kMaxParts];
    __shared__ uint64_t s_base[kMaxParts];  // global position of this tile's first element of b
    extern __shared__ __align__(16) uint64_t sc_dyn[];
    uint64_t* s_k = sc_dyn;                                                 // [kTile]
    uint32_t* s_v = reinterpret_cast<uint32_t*>(sc_dyn + kTile);            // [kTile]
    uint16_t* s_b = reinterpret_cast<uint16_t*>(s_v + kTile);               // [kTile]
    for (uint32_t i = threadIdx.x; i < kMaxParts; i += kThreads) {
        s_spl[i] = i + 1 < parts ? splitters[i] : ~0ull;
        for (int w = 0; w < kWarps; ++w) s_whist[w][i] = 0;
    }
    if (threadIdx.x == 0) {
        // segment b starts at the sum of the earlier totals, each rounded up to `align`
        // elements; block 0 fills the padding slots with the sentinel column {0, 0} (a cycle)
        uint64_t acc = 0;
        for (uint32_t b = 0; b < parts; ++b) {
            s_base[b] = acc + offsets[(uint64_t)blockIdx.x * parts + b];
            const uint64_t padded = (totals[b] + align - 1) / align * align;
            if (blockIdx.x == 0)
                for (uint64_t q = acc + totals[b]; q < acc + padded; ++q) {
                    keys_out[q] = 0;
                    vals_out[q] = 0;
                }
            acc += padded;
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t tile0 = (uint64_t)blockIdx.x * kTile;
    const uint32_t tn = (uint32_t)(count - tile0 < (uint64_t)kTile ? count - tile0 : kTile);
    const uint32_t wofs = warp * (32 * kItems) + lane;
    uint64_t kk[kItems];
    uint32_t vv[kItems], bk[kItems], rk[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {  // all loads in flight first
        const uint32_t pos = wofs + 32 * i;
        kk[i] = pos < tn ? keys[tile0 + pos] : 0ull;
        vv[i] = pos < tn ? vals[tile0 + pos] : 0u;
    }
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const uint32_t pos = wofs + 32 * i;
        bk[i] = pos < tn ? bucket_of(kk[i], s_spl, parts - 1) : 0u;
        // ATOMS resolves same-address lanes in lane order (device self-test), so the
        // returned count is the stable rank within this warp
        rk[i] = pos < tn ? atomicAdd(&s_whist[warp][bk[i]], 1u) : 0u;
    }
    __syncthreads();
    if (threadIdx.x < kMaxParts) {
        const uint32_t b = threadIdx.x;
        uint32_t acc = 0;
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t c = s_whist[w][b];
            s_whist[w][b] = acc;
            acc += c;
        }
        s_tstart[b] = acc;  // tile count of b (scanned below)
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t acc = 0;
        for (uint32_t b = 0; b < parts; ++b) {
            const uint32_t c = s_tstart[b];
            s_tstart[b] = acc;
            acc += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const uint32_t pos = wofs + 32 * i;
        if (pos < tn) {
            const uint32_t dst = s_tstart[bk[i]] + s_whist[warp][bk[i]] + rk[i];
            s_k[dst] = kk[i];
            s_v[dst] = vv[i];
            s_b[dst] = (uint16_t)bk[i];
        }
    }
    __syncthreads();
    for (uint32_t p = threadIdx.x; p < tn; p += kThreads) {
        const uint32_t b = s_b[p];
        const uint64_t dst = s_base[b] + (p - s_tstart[b]);
        keys_out[dst] = s_k[p];
        vals_out[dst] = s_v[p];
    }
}

}  // namespace

int launch_partition(const uint64_t* keys, const uint32_t* vals, uint64_t count,
                     const uint64_t* d_splitters, uint32_t parts, uint32_t* d_counts_scratch,
                     uint64_t* d_totals, uint64_t* d_bminmax, uint64_t* keys_out,
                     uint32_t* vals_out, cudaStream_t s, uint32_t align) {
    if (parts < 1 || parts > (uint32_t)kMaxParts) return -1;
    const uint64_t tiles = (count + kTile - 1) / kTile;
    cudaMemsetAsync(d_bminmax, 0xFF, sizeof(uint64_t) * parts, s);
    cudaMemsetAsync(d_bminmax + parts, 0, sizeof(uint64_t) * parts, s);
    if (tiles == 0) {
        cudaMemsetAsync(d_totals, 0, sizeof(uint64_t) * parts, s);
        return 1;
    }
    k7_count<<<(unsigned)tiles, kThreads, 0, s>>>(
        keys, count, d_splitters, parts, d_counts_scratch,
        reinterpret_cast<unsigned long long*>(d_bminmax),
        reinterpret_cast<unsigned long long*>(d_bminmax + parts));
    k7_scan<<<parts, 1024, 0, s>>>(d_counts_scratch, (uint32_t)tiles, parts, d_totals);
    constexpr size_t kScSmem = (size_t)kTile * (8 + 4 + 2);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k7_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kScSmem);
        configured = true;
    }
    k7_scatter<<<(unsigned)tiles, kThreads, kScSmem, s>>>(keys, vals, count, d_splitters, parts,
                                                    d_counts_scratch, d_totals, keys_out,
                                                    vals_out, align);
    return 3;
}

int launch_sample(const uint64_t* keys, uint64_t count, uint64_t s, uint64_t* out, cudaStream_t st) {
    if (s == 0 || count == 0) return 0;
    k7_sample<<<(unsigned)((s + 255) / 256), 256, 0, st>>>(keys, count, s, out);
    return 1;
}

int launch_gather_u32(const uint32_t* src, const uint32_t* idx, uint64_t m, uint32_t* out,
                      cudaStream_t st) {
    if (m == 0) return 0;
    k7_gather_u32<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(src, idx, m, out);
    return 1;
}

uint64_t partition_scratch_words(uint64_t count, uint32_t parts) {
    return ((count + kTile - 1) / kTile) * parts;
}

}  // namespace ph0b
