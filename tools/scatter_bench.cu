// How well does the B200 L2 merge scattered appends?  G CTAs each own one contiguous
// sub-region per bucket and append (u64 key, u32 val) records to a random bucket per
// element (positions from shared-memory atomics, no staging).  Reports effective GB/s of
// the 12 B/element written, for several fan-outs F.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

template <bool STAGED>
__global__ void scatter(uint64_t* keys, uint32_t* vals, uint64_t per_cta, uint32_t F,
                        uint64_t region) {
    extern __shared__ uint32_t cur[];  // [F]
    for (uint32_t b = threadIdx.x; b < F; b += blockDim.x) cur[b] = 0;
    __syncthreads();
    const uint64_t base = (uint64_t)blockIdx.x * region;  // this CTA's slice in every bucket
    const uint64_t stride = (uint64_t)gridDim.x * region;  // bucket stride
    uint32_t x = hash32(blockIdx.x * 1315423911u + threadIdx.x);
    for (uint64_t i = threadIdx.x; i < per_cta; i += blockDim.x) {
        x = x * 1664525u + 1013904223u;
        const uint32_t b = (x >> 8) % F;
        const uint32_t pos = atomicAdd(&cur[b], 1u);
        const uint64_t g = (uint64_t)b * stride + base + pos;
        keys[g] = ((uint64_t)x << 32) | i;
        vals[g] = x;
    }
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint64_t total = 1ull << 30;  // elements (12 GiB written)
    for (int ctas_per_sm : {1, 2, 4}) {
        const uint32_t G = sms * ctas_per_sm;
        for (uint32_t F : {256u, 1024u, 4096u, 16384u}) {
            const uint64_t per_cta = total / G;
            const uint64_t region = per_cta / F * 13 / 10 + 256;  // slack per (cta, bucket)
            const uint64_t cap = region * G * F;
            uint64_t* keys;
            uint32_t* vals;
            if (cudaMalloc(&keys, cap * 8) != cudaSuccess || cudaMalloc(&vals, cap * 4) != cudaSuccess) {
                printf("alloc failed F=%u\n", F);
                cudaGetLastError();
                continue;
            }
            cudaFuncSetAttribute(scatter<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
            scatter<false><<<G, 512, F * 4>>>(keys, vals, per_cta, F, region);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            scatter<false><<<G, 512, F * 4>>>(keys, vals, per_cta, F, region);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("ctas/SM %d  F %6u : %8.3f ms  %7.1f GB/s (12 B/elem)  err=%s\n", ctas_per_sm, F, ms,
                   total * 12.0 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
            cudaFree(keys);
            cudaFree(vals);
        }
    }
    return 0;
}
