// Per-key cost of the onesweep's in-SM building blocks on B200 (sm_100a), 256-thread CTAs,
// per-warp 256-bin digit counters, random digits: what the rank and next-digit histogram
// phases cost with shared-memory atomics vs bit-sliced ballots with register counters.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rb tools/rank_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

// MODE 0: ATOMS.ADD with return (the rank)            1: ATOMS.ADD no return (histogram)
// MODE 2: ballots -> peers, popc(peers&lt) (item rank) 3: ballots -> 8 register counters/lane
// MODE 4: 2 + 3 (rank + counts, no smem)               5: STS.64 random scatter
// MODE 6: STS.32 random scatter                        7: LDS.32 random gather
// MODE 8: STS.64 to 2 x STS.32 planes                  9: ALU baseline
template <int MODE>
__global__ void __launch_bounds__(256, 2) kern(uint32_t* out, int iters) {
    __shared__ uint32_t h[8][256];
    __shared__ uint64_t s64[2048];
    __shared__ uint32_t s32[4096];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    uint32_t x = hash32(blockIdx.x * blockDim.x + threadIdx.x);
    uint32_t acc = 0;
    uint32_t cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    for (int it = 0; it < iters; ++it) {
        x = x * 1664525u + 1013904223u;
        const uint32_t d = (x >> 13) & 255u;
        if (MODE == 0) {
            acc += atomicAdd(&h[warp][d], 1u);
        } else if (MODE == 1) {
            atomicAdd(&h[warp][d], 1u);
        } else if (MODE == 2 || MODE == 3 || MODE == 4) {
            uint32_t bal[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) bal[b] = __ballot_sync(0xffffffffu, (d >> b) & 1u);
            if (MODE != 3) {
                uint32_t p = 0xffffffffu;
#pragma unroll
                for (int b = 0; b < 8; ++b) p &= ((d >> b) & 1u) ? bal[b] : ~bal[b];
                acc += __popc(p & lt);
            }
            if (MODE != 2) {
                // lane owns digits 8*lane .. 8*lane+7: top 5 bits = lane, low 3 bits = j
                uint32_t m = 0xffffffffu;
#pragma unroll
                for (int b = 3; b < 8; ++b) m &= ((lane >> (b - 3)) & 1u) ? bal[b] : ~bal[b];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t l = ((j & 1) ? bal[0] : ~bal[0]) & ((j & 2) ? bal[1] : ~bal[1]) &
                                       ((j & 4) ? bal[2] : ~bal[2]);
                    cnt[j] += __popc(m & l);
                }
            }
        } else if (MODE == 5) {
            s64[(d << 3) | (x & 7u)] = x;
        } else if (MODE == 6) {
            s32[(d << 4) | (x & 15u)] = x;
        } else if (MODE == 7) {
            acc += s32[(d << 4) | (x & 15u)];
        } else if (MODE == 8) {
            const uint32_t q = (d << 4) | (x & 15u);
            s32[q] = x;
            reinterpret_cast<uint32_t*>(s64)[q] = x ^ 1u;
        } else {
            acc += d;
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += cnt[j];
    if (threadIdx.x == 0) out[blockIdx.x] = acc + h[0][0] + (uint32_t)s64[7] + s32[9];
}

template <int MODE>
void run(const char* name, int iters) {
    const int blocks = 148 * 2, threads = 256;
    uint32_t* out;
    cudaMalloc(&out, blocks * 4);
    kern<MODE><<<blocks, threads>>>(out, iters);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<MODE><<<blocks, threads>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double keys_per_sm = (double)blocks * threads * iters / 148;
    const double cyc = ms * 1e-3 * 1.965e9;
    printf("%-36s %8.3f ms  %.3f SM-cycles per key   C5 pass equiv %.2f ms\n", name, ms,
           cyc / keys_per_sm, cyc / keys_per_sm * 2.147e9 / 148 / 1.965e9 * 1e3);
    cudaFree(out);
}

int main() {
    const int it = 8192;
    run<9>("alu baseline", it);
    run<0>("ATOMS.ADD return (rank)", it);
    run<1>("ATOMS.ADD no return (histogram)", it);
    run<2>("ballots: peers + item rank", it);
    run<3>("ballots: 8 register counters/lane", it);
    run<4>("ballots: rank + counters", it);
    run<5>("STS.64 random scatter", it);
    run<6>("STS.32 random scatter", it);
    run<7>("LDS.32 random gather", it);
    run<8>("2 x STS.32 planes", it);
    return 0;
}
