// Microbenchmarks of the primitives the radix sort is built from (B200, sm_100a).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

template <int MODE>
__global__ void kern(uint32_t* out, int iters) {
    __shared__ uint32_t h[8][256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    uint32_t x = hash32(blockIdx.x * blockDim.x + threadIdx.x);
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        x = x * 1664525u + 1013904223u;
        const uint32_t d = (x >> 13) & 255u;
        if (MODE == 0) {          // ATOMS.ADD, random bins, per-warp histogram
            atomicAdd(&h[warp][d], 1u);
        } else if (MODE == 1) {   // ATOMS.ADD with return
            acc += atomicAdd(&h[warp][d], 1u);
        } else if (MODE == 2) {   // match.any
            acc += __match_any_sync(0xffffffffu, d);
        } else if (MODE == 3) {   // 8 ballots (bit-sliced peers)
            uint32_t p = 0xffffffffu;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const uint32_t bit = (d >> b) & 1u;
                const uint32_t bal = __ballot_sync(0xffffffffu, bit);
                p &= bit ? bal : ~bal;
            }
            acc += p;
        } else if (MODE == 4) {   // LDS + STS random (non-atomic RMW)
            h[warp][d] += 1u;
        } else if (MODE == 5) {   // ATOMS, all lanes same address
            atomicAdd(&h[warp][lane == 0 ? d : d], 1u);
        } else if (MODE == 6) {   // baseline: ALU only
            acc += d;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = acc + h[0][0];
}

template <int MODE>
float run(const char* name, int blocks, int threads, int iters) {
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
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double lane_ops = (double)blocks * threads * iters;
    const double cyc = ms * 1e-3 * clk * 1e3;  // at max clock
    printf("%-28s %8.3f ms  %.3f SM-cycles per lane-op  (%.1f warp-instr/cycle/SM)\n", name, ms,
           cyc * sms / lane_ops, lane_ops / 32 / (cyc * sms));
    cudaFree(out);
    return ms;
}

int main() {
    const int blocks = 148 * 8, threads = 256, iters = 4096;
    run<6>("alu baseline", blocks, threads, iters);
    run<0>("atoms add (no return)", blocks, threads, iters);
    run<1>("atoms add (return)", blocks, threads, iters);
    run<5>("atoms same-address", blocks, threads, iters);
    run<2>("match.any", blocks, threads, iters);
    run<3>("8x ballot peers", blocks, threads, iters);
    run<4>("lds+sts rmw", blocks, threads, iters);
    return 0;
}
