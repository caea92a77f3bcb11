// FP64 pipe peak on this B200 (the denominator of K1's FP64 roofline): independent chains of
// DADD, DMUL and DFMA, 8 per thread, every SM full of warps.  Reports FP64 instructions per
// second (one DADD / DMUL / DFMA = one instruction; a DFMA is 2 flops).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void __launch_bounds__(256) kern(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-9 + j;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (OP == 0) x[j] = __dadd_rn(x[j], a);
            else if (OP == 1) x[j] = __dmul_rn(x[j], b);
            else x[j] = __fma_rn(x[j], b, a);
        }
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == 123.456) out[0] = s;
}

template <int OP>
void run(const char* name) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256, iters = 20000;
    double* out;
    cudaMalloc(&out, 8);
    kern<OP><<<blocks, threads>>>(out, 100, 1e-7, 0.9999999);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<OP><<<blocks, threads>>>(out, iters, 1e-7, 0.9999999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double inst = (double)blocks * threads * iters * 8;
    printf("%-6s %8.3f ms  %.2f T FP64 instr/s  (%.1f per SM per clock at 1.965 GHz)  err=%s\n",
           name, ms, inst / ms * 1e-9, inst / (ms * 1e-3) / sms / 1.965e9,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main() {
    run<0>("DADD");
    run<1>("DMUL");
    run<2>("DFMA");
    return 0;
}
