// Does ATOMS resolve same-address lanes of one warp instruction in ascending lane order?
#include <cstdio>
#include <cstdint>
__global__ void k(unsigned long long* viol, unsigned long long* checks, int iters, int mask) {
    __shared__ uint32_t h[8][256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    uint32_t x = (blockIdx.x * 7919u + threadIdx.x * 104729u) ^ 0x9e3779b9u;
    unsigned long long v = 0, c = 0;
    for (int it = 0; it < iters; ++it) {
        x = x * 1664525u + 1013904223u;
        const uint32_t d = (x >> 11) & mask;
        const uint32_t old = atomicAdd(&h[warp][d], 1u);
        // compare with every other lane having the same digit
        for (int o = 0; o < 32; ++o) {
            const uint32_t od = __shfl_sync(0xffffffffu, d, o);
            const uint32_t oo = __shfl_sync(0xffffffffu, old, o);
            if (od == d && o < lane) { ++c; if (!(oo < old)) ++v; }
        }
    }
    atomicAdd(viol, v);
    atomicAdd(checks, c);
}
int main() {
    unsigned long long *v, *c;
    cudaMallocManaged(&v, 8); cudaMallocManaged(&c, 8);
    for (int mask : {1, 7, 255}) {
        *v = 0; *c = 0;
        k<<<148 * 4, 256>>>(v, c, 2000, mask);
        cudaDeviceSynchronize();
        printf("mask %3d: same-digit lane pairs checked %llu, order violations %llu\n", mask, *c, *v);
    }
}
