// On-device generate_uniform_cloud: restates
// /root/reference/proj/src/point_cloud.cpp:20-29 with the SplitMix64 stream of
// /root/reference/proj/include/ph0/splitmix64.hpp:20-43.  SplitMix64 is jumpable — draw k
// is mix64(seed + (k+1)·γ) — so every coordinate is computed independently; coordinates are
// consumed row by row (pts(i, j) for i, then j) and written column-major (Eigen storage).
// next_unit_open rejects draws whose top 53 bits are zero, which shifts every later
// coordinate by one draw: the kernel records such draws (probability 2^-53 each) and a
// second kernel re-maps the coordinates past them, so the output is exact in every case.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "kernels.h"

namespace ph0b {
namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr uint32_t kMaxZeros = 64;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t top53(uint64_t seed, uint64_t draw, uint64_t forced_zero) {
    return draw == forced_zero ? 0ull : mix64(seed + (draw + 1) * kGamma) >> 11;
}

// Pass 1: coordinate t from draw t (no rejection yet); zero draws in [0, total + kMaxZeros)
// are appended to zeros[] (count in zeros[kMaxZeros]).
__global__ void k8_uniform(uint64_t n, uint64_t dim, uint64_t seed, uint64_t forced_zero,
                           double* __restrict__ out, unsigned long long* __restrict__ zeros) {
    const uint64_t total = n * dim;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total + kMaxZeros;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t top = top53(seed, t, forced_zero);
        if (top == 0) {
            const unsigned long long slot = atomicAdd(&zeros[kMaxZeros], 1ull);
            if (slot < kMaxZeros) zeros[slot] = t;
        }
        if (t < total) {
            const uint64_t i = t / dim, j = t - i * dim;
            out[j * n + i] = (double)top * 0x1.0p-53;
        }
    }
}

// Pass 2 (only when a zero draw was seen): coordinate t takes the first non-zero draw
// t + c, c = number of zero draws at or before it (zeros sorted by the host launcher).
__global__ void k8_uniform_fix(uint64_t n, uint64_t dim, uint64_t seed, uint64_t forced_zero,
                               double* __restrict__ out, const unsigned long long* __restrict__ zeros,
                               uint32_t nz) {
    const uint64_t total = n * dim;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total;
         t += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t c = 0;
        while (c < nz && zeros[c] <= t + c) ++c;
        if (c == 0) continue;
        const uint64_t i = t / dim, j = t - i * dim;
        out[j * n + i] = (double)top53(seed, t + c, forced_zero) * 0x1.0p-53;
    }
}

}  // namespace

int launch_uniform_cloud(uint64_t n, uint64_t dim, uint64_t seed, double* d_out,
                         unsigned long long* d_zeros, unsigned long long* h_zeros,
                         cudaStream_t s, int num_sms) {
    static const uint64_t forced = [] {  // test hook: treat this draw index as a zero draw
        const char* e = getenv("PH0B_GEN_FORCE_ZERO");
        return e ? (uint64_t)strtoull(e, nullptr, 10) : ~0ull;
    }();
    const uint64_t total = n * dim;
    cudaMemsetAsync(d_zeros, 0, (kMaxZeros + 1) * sizeof(unsigned long long), s);
    uint64_t blocks = (total + kMaxZeros + 255) / 256;
    const uint64_t cap = (uint64_t)num_sms * 16;
    if (blocks > cap) blocks = cap;
    k8_uniform<<<(unsigned)blocks, 256, 0, s>>>(n, dim, seed, forced, d_out, d_zeros);
    cudaMemcpyAsync(h_zeros, d_zeros, (kMaxZeros + 1) * sizeof(unsigned long long),
                    cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return -1;
    const uint64_t nz = h_zeros[kMaxZeros];
    if (nz == 0) return 1;
    if (nz > kMaxZeros) return -2;
    for (uint64_t a = 1; a < nz; ++a)  // insertion sort of <= 64 indices
        for (uint64_t b = a; b > 0 && h_zeros[b - 1] > h_zeros[b]; --b) {
            const unsigned long long x = h_zeros[b];
            h_zeros[b] = h_zeros[b - 1];
            h_zeros[b - 1] = x;
        }
    cudaMemcpyAsync(d_zeros, h_zeros, nz * sizeof(unsigned long long), cudaMemcpyHostToDevice, s);
    k8_uniform_fix<<<(unsigned)blocks, 256, 0, s>>>(n, dim, seed, forced, d_out, d_zeros,
                                                    (uint32_t)nz);
    if (cudaStreamSynchronize(s) != cudaSuccess) return -1;
    return 2;
}

}  // namespace ph0b
