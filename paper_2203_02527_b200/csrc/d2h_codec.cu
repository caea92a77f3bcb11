// D over PCIe in half the bytes (overlapped host path).  D is strictly increasing, so the
// 64-bit patterns of consecutive lengths differ by small amounts: each 4096-value chunk is
// sent as its first pattern (u64) plus 32-bit deltas, and decoded on the host by a prefix
// sum (host_decode.cpp).  A chunk with any delta >= 2^32 is flagged raw and copied as is.
// Lossless: the host reconstructs the exact bit patterns of D (Filtration::scale).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace ph0b {
namespace {

constexpr int kEncThreads = 256;
constexpr int kEncPer = kD2HChunk / kEncThreads;  // 16 values per thread

__global__ void __launch_bounds__(kEncThreads)
    k9_encode(const uint64_t* __restrict__ d, uint64_t n, uint32_t* __restrict__ deltas,
              uint64_t* __restrict__ bases, uint8_t* __restrict__ raw) {
    const uint64_t c0 = (uint64_t)blockIdx.x * kD2HChunk;
    const uint32_t len = (uint32_t)(n - c0 < (uint64_t)kD2HChunk ? n - c0 : kD2HChunk);
    bool big = false;
#pragma unroll
    for (int j = 0; j < kEncPer; ++j) {
        const uint32_t i = (uint32_t)j * kEncThreads + threadIdx.x;
        if (i < len) {
            const uint64_t cur = d[c0 + i];
            const uint64_t prev = i > 0 ? d[c0 + i - 1] : cur;
            const uint64_t delta = cur - prev;
            big |= (delta >> 32) != 0;
            deltas[c0 + i] = (uint32_t)delta;
        }
    }
    const int any_big = __syncthreads_or(big ? 1 : 0);
    if (threadIdx.x == 0) {
        bases[blockIdx.x] = d[c0];
        raw[blockIdx.x] = any_big ? 1 : 0;
    }
}

// Bucket variant for the streamed host path: the slice is [lohi[0], lohi[1]) of d (device
// words written by the bucket's unique kernel), so the host can enqueue it before the
// bucket's |D| is known; the grid covers an upper bound and blocks past the end exit.
__global__ void __launch_bounds__(kEncThreads)
    k9_encode_bucket(const uint64_t* __restrict__ d, const uint64_t* __restrict__ lohi,
                     uint32_t* __restrict__ deltas, uint64_t* __restrict__ bases,
                     uint8_t* __restrict__ raw) {
    const uint64_t lo = lohi[0], n = lohi[1] - lo;
    const uint64_t c0 = (uint64_t)blockIdx.x * kD2HChunk;
    if (c0 >= n) return;
    const uint64_t* dd = d + lo;
    const uint32_t len = (uint32_t)(n - c0 < (uint64_t)kD2HChunk ? n - c0 : kD2HChunk);
    bool big = false;
#pragma unroll
    for (int j = 0; j < kEncPer; ++j) {
        const uint32_t i = (uint32_t)j * kEncThreads + threadIdx.x;
        if (i < len) {
            const uint64_t cur = dd[c0 + i];
            const uint64_t prev = i > 0 ? dd[c0 + i - 1] : cur;
            const uint64_t delta = cur - prev;
            big |= (delta >> 32) != 0;
            deltas[c0 + i] = (uint32_t)delta;
        }
    }
    const int any_big = __syncthreads_or(big ? 1 : 0);
    if (threadIdx.x == 0) {
        bases[blockIdx.x] = dd[c0];
        raw[blockIdx.x] = any_big ? 1 : 0;
    }
}

}  // namespace

int launch_d2h_encode_bucket(const double* d, const uint64_t* lohi, uint64_t n_upper,
                             uint32_t* deltas, uint64_t* bases, uint8_t* raw, cudaStream_t s) {
    if (n_upper == 0) return 0;
    const uint64_t chunks = (n_upper + kD2HChunk - 1) / kD2HChunk;
    k9_encode_bucket<<<(unsigned)chunks, kEncThreads, 0, s>>>(
        reinterpret_cast<const uint64_t*>(d), lohi, deltas, bases, raw);
    return 1;
}

int launch_d2h_encode(const double* d, uint64_t n, uint32_t* deltas, uint64_t* bases,
                      uint8_t* raw, cudaStream_t s) {
    if (n == 0) return 0;
    const uint64_t chunks = (n + kD2HChunk - 1) / kD2HChunk;
    k9_encode<<<(unsigned)chunks, kEncThreads, 0, s>>>(reinterpret_cast<const uint64_t*>(d), n,
                                                       deltas, bases, raw);
    return 1;
}

}  // namespace ph0b
