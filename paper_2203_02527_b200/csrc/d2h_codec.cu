// D over PCIe in ~40 % of its bytes (overlapped host path).  D is strictly increasing, so the
// 64-bit patterns of consecutive lengths differ by small amounts: each 1024-value chunk is
// sent as its first pattern (u64) plus 3- or 4-byte deltas (the narrowest width holding all
// of its deltas), and decoded on the host by a prefix sum (host_decode.cpp).  A chunk with
// any delta >= 2^32 is flagged raw and copied as is.  Lossless: the host reconstructs the
// exact bit patterns of D (Filtration::scale).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace ph0b {
namespace {

// ---- packed variant (the streamed host path): 1024-value chunks, each shipped as 3- or
// 4-byte deltas (width = bytes of its largest delta; 0 = raw, some delta >= 2^32), chunks
// concatenated; a scan gives every chunk's byte offset, and the offsets of piece boundaries
// (every kPackPiece chunks) go to mapped host memory so the host can size the copies.
constexpr int kPT = 256;                      // threads per chunk block, 4 values each
static_assert(kPackChunk == 4 * kPT, "4 values per thread");

__device__ __forceinline__ uint32_t chunk_len(uint64_t n, uint64_t c) {
    const uint64_t c0 = c * kPackChunk;
    return (uint32_t)(n - c0 < (uint64_t)kPackChunk ? n - c0 : kPackChunk);
}

__global__ void __launch_bounds__(kPT)
    k9p_widths(const uint64_t* __restrict__ d, const uint64_t* __restrict__ lohi,
               uint64_t* __restrict__ bases, uint8_t* __restrict__ widths) {
    const uint64_t lo = lohi[0], n = lohi[1] - lo;
    const uint64_t c0 = (uint64_t)blockIdx.x * kPackChunk;
    if (c0 >= n) return;
    const uint64_t* dd = d + lo + c0;
    const uint32_t len = chunk_len(n, blockIdx.x);
    uint64_t mx = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t i = 4 * threadIdx.x + j;
        if (i > 0 && i < len) {
            const uint64_t delta = dd[i] - dd[i - 1];
            mx = delta > mx ? delta : mx;
        }
    }
    const uint32_t big = __syncthreads_or((mx >> 32) != 0);
    const uint32_t wide = __syncthreads_or((mx >> 24) != 0);
    if (threadIdx.x == 0) {
        bases[blockIdx.x] = dd[0];
        widths[blockIdx.x] = big ? 0 : (wide ? 4 : 3);
    }
}

// One block: exclusive scan of the chunk sizes -> absolute byte offsets (device), offsets
// within each piece (u32, host metadata) and the piece boundaries (mapped host words).
__global__ void __launch_bounds__(1024)
    k9p_scan(const uint8_t* __restrict__ widths, const uint64_t* __restrict__ lohi,
             uint64_t* __restrict__ offs, uint32_t* __restrict__ poff,
             uint64_t* __restrict__ piece_off, uint32_t piece_chunks) {
    __shared__ uint64_t s_w[32];
    __shared__ uint64_t s_carry;
    const uint64_t n = lohi[1] - lohi[0];
    const uint64_t nch = (n + kPackChunk - 1) / kPackChunk;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    uint64_t piece_base = 0;
    for (uint64_t c0 = 0; c0 < nch; c0 += 1024) {
        const uint64_t c = c0 + threadIdx.x;
        const uint64_t sz = c < nch ? (uint64_t)widths[c] * chunk_len(n, c) : 0;
        uint64_t inc = sz;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) s_w[warp] = inc;
        __syncthreads();
        uint64_t wb = 0, tot = 0;
        for (int w = 0; w < 32; ++w) {
            wb += w < warp ? s_w[w] : 0;
            tot += s_w[w];
        }
        const uint64_t off = s_carry + wb + inc - sz;
        if (c < nch) {
            offs[c] = off;
            if (c % piece_chunks == 0) piece_off[c / piece_chunks] = off;
        }
        __syncthreads();
        if (threadIdx.x == 0) s_carry += tot;
        __syncthreads();
        (void)piece_base;
    }
    __syncthreads();
    if (threadIdx.x == 0) piece_off[(nch + piece_chunks - 1) / piece_chunks] = s_carry;
    // offsets within the piece (needs the piece starts written above)
    __syncthreads();
    for (uint64_t c = threadIdx.x; c < nch; c += 1024)
        poff[c] = (uint32_t)(offs[c] - offs[c - c % piece_chunks]);
}

__global__ void __launch_bounds__(kPT)
    k9p_pack(const uint64_t* __restrict__ d, const uint64_t* __restrict__ lohi,
             const uint8_t* __restrict__ widths, const uint64_t* __restrict__ offs,
             uint8_t* __restrict__ out) {
    const uint64_t lo = lohi[0], n = lohi[1] - lo;
    const uint64_t c0 = (uint64_t)blockIdx.x * kPackChunk;
    if (c0 >= n) return;
    const uint32_t w = widths[blockIdx.x];
    if (w == 0) return;  // raw chunk: shipped uncompressed
    const uint64_t* dd = d + lo + c0;
    const uint32_t len = chunk_len(n, blockIdx.x);
    uint32_t x[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t i = 4 * threadIdx.x + j;
        x[j] = (i > 0 && i < len) ? (uint32_t)(dd[i] - dd[i - 1]) : 0u;
    }
    if (4 * threadIdx.x >= len) return;
    // chunk sizes are multiples of 4 bytes except a bucket's last chunk: 4-byte stores
    uint32_t* o = reinterpret_cast<uint32_t*>(out + offs[blockIdx.x] + (uint64_t)w * 4 * threadIdx.x);
    if (w == 4) {
        o[0] = x[0];
        o[1] = x[1];
        o[2] = x[2];
        o[3] = x[3];
    } else {  // 4 x 24 bits -> 3 words, little-endian byte order
        o[0] = x[0] | (x[1] << 24);
        o[1] = (x[1] >> 8) | (x[2] << 16);
        o[2] = (x[2] >> 16) | (x[3] << 8);
    }
}

}  // namespace

int launch_d2h_pack_bucket(const double* d, const uint64_t* lohi, uint64_t n_upper,
                           uint64_t* bases, uint8_t* widths, uint64_t* offs, uint32_t* poff,
                           uint64_t* piece_off, uint32_t piece_chunks, uint8_t* out,
                           cudaStream_t s) {
    if (n_upper == 0) return 0;
    const uint64_t chunks = (n_upper + kPackChunk - 1) / kPackChunk;
    const uint64_t* dd = reinterpret_cast<const uint64_t*>(d);
    k9p_widths<<<(unsigned)chunks, kPT, 0, s>>>(dd, lohi, bases, widths);
    k9p_scan<<<1, 1024, 0, s>>>(widths, lohi, offs, poff, piece_off, piece_chunks);
    k9p_pack<<<(unsigned)chunks, kPT, 0, s>>>(dd, lohi, widths, offs, out);
    return 3;
}

}  // namespace ph0b
