// K1 — tiled upper-triangle pairwise-distance kernel (replaces pairwise_distances,
// /root/reference/proj/src/filtration.cpp:8-18).
//
// * The triangle of 128 x 128 point tiles (bu <= bv) is walked by a persistent grid; each
//   CTA stages the two 128-point tiles of X (coordinate-major, so one tile is a {128, d}
//   box) into shared memory with TMA (cp.async.bulk.tensor.2d + mbarrier), double
//   buffered so the next tile's load overlaps this tile's FP64 math.
// * Bit-exact with the reference: Eigen's norm() of a row difference of a col-major
//   MatrixXd is the sequential fold  acc = Δ0²; acc = acc + Δk²  followed by a correctly
//   rounded sqrt, compiled with no FMA (proj/CMakeLists.txt:8-10).  The
//   explicit __dsub_rn/__dmul_rn/__dadd_rn/__dsqrt_rn keep nvcc from contracting to DFMA.
// * Output is the reference's u-major edge order (filtration.cpp:14-15):
//   key[e] = bits(length) (monotone for lengths >= +0), val[e] = the column value of {u, v}
//   (u << 16 | v, or the edge index above N = 65536: colcodec.h).  Each warp
//   writes 32 consecutive edges of one row per store.  Running min/max key and the
//   histogram of the raw low key byte feed the radix sort's first pass.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace ph0b {
namespace {

constexpr int kTile = 128;      // points per tile side
constexpr int kThreads = 256;   // 8 warps
constexpr int kWarps = kThreads / 32;
constexpr int kRV = kTile / 32; // v columns per lane
constexpr int kMaxTmaDim = 32;  // TMA/smem path for d <= 32

// One CTA-tile of edges. XS: source of coordinates, laid out [k][stride] with the tile's
// first point at offset 0 (smem tile or global pointer).
template <int D>
__device__ __forceinline__ void tile_edges(const double* __restrict__ xu_src,
                                           const double* __restrict__ xv_src, uint64_t stride,
                                           int dd, uint32_t n, uint32_t u0, uint32_t v0,
                                           uint32_t u_lo, uint32_t u_hi, uint64_t e_off,
                                           uint64_t* __restrict__ keys,
                                           uint32_t* __restrict__ vals, uint64_t& kmin,
                                           uint64_t& kmax, uint32_t* sh_hist) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    constexpr bool kStatic = D > 0;
    constexpr int kRegD = (D > 0 && D <= 8) ? D : 1;
    // x_v coordinates for this lane's 4 columns, held in registers for small static d.
    double xv[kRV][kRegD];
    if constexpr (kStatic && D <= 8) {
#pragma unroll
        for (int r = 0; r < kRV; ++r)
#pragma unroll
            for (int k = 0; k < D; ++k) xv[r][k] = xv_src[k * stride + lane + 32 * r];
    }
    const int dim = kStatic ? D : dd;
    const uint64_t nn = n;
    for (int i = warp; i < kTile; i += kWarps) {
        const uint32_t u = u0 + i;
        if (u >= u_hi) break;
        if (u + 1 >= v0 + kTile) break;  // no v > u left in this tile (diagonal tiles)
        if (u < u_lo) continue;          // row outside this shard's row range
        const uint64_t base = row_base(u, nn) - u - 1 - e_off;
        double acc[kRV];
        if constexpr (kStatic && D <= 8) {
            double xu[D];
#pragma unroll
            for (int k = 0; k < D; ++k) xu[k] = xu_src[k * stride + i];
#pragma unroll
            for (int r = 0; r < kRV; ++r) {
                double t = __dsub_rn(xu[0], xv[r][0]);
                acc[r] = __dmul_rn(t, t);
#pragma unroll
                for (int k = 1; k < D; ++k) {
                    t = __dsub_rn(xu[k], xv[r][k]);
                    acc[r] = __dadd_rn(acc[r], __dmul_rn(t, t));
                }
            }
        } else {
            if (dim == 0) {
#pragma unroll
                for (int r = 0; r < kRV; ++r) acc[r] = 0.0;
            } else {
                const double xu0 = xu_src[i];
#pragma unroll
                for (int r = 0; r < kRV; ++r) {
                    const double t = __dsub_rn(xu0, xv_src[lane + 32 * r]);
                    acc[r] = __dmul_rn(t, t);
                }
#pragma unroll 4
                for (int k = 1; k < dim; ++k) {
                    const double xuk = xu_src[k * stride + i];
#pragma unroll
                    for (int r = 0; r < kRV; ++r) {
                        const double t = __dsub_rn(xuk, xv_src[k * stride + lane + 32 * r]);
                        acc[r] = __dadd_rn(acc[r], __dmul_rn(t, t));
                    }
                }
            }
        }
#pragma unroll
        for (int r = 0; r < kRV; ++r) {
            const uint32_t v = v0 + lane + 32 * r;
            if (v > u && v < n) {
                const double len = __dsqrt_rn(acc[r]);
                const uint64_t key = static_cast<uint64_t>(__double_as_longlong(len));
                const uint64_t e = base + v;
                keys[e] = key;
                vals[e] = col_value(u, v, e + e_off, nn);
                kmin = key < kmin ? key : kmin;
                kmax = key > kmax ? key : kmax;
                if (sh_hist) atomicAdd(&sh_hist[key & 0xFFu], 1u);
            }
        }
    }
}

__device__ __forceinline__ void finish_block(uint64_t kmin, uint64_t kmax, uint32_t* sh_hist,
                                             uint64_t* sh_min, uint64_t* sh_max,
                                             uint64_t* minmax, uint32_t* hist0) {
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t a = __shfl_xor_sync(0xffffffffu, kmin, o);
        const uint64_t b = __shfl_xor_sync(0xffffffffu, kmax, o);
        kmin = a < kmin ? a : kmin;
        kmax = b > kmax ? b : kmax;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        sh_min[warp] = kmin;
        sh_max[warp] = kmax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kWarps; ++w) {
            kmin = sh_min[w] < kmin ? sh_min[w] : kmin;
            kmax = sh_max[w] > kmax ? sh_max[w] : kmax;
        }
        if (kmin < *reinterpret_cast<volatile uint64_t*>(&minmax[0]))
            atomicMin(reinterpret_cast<unsigned long long*>(&minmax[0]), kmin);
        if (kmax > *reinterpret_cast<volatile uint64_t*>(&minmax[1]))
            atomicMax(reinterpret_cast<unsigned long long*>(&minmax[1]), kmax);
    }
    if (hist0)
        for (int b = threadIdx.x; b < 256; b += kThreads)
            if (sh_hist[b]) atomicAdd(&hist0[b], sh_hist[b]);
}

// Shared-memory TMA path, d <= 32 (D = 0: runtime d).  Two point-tile pairs in flight, each
// with a "full" mbarrier (TMA completion) and an "empty" one (every warp arrives when it is
// done with the pair): warps move from tile to tile on their own, and thread 0 refills a
// stage as soon as the last warp has left it — no CTA-wide barrier per tile (C5: 8.85 ->
// 7.59 ms; three stages 7.74 ms, four 7.73 ms).
template <int D>
constexpr int distance_stages() { return 2; }

template <int D>
__global__ void __launch_bounds__(kThreads)
    k1_distance_tma(const __grid_constant__ CUtensorMap tmap, uint32_t n, uint32_t dd,
                    uint32_t nb, uint32_t total_tiles, uint32_t t0, uint32_t u_lo, uint32_t u_hi,
                    uint64_t e_off, uint64_t* __restrict__ keys,
                    uint32_t* __restrict__ vals, uint64_t* minmax, uint32_t* hist0) {
    constexpr int S = distance_stages<D>();
    extern __shared__ __align__(128) double smem[];
    __shared__ uint64_t full[S], empty[S];
    __shared__ uint32_t sh_hist[256];
    __shared__ uint64_t sh_min[kWarps], sh_max[kWarps];
    const int dim = D > 0 ? D : (int)dd;
    const uint32_t tile_elems = kTile * dim;   // doubles per {128, d} box
    const uint32_t bytes = 2u * tile_elems * 8u;  // stage s: [u-tile | v-tile]
    auto stage = [&](int s_) { return smem + (size_t)s_ * 2 * tile_elems; };

    for (int b = threadIdx.x; b < 256; b += kThreads) sh_hist[b] = 0;
    if (threadIdx.x == 0) {
        for (int s_ = 0; s_ < S; ++s_) {
            mbar_init(&full[s_], 1);
            mbar_init(&empty[s_], kWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto issue = [&](uint32_t t, int s_) {
        uint32_t bu, bv;
        tile_coords(t + t0, nb, bu, bv);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&full[s_], bytes);
        tma_load_2d(stage(s_), &tmap, &full[s_], (int)(bu * kTile), 0);
        tma_load_2d(stage(s_) + tile_elems, &tmap, &full[s_], (int)(bv * kTile), 0);
    };
    if (threadIdx.x == 0)
        for (int s_ = 0; s_ < S - 1; ++s_) {
            const uint32_t t = blockIdx.x + (uint32_t)s_ * gridDim.x;
            if (t < total_tiles) issue(t, s_);
        }

    uint64_t kmin = ~0ull, kmax = 0;
    uint32_t it = 0;
    for (uint32_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++it) {
        const int s_ = (int)(it % S);
        mbar_wait(&full[s_], (it / S) & 1u);
        if (threadIdx.x == 0) {  // refill the stage left at iteration it - 1
            const uint32_t next = tile + (uint32_t)(S - 1) * gridDim.x;
            if (next < total_tiles) {
                const int sn = (int)((it + S - 1) % S);
                if (it >= 1) mbar_wait(&empty[sn], ((it - 1) / S) & 1u);
                issue(next, sn);
            }
        }
        uint32_t bu, bv;
        tile_coords(tile + t0, nb, bu, bv);
        tile_edges<D>(stage(s_), stage(s_) + tile_elems, kTile, dim, n, bu * kTile, bv * kTile,
                      u_lo, u_hi, e_off, keys, vals, kmin, kmax, hist0 ? sh_hist : nullptr);
        __syncwarp();
        if ((threadIdx.x & 31) == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s_]))
                         : "memory");
    }
    __syncthreads();
    finish_block(kmin, kmax, sh_hist, sh_min, sh_max, minmax, hist0);
}

// Global-memory path for d > 32 (reads X through L1/L2; same arithmetic and order).
__global__ void __launch_bounds__(kThreads)
    k1_distance_global(const double* __restrict__ xpad, uint64_t ldx, uint32_t n, uint32_t dd,
                       uint32_t nb, uint32_t total_tiles, uint32_t t0, uint32_t u_lo,
                       uint32_t u_hi, uint64_t e_off, uint64_t* __restrict__ keys,
                       uint32_t* __restrict__ vals, uint64_t* minmax, uint32_t* hist0) {
    __shared__ uint32_t sh_hist[256];
    __shared__ uint64_t sh_min[kWarps], sh_max[kWarps];
    for (int b = threadIdx.x; b < 256; b += kThreads) sh_hist[b] = 0;
    __syncthreads();
    uint64_t kmin = ~0ull, kmax = 0;
    for (uint32_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        uint32_t bu, bv;
        tile_coords(tile + t0, nb, bu, bv);
        tile_edges<0>(xpad + bu * kTile, xpad + bv * kTile, ldx, (int)dd, n, bu * kTile,
                      bv * kTile, u_lo, u_hi, e_off, keys, vals, kmin, kmax,
                      hist0 ? sh_hist : nullptr);
    }
    __syncthreads();
    finish_block(kmin, kmax, sh_hist, sh_min, sh_max, minmax, hist0);
}

// X (col-major with ld = n, or row-major) -> coordinate-major [d][ldx], zero padded;
// flags any non-finite coordinate (PointCloud ctor, point_cloud.cpp:15-18).
__global__ void k0_pack_points(const double* __restrict__ x, uint32_t layout, uint32_t n,
                               uint32_t d, double* __restrict__ xpad, uint64_t ldx,
                               uint32_t* nonfinite) {
    const uint64_t total = (uint64_t)d * ldx;
    for (uint64_t idx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = idx / ldx, i = idx % ldx;
        double v = 0.0;
        if (i < n) {
            v = layout == 0 ? x[k * n + i] : x[i * (uint64_t)d + k];
            if (!isfinite(v)) atomicOr(nonfinite, 1u);
        }
        xpad[idx] = v;
    }
}

}  // namespace

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

bool make_point_tmap(const double* xpad, uint64_t ldx, uint32_t d, CUtensorMap* map) {
    if (d < 1 || d > 256) return false;
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) return false;
    const cuuint64_t dims[2] = {ldx, d};
    const cuuint64_t strides[1] = {ldx * sizeof(double)};
    const cuuint32_t box[2] = {128u, d};
    const cuuint32_t estr[2] = {1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(xpad), dims, strides,
               box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace {

template <int D>
int launch_tma(const DistanceArgs& a, const CUtensorMap& map, uint32_t nb, uint32_t total,
               uint32_t t0, cudaStream_t s, int num_sms) {
    const uint32_t dim = D > 0 ? D : a.d;
    const size_t smem = 2ull * distance_stages<D>() * kTile * dim * sizeof(double);
    auto kern = k1_distance_tma<D>;
    const int per_sm = kernel_blocks_per_sm((const void*)kern, kThreads, smem);
    if (per_sm < 1) return 0;
    uint32_t grid = (uint32_t)num_sms * per_sm;
    if (grid > total) grid = total;
    kern<<<grid, kThreads, smem, s>>>(map, a.n, a.d, nb, total, t0, a.u_lo, a.u_hi, a.e_off,
                                      a.keys, a.vals, a.minmax, a.hist0);
    return 1;
}

}  // namespace

int launch_pack_points(const double* x, uint32_t layout, uint32_t n, uint32_t d, double* xpad,
                       uint64_t ldx, uint32_t* nonfinite_flag, cudaStream_t s) {
    const uint64_t total = (uint64_t)d * ldx;
    if (total == 0) return 0;
    uint32_t grid = (uint32_t)((total + 255) / 256);
    if (grid > 4096) grid = 4096;
    k0_pack_points<<<grid, 256, 0, s>>>(x, layout, n, d, xpad, ldx, nonfinite_flag);
    return 1;
}

int launch_distance(const DistanceArgs& a, cudaStream_t s, int num_sms) {
    if (a.n < 2 || a.u_hi <= a.u_lo) return 0;
    const uint32_t nb = (a.n + kTile - 1) / kTile;
    // tile rows bu_lo..bu_hi of the upper triangle (rowstart(b) = b*nb - b*(b-1)/2)
    auto rowstart = [nb](uint64_t b) { return b * nb - b * (b - 1) / 2; };
    const uint32_t bu_lo = a.u_lo / kTile, bu_hi = (a.u_hi - 1) / kTile;
    const uint32_t t0 = (uint32_t)rowstart(bu_lo);
    const uint32_t total = (uint32_t)(rowstart(bu_hi + 1) - t0);
    CUtensorMap map;
    if (a.d >= 1 && a.d <= (uint32_t)kMaxTmaDim && make_point_tmap(a.xpad, a.ldx, a.d, &map)) {
        switch (a.d) {
            case 1: return launch_tma<1>(a, map, nb, total, t0, s, num_sms);
            case 2: return launch_tma<2>(a, map, nb, total, t0, s, num_sms);
            case 3: return launch_tma<3>(a, map, nb, total, t0, s, num_sms);
            case 4: return launch_tma<4>(a, map, nb, total, t0, s, num_sms);
            case 8: return launch_tma<8>(a, map, nb, total, t0, s, num_sms);
            case 16: return launch_tma<16>(a, map, nb, total, t0, s, num_sms);
            default: return launch_tma<0>(a, map, nb, total, t0, s, num_sms);
        }
    }
    uint32_t grid = (uint32_t)num_sms * 4;
    if (grid > total) grid = total;
    k1_distance_global<<<grid, kThreads, 0, s>>>(a.xpad, a.ldx, a.n, a.d, nb, total, t0, a.u_lo,
                                                 a.u_hi, a.e_off, a.keys, a.vals, a.minmax,
                                                 a.hist0);
    return 1;
}

}  // namespace ph0b
