// TMA (cp.async.bulk.tensor) + mbarrier helpers and the triangle tile map shared by the
// distance kernels (distance.cu, msd_sort.cu).
#pragma once

#include <cuda.h>
#include <cstdint>

namespace ph0b {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// Tile t of the row-major upper triangle of an nb x nb tile grid -> (bu, bv), bu <= bv.
__device__ __forceinline__ void tile_coords(uint32_t t, uint32_t nb, uint32_t& bu, uint32_t& bv) {
    // rowstart(b) = b*nb - b*(b-1)/2
    const double B = 2.0 * nb + 1.0;
    int b = (int)((B - sqrt(B * B - 8.0 * (double)t)) * 0.5);
    if (b < 0) b = 0;
    auto rs = [nb](int x) { return (int64_t)x * nb - (int64_t)x * (x - 1) / 2; };
    while (b > 0 && rs(b) > (int64_t)t) --b;
    while (rs(b + 1) <= (int64_t)t) ++b;
    bu = (uint32_t)b;
    bv = (uint32_t)(b + ((int64_t)t - rs(b)));
}


// Sequential, unfused fold of the reference (Eigen redux of a row difference, then sqrt):
// acc = d0*d0; acc = acc + dk*dk; sqrt(acc) — explicit _rn intrinsics forbid DFMA contraction.
__device__ __forceinline__ double fold_sq(double acc, double a, double b) {
    const double t = __dsub_rn(a, b);
    return __dadd_rn(acc, __dmul_rn(t, t));
}
__device__ __forceinline__ double first_sq(double a, double b) {
    const double t = __dsub_rn(a, b);
    return __dmul_rn(t, t);
}

// Length bits of edge (u, v) straight from the padded coordinate-major cloud (used for
// samples and survivors; same fold as the tile kernels).
__device__ __forceinline__ uint64_t edge_key_global(const double* __restrict__ xpad, uint64_t ldx,
                                                    uint32_t d, uint32_t u, uint32_t v) {
    if (d == 0) return 0ull;
    double acc = first_sq(xpad[u], xpad[v]);
    for (uint32_t k = 1; k < d; ++k) acc = fold_sq(acc, xpad[k * ldx + u], xpad[k * ldx + v]);
    return static_cast<uint64_t>(__double_as_longlong(__dsqrt_rn(acc)));
}

}  // namespace ph0b
