// Column value of an edge (the boundary-matrix column {u, v}, u < v) as carried through the
// sort, shared by host and device code.  N <= 65536: u << 16 | v.  Above that ("edge-id
// mode", N <= 92682 so that K < 2^32): the u-major edge index e (filtration.cpp:14-15 order),
// with kColCycle standing for the cycle column {0, 0} (padding).  Decided by N alone, so every
// kernel and the host agree.
#pragma once

#include <cmath>
#include <cstdint>

#ifdef __CUDACC__
#define PH0B_HD __host__ __device__ __forceinline__
#else
#define PH0B_HD inline
#endif

namespace ph0b {

constexpr uint32_t kPackedMaxN = 65536;
constexpr uint32_t kColCycle = 0xFFFFFFFFu;

// Upper-triangle edge indexing in the reference's u-major order (filtration.cpp:14-15):
// e(u, v) = u*(2N-u-1)/2 + (v-u-1) for u < v.
PH0B_HD uint64_t row_base(uint64_t u, uint64_t n) { return u * (2 * n - u - 1) / 2; }

PH0B_HD bool col_ids(uint64_t n) { return n > kPackedMaxN; }
PH0B_HD uint32_t col_cycle(uint64_t n) { return col_ids(n) ? kColCycle : 0u; }

PH0B_HD uint32_t col_value(uint32_t u, uint32_t v, uint64_t e_global, uint64_t n) {
    return col_ids(n) ? (uint32_t)e_global : ((u << 16) | v);
}

PH0B_HD void col_rows(uint32_t c, uint64_t n, uint32_t& u, uint32_t& v) {
    if (!col_ids(n)) {
        u = c >> 16;
        v = c & 0xFFFFu;
        return;
    }
    if (c == kColCycle) {
        u = v = 0;
        return;
    }
    // the largest u with row_base(u) <= c: the smaller root of u^2 - (2N-1)u + 2c = 0, then
    // exact integer fix-ups (the double estimate is off by at most one row)
    const double b = 2.0 * (double)n - 1.0;
    const double t = b * b - 8.0 * (double)c;
    uint64_t r = (uint64_t)((b - sqrt(t > 0.0 ? t : 0.0)) * 0.5);
    while (r > 0 && row_base(r, n) > c) --r;
    while (r + 1 < n && row_base(r + 1, n) <= c) ++r;
    u = (uint32_t)r;
    v = (uint32_t)(c - row_base(r, n) + r + 1);
}

}  // namespace ph0b
