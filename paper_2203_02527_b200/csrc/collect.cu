// K5 — barcode collect (replaces extract_barcode, /root/reference/proj/src/reduction.cpp:140-150).
//
// The reduction leaves the surviving column ids unordered; they are put in filtration order
// with the same onesweep radix sort (keys only), then each survivor j becomes the interval
// (0, grade_j, scale[grade_j - 1]) with grade_j = 1 + lower_bound(D, length_j) — D is strictly
// increasing and contains length_j, so this is exactly the grade build_filtration assigned
// (filtration.cpp:29-33).  essential_count = N - #finite (reduction.cpp:148) is done on host.
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace ph0b {
namespace {

__global__ void k5_widen(const uint32_t* __restrict__ in, uint32_t m, uint64_t* __restrict__ out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
        out[i] = in[i];
}

__global__ void k5_narrow(const uint64_t* __restrict__ in, uint32_t m, uint32_t* __restrict__ out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
        out[i] = (uint32_t)in[i];
}

__global__ void k5_map(const uint64_t* __restrict__ cols_sorted, uint32_t m,
                       const uint64_t* __restrict__ sorted_keys, const double* __restrict__ scale,
                       const uint64_t* __restrict__ n_scale, uint64_t grade_offset,
                       uint32_t* __restrict__ surv_sorted,
                       uint64_t* __restrict__ death_grade, double* __restrict__ death_length) {
    const uint64_t* dbits = reinterpret_cast<const uint64_t*>(scale);
    const uint64_t ns = *n_scale;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        const uint64_t j = cols_sorted[i];
        const uint64_t key = sorted_keys[j];
        uint64_t lo = 0, hi = ns;  // first index with D[idx] >= key
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (dbits[mid] < key)
                lo = mid + 1;
            else
                hi = mid;
        }
        death_grade[i] = grade_offset + lo + 1;
        death_length[i] = __longlong_as_double((long long)key);
        surv_sorted[i] = (uint32_t)j;
    }
}

// Reduced support {x, low} (x < low) of each surviving column, in filtration order — the
// column the reference's reduce() leaves in M (reduction.cpp:33-49) — and its claimed low
// (reduction.cpp:44-45).  Supports stay 2-sparse (boundary_matrix.cpp:22-24): reducing {a, c}
// (a < c) against the earlier column that claimed row c, whose support is {parent(c), c},
// gives {a, parent(c)}; the walk ends when the larger row is unclaimed, and that column then
// claims it.  Only surviving columns claim rows, so replaying the walk over the N-1 survivors
// in filtration order reproduces the reference's pivot table and reduced columns exactly
// (the cycle columns end empty).  One thread, parent table in shared memory: a parity
// surface, not on the hot path.
// kWide (N > 65536): rows do not fit u16 and the table does not fit shared memory — a u32
// parent table in global memory (gparent, n entries).
template <bool kWide>
__global__ void k5_reduced_supports(const uint32_t* __restrict__ surv_sorted, uint32_t m,
                                    const uint32_t* __restrict__ uv, uint32_t n,
                                    uint32_t* __restrict__ xs, uint32_t* __restrict__ lows,
                                    uint32_t* __restrict__ err, uint32_t* __restrict__ gparent) {
    extern __shared__ uint16_t s_parent[];  // parent[r] == r: row r is unclaimed
    for (uint32_t v = threadIdx.x; v < n; v += blockDim.x) {
        if (kWide)
            gparent[v] = v;
        else
            s_parent[v] = (uint16_t)v;
    }
    if (kWide) __threadfence_block();
    __syncthreads();
    if (threadIdx.x != 0) return;
    auto parent = [&](uint32_t r) -> uint32_t { return kWide ? gparent[r] : s_parent[r]; };
    uint32_t bad = 0;
    for (uint32_t i = 0; i < m; ++i) {
        uint32_t a, c;
        col_rows(uv[surv_sorted[i]], n, a, c);
        if (a > c) {
            const uint32_t t = a;
            a = c;
            c = t;
        }
        while (parent(c) != c) {  // row c claimed by an earlier column {parent(c), c}
            const uint32_t p = parent(c);
            if (p == a) {  // the column would empty: not a survivor (cannot happen)
                bad = 1;
                break;
            }
            c = p > a ? p : a;
            a = p > a ? a : p;
        }
        if (kWide)
            gparent[c] = a;
        else
            s_parent[c] = (uint16_t)a;
        lows[i] = c;
        if (xs) xs[i] = a;
    }
    if (err) *err = bad;
}

}  // namespace

// a.surv: unordered survivors; a.surv_scratch reinterpreted as 2 x m u64 ping-pong is not
// enough room, so the caller passes u64 scratch through SortArgs (see pipeline).
int launch_collect_map(const uint64_t* cols_sorted, uint32_t m, const uint64_t* sorted_keys,
                       const double* scale, const uint64_t* n_scale, uint64_t grade_offset,
                       uint32_t* surv_sorted, uint64_t* death_grade, double* death_length,
                       cudaStream_t s) {
    if (m == 0) return 0;
    const unsigned grid = (m + 255) / 256;
    k5_map<<<grid, 256, 0, s>>>(cols_sorted, m, sorted_keys, scale, n_scale, grade_offset,
                                surv_sorted, death_grade, death_length);
    return 1;
}

int launch_narrow(const uint64_t* in, uint32_t m, uint32_t* out, cudaStream_t s) {
    if (m == 0) return 0;
    k5_narrow<<<(m + 255) / 256, 256, 0, s>>>(in, m, out);
    return 1;
}

int launch_widen(const uint32_t* in, uint32_t m, uint64_t* out, cudaStream_t s) {
    if (m == 0) return 0;
    k5_widen<<<(m + 255) / 256, 256, 0, s>>>(in, m, out);
    return 1;
}

int launch_reduced_supports(const uint32_t* surv_sorted, uint32_t m, const uint32_t* uv,
                            uint32_t n, uint32_t* xs, uint32_t* lows, uint32_t* err,
                            uint32_t* scratch, cudaStream_t s) {
    if (m == 0) return 0;
    if (col_ids(n)) {
        k5_reduced_supports<true><<<1, 1024, 0, s>>>(surv_sorted, m, uv, n, xs, lows, err,
                                                     scratch);
        return 1;
    }
    const size_t smem = sizeof(uint16_t) * ((n + 1) & ~1u);
    if (kernel_blocks_per_sm((const void*)k5_reduced_supports<false>, 1024, smem) < 1) return -1;
    k5_reduced_supports<false><<<1, 1024, smem, s>>>(surv_sorted, m, uv, n, xs, lows, err,
                                                      nullptr);
    return 1;
}

}  // namespace ph0b
