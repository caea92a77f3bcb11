// Multi-GPU splitter partition: each rank computes the edges of its own
// row range (u-major), then stably partitions them into P contiguous segments by global
// splitters on the length key; segment j goes to rank j in the all-to-all exchange.
// Because rank r owns rows [U_r, U_{r+1}) with U increasing, and every segment keeps the
// u-major order, the data a rank receives (sources concatenated in rank order) is again in
// u-major order, so the local stable radix sort yields exactly the global (length, u, v)
// order restricted to that rank's key range — no merge step is needed.
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace ph0b {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;
constexpr int kMaxParts = 256;

__device__ __forceinline__ uint32_t bucket_of(uint64_t key, const uint64_t* spl, uint32_t nspl) {
    // number of splitters <= key (upper_bound): keys equal to a splitter go right, so equal
    // lengths always land in the same bucket
    uint32_t lo = 0, hi = nspl;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (spl[mid] <= key)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint32_t block_scan_256(uint32_t x, uint32_t* sh_warp,
                                                 uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) sh_warp[warp] = inc;
    __syncthreads();
    uint32_t wb = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        const uint32_t t = sh_warp[w];
        wb += (w < warp) ? t : 0u;
        tot += t;
    }
    if (total) *total = tot;
    return wb + inc - x;
}

// Bucket lookup table over the top kCellBits of (key - kmin): per cell, the bucket of its
// lowest key, with kSplitIn set when a splitter falls inside the cell — then the few
// splitters from that bucket on are compared (a binary search only past three of them).
// Built on the host per partition (build_cell_table).  (2^11 cells keep k7_scatter at 3 CTAs
// per SM; with 2^12 cells and a binary search for every key of a splitter cell, C5's host
// partition spent a quarter of its stall samples in that search.)
constexpr int kCellBits = 11;
constexpr int kCells = 1 << kCellBits;
constexpr uint16_t kSplitIn = 0x8000;

struct CellMap {
    uint64_t kmin;
    uint32_t shift;  // cell = (key - kmin) >> shift
};

__device__ __forceinline__ uint32_t bucket_from(uint64_t key, const uint64_t* spl, uint32_t lo,
                                                uint32_t nspl) {
    uint32_t hi = nspl;  // upper_bound over spl[lo, nspl)
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (spl[mid] <= key)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint32_t bucket_fast(uint64_t key, const uint16_t* s_cell,
                                                const uint64_t* s_spl, uint32_t nspl,
                                                CellMap cm) {
    const uint64_t rel = key - cm.kmin;
    const uint64_t c = rel >> cm.shift;
    if (c >= (uint64_t)kCells) return bucket_of(key, s_spl, nspl);
    const uint32_t e = s_cell[c];
    uint32_t b = e & ~(uint32_t)kSplitIn;
    if (e & kSplitIn) {
#pragma unroll
        for (int t = 0; t < 3; ++t) b += (b < nspl && s_spl[b] <= key) ? 1u : 0u;
        if (b < nspl && s_spl[b] <= key) b = bucket_from(key, s_spl, b, nspl);
    }
    return b;
}

// Per-tile bucket counts, bucket-major (counts[b * tiles + t], one block per tile); one ATOMS
// per key (the bucket key ranges themselves come from the splitters, so no per-key min/max
// is needed).
__global__ void __launch_bounds__(kThreads)
    k7_count(const uint64_t* __restrict__ keys, uint64_t count, const uint64_t* __restrict__ splitters,
             uint32_t parts, uint32_t* __restrict__ counts, const uint16_t* __restrict__ cells,
             CellMap cm) {
    __shared__ uint64_t s_spl[kMaxParts];
    __shared__ uint32_t s_cnt[kMaxParts];
    __shared__ uint16_t s_cell[kCells];
    for (uint32_t i = threadIdx.x; i < kMaxParts; i += kThreads) {
        s_spl[i] = i + 1 < parts ? splitters[i] : ~0ull;
        s_cnt[i] = 0;
    }
    for (uint32_t i = threadIdx.x; i < kCells / 8; i += kThreads)
        reinterpret_cast<uint4*>(s_cell)[i] = reinterpret_cast<const uint4*>(cells)[i];
    const uint64_t base = (uint64_t)blockIdx.x * kTile;
    const uint32_t tn = (uint32_t)(count - base < (uint64_t)kTile ? count - base : kTile);
    uint64_t k[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const uint32_t j = (uint32_t)i * kThreads + threadIdx.x;
        k[i] = j < tn ? keys[base + j] : 0ull;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kItems; ++i)
        if ((uint32_t)i * kThreads + threadIdx.x < tn)
            atomicAdd(&s_cnt[bucket_fast(k[i], s_cell, s_spl, parts - 1, cm)], 1u);
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < parts; b += kThreads)
        counts[(uint64_t)b * gridDim.x + blockIdx.x] = s_cnt[b];
}

// Evenly spaced sample of keys[0..count) (splitter selection).
__global__ void k7_sample(const uint64_t* __restrict__ keys, uint64_t count, uint64_t s,
                          uint64_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < s;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = keys[(i * count) / s + (count / s) / 2];
}

__global__ void k7_gather_u32(const uint32_t* __restrict__ src, const uint32_t* __restrict__ idx,
                              uint64_t m, uint32_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = src[idx[i]];
}

// One block per bucket: exclusive scan of that bucket's (contiguous) per-tile counts, in
// place, and its total.  Warp w walks a contiguous chunk 32 counts at a time.
__global__ void __launch_bounds__(1024)
    k7_scan(uint32_t* __restrict__ counts, uint32_t tiles, uint32_t parts,
            uint64_t* __restrict__ totals) {
    __shared__ uint64_t s_tot[32];
    const uint32_t bk = blockIdx.x;
    uint32_t* c = counts + (uint64_t)bk * tiles;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t per = ((tiles + 31) / 32 + 31) / 32 * 32;
    const uint32_t b = warp * per;
    const uint32_t e = b + per < tiles ? b + per : tiles;
    uint64_t tot = 0;
    constexpr int kU = 8;  // independent loads in flight per lane
    for (uint32_t t0 = b; t0 < e; t0 += 32 * kU) {
        uint32_t x[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t t = t0 + 32 * u + lane;
            x[u] = t < e ? c[t] : 0u;
        }
        uint32_t sum = 0;
#pragma unroll
        for (int u = 0; u < kU; ++u) sum += x[u];
        tot += __reduce_add_sync(0xffffffffu, sum);
    }
    if (lane == 0) s_tot[warp] = tot;
    __syncthreads();
    uint64_t carry = 0, all = 0;
    for (int w = 0; w < 32; ++w) {
        carry += w < warp ? s_tot[w] : 0u;
        all += s_tot[w];
    }
    for (uint32_t t0 = b; t0 < e; t0 += 32 * kU) {
        uint32_t x[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t t = t0 + 32 * u + lane;
            x[u] = t < e ? c[t] : 0u;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t t = t0 + 32 * u + lane;
            uint32_t inc = x[u];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            if (t < e) c[t] = (uint32_t)(carry + inc - x[u]);
            carry += __shfl_sync(0xffffffffu, inc, 31);
        }
    }
    if (threadIdx.x == 0) totals[bk] = all;
}

// One block: padded segment starts (segments begin on `align`-element boundaries), the
// sentinel column {0, 0} (pad_val, colcodec.h) in the padding slots, and each segment's key bounds: segment b
// holds keys in [splitter[b-1], splitter[b]) within the local range [kmin, kmax].
__global__ void k7_layout(const uint64_t* __restrict__ totals, const uint64_t* __restrict__ splitters,
                          uint32_t parts, uint32_t align, uint64_t kmin, uint64_t kmax,
                          uint64_t* __restrict__ starts, uint64_t* __restrict__ bminmax,
                          uint64_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
                          uint32_t pad_val) {
    __shared__ uint64_t s_start[kMaxParts + 1];
    if (threadIdx.x == 0) {
        uint64_t acc = 0;
        for (uint32_t b = 0; b < parts; ++b) {
            s_start[b] = acc;
            acc += (totals[b] + align - 1) / align * align;
        }
        s_start[parts] = acc;
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < parts; b += blockDim.x) {
        starts[b] = s_start[b];
        const uint64_t lo = b > 0 && splitters[b - 1] > kmin ? splitters[b - 1] : kmin;
        const uint64_t hi = b + 1 < parts && splitters[b] - 1 < kmax ? splitters[b] - 1 : kmax;
        bminmax[b] = lo;
        bminmax[parts + b] = hi;
        for (uint64_t q = s_start[b] + totals[b]; q < s_start[b + 1]; ++q) {
            keys_out[q] = 0;
            vals_out[q] = pad_val;
        }
    }
}

// Stable scatter of one 4096-element tile into its segments: ranks from per-warp shared
// histograms (ATOMS lane order = stable), the tile staged in shared memory in segment order,
// then written out so consecutive threads write consecutive positions of each segment run.
__global__ void __launch_bounds__(kThreads, 3)
    k7_scatter(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals, uint64_t count,
               const uint64_t* __restrict__ splitters, uint32_t parts,
               const uint32_t* __restrict__ offsets, const uint64_t* __restrict__ starts,
               uint64_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
               const uint16_t* __restrict__ cells, CellMap cm, uint32_t skip_bucket,
               const uint64_t* __restrict__ peer_k, const uint64_t* __restrict__ peer_v) {
    __shared__ uint64_t s_spl[kMaxParts];
    // peer mode (peer_k != null): bucket b goes straight into its destination rank's receive
    // buffer (NVLink P2P stores through a CUDA IPC mapping); peer_k/peer_v[b] are byte
    // addresses already offset so that local layout position q lands at q * 8 / q * 4
    __shared__ uint64_t s_pk[kMaxParts], s_pv[kMaxParts];
    __shared__ uint16_t s_cell[kCells];
    __shared__ uint32_t s_whist[kWarps][kMaxParts];
    __shared__ uint32_t s_tstart[kMaxParts];
    __shared__ uint64_t s_base[kMaxParts];  // global position of this tile's first element of b
    __shared__ uint32_t s_scan[kWarps];
    extern __shared__ __align__(16) uint64_t sc_dyn[];
    uint64_t* s_k = sc_dyn;                                                 // [kTile]
    uint32_t* s_v = reinterpret_cast<uint32_t*>(sc_dyn + kTile);            // [kTile]
    uint8_t* s_b = reinterpret_cast<uint8_t*>(s_v + kTile);                 // [kTile]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t tile0 = (uint64_t)blockIdx.x * kTile;
    const uint32_t tn = (uint32_t)(count - tile0 < (uint64_t)kTile ? count - tile0 : kTile);
    const uint32_t wofs = warp * (32 * kItems) + lane;
    uint64_t kk[kItems];
    uint32_t vv[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {  // all loads in flight first
        const uint32_t pos = wofs + 32 * i;
        kk[i] = pos < tn ? keys[tile0 + pos] : 0ull;
        vv[i] = pos < tn ? vals[tile0 + pos] : 0u;
    }
    // kThreads == kMaxParts: thread b owns bucket b in the per-bucket steps
    s_spl[tid] = (uint32_t)tid + 1 < parts ? splitters[tid] : ~0ull;
    if (peer_k) {
        s_pk[tid] = (uint32_t)tid < parts ? peer_k[tid] : 0ull;
        s_pv[tid] = (uint32_t)tid < parts ? peer_v[tid] : 0ull;
    }
    for (uint32_t i = tid; i < kCells / 8; i += kThreads)
        reinterpret_cast<uint4*>(s_cell)[i] = reinterpret_cast<const uint4*>(cells)[i];
    const uint64_t my_base =
        (uint32_t)tid < parts ? starts[tid] + offsets[(uint64_t)tid * gridDim.x + blockIdx.x] : 0ull;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s_whist[w][tid] = 0;
    __syncthreads();
    uint32_t br[kItems];  // bucket << 16 | rank within the warp (rank < 512)
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const uint32_t pos = wofs + 32 * i;
        const uint32_t b = pos < tn ? bucket_fast(kk[i], s_cell, s_spl, parts - 1, cm) : 0u;
        // ATOMS resolves same-address lanes in lane order (device self-test), so the
        // returned count is the stable rank within this warp
        br[i] = (b << 16) | (pos < tn ? atomicAdd(&s_whist[warp][b], 1u) : 0u);
    }
    __syncthreads();
    uint32_t acc = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        const uint32_t c = s_whist[w][tid];
        s_whist[w][tid] = acc;
        acc += c;
    }
    const uint32_t tstart = block_scan_256(acc, s_scan, nullptr);
    s_tstart[tid] = tstart;
    s_base[tid] = my_base - tstart;  // global position of tile slot p of bucket b = base + p
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s_whist[w][tid] += tstart;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const uint32_t pos = wofs + 32 * i;
        if (pos < tn) {
            const uint32_t dst = s_whist[warp][br[i] >> 16] + (br[i] & 0xFFFFu);
            s_k[dst] = kk[i];
            s_v[dst] = vv[i];
            s_b[dst] = (uint8_t)(br[i] >> 16);
        }
    }
    __syncthreads();
#pragma unroll 4
    for (int i = 0; i < kItems; ++i) {
        const uint32_t p = (uint32_t)i * kThreads + tid;
        if (p < tn && s_b[p] != skip_bucket) {
            const uint32_t b = s_b[p];
            const uint64_t dst = s_base[b] + p;
            if (peer_k) {
                reinterpret_cast<uint64_t*>(s_pk[b])[dst] = s_k[p];
                reinterpret_cast<uint32_t*>(s_pv[b])[dst] = s_v[p];
            } else {
                keys_out[dst] = s_k[p];
                vals_out[dst] = s_v[p];
            }
        }
    }
}

// Stable extraction of one segment (keys in [lo_b, hi_b]) into its place in the partition
// output, ahead of the full scatter, so that segment can be sorted while the rest is still
// being partitioned (overlapped host path).  Same tiles and offsets as k7_count/k7_scan.
__global__ void __launch_bounds__(kThreads)
    k7_select(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals, uint64_t count,
              uint32_t parts, uint32_t b, const uint32_t* __restrict__ offsets,
              const uint64_t* __restrict__ starts, const uint64_t* __restrict__ bminmax,
              uint64_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out) {
    __shared__ uint32_t s_wt[kWarps];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t tile0 = (uint64_t)blockIdx.x * kTile;
    const uint32_t tn = (uint32_t)(count - tile0 < (uint64_t)kTile ? count - tile0 : kTile);
    const uint64_t lo = bminmax[b], hi = bminmax[parts + b];
    const uint32_t wofs = warp * (32 * kItems) + lane;
    uint64_t k[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const uint32_t pos = wofs + 32 * i;
        k[i] = pos < tn ? keys[tile0 + pos] : ~0ull;
    }
    uint32_t ball[kItems], total = 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const uint32_t pos = wofs + 32 * i;
        ball[i] = __ballot_sync(0xffffffffu, pos < tn && k[i] >= lo && k[i] <= hi);
        total += __popc(ball[i]);
    }
    if (lane == 0) s_wt[warp] = total;
    __syncthreads();
    uint32_t wb = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) wb += (w < warp) ? s_wt[w] : 0u;
    uint64_t run = starts[b] + offsets[(uint64_t)b * gridDim.x + blockIdx.x] + wb;
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        if ((ball[i] >> lane) & 1u) {
            const uint64_t dst = run + __popc(ball[i] & lt);
            keys_out[dst] = k[i];
            vals_out[dst] = vals[tile0 + wofs + 32 * i];
        }
        run += __popc(ball[i]);
    }
}

// Sentinel column {0, 0} (key 0) in the padding slots [start_b + total_b, pad(...)) of every
// segment of (keys, vals) — a buffer other than the one k7_layout padded.
__global__ void k7_pad_fill(const uint64_t* __restrict__ totals, const uint64_t* __restrict__ starts,
                            uint32_t parts, uint32_t align, uint64_t* __restrict__ keys,
                            uint32_t* __restrict__ vals, uint32_t pad_val) {
    for (uint32_t b = threadIdx.x; b < parts; b += blockDim.x) {
        const uint64_t e = starts[b] + (totals[b] + align - 1) / align * align;
        for (uint64_t q = starts[b] + totals[b]; q < e; ++q) {
            keys[q] = 0;
            vals[q] = pad_val;
        }
    }
}

}  // namespace

namespace {
// Host: the cell -> bucket table for splitters h_spl[parts-1] over keys in [kmin, kmax].
CellMap build_cell_table(const uint64_t* h_spl, uint32_t parts, uint64_t kmin, uint64_t kmax,
                         uint16_t* table) {
    const uint64_t span = kmax >= kmin ? kmax - kmin : 0;
    const uint32_t bits = span ? 64u - (uint32_t)__builtin_clzll(span) : 0u;
    CellMap cm{kmin, bits > (uint32_t)kCellBits ? bits - kCellBits : 0u};
    auto ub = [&](uint64_t key) {  // upper_bound over the splitters
        uint32_t lo = 0, hi = parts - 1;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (h_spl[mid] <= key) lo = mid + 1; else hi = mid;
        }
        return lo;
    };
    for (uint32_t c = 0; c < (uint32_t)kCells; ++c) {
        const uint64_t lo_rel = (uint64_t)c << cm.shift;
        if (lo_rel > span) {  // (no key falls here; scanning from the last bucket is exact)
            table[c] = (uint16_t)(ub(kmax) | kSplitIn);
            continue;
        }
        const uint64_t hi_rel = ((uint64_t)(c + 1) << cm.shift) - 1;
        const uint64_t lo_key = kmin + lo_rel;
        const uint64_t hi_key = hi_rel > span ? kmax : kmin + hi_rel;
        const uint32_t a = ub(lo_key), b = ub(hi_key);
        table[c] = (uint16_t)(a | (a == b ? 0u : (uint32_t)kSplitIn));
    }
    return cm;
}
}  // namespace

size_t partition_table_bytes() { return kCells * sizeof(uint16_t); }

int launch_partition_count(const uint64_t* keys, uint64_t count, const uint64_t* d_splitters,
                           uint32_t parts, uint32_t* d_counts_scratch, uint64_t* d_totals,
                           uint64_t* d_bminmax, uint64_t* keys_out, uint32_t* vals_out,
                           cudaStream_t s, uint32_t align, uint64_t kmin, uint64_t kmax,
                           const uint64_t* h_splitters, uint16_t* d_table, uint32_t pad_val) {
    static_assert(kThreads == kMaxParts, "one thread per bucket in k7_scatter");
    if (parts < 1 || parts > (uint32_t)kMaxParts) return -1;
    const uint64_t tiles = (count + kTile - 1) / kTile;
    static thread_local std::vector<uint16_t> h_table(kCells);
    const CellMap cm = build_cell_table(h_splitters, parts, kmin, kmax, h_table.data());
    // pageable source: the copy is staged before the call returns, so reuse is safe
    cudaMemcpyAsync(d_table, h_table.data(), kCells * sizeof(uint16_t), cudaMemcpyHostToDevice, s);
    int l = 1;
    if (tiles == 0) {
        cudaMemsetAsync(d_totals, 0, sizeof(uint64_t) * parts, s);
    } else {
        k7_count<<<(unsigned)tiles, kThreads, 0, s>>>(keys, count, d_splitters, parts,
                                                      d_counts_scratch, d_table, cm);
        k7_scan<<<parts, 1024, 0, s>>>(d_counts_scratch, (uint32_t)tiles, parts, d_totals);
        l = 3;
    }
    // d_totals has room for 2 * parts words: [totals | segment starts]
    k7_layout<<<1, 256, 0, s>>>(d_totals, d_splitters, parts, align, kmin, kmax,
                                d_totals + parts, d_bminmax, keys_out, vals_out, pad_val);
    return l;
}

int launch_partition_select(const uint64_t* keys, const uint32_t* vals, uint64_t count,
                            uint32_t parts, uint32_t bucket, const uint32_t* d_counts_scratch,
                            const uint64_t* d_totals, const uint64_t* d_bminmax,
                            uint64_t* keys_out, uint32_t* vals_out, cudaStream_t s) {
    const uint64_t tiles = (count + kTile - 1) / kTile;
    if (tiles == 0) return 0;
    k7_select<<<(unsigned)tiles, kThreads, 0, s>>>(keys, vals, count, parts, bucket,
                                                   d_counts_scratch, d_totals + parts, d_bminmax,
                                                   keys_out, vals_out);
    return 1;
}

int launch_partition_scatter(const uint64_t* keys, const uint32_t* vals, uint64_t count,
                             const uint64_t* d_splitters, uint32_t parts,
                             const uint32_t* d_counts_scratch, const uint64_t* d_totals,
                             uint64_t* keys_out, uint32_t* vals_out, cudaStream_t s,
                             uint64_t kmin, uint64_t kmax, const uint16_t* d_table,
                             uint32_t skip_bucket, const uint64_t* d_peer_k,
                             const uint64_t* d_peer_v) {
    const uint64_t tiles = (count + kTile - 1) / kTile;
    if (tiles == 0) return 0;
    const uint64_t span = kmax >= kmin ? kmax - kmin : 0;
    const uint32_t bits = span ? 64u - (uint32_t)__builtin_clzll(span) : 0u;
    const CellMap cm{kmin, bits > (uint32_t)kCellBits ? bits - kCellBits : 0u};
    constexpr size_t kScSmem = (size_t)kTile * (8 + 4 + 1);
    // one tile per CTA: the block scheduler overlaps a new tile's loads with finishing tiles
    // (a persistent grid over the same tiles measured 19.1 ms vs 14.0 at C5)
    if (kernel_blocks_per_sm((const void*)k7_scatter, kThreads, kScSmem) < 1) return -1;
    k7_scatter<<<(unsigned)tiles, kThreads, kScSmem, s>>>(keys, vals, count, d_splitters, parts,
                                                          d_counts_scratch, d_totals + parts,
                                                          keys_out, vals_out, d_table, cm,
                                                          skip_bucket, d_peer_k, d_peer_v);
    return 1;
}

int launch_partition_pad(const uint64_t* d_totals, uint32_t parts, uint32_t align,
                         uint64_t* keys, uint32_t* vals, cudaStream_t s, uint32_t pad_val) {
    k7_pad_fill<<<1, 256, 0, s>>>(d_totals, d_totals + parts, parts, align, keys, vals,
                                  pad_val);
    return 1;
}

int launch_partition(const uint64_t* keys, const uint32_t* vals, uint64_t count,
                     const uint64_t* d_splitters, uint32_t parts, uint32_t* d_counts_scratch,
                     uint64_t* d_totals, uint64_t* d_bminmax, uint64_t* keys_out,
                     uint32_t* vals_out, cudaStream_t s, uint32_t align, uint64_t kmin,
                     uint64_t kmax, const uint64_t* h_splitters, uint16_t* d_table) {
    const int l = launch_partition_count(keys, count, d_splitters, parts, d_counts_scratch,
                                         d_totals, d_bminmax, keys_out, vals_out, s, align, kmin,
                                         kmax, h_splitters, d_table);
    if (l < 0) return l;
    const int sc = launch_partition_scatter(keys, vals, count, d_splitters, parts, d_counts_scratch,
                                        d_totals, keys_out, vals_out, s, kmin, kmax, d_table,
                                        ~0u, nullptr, nullptr);
    return sc < 0 ? sc : l + sc;
}

int launch_sample(const uint64_t* keys, uint64_t count, uint64_t s, uint64_t* out, cudaStream_t st) {
    if (s == 0 || count == 0) return 0;
    k7_sample<<<(unsigned)((s + 255) / 256), 256, 0, st>>>(keys, count, s, out);
    return 1;
}

int launch_gather_u32(const uint32_t* src, const uint32_t* idx, uint64_t m, uint32_t* out,
                      cudaStream_t st) {
    if (m == 0) return 0;
    k7_gather_u32<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(src, idx, m, out);
    return 1;
}

uint64_t partition_scratch_words(uint64_t count, uint32_t parts) {
    return ((count + kTile - 1) / kTile) * parts;
}

}  // namespace ph0b
