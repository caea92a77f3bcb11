// Per-device launch attributes of the kernels with dynamic shared memory (the opt-in above
// 48 KB), and their occupancy.  cudaFuncSetAttribute acts on the CURRENT device's context, so
// a process that runs on device 1 after device 0 (ph0b_options.device, one context per
// device, the multi-device path) must opt in again there: the result is cached per
// (device, kernel, smem, threads) under a lock, and a cache entry is published only once
// both calls have returned.
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <tuple>

#include "kernels.h"

namespace ph0b {

int kernel_blocks_per_sm(const void* kern, int threads, size_t smem) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    using Key = std::tuple<int, const void*, size_t, int>;
    static std::mutex mu;
    static std::map<Key, int> cache;
    // the opt-in is a per-kernel maximum: it is only ever raised, so a launch with less
    // shared memory never lowers it under a cached larger size (kernels whose shared memory
    // depends on N or d are launched with several sizes)
    static std::map<std::pair<int, const void*>, size_t> opted;
    const Key key{dev, kern, smem, threads};
    std::lock_guard<std::mutex> lock(mu);
    const auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    size_t& cur = opted[{dev, kern}];
    // (the opt-in also covers dynamic + static shared memory crossing 48 KB together)
    if (smem > cur) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess) {
            cudaGetLastError();
            return 0;  // not cached: a later call may retry
        }
        cur = smem;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) !=
        cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    cache.emplace(key, per_sm);
    return per_sm;
}

int device_sm_count() {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    return n;
}

}  // namespace ph0b
