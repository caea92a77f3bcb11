// Page-locked host memory for the D stream (ring, chunk metadata, result and caller buffers):
// anonymous memory on transparent huge pages, then cudaHostRegister (cudaHostAlloc if that
// fails, or with PH0B_HOST_THP=0).  With cudaHostAlloc the C5 host-path e2e of the same code
// was ~182 ms in most processes and 204-233 ms in some (2 of 10 in a row on one box, and most
// of the round's earlier bench processes); on huge pages 10 of 10 ran at 181-192 ms
// (tools/ab_host_thp.sh, profiles/host_thp_r02.txt).
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>

#include "kernels.h"

namespace ph0b {
namespace {
std::mutex g_mu;
std::map<void*, size_t>& registered() {
    static auto* m = new std::map<void*, size_t>();  // (never destroyed: frees may come late)
    return *m;
}
bool use_thp() {
    static const bool v = [] {
        const char* e = getenv("PH0B_HOST_THP");
        return !(e && e[0] == '0');
    }();
    return v;
}
}  // namespace

void* pinned_alloc(size_t bytes) {
    bytes = bytes ? bytes : 1;
    if (use_thp()) {
        const size_t len = (bytes + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1);
        void* p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (p != MAP_FAILED) {
            madvise(p, len, MADV_HUGEPAGE);
            if (cudaHostRegister(p, len, cudaHostRegisterDefault) == cudaSuccess) {
                std::lock_guard<std::mutex> lk(g_mu);
                registered()[p] = len;
                return p;
            }
            cudaGetLastError();
            munmap(p, len);
        }
    }
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}

void pinned_free(void* p) {
    if (!p) return;
    size_t len = 0;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = registered().find(p);
        if (it != registered().end()) {
            len = it->second;
            registered().erase(it);
        }
    }
    if (len) {
        cudaHostUnregister(p);
        munmap(p, len);
    } else {
        cudaFreeHost(p);
    }
}

}  // namespace ph0b
