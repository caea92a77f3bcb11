// D2H microbenchmark for the streamed ring (tools only): throughput of P-MiB copies on S
// streams, with/without stream memory ops (cuStreamWaitValue32 / cuStreamWriteValue32).
// nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/ring_bench.cu -o tools/ring_bench -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <immintrin.h>

#include <chrono>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

int main(int argc, char** argv) {
    const double total_gb = 8.0;
    cudaSetDevice(0);
    const size_t total = (size_t)(total_gb * (1ull << 30));
    void* d;
    cudaMalloc(&d, total);
    cudaMemset(d, 1, total);
    void* h_big;
    cudaHostAlloc(&h_big, total, cudaHostAllocDefault);
    uint32_t* flags;
    cudaHostAlloc((void**)&flags, 4096 * 4, cudaHostAllocMapped);
    for (int i = 0; i < 4096; ++i) flags[i] = 0;
    CUdeviceptr dflags;
    cudaHostGetDevicePointer((void**)&dflags, flags, 0);
    std::vector<cudaStream_t> ss(8);
    for (auto& s : ss) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    if (argc > 1) {  // contention: DMA into a small ring while T threads NT-write 2x the bytes
        const int T = atoi(argv[1]);
        const size_t ring = (size_t)atoi(argc > 2 ? argv[2] : "32") << 20;
        const size_t P = 8ull << 20, n = total / P;
        const size_t out_bytes = 2 * total;
        char* out = (char*)aligned_alloc(64, out_bytes);
        memset(out, 0, out_bytes);
        for (int rep = 0; rep < 3; ++rep) {
            cudaDeviceSynchronize();
            auto t0 = std::chrono::steady_clock::now();
            cudaEventRecord(e0, ss[0]);
            for (size_t i = 0; i < n; ++i)
                cudaMemcpyAsync((char*)h_big + (i * P) % ring, (char*)d + i * P, P,
                                cudaMemcpyDeviceToHost, ss[i % 2]);
            cudaEventRecord(e1, ss[0]);
            std::vector<std::thread> th;
            for (int t = 0; t < T; ++t)
                th.emplace_back([=] {
                    const size_t per = out_bytes / T / 64 * 64;
                    __m512i v = _mm512_set1_epi64(t);
                    for (char* p = out + t * per; p < out + (t + 1) * per; p += 64)
                        _mm512_stream_si512((__m512i*)p, v);
                    _mm_sfence();
                });
            for (auto& x : th) x.join();
            const double cpu = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            cudaDeviceSynchronize();
            const double all = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("T=%d ring %zu MiB: DMA %.1f GB/s alone-equivalent (%.1f ms stream0), CPU NT %.1f GB/s (%.1f ms), all %.1f ms\n",
                   T, ring >> 20, total / (all * 1e6), ms, out_bytes / (cpu * 1e6), cpu, all);
        }
        return 0;
    }
    const int pieces_mib[] = {1, 2, 4, 8, 32};
    for (int mode = 0; mode < 4; ++mode) {  // 0 plain, 1 +write, 2 +wait, 3 +wait+write
        for (int S : {1, 2, 4, 8}) {
            for (int pm : pieces_mib) {
                const size_t P = (size_t)pm << 20;
                const size_t n = total / P;
                // ring of 32 MiB for the destination when mode>0 (as the product), else big
                const size_t ring = 32ull << 20;
                cudaDeviceSynchronize();
                auto t0 = std::chrono::steady_clock::now();
                cudaEventRecord(e0, ss[0]);
                for (int i = 1; i < S; ++i) cudaStreamWaitEvent(ss[i], e0, 0);
                for (size_t i = 0; i < n; ++i) {
                    cudaStream_t s = ss[i % S];
                    if (mode >= 2) cuStreamWaitValue32((CUstream)s, dflags, 0, CU_STREAM_WAIT_VALUE_EQ);
                    char* dst = (char*)h_big + (i * P) % ring;
                    cudaMemcpyAsync(dst, (char*)d + i * P, P, cudaMemcpyDeviceToHost, s);
                    if (mode == 1 || mode == 3)
                        cuStreamWriteValue32((CUstream)s, dflags + 4 * (1 + i % 1000), (uint32_t)i, 0);
                }
                auto t1 = std::chrono::steady_clock::now();
                for (int i = 1; i < S; ++i) {
                    cudaEvent_t x;
                    cudaEventCreate(&x);
                    cudaEventRecord(x, ss[i]);
                    cudaStreamWaitEvent(ss[0], x, 0);
                    cudaEventDestroy(x);
                }
                cudaEventRecord(e1, ss[0]);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                const double enq = std::chrono::duration<double, std::milli>(t1 - t0).count();
                printf("mode %d S=%d piece %2d MiB: %7.1f ms  %5.1f GB/s  (enqueue %6.1f ms, %zu pieces)\n",
                       mode, S, pm, ms, n * P / ms / 1e6, enq, n);
                fflush(stdout);
            }
        }
    }
    return 0;
}
