// Host memory write bandwidth with non-temporal 64-byte stores, T threads (tools only).
// g++ -O2 -mavx512f tools/host_ntbw.cpp -o tools/host_ntbw -lpthread
#include <immintrin.h>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
int main(int argc, char** argv) {
    const size_t total = 16ull << 30;
    char* buf = (char*)aligned_alloc(64, total);
    memset(buf, 0, total);  // fault the pages in
    for (int T : {1, 2, 4, 8, 12, 15, 16}) {
        for (int rep = 0; rep < 2; ++rep) {
            auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> th;
            for (int t = 0; t < T; ++t)
                th.emplace_back([=] {
                    const size_t per = total / T / 64 * 64;
                    __m512i v = _mm512_set1_epi64(t);
                    for (char* p = buf + t * per; p < buf + (t + 1) * per; p += 64)
                        _mm512_stream_si512((__m512i*)p, v);
                    _mm_sfence();
                });
            for (auto& x : th) x.join();
            const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            printf("T=%2d NT write %.1f GB/s\n", T, total / s / 1e9);
        }
    }
}
