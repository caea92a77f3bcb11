// Host decoder of the compressed D stream; see host_decode.h and d2h_codec.cu.
#include "host_decode.h"

#include <immintrin.h>
#include <sys/resource.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>

namespace ph0b {

namespace {

struct Chunk {
    const uint32_t* deltas;
    uint64_t base;
    uint64_t* out;
    uint32_t len;
};

__attribute__((target("avx2"))) void decode_avx2(const Chunk& t) {
    uint64_t acc = t.base;
    uint64_t* out = t.out;
    const uint32_t* d = t.deltas;
    uint32_t i = 0;
    out[0] = acc;
    i = 1;
    // scalar until the output is 32-byte aligned, then 4 values per non-temporal store (the
    // decoded D is not read again by this process: streaming stores skip the cache fill)
    while (i < t.len && (reinterpret_cast<uintptr_t>(out + i) & 31u)) {
        acc += d[i];
        out[i++] = acc;
    }
    for (; i + 4 <= t.len; i += 4) {
        const uint64_t a0 = acc + d[i];
        const uint64_t a1 = a0 + d[i + 1];
        const uint64_t a2 = a1 + d[i + 2];
        const uint64_t a3 = a2 + d[i + 3];
        acc = a3;
        _mm256_stream_si256(reinterpret_cast<__m256i*>(out + i),
                            _mm256_set_epi64x((long long)a3, (long long)a2, (long long)a1,
                                              (long long)a0));
    }
    for (; i < t.len; ++i) {
        acc += d[i];
        out[i] = acc;
    }
    _mm_sfence();
}

void decode_scalar(const Chunk& t) {
    uint64_t acc = t.base;
    t.out[0] = acc;
    for (uint32_t i = 1; i < t.len; ++i) {
        acc += t.deltas[i];
        t.out[i] = acc;
    }
}

}  // namespace

void decode_chunk(const DecodeTask& t) {
    static const bool avx2 = __builtin_cpu_supports("avx2");
    for (uint64_t j = 0, s0 = 0; s0 < t.n; ++j, s0 += t.chunk) {
        if (t.raw[j]) continue;
        const Chunk c{t.deltas + s0, t.bases[j], t.out + s0,
                      (uint32_t)(t.n - s0 < t.chunk ? t.n - s0 : t.chunk)};
        if (avx2)
            decode_avx2(c);
        else
            decode_scalar(c);
    }
}

DecodePool::DecodePool(unsigned threads) {
    for (unsigned i = 0; i < std::max(1u, threads); ++i) workers_.emplace_back([this] { run(); });
}

DecodePool::~DecodePool() {
    {
        std::lock_guard<std::mutex> lk(mu_);
        stop_ = true;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
}

void DecodePool::submit(const std::vector<DecodeTask>& tasks) {
    if (tasks.empty()) return;
    {
        std::lock_guard<std::mutex> lk(mu_);
        for (const auto& t : tasks) queue_.push_back(t);
        pending_ += tasks.size();
    }
    cv_.notify_all();
}

void DecodePool::wait() {
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
}

void DecodePool::run() {
    // below the orchestrating thread: the GPU's next launches must not wait for a core
    setpriority(PRIO_PROCESS, (id_t)syscall(SYS_gettid), 5);
    for (;;) {
        DecodeTask t;
        {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [this] { return stop_ || !queue_.empty(); });
            if (stop_ && queue_.empty()) return;
            t = queue_.front();
            queue_.pop_front();
        }
        decode_chunk(t);
        {
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_cv_.notify_all();
        }
    }
}

}  // namespace ph0b
