// Host decoder of the compressed D stream; see host_decode.h and d2h_codec.cu.
#include "host_decode.h"

#include <immintrin.h>
#include <sys/resource.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>

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

// 8 values per step: widen 8 deltas to u64, in-register prefix sum (3 lane shifts), add the
// running value, one 64-byte non-temporal store.
__attribute__((target("avx512f"))) void decode_avx512(const Chunk& t) {
    uint64_t acc = t.base;
    uint64_t* out = t.out;
    const uint32_t* d = t.deltas;
    out[0] = acc;
    uint32_t i = 1;
    while (i < t.len && (reinterpret_cast<uintptr_t>(out + i) & 63u)) {
        acc += d[i];
        out[i++] = acc;
    }
    if (i + 8 <= t.len) {
        const __m512i z = _mm512_setzero_si512();
        const __m512i last = _mm512_set1_epi64(7);
        __m512i run = _mm512_set1_epi64((long long)acc);
        for (; i + 8 <= t.len; i += 8) {
            __m512i x = _mm512_cvtepu32_epi64(_mm256_loadu_si256(reinterpret_cast<const __m256i*>(d + i)));
            x = _mm512_add_epi64(x, _mm512_alignr_epi64(x, z, 7));
            x = _mm512_add_epi64(x, _mm512_alignr_epi64(x, z, 6));
            x = _mm512_add_epi64(x, _mm512_alignr_epi64(x, z, 4));
            x = _mm512_add_epi64(x, run);
            run = _mm512_permutexvar_epi64(last, x);
            _mm512_stream_si512(reinterpret_cast<__m512i*>(out + i), x);
        }
        acc = (uint64_t)_mm_cvtsi128_si64(_mm512_castsi512_si128(run));
    }
    for (; i < t.len; ++i) {
        acc += d[i];
        out[i] = acc;
    }
    _mm_sfence();
}

// 3-byte deltas (packed chunks): 8 per step, widened to 32-bit lanes with one byte permute,
// then the same prefix sum as decode_avx512.  Reads up to 8 bytes past the chunk's data
// (the ring slots carry slack).
inline uint32_t load24(const uint8_t* p) {
    uint32_t x;
    std::memcpy(&x, p, 4);
    return x & 0xFFFFFFu;
}

__attribute__((target("avx512f,avx512vl,avx512vbmi"))) void decode3_avx512(const uint8_t* d,
                                                                           uint64_t base,
                                                                           uint64_t* out,
                                                                           uint32_t len) {
    uint64_t acc = base;
    out[0] = acc;
    uint32_t i = 1;
    while (i < len && (reinterpret_cast<uintptr_t>(out + i) & 63u)) {
        acc += load24(d + 3 * i);
        out[i++] = acc;
    }
    if (i + 8 <= len) {
        const __m512i z = _mm512_setzero_si512();
        const __m512i last = _mm512_set1_epi64(7);
        const __m256i idx = _mm256_setr_epi8(0, 1, 2, 0, 3, 4, 5, 0, 6, 7, 8, 0, 9, 10, 11, 0, 12,
                                             13, 14, 0, 15, 16, 17, 0, 18, 19, 20, 0, 21, 22, 23, 0);
        const __m256i m24 = _mm256_set1_epi32(0xFFFFFF);
        __m512i run = _mm512_set1_epi64((long long)acc);
        for (; i + 8 <= len; i += 8) {
            const __m256i raw = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(d + 3 * i));
            const __m256i x32 = _mm256_and_si256(_mm256_permutexvar_epi8(idx, raw), m24);
            __m512i x = _mm512_cvtepu32_epi64(x32);
            x = _mm512_add_epi64(x, _mm512_alignr_epi64(x, z, 7));
            x = _mm512_add_epi64(x, _mm512_alignr_epi64(x, z, 6));
            x = _mm512_add_epi64(x, _mm512_alignr_epi64(x, z, 4));
            x = _mm512_add_epi64(x, run);
            run = _mm512_permutexvar_epi64(last, x);
            _mm512_stream_si512(reinterpret_cast<__m512i*>(out + i), x);
        }
        acc = (uint64_t)_mm_cvtsi128_si64(_mm512_castsi512_si128(run));
    }
    for (; i < len; ++i) {
        acc += load24(d + 3 * i);
        out[i] = acc;
    }
    _mm_sfence();
}

void decode3_scalar(const uint8_t* d, uint64_t base, uint64_t* out, uint32_t len) {
    uint64_t acc = base;
    out[0] = acc;
    for (uint32_t i = 1; i < len; ++i) {
        acc += load24(d + 3 * i);
        out[i] = acc;
    }
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
    static const int isa = __builtin_cpu_supports("avx512f") ? 2 : __builtin_cpu_supports("avx2") ? 1 : 0;
    static const bool vbmi = __builtin_cpu_supports("avx512vbmi") &&
                             __builtin_cpu_supports("avx512vl");
    if (t.widths) {  // packed chunks
        for (uint64_t j = 0, s0 = 0; s0 < t.n; ++j, s0 += t.chunk) {
            const uint32_t w = t.widths[j];
            if (w == 0) continue;
            const uint32_t len = (uint32_t)(t.n - s0 < t.chunk ? t.n - s0 : t.chunk);
            const uint8_t* src = t.packed + t.poff[j];
            if (w == 3) {
                if (vbmi)
                    decode3_avx512(src, t.bases[j], t.out + s0, len);
                else
                    decode3_scalar(src, t.bases[j], t.out + s0, len);
                continue;
            }
            const Chunk c{reinterpret_cast<const uint32_t*>(src), t.bases[j], t.out + s0, len};
            if (isa == 2)
                decode_avx512(c);
            else if (isa == 1)
                decode_avx2(c);
            else
                decode_scalar(c);
        }
        return;
    }
    for (uint64_t j = 0, s0 = 0; s0 < t.n; ++j, s0 += t.chunk) {
        if (t.raw[j]) continue;
        const Chunk c{t.deltas + s0, t.bases[j], t.out + s0,
                      (uint32_t)(t.n - s0 < t.chunk ? t.n - s0 : t.chunk)};
        if (isa == 2)
            decode_avx512(c);
        else if (isa == 1)
            decode_avx2(c);
        else
            decode_scalar(c);
    }
}

std::atomic<uint64_t> g_wait_ns{0}, g_decode_ns{0}, g_pieces{0};

void decode_stats(uint64_t* wait_ns, uint64_t* decode_ns, uint64_t* pieces, bool reset) {
    *wait_ns = g_wait_ns.load();
    *decode_ns = g_decode_ns.load();
    *pieces = g_pieces.load();
    if (reset) {
        g_wait_ns = 0;
        g_decode_ns = 0;
        g_pieces = 0;
    }
}

void decode_piece(const DecodeTask& t) {
    const auto t0 = std::chrono::steady_clock::now();
    // the copy engine flags the slot after the piece (and, earlier in the same stream, the
    // bucket's chunk bases and raw flags) has landed
    std::chrono::steady_clock::time_point deadline{};
    for (uint32_t spins = 0; __atomic_load_n(t.ready, __ATOMIC_ACQUIRE) != t.gen; ++spins) {
        if (spins < 4096) {
            _mm_pause();
            continue;
        }
        std::this_thread::yield();
        if ((spins & 1023u) != 0) continue;
        const auto now = std::chrono::steady_clock::now();
        if (spins == 4096) {
            deadline = now + std::chrono::seconds(60);
        } else if (now > deadline) {  // the copy stream is dead (device fault): give up
            *t.overflow = 2;
            if (t.done->fetch_add(1) + 1 == (uint64_t)t.gen * t.nsub)
                __atomic_store_n(t.freed, t.gen, __ATOMIC_RELEASE);
            return;
        }
    }
    const auto t1 = std::chrono::steady_clock::now();
    const uint64_t lo = t.bounds[0], hi = t.bounds[1];
    const uint64_t nb = hi > lo ? hi - lo : 0;
    if (t.v0 < nb) {
        const uint64_t v1 = t.v0 + t.n < nb ? t.v0 + t.n : nb;
        if (lo + v1 > t.capacity) {
            *t.overflow = 1;
        } else {
            DecodeTask c = t;
            c.out = t.out + lo + t.v0;
            c.n = v1 - t.v0;
            decode_chunk(c);
        }
    }
    if (t.done->fetch_add(1, std::memory_order_acq_rel) + 1 == (uint64_t)t.gen * t.nsub)
        __atomic_store_n(t.freed, t.gen, __ATOMIC_RELEASE);
    const auto t2 = std::chrono::steady_clock::now();
    g_wait_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
    g_decode_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(t2 - t1).count();
    ++g_pieces;
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
        if (t.ready)
            decode_piece(t);
        else
            decode_chunk(t);
        {
            std::lock_guard<std::mutex> lk(mu_);
            if (--pending_ == 0) done_cv_.notify_all();
        }
    }
}

}  // namespace ph0b
