// Host-side decoder of the compressed D stream (d2h_codec.cu): a small pool of threads that
// prefix-sum 32-bit deltas back into the 64-bit patterns of D, writing the caller's buffer
// with non-temporal stores.  Internal header.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

namespace ph0b {

// A run of consecutive chunks of one bucket: chunk j covers values [j*chunk, ...) of
// deltas/out; raw chunks (shipped uncompressed) are skipped.
struct DecodeTask {
    const uint32_t* deltas;  // [n] (each chunk's first entry unused)
    const uint64_t* bases;   // [nchunks] pattern of each chunk's first value
    const uint8_t* raw;      // [nchunks] 1 = chunk shipped raw
    uint64_t* out;           // [n]
    uint64_t n;              // values covered
    uint32_t chunk;          // values per chunk
};

class DecodePool {
public:
    explicit DecodePool(unsigned threads);
    ~DecodePool();
    void submit(const std::vector<DecodeTask>& tasks);
    void wait();  // until every submitted task is done
    unsigned threads() const { return (unsigned)workers_.size(); }

private:
    void run();
    std::vector<std::thread> workers_;
    std::deque<DecodeTask> queue_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    uint64_t pending_ = 0;
    bool stop_ = false;
};

void decode_chunk(const DecodeTask& t);

}  // namespace ph0b
