// Host-side decoder of the compressed D stream (d2h_codec.cu): a small pool of threads that
// prefix-sum 32-bit deltas back into the 64-bit patterns of D, writing the caller's buffer
// with non-temporal stores.  Internal header.
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

namespace ph0b {

// A run of consecutive chunks of one bucket: chunk j covers values [j*chunk, ...) of
// deltas/out; raw chunks (shipped uncompressed) are skipped.
//
// Streamed pieces (`ready` set): the deltas sit in a slot of the pinned staging ring, which
// the copy engine fills and then flags by writing `gen` into *ready (a stream memory
// operation after the copy).  The worker spins until *ready == gen, decodes, and hands the
// slot back with *freed = gen (the copy engine's next fill of that slot waits for it).  The
// value range is only known on the device when the piece is enqueued: it is resolved from
// the bucket's published D bounds (`bounds[0..1]`, mapped host words) at decode time as
// values [v0, min(v0 + n, hi - lo)) of the bucket, written to out_base + lo + v0.
struct DecodeTask {
    const uint32_t* deltas;  // [n] (each chunk's first entry unused)
    const uint64_t* bases;   // [nchunks] pattern of each chunk's first value
    const uint8_t* raw;      // [nchunks] 1 = chunk shipped raw
    uint64_t* out;           // [n] (streamed pieces: out_base)
    uint64_t n;              // values covered (streamed pieces: upper bound)
    uint32_t chunk;          // values per chunk
    const volatile uint32_t* ready = nullptr;
    volatile uint32_t* freed = nullptr;
    uint32_t gen = 0;
    const volatile uint64_t* bounds = nullptr;
    uint64_t v0 = 0;
    uint64_t capacity = 0;   // entries of out_base
    volatile int* overflow = nullptr;  // set when lo + v1 > capacity (nothing written)
    // a piece is decoded by `nsub` tasks (sub-ranges of its chunks); the slot's monotone
    // completion counter reaches gen * nsub when the last one finishes, which frees the slot
    std::atomic<uint64_t>* done = nullptr;
    uint32_t nsub = 1;
    // packed chunks (widths != null): chunk j's deltas are widths[j] bytes each (3 or 4; 0 =
    // raw, skipped) at packed + poff[j]; `deltas` and `raw` are unused
    const uint8_t* widths = nullptr;
    const uint32_t* poff = nullptr;
    const uint8_t* packed = nullptr;
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
// A streamed piece: wait for its slot, decode the resolved range, release the slot.
void decode_piece(const DecodeTask& t);
// diagnostics (PH0B_TRACE): summed wait-for-slot and decode times of streamed pieces
void decode_stats(uint64_t* wait_ns, uint64_t* decode_ns, uint64_t* pieces, bool reset);

}  // namespace ph0b
