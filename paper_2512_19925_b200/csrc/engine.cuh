// Pieces shared by the segment API (engine.cu) and the driver (driver.cu).
#pragma once

#include <cstdlib>

#include "device_state.cuh"
#include "transport.cuh"

namespace hwwg {

int bit_length(unsigned long long v);

// Arena of the history-parallel exact path's tally log (transport.cuh ExactLog).
// blocks[0] is the per-segment block allocator, blocks[1] the largest demand
// seen since reset_need() (overflowing histories record it), so a step that
// overflowed replays once with an arena of the right size.
struct ExactLogBuf {
  DevBuf<unsigned> slot, next, first, count;
  DevBuf<double> val;
  DevBuf<unsigned long long> blocks;
  unsigned long long cap = 0;
  bool off = std::getenv("HWWG_EXACT_CHUNKS") != nullptr;  // diagnostic: chunk-serial kernel
  void reset_need(cudaStream_t s) {
    blocks.reserve(2);
    HWWG_CUDA(cudaMemsetAsync(blocks.p, 0, 2 * sizeof(unsigned long long), s));
  }
  void ensure_blocks(unsigned long long want) {
    want = std::min<unsigned long long>(want, 0xfffffff0ULL);
    if (want <= cap) return;
    slot.reserve(want * kLogBlock);
    val.reserve(want * kLogBlock);
    next.reserve(want);
    cap = want;
  }
  // The demand recorded by overflowing histories (synchronous read).
  unsigned long long need(cudaStream_t s) {
    unsigned long long v = 0;
    HWWG_CUDA(cudaMemcpyAsync(&v, blocks.p + 1, sizeof v, cudaMemcpyDeviceToHost, s));
    HWWG_CUDA(cudaStreamSynchronize(s));
    return v;
  }
  ExactLog view(uint64_t n) {
    ExactLog L{};
    if (off || n == 0) return L;
    blocks.reserve(2);
    ensure_blocks(std::max<unsigned long long>(65536, 4 * (unsigned long long)n));
    first.reserve(n);
    count.reserve(n);
    L.slot = slot.p;
    L.val = val.p;
    L.next = next.p;
    L.first = first.p;
    L.count = count.p;
    L.blocks = blocks.p;
    L.cap_blocks = cap;
    return L;
  }
};

// Census staging: records appended with (history << 24 | emission) keys, then
// radix-sorted into the reference's history-major depth-first order.
struct CensusStage {
  DevBuf<hwwg_particle> records;
  DevBuf<unsigned long long> keys, keys_alt;
  DevBuf<unsigned> idx, idx_alt;
  DevBuf<char> temp;
  size_t temp_bytes = 0;
  void ensure(uint64_t cap);
  void sort_into(hwwg_particle* out, uint64_t n, unsigned long long max_key, cudaStream_t s);
};

}  // namespace hwwg
