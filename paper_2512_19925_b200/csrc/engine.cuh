// Pieces shared by the segment API (engine.cu) and the driver (driver.cu).
#pragma once

#include "device_state.cuh"

namespace hwwg {

int bit_length(unsigned long long v);

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
