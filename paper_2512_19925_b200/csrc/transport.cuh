// Launch interfaces of the transport kernels (transport_exact.cu,
// transport_fast.cu).
#pragma once

#include "common.cuh"

namespace hwwg {

// The reference's OpenMP chunk (run_segment_parallel's default chunk_size,
// proj/include/hww/transport.hpp:117-120).
constexpr int kChunk = 256;

// Chunk-private TallySets of one exact-mode segment: per chunk `stride`
// doubles = track I | census phi,J,F 3I | edge I+1 | bclosure 2 | leak,aborted 2
// | census_weight_batch B | track_flux_batch span*I (batches b0..b0+span-1).
struct ChunkLayout {
  double* base;
  size_t stride;
  int count;
  int span;
};
ChunkLayout chunk_layout(uint64_t n, uint64_t h_begin, uint64_t H, int I, int B);

// Tally log of the history-parallel exact path: every history (one thread)
// appends its fp64 contributions (chunk-layout slot, value) in event order to
// its own chain of kLogBlock-entry blocks; a replay kernel then adds each
// chunk's entries in history and event order — the reference's chunk-
// sequential summation — so the physics runs one thread per history instead
// of one per 256-history chunk.
constexpr int kLogBlock = 32;
constexpr int kLogOverflow = -100;  // DevError code: the arena was too small (replay)
struct ExactLog {
  unsigned* slot;                 // cap_blocks * kLogBlock
  double* val;                    // cap_blocks * kLogBlock
  unsigned* next;                 // cap_blocks: next block of the same history
  unsigned* first;                // per history: first block (or ~0u)
  unsigned* count;                // per history: entries
  unsigned long long* blocks;     // allocated blocks (zeroed per segment)
  unsigned long long cap_blocks;
};

// One exact-mode segment: histories [h_begin, h_begin + n) of a step.
struct ExactArgs {
  const hwwg_particle* src;  // n source particles (AoS, device)
  uint64_t n;
  unsigned long long h_begin;
  MeshView mesh;
  double t_begin, t_end, inv_dt;
  uint64_t seed;
  uint64_t step;
  uint64_t H;  // histories_total (batch assignment)
  int B;
  const double* centers;  // NULL: analog
  const int* active;      // optional device flag gating the windows (lww/hww)
  double rho;
  TallyPtrs t;            // running tallies (accumulated in reference order)
  ChunkLayout chunks;
  hwwg_particle* census;            // staging records
  unsigned long long* census_keys;  // history << 24 | emission index
  unsigned long long* census_count;
  uint64_t census_cap;
  DevError* err;
  ExactLog log;  // slot == null: the chunk-serial kernel
};

void launch_exact_segment(const ExactArgs& a, cudaStream_t s);
// Whether a segment with this chunk layout takes the history-parallel path
// (the chunk accumulators of one chunk fit a warp's shared memory).

struct CensusSortArgs {
  const hwwg_particle* records;
  unsigned long long* keys_in;
  unsigned long long* keys_out;
  unsigned* idx_in;
  unsigned* idx_out;
  hwwg_particle* out;
  uint64_t n;
  int begin_bit, end_bit;
  void* temp;
  size_t temp_bytes;
};

size_t census_sort_temp_bytes(uint64_t n);
void sort_census(const CensusSortArgs& a, cudaStream_t s);

}  // namespace hwwg
