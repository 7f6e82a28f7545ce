// Launch interfaces of the transport kernels (see transport_exact.cu,
// transport_fast.cu).
#pragma once

#include "common.cuh"

namespace hwwg {

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
  TallyPtrs t;
  hwwg_particle* census;            // staging records
  unsigned long long* census_keys;  // history << 24 | emission index
  unsigned long long* census_count;
  uint64_t census_cap;
  DevError* err;
};

void launch_exact_segment(const ExactArgs& a, cudaStream_t s);

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
