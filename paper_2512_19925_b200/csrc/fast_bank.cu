// Throughput-mode bank kernels: the parallel comb (population control at step
// start, proj/src/popctrl.cpp:7-42) and bank format conversions.
//
// The comb keeps the reference's estimator — teeth spaced W/target apart with
// one random offset walk the cumulative-weight axis of the bank — but the
// cumulative weights come from a parallel fp64 scan (CUB decoupled look-back,
// deterministic for a given bank order) instead of a serial walk, and each
// tooth finds its particle by binary search. Teeth land in bank order, so the
// new source stays grouped by parent history.
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "fast.cuh"
#include "rng.cuh"

namespace hwwg {

namespace {

__global__ void k_extract_w(FastBank b, uint64_t n, double* w) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) w[i] = b.wt[i].x;
}

__global__ void k_comb_scalars(const double* prefix, uint64_t n, uint64_t target, uint64_t seed,
                               uint64_t stream, double* sc) {
  const double W = prefix[n - 1];
  const double spacing = W / (double)target;
  Xoshiro r;
  r.seed(seed, stream);
  sc[0] = W;
  sc[1] = spacing;
  sc[2] = r.uniform() * spacing;
  sc[3] = spacing * (double)target;
}

__global__ void k_comb_teeth(FastCombArgs a) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= a.target) return;
  const double spacing = a.scalars[1];
  const double T = a.scalars[2] + (double)k * spacing;
  uint64_t lo = 0, hi = a.n;  // first index with T < prefix[idx]
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (T < a.prefix[mid]) hi = mid;
    else lo = mid + 1;
  }
  uint64_t s = lo < a.n ? lo : a.n - 1;
  // a tooth stranded by round-off copies the last real particle (popctrl.cpp:31-37),
  // skipping the zero-weight holes at the tail of census chunks
  if (lo >= a.n)
    while (s > 0 && a.bank.wt[s].x <= 0.0) --s;
  a.out.xm[k] = a.bank.xm[s];
  const double2 wt = a.bank.wt[s];
  a.out.wt[k] = make_double2(spacing, wt.y);
  const uint4 m = a.bank.meta[s];
  // fresh identity for the new step: history = tooth index, key 0, draw 0
  a.out.meta[k] = make_uint4(m.x & 0xffffu, (unsigned)k, 0u, 0u);
}

__global__ void k_local_total(const double* prefix, uint64_t n, double* sc) {
  sc[0] = n ? prefix[n - 1] : 0.0;
}

__global__ void k_comb_teeth_range(FastCombArgs a, double spacing, double offset, double origin,
                                   uint64_t k_lo, uint64_t k_hi, FastBank out) {
  const uint64_t k = k_lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= k_hi) return;
  const double T = offset + (double)k * spacing;
  uint64_t lo = 0, hi = a.n;  // first local particle with T < origin + prefix
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (T < origin + a.prefix[mid]) hi = mid;
    else lo = mid + 1;
  }
  uint64_t s = lo < a.n ? lo : a.n - 1;
  if (lo >= a.n)
    while (s > 0 && a.bank.wt[s].x <= 0.0) --s;
  const uint64_t o = k - k_lo;
  out.xm[o] = a.bank.xm[s];
  out.wt[o] = make_double2(spacing, a.bank.wt[s].y);
  out.meta[o] = make_uint4(a.bank.meta[s].x & 0xffffu, (unsigned)k, 0u, 0u);
}

__global__ void k_fill_holes(FastBank c, uint64_t cap, const unsigned long long* cur, int warps,
                             double x_fill, double t_fill) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= warps) return;
  const unsigned long long end = cur[2 * w + 1] < cap ? cur[2 * w + 1] : cap;
  for (unsigned long long s = cur[2 * w]; s < end; ++s) {
    c.xm[s] = make_double2(x_fill, 0.5);
    c.wt[s] = make_double2(0.0, t_fill);
    c.meta[s] = make_uint4(0u, 0u, 0u, 0u);
  }
}

// Drop zero-weight holes while converting to AoS (order is free in this mode).
__global__ void k_compact_aos(FastBank in, uint64_t n, hwwg_particle* out,
                              unsigned long long* count) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool keep = i < n && in.wt[i].x > 0.0;
  const unsigned mask = __ballot_sync(0xffffffffu, keep);
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == 0 && mask) base = atomicAdd(count, (unsigned long long)__popc(mask));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (keep) {
    const unsigned long long j = base + __popc(mask & ((1u << lane) - 1u));
    double2* o = reinterpret_cast<double2*>(out) + 2 * j;
    o[0] = in.xm[i];
    o[1] = in.wt[i];
  }
}

__global__ void k_track_from_batches(TallyPtrs t, int I, int B) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= I) return;
  double s = 0.0;
  for (int b = 0; b < B; ++b) s += t.track_flux_batch[(size_t)b * I + i];
  t.track_flux[i] = s;
}

__global__ void k_fast_to_aos(FastBank in, uint64_t n, hwwg_particle* out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2* o = reinterpret_cast<double2*>(out) + 2 * i;
  o[0] = in.xm[i];
  o[1] = in.wt[i];
}

}  // namespace

size_t fast_comb_temp_bytes(uint64_t n) {
  size_t bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, bytes, (const double*)nullptr, (double*)nullptr, (int)n);
  return bytes;
}

void launch_fast_comb(const FastCombArgs& a, cudaStream_t s) {
  const unsigned bn = (unsigned)((a.n + 255) / 256);
  k_extract_w<<<bn, 256, 0, s>>>(a.bank, a.n, a.prefix);
  size_t bytes = a.temp_bytes;
  HWWG_CUDA(cub::DeviceScan::InclusiveSum(a.temp, bytes, a.prefix, a.prefix, (int)a.n, s));
  k_comb_scalars<<<1, 1, 0, s>>>(a.prefix, a.n, a.target, a.seed, a.stream, a.scalars);
  k_comb_teeth<<<(unsigned)((a.target + 255) / 256), 256, 0, s>>>(a);
  HWWG_CUDA(cudaGetLastError());
}

void launch_fast_comb_local_scan(const FastCombArgs& a, cudaStream_t s) {
  if (a.n) {
    k_extract_w<<<(unsigned)((a.n + 255) / 256), 256, 0, s>>>(a.bank, a.n, a.prefix);
    size_t bytes = a.temp_bytes;
    HWWG_CUDA(cub::DeviceScan::InclusiveSum(a.temp, bytes, a.prefix, a.prefix, (int)a.n, s));
  }
  k_local_total<<<1, 1, 0, s>>>(a.prefix, a.n, a.scalars);
  HWWG_CUDA(cudaGetLastError());
}

void launch_fast_comb_teeth_range(const FastCombArgs& a, double spacing, double offset,
                                  double origin, uint64_t k_lo, uint64_t k_hi, FastBank out,
                                  cudaStream_t s) {
  const uint64_t n = k_hi - k_lo;
  if (!n || !a.n) return;
  k_comb_teeth_range<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, spacing, offset, origin,
                                                                 k_lo, k_hi, out);
  HWWG_CUDA(cudaGetLastError());
}

void launch_fill_census_holes(FastBank census, uint64_t cap, const unsigned long long* warp_cursor,
                              int warps, double x_fill, double t_fill, cudaStream_t s) {
  k_fill_holes<<<(warps + 127) / 128, 128, 0, s>>>(census, cap, warp_cursor, warps, x_fill, t_fill);
  HWWG_CUDA(cudaGetLastError());
}

void launch_fast_compact_aos(FastBank in, uint64_t n, hwwg_particle* out,
                             unsigned long long* count, cudaStream_t s) {
  HWWG_CUDA(cudaMemsetAsync(count, 0, sizeof(unsigned long long), s));
  if (!n) return;
  k_compact_aos<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(in, n, out, count);
  HWWG_CUDA(cudaGetLastError());
}

void launch_track_from_batches(TallyPtrs t, int I, int B, cudaStream_t s) {
  k_track_from_batches<<<(I + 255) / 256, 256, 0, s>>>(t, I, B);
  HWWG_CUDA(cudaGetLastError());
}

void launch_fast_to_aos(FastBank in, uint64_t n, hwwg_particle* out, cudaStream_t s) {
  if (!n) return;
  k_fast_to_aos<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(in, n, out);
  HWWG_CUDA(cudaGetLastError());
}

}  // namespace hwwg
