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
  const uint64_t s = lo < a.n ? lo : a.n - 1;
  a.out.xm[k] = a.bank.xm[s];
  const double2 wt = a.bank.wt[s];
  a.out.wt[k] = make_double2(spacing, wt.y);
  const uint4 m = a.bank.meta[s];
  // fresh identity for the new step: history = tooth index, key 0, draw 0
  a.out.meta[k] = make_uint4(m.x & 0xffffu, (unsigned)k, 0u, 0u);
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
