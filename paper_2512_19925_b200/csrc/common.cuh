// Shared device-side data layout of the hwwg engine.
//
// HBM layout:
//   * per-cell table CellInfo[I] (48 B: sigma_t, sigma_s, sigma_f, nu_f, speed,
//     1/dx) + edges[I+1]: read-only, L1/L2 resident (<= 200 KB at I = 4000);
//   * tally slab: one contiguous fp64 block (TallyPtrs views into it) so a
//     step's tallies reset with one memset and reduce with one collective;
//   * particle banks: AoS hwwg_particle (32 B) in exact mode — the comb and the
//     drop-in boundary speak the reference's AoS Particle — and SoA 48 B
//     records (double2 {x,mu}, double2 {w,t}, uint4 {cell,hist,key,ctr}) in
//     the event-based Philox mode.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <string>

#include "capi_util.h"
#include "hwwg.h"

namespace hwwg {

struct CellInfo {
  double sigma_t, sigma_s, sigma_f, nu_f, speed, inv_dx;
  double inv_sigma_t, inv_speed, inv_sigma_s;  // throughput mode only (exact mode divides)
};

// Views into the device tally slab (== hww::TallySet, tally.hpp:16-45).
struct TallyPtrs {
  double* track_flux;           // I
  double* track_flux_batch;     // B*I
  double* census_phi;           // I
  double* census_current;       // I
  double* census_closure;       // I
  double* census_weight_batch;  // B
  double* edge_current;         // I+1
  double* boundary_closure;     // 2: left, right
  unsigned long long* tracks;   // I   (tracks_per_cell)
  unsigned long long* ucount;   // 11: 9 StepCounters u64 + histories_scored + grazing_discarded
  double* dcount;               // 2: leakage_weight, aborted_weight
};

enum UCounter {
  kCollisions = 0,
  kSplits,
  kSplitDaughters,
  kCappedSplits,
  kRouletteKills,
  kRouletteSurvivals,
  kCensusCount,
  kEventCapAborts,
  kNanAborts,
  kHistoriesScored,
  kGrazingDiscarded,
  kNumUCounters
};

// Mesh + materials as the kernels see them.
struct MeshView {
  const double* edges;
  const CellInfo* cells;
  int I;
  int uniform;
  double x_min, x_max, w0;
};

// Device error record: first failing history and its code.
struct DevError {
  int code;  // 0 ok, HWWG_EINVAL, HWWG_ESTACK
  int pad;
  unsigned long long history;
};

#define HWWG_CUDA(call)                                                                \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      throw ::hwwg::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_));     \
  } while (0)

// Device-side bounds checks of the builds with -DHWWG_CHECKS
// (_build_checked/, tests/test_gpu_checked.py): a failed check prints its
// site and traps, which fails the launch. compute-sanitizer is not available
// on the GPU pool, so these stand in for memcheck on the indices that matter.
#ifdef HWWG_CHECKS
#define HWWG_CHECK(cond)                                                               \
  do {                                                                                 \
    if (!(cond)) {                                                                     \
      printf("HWWG_CHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__,  \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                             \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
#else
#define HWWG_CHECK(cond) \
  do {                   \
  } while (0)
#endif

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device setting: the
// size configured so far is cached per device ordinal (a process may drive
// several GPUs), under a lock (loopback ranks are host threads).
constexpr int kMaxDevices = 64;
struct DynSmemCache {
  size_t size[kMaxDevices] = {};
};
template <class Kernel>
inline void ensure_dyn_smem(Kernel k, size_t smem, DynSmemCache& cache) {
  static std::mutex m;
  int dev = 0;
  HWWG_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  std::lock_guard<std::mutex> lk(m);
  if (smem <= cache.size[dev]) return;
  HWWG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cache.size[dev] = smem;
}

// mesh.cpp:26-40 on the device: uniform fast path with +-1 guards, else
// upper_bound; -1 when x lies outside [x_min, x_max].
__device__ __forceinline__ int locate_cell(const MeshView& m, double x) {
  if (x < m.x_min || x > m.x_max) return -1;
  if (x == m.x_max) return m.I - 1;
  if (m.uniform) {
    int c = (int)__ddiv_rn(__dsub_rn(x, m.x_min), m.w0);
    if (c >= m.I) c = m.I - 1;
    if (x < m.edges[c]) --c;
    else if (x >= m.edges[c + 1]) ++c;
    return c;
  }
  int a = 0, b = m.I + 1;
  while (a < b) {
    const int mid = (a + b) >> 1;
    if (m.edges[mid] > x) b = mid;
    else a = mid + 1;
  }
  return a - 1;
}

// tally.hpp:130-134
__device__ __forceinline__ int batch_of(uint64_t h, uint64_t H, int B) {
  if (H == 0) return 0;
  const int b = (int)(h * (uint64_t)B / H);
  return b < B ? b : B - 1;
}

// Warp-aggregated reservation of one slot per calling lane on a global
// counter: one atomic per group of converged lanes instead of one per lane.
__device__ __forceinline__ unsigned long long warp_reserve1(unsigned long long* ctr) {
  const unsigned mask = __activemask();
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(mask) - 1;
  const unsigned rank = __popc(mask & ((1u << lane) - 1u));
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(ctr, (unsigned long long)__popc(mask));
  base = __shfl_sync(mask, base, leader);
  return base + rank;
}

}  // namespace hwwg
