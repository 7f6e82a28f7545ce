// Exact-mode history kernel: bit-exact replay of hww::advance_history
// (proj/src/transport.cpp:81-192) on sm_100a, one history per thread.
//
// Why one history per thread: the reference's daughters share their parent
// history's flight/window streams and run depth-first on a LIFO stack
// (transport.cpp:100-107, 199-202), so a history's event sequence is
// inherently serial. The stack is run-length encoded: a split pushes its
// n-1 identical copies as ONE run (entry, n-1) (transport.cpp:65-66), so the
// pop order is the reference's while storage is O(split events) — measured
// depth <= 9 runs on BASELINE configs 1/2/4/5 (oracle diagnostics), 64 here.
//
// Arithmetic parity: this translation unit is compiled with -fmad=false (no
// FMA contraction, like the reference's x86-64 baseline build), divisions are
// IEEE div.rn, and log is the bit-exact libm replay in libm_log.h. Census
// records are appended with a (history << 24 | emission index) key and sorted
// afterwards, which restores the reference's history-major, depth-first order
// (transport.cpp:146, 233-236).
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "rng.cuh"
#include "transport.cuh"

namespace hwwg {

namespace {

constexpr int kMaxRuns = 64;
constexpr uint64_t kMaxEventsPerHistory = 1000000ULL;  // transport.hpp:97
constexpr double kMaxSplitDaughters = 1000000.0;        // ww.hpp:53
constexpr double kGrazingMu = 1e-10;                    // tally.hpp:48

struct Run {
  double x, mu, w, t;
  int cell;
  unsigned count;
};

struct Local {
  unsigned long long u[kNumUCounters];
  double leak, aborted;
};

__device__ __forceinline__ void set_error(DevError* e, int code, unsigned long long h) {
  if (atomicCAS(&e->code, 0, code) == 0) e->history = h;
}

struct History {
  const ExactArgs& a;
  Local& c;
  Run* stk;
  int sp;
  Xoshiro flight, win;
  unsigned long long h;

  __device__ __forceinline__ bool push(double x, double mu, double w, double t, int cell,
                                       unsigned count) {
    if (sp == kMaxRuns) {
      set_error(a.err, HWWG_ESTACK, h);
      return false;
    }
    stk[sp] = Run{x, mu, w, t, cell, count};
    ++sp;
    return true;
  }

  // ww.cpp:46-72 + transport.cpp:54-77 applied in place; false = particle dies.
  __device__ __forceinline__ bool window_game(double x, double mu, double& w, double t,
                                              int cell) {
    const double center = a.centers[cell];
    const double floor_ = center / a.rho;
    const double ceil_ = center * a.rho;
    if (w > ceil_) {
      double n = ceil(w / center);
      if (n > kMaxSplitDaughters) {
        n = kMaxSplitDaughters;
        ++c.u[kCappedSplits];
      }
      const int daughters = (int)n;
      ++c.u[kSplits];
      c.u[kSplitDaughters] += (unsigned long long)(daughters - 1);
      w = w / n;
      if (daughters > 1 && !push(x, mu, w, t, cell, (unsigned)(daughters - 1))) {
        sp = 0;
        return false;
      }
      return true;
    }
    if (w < floor_) {
      const double survival = w / center;
      if (win.uniform() < survival) {
        ++c.u[kRouletteSurvivals];
        w = center;
        return true;
      }
      ++c.u[kRouletteKills];
      return false;
    }
    return true;
  }
};

__device__ void run_history(const ExactArgs& a, uint64_t i, Local& c, Run* stk) {
  const unsigned long long h = a.h_begin + i;
  const double2 s0 = reinterpret_cast<const double2*>(a.src)[2 * i];
  const double2 s1 = reinterpret_cast<const double2*>(a.src)[2 * i + 1];
  // transport.cpp:91-98
  if (!isfinite(s0.x) || !isfinite(s1.x) || s1.x <= 0.0) {
    ++c.u[kNanAborts];
    return;
  }
  const int start_cell = locate_cell(a.mesh, s0.x);
  if (start_cell < 0 || !(s1.y >= a.t_begin && s1.y < a.t_end)) {
    set_error(a.err, HWWG_EINVAL, h);
    return;
  }

  History hs{a, c, stk, 0, {}, {}, h};
  hs.flight.seed(a.seed, stream_id(a.step, h, kFlight));  // transport.cpp:199-202
  hs.win.seed(a.seed, stream_id(a.step, h, kWindow));
  const int batch = batch_of(h, a.H, a.B);
  const bool windows = a.centers != nullptr && (a.active == nullptr || *a.active != 0);
  const int I = a.mesh.I;
  const double* edges = a.mesh.edges;
  const TallyPtrs& T = a.t;

  hs.push(s0.x, s0.y, s1.x, s1.y, start_cell, 1u);
  unsigned long long events = 0;
  unsigned seq = 0;

  while (hs.sp > 0) {
    Run& top = stk[hs.sp - 1];
    double x = top.x, mu = top.mu, w = top.w, t = top.t;
    int cell = top.cell;
    if (--top.count == 0) --hs.sp;

    bool alive = true;
    while (alive) {
      if (++events > kMaxEventsPerHistory) {  // transport.cpp:111-118
        ++c.u[kEventCapAborts];
        c.aborted += w;
        for (int r = 0; r < hs.sp; ++r)
          for (unsigned j = 0; j < stk[r].count; ++j) c.aborted += stk[r].w;
        hs.sp = 0;
        break;
      }
      const CellInfo ci = a.mesh.cells[cell];
      const double d_census = ci.speed * (a.t_end - t);
      const double d_collision = -hwwg_libm_log(hs.flight.uniform()) / ci.sigma_t;
      double d_boundary = __longlong_as_double(0x7ff0000000000000LL);
      int edge = -1;
      if (mu > 0.0) {
        edge = cell + 1;
        d_boundary = (edges[edge] - x) / mu;
      } else if (mu < 0.0) {
        edge = cell;
        d_boundary = (edges[edge] - x) / mu;
      }
      double d = d_census;  // std::min({...}) keeps the first smallest
      if (d_collision < d) d = d_collision;
      if (d_boundary < d) d = d_boundary;

      if (d > 0.0) {  // score_track, tally.hpp:51-56
        const double sc = w * d * (ci.inv_dx * a.inv_dt);
        atomicAdd(&T.track_flux[cell], sc);
        atomicAdd(&T.track_flux_batch[(size_t)batch * I + cell], sc);
        atomicAdd(&T.tracks[cell], 1ULL);
      }

      if (d == d_census) {  // transport.cpp:141-149
        x += d * mu;
        t = a.t_end;
        const double base = ci.speed * w * ci.inv_dx;  // score_census, tally.hpp:65-72
        atomicAdd(&T.census_phi[cell], base);
        atomicAdd(&T.census_current[cell], base * mu);
        atomicAdd(&T.census_closure[cell], base * (1.0 / 3.0 - mu * mu));
        atomicAdd(&T.census_weight_batch[batch], w);
        ++c.u[kCensusCount];
        const unsigned long long slot = warp_reserve1(a.census_count);
        if (slot < a.census_cap) {
          double2* dst = reinterpret_cast<double2*>(a.census) + 2 * slot;
          dst[0] = make_double2(x, mu);
          dst[1] = make_double2(w, t);
          a.census_keys[slot] = (h << 24) | seq;
        }
        ++seq;
        alive = false;
        continue;
      }

      if (d == d_boundary) {  // transport.cpp:151-164
        x = edges[edge];
        t += d / ci.speed;
        const bool domain = edge == 0 || edge == I;
        atomicAdd(&T.edge_current[edge], (mu > 0 ? w : -w) * a.inv_dt);  // tally.hpp:77-92
        if (domain) {
          const double amu = mu > 0 ? mu : -mu;
          if (amu < kGrazingMu) {
            ++c.u[kGrazingDiscarded];
          } else {
            atomicAdd(&T.boundary_closure[edge == 0 ? 0 : 1], w * (0.5 - amu) / amu * a.inv_dt);
          }
          c.leak += w;
          alive = false;
          continue;
        }
        cell += mu > 0.0 ? 1 : -1;
        if (windows) alive = hs.window_game(x, mu, w, t, cell);
        continue;
      }

      // collision, transport.cpp:166-190; sample_collision :29-40
      x += d * mu;
      t += d / ci.speed;
      ++c.u[kCollisions];
      const double xi = hs.flight.uniform() * ci.sigma_t;
      if (xi < ci.sigma_s) {
        mu = hs.flight.uniform_pm1();
        if (windows) alive = hs.window_game(x, mu, w, t, cell);
      } else if (xi < ci.sigma_s + ci.sigma_f) {
        const double fl = floor(ci.nu_f);
        const double frac = ci.nu_f - fl;
        int ns = (int)fl;
        if (frac > 0.0 && hs.flight.uniform() < frac) ++ns;
        for (int s = 0; s < ns; ++s) {
          double ws = w;
          const double mus = hs.flight.uniform_pm1();
          if (!windows || hs.window_game(x, mus, ws, t, cell)) {
            if (!hs.push(x, mus, ws, t, cell, 1u)) {
              hs.sp = 0;
              break;
            }
          }
        }
        alive = false;
      } else {
        alive = false;
      }
    }
  }
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(128) k_exact_histories(ExactArgs a) {
  Run stk[kMaxRuns];
  Local c;
#pragma unroll
  for (int k = 0; k < kNumUCounters; ++k) c.u[k] = 0;
  c.leak = 0.0;
  c.aborted = 0.0;
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < a.n) run_history(a, i, c, stk);
  __syncwarp();
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < kNumUCounters; ++k) {
    const unsigned long long v = warp_sum_u64(c.u[k]);
    if (lane == 0 && v) atomicAdd(&a.t.ucount[k], v);
  }
  const double leak = warp_sum_f64(c.leak);
  const double ab = warp_sum_f64(c.aborted);
  if (lane == 0) {
    if (leak != 0.0) atomicAdd(&a.t.dcount[0], leak);
    if (ab != 0.0) atomicAdd(&a.t.dcount[1], ab);
  }
}

__global__ void k_iota(unsigned* v, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (unsigned)i;
}

__global__ void k_gather(const hwwg_particle* __restrict__ src, const unsigned* __restrict__ idx,
                         hwwg_particle* __restrict__ dst, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const double2* s = reinterpret_cast<const double2*>(src) + 2 * (uint64_t)idx[i];
    double2* d = reinterpret_cast<double2*>(dst) + 2 * i;
    d[0] = s[0];
    d[1] = s[1];
  }
}

}  // namespace

void launch_exact_segment(const ExactArgs& a, cudaStream_t s) {
  if (a.n == 0) return;
  const unsigned threads = 128;
  const uint64_t blocks = (a.n + threads - 1) / threads;
  k_exact_histories<<<(unsigned)blocks, threads, 0, s>>>(a);
  HWWG_CUDA(cudaGetLastError());
}

size_t census_sort_temp_bytes(uint64_t n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (const unsigned*)nullptr,
                                  (unsigned*)nullptr, (int)n, 0, 64);
  return bytes;
}

void sort_census(const CensusSortArgs& a, cudaStream_t s) {
  if (a.n == 0) return;
  const unsigned threads = 256;
  const unsigned blocks = (unsigned)((a.n + threads - 1) / threads);
  k_iota<<<blocks, threads, 0, s>>>(a.idx_in, a.n);
  size_t bytes = a.temp_bytes;
  HWWG_CUDA(cub::DeviceRadixSort::SortPairs(a.temp, bytes, a.keys_in, a.keys_out, a.idx_in,
                                            a.idx_out, (int)a.n, a.begin_bit, a.end_bit, s));
  k_gather<<<blocks, threads, 0, s>>>(a.records, a.idx_out, a.out, a.n);
  HWWG_CUDA(cudaGetLastError());
}

}  // namespace hwwg
