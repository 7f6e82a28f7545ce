// Time-dependent discrete-ordinates (S_N) reference solver on the device
// (SURVEY.md §8(f4)): hww::sn_solve (proj/src/reference.cpp:151-233) and
// hww::compute_reference (reference.cpp:302-372), the deterministic reference
// the error diagnostics compare Monte Carlo steps against.
//
// The reference sweeps one direction at a time through every fine cell, per
// source iteration, per fine time step — at config 4 (20000 fine cells, 2000
// fine steps, S16) that is three minutes of host time. Here the whole solve is
// ONE persistent cooperative launch, one CTA per direction:
//
//   * sweep: the diamond-difference recurrence psi_{i+1} = (s_i dx + (|mu| -
//     h_i) psi_i) / (|mu| + h_i) is affine in psi_i, so a CTA splits its
//     direction's cells into per-thread runs, composes each run's affine map,
//     scans the maps across the block (warp shuffles + one smem pass), and
//     every thread then replays its run from its exact incoming flux with the
//     reference's own formula;
//   * reduce: after a grid barrier, each CTA forms phi = sum_k w_k psi_k for
//     its share of cells in the reference's direction order, and the residual
//     max|dphi| / max|phi| by atomicMax over non-negative doubles;
//   * projection: the CTA that owns a tally cell's fine cells projects the
//     layer (width-weighted) and accumulates the trapezoid interval averages in
//     the reference's order.
//
// Everything but the sweep's run-start fluxes (scan-composed, a few ulp) runs
// in the reference's arithmetic order with FMA contraction off (-fmad=false),
// so results match hww::compute_reference to ~1e-13 relative unless a step's
// residual sits on the 1e-9 tolerance (tests/test_gpu_sn.py).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "capi_util.h"
#include "common.cuh"
#include "device_state.cuh"
#include "driver_host.h"
#include "reference_io.h"
#include "sn.cuh"

namespace cg = cooperative_groups;

namespace hwwg {
namespace {

constexpr int kSnThreads = 1024;
constexpr int kSnWarps = kSnThreads / 32;
constexpr int kSnMaxOrder = 256;
constexpr unsigned kFull = 0xffffffffu;

struct SnArgs {
  int K, cells, steps;
  const double* mu;       // K
  const double* wq;       // K
  const double* dx;       // cells
  const double* speed;    // cells
  const double* sig_t;    // cells
  const double* sig_src;  // cells: sigma_s + nu_f * sigma_f
  const double* layers;   // steps+1
  const double* inc_left;
  const double* inc_right;
  const double* q_rows;
  const int* q_index;     // steps+1
  double* psi_a;          // K*cells: psi0 on entry
  double* psi_b;          // K*cells
  double* phi;            // cells
  double* phi_fine;       // (steps+1)*cells or null
  int* iterations;        // steps+1
  // projection
  int tally, sr, ratio;   // tally cells; fine cells per tally cell; fine steps per tally step
  const double* tally_w;  // tally widths (null: no projection)
  double* phi_layer;      // (steps/ratio+1)*tally
  double* phi_interval;   // (steps/ratio)*tally, zeroed
  double tol;
  int max_iter;
  unsigned long long* slots;  // [2][2]: max|dphi|, max|phi| by iteration parity
  int* err_step;              // 0: converged everywhere
  double* err_residual;
};

struct Affine {
  double a, b;  // psi_out = a * psi_in + b
};

// `first` then `second`
__device__ __forceinline__ Affine then(Affine first, Affine second) {
  return {second.a * first.a, second.a * first.b + second.b};
}

// exclusive scan of the threads' maps in thread order (identity for thread 0)
__device__ Affine block_exclusive_scan(Affine v, Affine* s_warp) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  Affine inc = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double pa = __shfl_up_sync(kFull, inc.a, off);
    const double pb = __shfl_up_sync(kFull, inc.b, off);
    if (lane >= off) inc = then(Affine{pa, pb}, inc);
  }
  if (lane == 31) s_warp[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    Affine w = lane < kSnWarps ? s_warp[lane] : Affine{1.0, 0.0};
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const double pa = __shfl_up_sync(kFull, w.a, off);
      const double pb = __shfl_up_sync(kFull, w.b, off);
      if (lane >= off) w = then(Affine{pa, pb}, w);
    }
    if (lane < kSnWarps) s_warp[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  const Affine warp_pre = wid > 0 ? s_warp[wid - 1] : Affine{1.0, 0.0};
  const double ea = __shfl_up_sync(kFull, inc.a, 1);
  const double eb = __shfl_up_sync(kFull, inc.b, 1);
  const Affine lane_pre = lane > 0 ? Affine{ea, eb} : Affine{1.0, 0.0};
  __syncthreads();  // s_warp is reused by the next sweep
  return then(warp_pre, lane_pre);
}

// One direction's sweep (moment_sweep's inner loops, reference.cpp:98-139):
// writes the cell-average angular flux of direction k into work.
__device__ void sweep(const SnArgs& a, int k, double mu, const double* prev, double* work,
                      double dt, const double* q, Affine* s_warp) {
  const int n = a.cells;
  const double amu = fabs(mu);
  const bool fwd = mu > 0.0;
  const double bnd = fwd ? a.inc_left[k] : a.inc_right[k];
  const int per = (n + kSnThreads - 1) / kSnThreads;
  const int j0 = min((int)threadIdx.x * per, n), j1 = min(j0 + per, n);
  const double* prow = prev + (size_t)k * n;
  double* wrow = work + (size_t)k * n;
  const double* phi = a.phi;
  // the reference's per-cell terms, same expressions
  auto terms = [&](int i, double& num, double& lin, double& den) {
    const double dx = a.dx[i];
    const double tau = 1.0 / (a.speed[i] * dt);
    const double sig_eff = a.sig_t[i] + tau;
    const double src = 0.5 * (a.sig_src[i] * phi[i] + (q ? q[i] : 0.0)) + tau * prow[i];
    num = src * dx;
    lin = amu - 0.5 * sig_eff * dx;
    den = amu + 0.5 * sig_eff * dx;
  };
  Affine acc{1.0, 0.0};
  for (int j = j0; j < j1; ++j) {
    const int i = fwd ? j : n - 1 - j;
    double num, lin, den;
    terms(i, num, lin, den);
    const double inv = 1.0 / den;
    acc = then(acc, Affine{lin * inv, num * inv});
  }
  const Affine pre = block_exclusive_scan(acc, s_warp);
  double psi = pre.a * bnd + pre.b;
  if (j0 == 0) psi = bnd;  // the boundary run starts from the incoming flux itself
  for (int j = j0; j < j1; ++j) {
    const int i = fwd ? j : n - 1 - j;
    double num, lin, den;
    terms(i, num, lin, den);
    const double next = (num + lin * psi) / den;
    wrow[i] = 0.5 * (psi + next);
    psi = next;
  }
}

__device__ __forceinline__ void owned_range(const SnArgs& a, int& c0, int& c1) {
  const long long G = gridDim.x, b = blockIdx.x;
  c0 = (int)((long long)a.tally * b / G);
  c1 = (int)((long long)a.tally * (b + 1) / G);
}

__device__ double block_max(double v, double* s_red) {
  for (int off = 16; off; off >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, off));
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double w = threadIdx.x < kSnWarps ? s_red[threadIdx.x] : 0.0;
    for (int off = 16; off; off >>= 1) w = fmax(w, __shfl_xor_sync(kFull, w, off));
    if (threadIdx.x == 0) s_red[0] = w;
  }
  __syncthreads();
  const double r = s_red[0];
  __syncthreads();
  return r;
}

// phi = sum_k w_k psi_k over this CTA's fine cells (sn_solve's phi_new loop,
// reference.cpp:196-201: k ascending from 0.0); with `resid`, the CTA's
// max|phi_new - phi| and max|phi_new| go to slots[0..1] by atomicMax.
__device__ void reduce_phi(const SnArgs& a, const double* psi, const double* s_w, bool resid,
                           unsigned long long* slot, double* fine_out, double* s_red) {
  int c0, c1;
  owned_range(a, c0, c1);
  const int f0 = c0 * a.sr, f1 = c1 * a.sr, n = a.cells;
  double dmax = 0.0, smax = 0.0;
  for (int f = f0 + threadIdx.x; f < f1; f += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < a.K; ++k) s += s_w[k] * psi[(size_t)k * n + f];
    if (resid) {
      dmax = fmax(dmax, fabs(s - a.phi[f]));
      smax = fmax(smax, fabs(s));
    }
    a.phi[f] = s;
    if (fine_out) fine_out[f] = s;
  }
  if (resid) {
    dmax = block_max(dmax, s_red);
    smax = block_max(smax, s_red);
    if (threadIdx.x == 0) {
      atomicMax(slot, (unsigned long long)__double_as_longlong(dmax));
      atomicMax(slot + 1, (unsigned long long)__double_as_longlong(smax));
    }
  }
}

// hww::project for fine layer m (reference.cpp:279-297): the tally cells whose
// fine cells this CTA reduced (call after a __syncthreads).
__device__ void project_layer(const SnArgs& a, int m) {
  if (!a.tally_w) return;
  int c0, c1;
  owned_range(a, c0, c1);
  const int steps = a.steps / a.ratio;
  const int step_right = m / a.ratio;
  const double half = 0.5 / a.ratio;
  const bool interior = (m % a.ratio) != 0;
  for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
    double v = 0.0;
    for (int f = c * a.sr; f < (c + 1) * a.sr; ++f) v += a.phi[f] * a.dx[f];
    v /= a.tally_w[c];
    if (!interior) a.phi_layer[(size_t)step_right * a.tally + c] = v;
    if (interior) {
      a.phi_interval[(size_t)step_right * a.tally + c] += v / a.ratio;
    } else {
      if (step_right >= 1) a.phi_interval[(size_t)(step_right - 1) * a.tally + c] += v * half;
      if (step_right < steps) a.phi_interval[(size_t)step_right * a.tally + c] += v * half;
    }
  }
}

__global__ void __launch_bounds__(kSnThreads, 1) k_sn_solve(SnArgs a) {
  __shared__ Affine s_warp[kSnWarps];
  __shared__ double s_red[kSnWarps];
  __shared__ double s_mu[kSnMaxOrder], s_w[kSnMaxOrder];
  cg::grid_group grid = cg::this_grid();
  for (int k = threadIdx.x; k < a.K; k += blockDim.x) {
    s_mu[k] = a.mu[k];
    s_w[k] = a.wq[k];
  }
  __syncthreads();
  const int n = a.cells;
  // layer 0: moments of psi0 (reference.cpp:174-189)
  reduce_phi(a, a.psi_a, s_w, false, nullptr, a.phi_fine, s_red);
  __syncthreads();
  project_layer(a, 0);
  grid.sync();

  double* prev = a.psi_a;
  double* work = a.psi_b;
  unsigned gi = 0;  // global residual-iteration count: slot parity
  for (int step = 1; step <= a.steps; ++step) {
    const double dt = a.layers[step] - a.layers[step - 1];
    const int qi = a.q_index ? a.q_index[step] : -1;
    const double* q = qi >= 0 ? a.q_rows + (size_t)qi * n : nullptr;
    int it = 0;
    bool converged = false;
    double residual = 0.0;
    for (; it < a.max_iter; ++it) {
      for (int k = blockIdx.x; k < a.K; k += gridDim.x)
        sweep(a, k, s_mu[k], prev, work, dt, q, s_warp);
      grid.sync();
      unsigned long long* slot = a.slots + 2 * (gi & 1);
      if (blockIdx.x == 0 && threadIdx.x == 0) {  // the other slot was read before this sync
        a.slots[2 * ((gi + 1) & 1)] = 0ull;
        a.slots[2 * ((gi + 1) & 1) + 1] = 0ull;
      }
      reduce_phi(a, work, s_w, true, slot, nullptr, s_red);
      grid.sync();
      const double diff = __longlong_as_double((long long)__ldcg(slot));
      const double scale = __longlong_as_double((long long)__ldcg(slot + 1));
      ++gi;
      residual = scale > 0.0 ? diff / scale : diff;
      if (residual <= a.tol) {
        converged = true;
        break;
      }
    }
    if (!converged) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        *a.err_step = step;
        *a.err_residual = residual;
      }
      return;  // uniform across the grid
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) a.iterations[step] = it + 1;
    // moments consistent with the converged flux: one more sweep (reference.cpp:217-221)
    for (int k = blockIdx.x; k < a.K; k += gridDim.x)
      sweep(a, k, s_mu[k], prev, work, dt, q, s_warp);
    grid.sync();
    reduce_phi(a, work, s_w, false, nullptr,
               a.phi_fine ? a.phi_fine + (size_t)step * n : nullptr, s_red);
    __syncthreads();
    project_layer(a, step);
    double* t = prev;
    prev = work;
    work = t;
    grid.sync();
  }
}

template <class T>
void upload(DevBuf<T>& b, const std::vector<T>& v, cudaStream_t s) {
  b.reserve(std::max<size_t>(v.size(), 1));
  if (!v.empty())
    HWWG_CUDA(cudaMemcpyAsync(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
}

}  // namespace

void gauss_legendre(int n, double* mu, double* weight) {
  if (n < 2 || n % 2 != 0) throw ApiError(HWWG_EINVAL, "quadrature order must be even and >= 2");
  constexpr double kPi = 3.141592653589793;  // std::numbers::pi
  for (int i = 0; i < n / 2; ++i) {
    // Newton iteration from the Chebyshev estimate of the i-th root
    double x = std::cos(kPi * (i + 0.75) / (n + 0.5));
    double dp = 0.0;
    for (int iter = 0; iter < 100; ++iter) {
      double p0 = 1.0, p1 = x;
      for (int l = 2; l <= n; ++l) {
        const double p2 = ((2 * l - 1) * x * p1 - (l - 1) * p0) / l;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (x * p1 - p0) / (x * x - 1.0);
      const double dx = p1 / dp;
      x -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    const double w = 2.0 / ((1.0 - x * x) * dp * dp);
    mu[i] = -x;
    mu[n - 1 - i] = x;
    weight[i] = w;
    weight[n - 1 - i] = w;
  }
}

void sn_solve_device(const SnHostProblem& p, int device, cudaStream_t s, double* phi_fine,
                     int* iterations, double* phi_layer, double* phi_interval) {
  const int K = p.order;
  if (K < 2 || K % 2 != 0) throw ApiError(HWWG_EINVAL, "quadrature order must be even and >= 2");
  if (K > kSnMaxOrder) throw ApiError(HWWG_EINVAL, "quadrature order above 256 is not supported");
  const int n = (int)p.edges.size() - 1;
  const int steps = (int)p.layers.size() - 1;
  if (n < 1) throw ApiError(HWWG_EINVAL, "mesh needs at least one cell");
  if (steps < 1) throw ApiError(HWWG_EINVAL, "time grid needs at least one step");
  if (p.psi0.size() != (size_t)K * n)
    throw ApiError(HWWG_EINVAL, "psi0 size does not match quadrature order and mesh");
  if (p.inc_left.size() != (size_t)K || p.inc_right.size() != (size_t)K)
    throw ApiError(HWWG_EINVAL, "incoming flux arrays must match quadrature order");
  if (p.materials.size() != (size_t)n)
    throw ApiError(HWWG_EINVAL, "materials and source must have one entry per cell");
  for (int i = 0; i < n; ++i)
    if (!(p.edges[i + 1] > p.edges[i]))
      throw ApiError(HWWG_EINVAL, "mesh edges must be strictly increasing");
  for (int m = 1; m <= steps; ++m)
    if (!(p.layers[m] > p.layers[m - 1]))
      throw ApiError(HWWG_EINVAL, "time layers must be strictly increasing");
  const bool project = p.tally_cells > 0;
  if (project && ((long long)p.tally_cells * p.sr != n || steps % p.ratio != 0))
    throw ApiError(HWWG_EINVAL, "fine grids must nest the tally grids");

  std::vector<double> mu(K), w(K);
  gauss_legendre(K, mu.data(), w.data());
  std::vector<double> dx(n), speed(n), sig_t(n), sig_src(n);
  for (int i = 0; i < n; ++i) {
    const hwwg_material& m = p.materials[i];
    dx[i] = p.edges[i + 1] - p.edges[i];
    speed[i] = m.speed;
    sig_t[i] = m.sigma_t;
    sig_src[i] = m.sigma_s + m.nu_f * m.sigma_f;  // reference.cpp:106-107 grouping
  }
  std::vector<double> tw;
  if (project) {
    tw.resize(p.tally_cells);
    for (int c = 0; c < p.tally_cells; ++c) tw[c] = p.tally_edges[c + 1] - p.tally_edges[c];
  }
  const int N = project ? steps / p.ratio : 0;

  HWWG_CUDA(cudaSetDevice(device));
  DevBuf<double> d_mu, d_w, d_dx, d_speed, d_sig_t, d_sig_src, d_layers, d_il, d_ir, d_q, d_psi_a,
      d_psi_b, d_phi, d_fine, d_tw, d_lay, d_itv, d_res;
  DevBuf<int> d_qi, d_iters, d_err;
  DevBuf<unsigned long long> d_slots;
  upload(d_mu, mu, s);
  upload(d_w, w, s);
  upload(d_dx, dx, s);
  upload(d_speed, speed, s);
  upload(d_sig_t, sig_t, s);
  upload(d_sig_src, sig_src, s);
  upload(d_layers, p.layers, s);
  upload(d_il, p.inc_left, s);
  upload(d_ir, p.inc_right, s);
  upload(d_q, p.q_rows, s);
  upload(d_qi, p.q_index, s);
  upload(d_psi_a, p.psi0, s);
  d_psi_b.reserve((size_t)K * n);
  d_phi.reserve(n);
  if (phi_fine) d_fine.reserve((size_t)(steps + 1) * n);
  d_iters.reserve(steps + 1);
  HWWG_CUDA(cudaMemsetAsync(d_iters.p, 0, (steps + 1) * sizeof(int), s));
  if (project) {
    upload(d_tw, tw, s);
    d_lay.reserve((size_t)(N + 1) * p.tally_cells);
    d_itv.reserve((size_t)N * p.tally_cells);
    HWWG_CUDA(cudaMemsetAsync(d_itv.p, 0, (size_t)N * p.tally_cells * 8, s));
  }
  d_slots.reserve(4);
  HWWG_CUDA(cudaMemsetAsync(d_slots.p, 0, 4 * 8, s));
  d_err.reserve(1);
  HWWG_CUDA(cudaMemsetAsync(d_err.p, 0, sizeof(int), s));
  d_res.reserve(1);

  SnArgs a{};
  a.K = K;
  a.cells = n;
  a.steps = steps;
  a.mu = d_mu.p;
  a.wq = d_w.p;
  a.dx = d_dx.p;
  a.speed = d_speed.p;
  a.sig_t = d_sig_t.p;
  a.sig_src = d_sig_src.p;
  a.layers = d_layers.p;
  a.inc_left = d_il.p;
  a.inc_right = d_ir.p;
  a.q_rows = p.q_rows.empty() ? nullptr : d_q.p;
  a.q_index = p.q_rows.empty() ? nullptr : d_qi.p;
  a.psi_a = d_psi_a.p;
  a.psi_b = d_psi_b.p;
  a.phi = d_phi.p;
  a.phi_fine = phi_fine ? d_fine.p : nullptr;
  a.iterations = d_iters.p;
  a.tally = project ? p.tally_cells : n;
  a.sr = project ? p.sr : 1;
  a.ratio = project ? p.ratio : 1;
  a.tally_w = project ? d_tw.p : nullptr;
  a.phi_layer = project ? d_lay.p : nullptr;
  a.phi_interval = project ? d_itv.p : nullptr;
  a.tol = p.tolerance;
  a.max_iter = p.max_iterations;
  a.slots = d_slots.p;
  a.err_step = d_err.p;
  a.err_residual = d_res.p;

  // one CTA per direction, all co-resident (cooperative launch checks it)
  void* args[] = {&a};
  HWWG_CUDA(cudaLaunchCooperativeKernel((const void*)k_sn_solve, dim3(K), dim3(kSnThreads), args,
                                        0, s));
  int err_step = 0;
  double residual = 0.0;
  HWWG_CUDA(cudaMemcpyAsync(&err_step, d_err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  HWWG_CUDA(cudaMemcpyAsync(&residual, d_res.p, 8, cudaMemcpyDeviceToHost, s));
  if (phi_fine)
    HWWG_CUDA(cudaMemcpyAsync(phi_fine, d_fine.p, (size_t)(steps + 1) * n * 8,
                              cudaMemcpyDeviceToHost, s));
  if (iterations)
    HWWG_CUDA(cudaMemcpyAsync(iterations, d_iters.p, (steps + 1) * sizeof(int),
                              cudaMemcpyDeviceToHost, s));
  if (project && phi_layer)
    HWWG_CUDA(cudaMemcpyAsync(phi_layer, d_lay.p, (size_t)(N + 1) * p.tally_cells * 8,
                              cudaMemcpyDeviceToHost, s));
  if (project && phi_interval)
    HWWG_CUDA(cudaMemcpyAsync(phi_interval, d_itv.p, (size_t)N * p.tally_cells * 8,
                              cudaMemcpyDeviceToHost, s));
  HWWG_CUDA(cudaStreamSynchronize(s));
  if (err_step) {
    std::ostringstream msg;  // reference.cpp:207-212
    msg << "source iteration did not converge at step " << err_step << ": residual " << residual
        << " after " << p.max_iterations << " iterations";
    throw ApiError(HWWG_ESINGULAR, msg.str());
  }
}

SnHostProblem reference_problem(const hwwg_run_config& c, int space_refine, int time_refine,
                                int sn_order) {
  if (space_refine < 1 || time_refine < 1)
    throw ApiError(HWWG_EINVAL, "refinement factors must be >= 1");
  if (c.cells < 1 || !(c.x_min < c.x_max) || c.time_steps < 1)
    throw ApiError(HWWG_EINVAL, "invalid mesh or time grid");
  const int I = c.cells;
  SnHostProblem p;
  p.order = sn_order;
  // tally mesh (mesh.cpp:42-50), the driver's construction
  p.tally_edges.resize(I + 1);
  const double tw = (c.x_max - c.x_min) / I;
  for (int e = 0; e <= I; ++e) p.tally_edges[e] = c.x_min + e * tw;
  p.tally_edges[I] = c.x_max;
  std::vector<hwwg_material> tmat(I, hwwg_material{c.sigma_t, c.sigma_s, c.sigma_f, c.nu_f, c.speed});
  if (c.n_regions > 0)  // config-3 regions, the driver's rule (first x_hi above the centre)
    for (int i = 0; i < I; ++i) {
      const double xc = 0.5 * (p.tally_edges[i] + p.tally_edges[i + 1]);
      int r = 0;
      while (r < c.n_regions - 1 && !(xc < c.region_x_hi[r])) ++r;
      const double* m = c.region_mat[r];
      tmat[i] = hwwg_material{m[0], m[1], m[2], m[3], m[4]};
    }
  // pulse_problem (reference.cpp:302-326): space_refine fine cells per tally cell
  p.edges.reserve((size_t)I * space_refine + 1);
  for (int cc = 0; cc < I; ++cc) {
    const double x0 = p.tally_edges[cc];
    const double w = (p.tally_edges[cc + 1] - p.tally_edges[cc]) / space_refine;
    for (int s = 0; s < space_refine; ++s) p.edges.push_back(x0 + s * w);
  }
  p.edges.push_back(c.x_max);
  const int n = (int)p.edges.size() - 1;
  for (int i = 1; i <= n; ++i)
    if (!(p.edges[i] > p.edges[i - 1]))
      throw ApiError(HWWG_EINVAL, "mesh edges must be strictly increasing");
  p.materials.resize(n);
  for (int f = 0; f < n; ++f) p.materials[f] = tmat[f / space_refine];
  const int steps = c.time_steps * time_refine;
  p.layers.resize(steps + 1);
  uniform_layers(c.t_end, steps, p.layers.data());
  p.tally_cells = I;
  p.sr = space_refine;
  p.ratio = time_refine;
  p.inc_left.assign(sn_order, 0.0);
  p.inc_right.assign(sn_order, 0.0);
  p.psi0.assign((size_t)sn_order * n, 0.0);
  if (sn_order < 2 || sn_order % 2 != 0)
    throw ApiError(HWWG_EINVAL, "quadrature order must be even and >= 2");
  // load_pulse_ic (reference.cpp:330-356)
  if (!c.no_pulse) {
    const int cell = locate_host(p.edges, c.x0);
    if (cell < 0) throw ApiError(HWWG_EINVAL, "pulse position outside the mesh");
    const double tol = 1e-12 * (p.edges[n] - p.edges[0]);
    int on_edge = -1;
    for (int e = 1; e < n; ++e)
      if (std::abs(p.edges[e] - c.x0) <= tol) {
        on_edge = e;
        break;
      }
    struct Part {
      int cell;
      double frac;
    };
    std::vector<Part> parts;
    if (on_edge >= 0) {
      parts.push_back({on_edge - 1, 0.5});
      parts.push_back({on_edge, 0.5});
    } else {
      parts.push_back({cell, 1.0});
    }
    for (const auto& part : parts) {
      const double psi = 0.5 * p.materials[part.cell].speed * c.strength * part.frac /
                         (p.edges[part.cell + 1] - p.edges[part.cell]);
      for (int k = 0; k < sn_order; ++k) p.psi0[(size_t)k * n + part.cell] = psi;
    }
  }
  // config-3 volumetric source: the LOSM's per-step emission (volume_q_host) on
  // the fine grid, as a density (per unit length) for the transport source
  if (c.vol_rate > 0.0) {
    p.q_index.assign(steps + 1, -1);
    std::vector<double> row(n);
    for (int m = 1; m <= steps; ++m) {
      const double ta = std::max(p.layers[m - 1], c.vol_t_lo);
      const double tb = std::min(p.layers[m], c.vol_t_hi);
      if (!(tb > ta)) continue;
      volume_q_host(p.edges.data(), n, c.vol_x_lo, c.vol_x_hi, ta, tb,
                    p.layers[m] - p.layers[m - 1], c.vol_rate, row.data());
      for (int f = 0; f < n; ++f) row[f] /= p.edges[f + 1] - p.edges[f];
      p.q_index[m] = (int)(p.q_rows.size() / n);
      p.q_rows.insert(p.q_rows.end(), row.begin(), row.end());
    }
  }
  return p;
}

}  // namespace hwwg
