// Device low-order pipeline, finalize and comb (see low_order.cuh).
//
// Single-CTA kernels: the per-update work is O(I) with I <= 4000, far below one
// wave, so one CTA that keeps every intermediate in L1/L2 (and the system in
// shared memory when it fits) beats any multi-kernel split, and there is no
// host round-trip between snapshot, filter, solve and centres.
//
// Parity: compiled with -fmad=false; assembly follows losm.cpp:68-139 term by
// term, the pivoted elimination follows banded.cpp:8-38 on one thread (the
// recurrence is serial), the moving average sums l = -k..k in order and
// divides once (filters.cpp:11-24).
#include <cfloat>

#include "common.cuh"
#include "libm_log.h"
#include <cmath>
#include <cstdlib>
#include <vector>

#include "fast.cuh"
#include "low_order.cuh"
#include "rng.cuh"

namespace hwwg {

namespace {

constexpr int kCtaThreads = 512;

__device__ __forceinline__ double ghost_width(const double* edges, int I, int i) {
  return (i <= 0 || i >= I + 1) ? 0.0 : edges[i] - edges[i - 1];  // mesh.hpp:30-33
}

__device__ __forceinline__ double removal_of(const CellInfo& c) {
  return c.sigma_t - c.sigma_s - c.nu_f * c.sigma_f;  // material.hpp:15
}

// losm.cpp:68-139: rows of the interleaved (phi_0, J_0, ..., J_I, phi_I+1) system.
__device__ void assemble_rows(int I, const double* edges, const CellInfo* cells,
                              const double* phi_prev, const double* J_prev, double J_L,
                              double J_R, const double* Fs, double PLs, double PRs,
                              const double* F_prev, double theta, double dt, const double* q,
                              double* lo, double* di, double* up, double* rh) {
  const int n = 2 * I + 3;
  for (int m = threadIdx.x; m < n; m += blockDim.x) {
    double l = 0.0, d = 0.0, u = 0.0, r = 0.0;
    if (m == 0) {  // left boundary: J_0 + phi_0/2 = 2 J_L + P_L
      d = 0.5;
      u = 1.0;
      r = 2.0 * J_L + PLs;
    } else if (m == n - 1) {  // right boundary: J_I - phi_I+1/2 = 2 J_R - P_R
      l = 1.0;
      d = -0.5;
      r = 2.0 * J_R - PRs;
    } else if ((m & 1) == 0) {  // balance over cell i
      const int i = m >> 1;
      const double dx = ghost_width(edges, I, i);
      const CellInfo c = cells[i - 1];
      const double tau = dx / (c.speed * dt);
      const double rem = removal_of(c);
      const double qi = q ? q[i - 1] : 0.0;
      l = -theta;
      d = tau + theta * rem * dx;
      u = theta;
      r = tau * phi_prev[i] + theta * qi +
          (theta - 1.0) * (J_prev[i] - J_prev[i - 1] + rem * dx * phi_prev[i] - qi);
    } else {  // first moment over the half cells around edge i
      const int i = (m - 1) >> 1;
      const double dx_l = ghost_width(edges, I, i);
      const double dx_r = ghost_width(edges, I, i + 1);
      const double dx_hat = 0.5 * (dx_r + dx_l);
      double num_sig = 0.0, num_vel = 0.0;
      if (dx_l > 0.0) {
        num_sig += cells[i - 1].sigma_t * dx_l;
        num_vel += dx_l / cells[i - 1].speed;
      }
      if (dx_r > 0.0) {
        num_sig += cells[i].sigma_t * dx_r;
        num_vel += dx_r / cells[i].speed;
      }
      const double sig_hat = num_sig / (dx_l + dx_r);
      const double inv_speed_hat = num_vel / (dx_l + dx_r);
      const double tau = dx_hat * inv_speed_hat / dt;
      l = -theta / 3.0;
      d = tau + theta * sig_hat * dx_hat;
      u = theta / 3.0;
      r = tau * J_prev[i] + theta * (Fs[i + 1] - Fs[i]) +
          (theta - 1.0) * ((phi_prev[i + 1] - phi_prev[i]) / 3.0 + sig_hat * dx_hat * J_prev[i] -
                           (F_prev[i + 1] - F_prev[i]));
    }
    lo[m] = l;
    di[m] = d;
    up[m] = u;
    rh[m] = r;
  }
}

// banded.cpp:8-38 on one thread. Returns 0, or 1 + pivot row when singular.
//
// Same operations in the same order as the reference, restructured for a
// GPU thread: the pivot row being eliminated lives in registers (at step k,
// fill[k] is always still 0 and row k+1 is untouched by earlier steps), the
// next row's inputs are loaded one step ahead (they do not depend on the
// recurrence), and only finished rows are stored. The serial chain is then
// one division and one fma per row instead of a global-memory round trip.
__device__ int solve_pivoted_serial(int n, const double* __restrict__ a, double* __restrict__ b,
                                    double* __restrict__ c, double* __restrict__ r,
                                    double* __restrict__ fill, double* __restrict__ x) {
  double bk = b[0], ck = c[0], rk = r[0], fk = 0.0;  // pivot row k
  double na = n > 1 ? a[1] : 0.0, nb = n > 1 ? b[1] : 0.0, nc = n > 1 ? c[1] : 0.0,
         nr = n > 1 ? r[1] : 0.0;  // row k+1 (original)
  for (int k = 0; k + 1 < n; ++k) {
    double a1 = na, b1 = nb, c1 = nc, r1 = nr;
    if (k + 2 < n) {  // prefetch row k+2
      na = a[k + 2];
      nb = b[k + 2];
      nc = c[k + 2];
      nr = r[k + 2];
    }
    if (fabs(a1) > fabs(bk)) {
      double t;
      t = bk; bk = a1; a1 = t;
      t = ck; ck = b1; b1 = t;
      if (k + 2 < n) { t = fk; fk = c1; c1 = t; }
      t = rk; rk = r1; r1 = t;
    }
    if (bk == 0.0) return 1 + k;
    const double m = a1 / bk;
    b1 -= m * ck;
    if (k + 2 < n) c1 -= m * fk;
    r1 -= m * rk;
    b[k] = bk;
    c[k] = ck;
    fill[k] = fk;
    r[k] = rk;
    bk = b1;
    ck = c1;
    rk = r1;
    fk = 0.0;
  }
  b[n - 1] = bk;
  c[n - 1] = ck;
  r[n - 1] = rk;
  fill[n - 1] = 0.0;
  if (bk == 0.0) return n;
  double x2 = r[n - 1] / b[n - 1];
  x[n - 1] = x2;
  if (n < 2) return 0;
  double x1 = (r[n - 2] - c[n - 2] * x2) / b[n - 2];
  x[n - 2] = x1;
  double pr = 0, pc = 0, pf = 0, pb = 0;
  if (n >= 3) { pr = r[n - 3]; pc = c[n - 3]; pf = fill[n - 3]; pb = b[n - 3]; }
  for (int k = n - 3; k >= 0; --k) {
    const double rr = pr, cc = pc, ff = pf, bb = pb;
    if (k > 0) { pr = r[k - 1]; pc = c[k - 1]; pf = fill[k - 1]; pb = b[k - 1]; }
    const double xk = (rr - cc * x1 - ff * x2) / bb;
    x[k] = xk;
    x2 = x1;
    x1 = xk;
  }
  return 0;
}

// Throughput-mode solve of the same system (not bit-identical to banded.cpp):
// the first-moment rows give J_i = p_i - q_i phi_i - s_i phi_{i+1}; substituting
// them into the balance and boundary rows leaves an (I+2) tridiagonal system in
// phi that is an M-matrix for non-multiplying media (diagonally dominant, no
// pivoting needed), solved by parallel cyclic reduction in shared memory:
// ceil(log2(I+2)) steps instead of a 2I+3-long serial recurrence.
constexpr int kPcrRowsPerThread = 16;

__device__ int solve_schur_pcr(int I, const double* __restrict__ lo, const double* __restrict__ di,
                               const double* __restrict__ up, const double* __restrict__ rh,
                               double* __restrict__ x, double* sm) {
  const int N = I + 2;
  double* A = sm;
  double* D = A + N;
  double* C = D + N;
  double* R = C + N;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const int m = 2 * i;
    double a = 0.0, d = di[m], c = 0.0, r = rh[m];
    if (i > 0) {  // J_{i-1} from moment row 2i-1
      const int mm = m - 1;
      const double inv = 1.0 / di[mm];
      const double p = rh[mm] * inv, q = lo[mm] * inv, s = up[mm] * inv;
      a = -lo[m] * q;
      d -= lo[m] * s;
      r -= lo[m] * p;
    }
    if (i < N - 1) {  // J_i from moment row 2i+1
      const int mp = m + 1;
      const double inv = 1.0 / di[mp];
      const double p = rh[mp] * inv, q = lo[mp] * inv, s = up[mp] * inv;
      d -= up[m] * q;
      c = -up[m] * s;
      r -= up[m] * p;
    }
    A[i] = a;
    D[i] = d;
    C[i] = c;
    R[i] = r;
  }
  __syncthreads();
  for (int s = 1; s < N; s <<= 1) {
    double na[kPcrRowsPerThread], nd[kPcrRowsPerThread], nc[kPcrRowsPerThread],
        nr[kPcrRowsPerThread];
    int k = 0;
    for (int i = threadIdx.x; i < N && k < kPcrRowsPerThread; i += blockDim.x, ++k) {
      double a = 0.0, d = D[i], c = 0.0, r = R[i];
      if (i - s >= 0) {
        const double al = -A[i] / D[i - s];
        a = al * A[i - s];
        d += al * C[i - s];
        r += al * R[i - s];
      }
      if (i + s < N) {
        const double ga = -C[i] / D[i + s];
        c = ga * C[i + s];
        d += ga * A[i + s];
        r += ga * R[i + s];
      }
      na[k] = a;
      nd[k] = d;
      nc[k] = c;
      nr[k] = r;
    }
    __syncthreads();
    k = 0;
    for (int i = threadIdx.x; i < N && k < kPcrRowsPerThread; i += blockDim.x, ++k) {
      A[i] = na[k];
      D[i] = nd[k];
      C[i] = nc[k];
      R[i] = nr[k];
    }
    __syncthreads();
  }
  int bad = 0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    if (D[i] == 0.0 || !isfinite(D[i])) bad = 1;
    x[2 * i] = R[i] / D[i];
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= I; i += blockDim.x) {  // back out the currents
    const int mp = 2 * i + 1;
    x[mp] = (rh[mp] - lo[mp] * x[2 * i] - up[mp] * x[2 * i + 2]) / di[mp];
  }
  return __syncthreads_or(bad);
}

// ---- cached factorization (throughput mode) --------------------------------
// The LOSM matrix depends on the mesh, the materials, theta and dt only, so the
// Schur complement and every PCR level's elimination multipliers are computed
// once (per theta/dt) and each later solve only carries the right-hand side
// through them: two fmas per row and level, no divisions. The cached values
// are the ones solve_schur_pcr computes, so results are identical to it.
constexpr int kFacLevels = 9;  // PCR levels for N = I + 2 <= 512 (one row per thread)

struct FacView {
  double *tau_b, *remdx_b, *lo_b, *di_b, *up_b;           // balance/boundary rows (N)
  double *tau_m, *sdx_m, *lo_m, *di_m, *up_m, *inv_m;     // moment rows (I + 1)
  double *al, *ga;                                        // [kFacLevels][N]
  double* dfin;                                           // N
  double* bad;                                            // 1
};

__host__ __device__ inline size_t fac_words_for(int I) {
  const size_t N = (size_t)I + 2, E = (size_t)I + 1;
  return 5 * N + 6 * E + 2 * (size_t)kFacLevels * N + N + 1;
}

__device__ FacView fac_view(double* f, int I) {
  const int N = I + 2, E = I + 1;
  FacView v;
  v.tau_b = f; f += N;
  v.remdx_b = f; f += N;
  v.lo_b = f; f += N;
  v.di_b = f; f += N;
  v.up_b = f; f += N;
  v.tau_m = f; f += E;
  v.sdx_m = f; f += E;
  v.lo_m = f; f += E;
  v.di_m = f; f += E;
  v.up_m = f; f += E;
  v.inv_m = f; f += E;
  v.al = f; f += (size_t)kFacLevels * N;
  v.ga = f; f += (size_t)kFacLevels * N;
  v.dfin = f; f += N;
  v.bad = f;
  return v;
}

// Builds the cache (same formulas and operation order as assemble_rows and
// solve_schur_pcr; the matrix rows come from the assembled system lo/di/up).
__device__ void build_factorization(int I, const double* edges, const CellInfo* cells,
                                    double theta, double dt, const double* lo, const double* di,
                                    const double* up, FacView F, double* sm) {
  const int N = I + 2, n = 2 * I + 3;
  double* A = sm;
  double* D = A + N;
  double* C = D + N;
  const int i = threadIdx.x;
  if (i < N) {
    // RHS constants of the balance row (losm.cpp:68-139 via assemble_rows)
    double tau = 0.0, remdx = 0.0;
    if (i >= 1 && i <= I) {
      const double dx = ghost_width(edges, I, i);
      const CellInfo c = cells[i - 1];
      tau = dx / (c.speed * dt);
      remdx = removal_of(c) * dx;
    }
    F.tau_b[i] = tau;
    F.remdx_b[i] = remdx;
    const int m = 2 * i;
    F.lo_b[i] = lo[m];
    F.di_b[i] = di[m];
    F.up_b[i] = up[m];
    if (i <= I) {  // moment row 2i+1
      const int mp = m + 1;
      const double dx_l = ghost_width(edges, I, i);
      const double dx_r = ghost_width(edges, I, i + 1);
      const double dx_hat = 0.5 * (dx_r + dx_l);
      double num_sig = 0.0, num_vel = 0.0;
      if (dx_l > 0.0) {
        num_sig += cells[i - 1].sigma_t * dx_l;
        num_vel += dx_l / cells[i - 1].speed;
      }
      if (dx_r > 0.0) {
        num_sig += cells[i].sigma_t * dx_r;
        num_vel += dx_r / cells[i].speed;
      }
      const double sig_hat = num_sig / (dx_l + dx_r);
      const double inv_speed_hat = num_vel / (dx_l + dx_r);
      F.tau_m[i] = dx_hat * inv_speed_hat / dt;
      F.sdx_m[i] = sig_hat * dx_hat;
      F.lo_m[i] = lo[mp];
      F.di_m[i] = di[mp];
      F.up_m[i] = up[mp];
      F.inv_m[i] = 1.0 / di[mp];
    }
    // Schur complement rows (solve_schur_pcr)
    double a = 0.0, d = di[m], c = 0.0;
    if (i > 0) {
      const int mm = m - 1;
      const double inv = 1.0 / di[mm];
      const double q = lo[mm] * inv, s = up[mm] * inv;
      a = -lo[m] * q;
      d -= lo[m] * s;
    }
    if (i < N - 1) {
      const int mp = m + 1;
      const double inv = 1.0 / di[mp];
      const double q = lo[mp] * inv, s = up[mp] * inv;
      d -= up[m] * q;
      c = -up[m] * s;
    }
    A[i] = a;
    D[i] = d;
    C[i] = c;
  }
  (void)n;
  __syncthreads();
  int l = 0;
  for (int s = 1; s < N; s <<= 1, ++l) {
    double na = 0.0, nd = 0.0, nc = 0.0;
    if (i < N) {
      double a = 0.0, d = D[i], c = 0.0, al = 0.0, ga = 0.0;
      if (i - s >= 0) {
        al = -A[i] / D[i - s];
        a = al * A[i - s];
        d += al * C[i - s];
      }
      if (i + s < N) {
        ga = -C[i] / D[i + s];
        c = ga * C[i + s];
        d += ga * A[i + s];
      }
      F.al[(size_t)l * N + i] = al;
      F.ga[(size_t)l * N + i] = ga;
      na = a;
      nd = d;
      nc = c;
    }
    __syncthreads();
    if (i < N) {
      A[i] = na;
      D[i] = nd;
      C[i] = nc;
    }
    __syncthreads();
  }
  int bad = 0;
  if (i < N) {
    F.dfin[i] = D[i];
    if (D[i] == 0.0 || !isfinite(D[i])) bad = 1;
  }
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) *F.bad = bad ? 1.0 : 0.0;
  __syncthreads();
}

// One solve through the cached factorization: RHS of assemble_rows (J_L = J_R
// = 0, as the driver calls it; q the config-3 source or null), the Schur RHS, the PCR levels, phi
// and the currents into x (interleaved like the full system). Returns nonzero
// when the factorization is singular.
__device__ int solve_cached(int I, FacView F, const double* phi_prev, const double* J_prev,
                            const double* Fs, double PLs, double PRs, const double* F_prev,
                            double theta, const double* q, double* x, double* sm) {
  const int N = I + 2;
  double* P = sm;       // N: moment-row RHS * inv diagonal
  double* R0 = P + N;   // N
  double* R1 = R0 + N;  // N
  double* RM = R1 + N;  // N: moment-row RHS
  const int i = threadIdx.x;
  double al[kFacLevels], ga[kFacLevels];
#pragma unroll
  for (int l = 0; l < kFacLevels; ++l) {
    al[l] = i < N ? F.al[(size_t)l * N + i] : 0.0;
    ga[l] = i < N ? F.ga[(size_t)l * N + i] : 0.0;
  }
  double rb = 0.0;
  if (i < N) {
    const double qi = (q && i >= 1 && i <= I) ? q[i - 1] : 0.0;
    if (i == 0) rb = 2.0 * 0.0 + PLs;
    else if (i == N - 1) rb = 2.0 * 0.0 - PRs;
    else
      rb = F.tau_b[i] * phi_prev[i] + theta * qi +
           (theta - 1.0) * (J_prev[i] - J_prev[i - 1] + F.remdx_b[i] * phi_prev[i] - qi);
    if (i <= I) {
      const double rm = F.tau_m[i] * J_prev[i] + theta * (Fs[i + 1] - Fs[i]) +
                        (theta - 1.0) * ((phi_prev[i + 1] - phi_prev[i]) / 3.0 +
                                         F.sdx_m[i] * J_prev[i] - (F_prev[i + 1] - F_prev[i]));
      RM[i] = rm;
      P[i] = rm * F.inv_m[i];
    }
  }
  __syncthreads();
  if (i < N) {
    double r = rb;
    if (i > 0) r -= F.lo_b[i] * P[i - 1];
    if (i < N - 1) r -= F.up_b[i] * P[i];
    R0[i] = r;
  }
  __syncthreads();
  double* Rc = R0;
  double* Rn = R1;
  int l = 0;
#pragma unroll
  for (int lv = 0; lv < kFacLevels; ++lv) {
    const int s = 1 << lv;
    if (s >= N) break;
    if (i < N) {
      double r = Rc[i];
      if (i - s >= 0) r += al[lv] * Rc[i - s];
      if (i + s < N) r += ga[lv] * Rc[i + s];
      Rn[i] = r;
    }
    __syncthreads();
    double* t = Rc;
    Rc = Rn;
    Rn = t;
    ++l;
  }
  if (i < N) x[2 * i] = Rc[i] / F.dfin[i];
  __syncthreads();
  if (i <= I) {
    const int mp = 2 * i + 1;
    x[mp] = (RM[i] - F.lo_m[i] * x[2 * i] - F.up_m[i] * x[2 * i + 2]) / F.di_m[i];
  }
  __syncthreads();
  return *F.bad != 0.0;
}

// Block max of per-thread partial maxima. The partials start at 0.0 and only
// grow through '>' (ww.cpp:13-15), so NaN never enters and max is exact.
__device__ double block_max(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  const double r = red[0];
  __syncthreads();
  return r;
}

// ww.cpp:8-32 over the block; returns true on uniform fallback.
__device__ bool build_centers_cta(const double* phi, int n, double eps_min, double* centers,
                                  double* red) {
  double mx = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (phi[i] > mx) mx = phi[i];
  mx = block_max(mx, red);
  const bool fallback = !(mx > 0.0) || !isfinite(mx);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (fallback) {
      centers[i] = 1.0;
    } else {
      const double cl = phi[i] > 0.0 ? phi[i] : 0.0;
      centers[i] = (cl / mx) * (1.0 - eps_min) + eps_min;
    }
  }
  __syncthreads();
  return fallback;
}

// filters.cpp:11-24, out-of-place over the block.
__device__ void moving_average_cta(const double* g, int M, int k, double* out) {
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    int km = k;
    if (m < km) km = m;
    if (M - 1 - m < km) km = M - 1 - m;
    double sum = 0.0;
    for (int l = -km; l <= km; ++l) sum += g[m + l];
    out[m] = sum / (2 * km + 1);
  }
  __syncthreads();
}

// In-place MA via scratch: filter_cell_avg_with_boundary (interior) or filter_edge (all).
__device__ void filter_inplace(double* g, int len, int interior, int k, double* tmp) {
  if (k <= 0) return;
  if (interior) {
    if (len <= 2) return;
    moving_average_cta(g + 1, len - 2, k, tmp);
    for (int i = threadIdx.x; i < len - 2; i += blockDim.x) g[i + 1] = tmp[i];
  } else {
    moving_average_cta(g, len, k, tmp);
    for (int i = threadIdx.x; i < len; i += blockDim.x) g[i] = tmp[i];
  }
  __syncthreads();
}

// filters.cpp:26-52 fourier_lowpass over the block, in place (via scratch).
// tab = fourier_tables(M) from the host: [fwd cos | fwd sin | inv cos | inv sin],
// each M*M laid out [m][j], the libm cos/sin of the reference's angles
// (-w0*j*m and w0*j*m), so the device never evaluates a transcendental. The
// spectrum sums run over m in order and the synthesis over j in order with the
// zero-mode skip, complex products as (ac - bd, ad + bc): the reference's
// operations in the reference's order.
__device__ void fourier_cta(double* g, int M, int cutoff, const double* __restrict__ tab,
                            double* tmp) {
  if (M <= 1) return;
  const size_t MM = (size_t)M * M;
  const double* fc = tab;
  const double* fs = tab + MM;
  const double* ic = tab + 2 * MM;
  const double* is = tab + 3 * MM;
  double* sre = tmp;
  double* sim = tmp + M;
  double* out = tmp + 2 * M;
  for (int j = threadIdx.x; j < M; j += blockDim.x) {
    double re = 0.0, im = 0.0;
    if (min(j, M - j) <= cutoff) {
      for (int m = 0; m < M; ++m) {
        const double gm = g[m];
        re = re + gm * fc[(size_t)m * M + j];
        im = im + gm * fs[(size_t)m * M + j];
      }
    }
    sre[j] = re;
    sim[j] = im;
  }
  __syncthreads();
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    double re = 0.0;
    for (int j = 0; j < M; ++j) {
      const double a = sre[j], b = sim[j];
      if (a == 0.0 && b == 0.0) continue;
      const double c = ic[(size_t)j * M + m], d = is[(size_t)j * M + m];
      re = re + (a * c - b * d);
    }
    out[m] = re / M;
  }
  __syncthreads();
  for (int m = threadIdx.x; m < M; m += blockDim.x) g[m] = out[m];
  __syncthreads();
}

// The step's filter: moving average (k > 0), Fourier low-pass (tab != null), or none.
__device__ void filter_any(double* g, int len, int interior, const LowOrderArgs& a, double* tmp) {
  if (a.fourier_tab_cell) {
    if (interior) {
      if (len > 2) fourier_cta(g + 1, len - 2, a.fourier_cutoff, a.fourier_tab_cell, tmp);
    } else {
      fourier_cta(g, len, a.fourier_cutoff, a.fourier_tab_edge, tmp);
    }
    return;
  }
  filter_inplace(g, len, interior, a.ma_k, tmp);
}

__device__ bool all_finite(const double* v, int n) {
  bool bad = false;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (!isfinite(v[i])) bad = true;
  return __syncthreads_or(bad ? 1 : 0) == 0;
}

// HWWG_LOSM_DEBUG: per-phase clock64 stamps of one update (thread 0, printf)
__device__ unsigned long long g_lp[24];
#define LP(k)                                              \
  do {                                                     \
    if (a.debug && threadIdx.x == 0) g_lp[k] = clock64();  \
  } while (0)

// driver.cpp:72-95 hybrid_windows + ww.cpp build_centers, given prepared
// inputs. Solves into the sys scratch; on failure keeps the previous windows.
__device__ __noinline__ void solve_and_center(const LowOrderArgs& a, const double* Fs, double PLs, double PRs,
                                 bool implicit, double* red) {
  const LowOrderState& s = a.s;
  const int I = a.I, n = 2 * I + 3;
  double* lo = s.sys;
  double* di = lo + n;
  double* up = di + n;
  double* rh = up + n;
  double* fill = rh + n;
  double* x = fill + n;
  __shared__ int status;
  LP(3);
  // check_inputs (losm.cpp:43-66): finite previous state and lagged closures
  const bool ok_in = all_finite(s.phi_prev, I + 2) && all_finite(s.J_prev, I + 1) &&
                     all_finite(s.F_prev, I + 2);
  LP(4);
  const bool cached = a.fast_solve && s.fac != nullptr && I + 2 <= (int)blockDim.x &&
                      I + 2 <= (1 << kFacLevels);
  // factorization state word: 0 ok, 1 singular, 2 not built for the current
  // (theta, dt) — a refactor request invalidates first, so a solve skipped on
  // bad inputs leaves the cache marked unbuilt rather than stale
  bool rebuild = false;
  if (cached) {
    const FacView F = fac_view(s.fac, I);
    if (a.refactor && threadIdx.x == 0) *F.bad = 2.0;
    __syncthreads();
    rebuild = *F.bad == 2.0;
    __syncthreads();
  }
  if (ok_in && cached && !rebuild) {
    extern __shared__ double dyn[];
    const int bad = solve_cached(I, fac_view(s.fac, I), s.phi_prev, s.J_prev, Fs, PLs, PRs,
                                 s.F_prev, a.theta, a.q, x, dyn);
    LP(6);
    if (threadIdx.x == 0) status = bad ? 2 : 0;
  } else if (ok_in) {
    assemble_rows(I, a.edges, a.cells, s.phi_prev, s.J_prev, 0.0, 0.0, Fs, PLs, PRs, s.F_prev,
                  a.theta, a.dt, a.q, lo, di, up, rh);
    __syncthreads();
    LP(5);
    if (cached) {  // (re)build: record the factorization, then solve as before
      extern __shared__ double dyn[];
      build_factorization(I, a.edges, a.cells, a.theta, a.dt, lo, di, up, fac_view(s.fac, I), dyn);
    }
    if (a.fast_solve) {
      extern __shared__ double dyn[];
      const int bad = solve_schur_pcr(I, lo, di, up, rh, x, dyn);
      LP(6);
      if (threadIdx.x == 0) status = bad ? 2 : 0;
    } else if (threadIdx.x == 0) {
      status = solve_pivoted_serial(n, lo, di, up, rh, fill, x) ? 2 : 0;
    }
  } else if (threadIdx.x == 0) {
    status = 1;
  }
  __syncthreads();
  const int st = status;
  if (st == 0) {
    for (int i = threadIdx.x; i < I; i += blockDim.x) s.phi_hybrid[i] = x[2 * (i + 1)];
    __syncthreads();
    LP(7);
    build_centers_cta(s.phi_hybrid, I, a.eps_min, s.centers, red);
    LP(8);
    if (threadIdx.x == 0) {
      s.flags[0] = 1;
      s.flags[1] = 1;
      if (implicit) ++s.flags[2];
    }
  } else {
    const bool was_active = s.flags[0] != 0;
    __syncthreads();
    if (!was_active)
      for (int i = threadIdx.x; i < I; i += blockDim.x) s.centers[i] = 1.0;
    if (threadIdx.x == 0) {
      s.flags[0] = 1;
      s.flags[3] = 1;
    }
  }
  if (threadIdx.x == 0) s.flags[4] = st;
}

// Shared-memory residency for the whole update (when it fits, host-decided via
// a.smem_state): the phases below are separated by block barriers, and with
// the state, the 2I+3 system and the filter scratch in global memory every
// phase paid an L2 round trip. Same operations on the same values either way.
constexpr int kSmemStateMaxI = 1200;

__device__ __noinline__ void low_order_update_body(const LowOrderArgs& a);

__global__ void __launch_bounds__(kCtaThreads) k_low_order_update(LowOrderArgs a) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent launch
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // (see k_losm_mid_fast)
  if (a.pool_ctl && threadIdx.x == 0) fast_pool_reset(a.pool_ctl, a.pool_src_head, a.pool_span);
  if (a.backup_centers) {  // the step-start windows backup, then the record flags
    for (int i = threadIdx.x; i < a.I; i += blockDim.x) a.backup_centers[i] = a.s.centers[i];
    if (threadIdx.x < 8) a.backup_flags[threadIdx.x] = a.s.flags[threadIdx.x];
    __syncthreads();
    if (threadIdx.x >= 1 && threadIdx.x <= 4) a.s.flags[threadIdx.x] = 0;
    __syncthreads();
  }
  if (!a.smem_state) {
    low_order_update_body(a);
    return;
  }
  extern __shared__ double dyn[];
  LP(0);
  const int I = a.I;
  const LowOrderState g = a.s;
  // dyn = [PCR scratch 4(I+2) | sys 6n | phi_prev | F_prev | F_now (I+2 each) | J_prev I+1 | phi_hybrid I]
  double* q = dyn + (a.fast_solve ? (size_t)4 * (I + 2) : 0);
  a.s.sys = q; q += (size_t)6 * (2 * I + 3);
  a.s.phi_prev = q; q += I + 2;
  a.s.F_prev = q; q += I + 2;
  a.s.F_now = q; q += I + 2;
  a.s.J_prev = q; q += I + 1;
  a.s.phi_hybrid = q;
  for (int i = threadIdx.x; i < I + 2; i += blockDim.x) {
    a.s.phi_prev[i] = g.phi_prev[i];
    a.s.F_prev[i] = g.F_prev[i];
  }
  for (int i = threadIdx.x; i < I + 1; i += blockDim.x) a.s.J_prev[i] = g.J_prev[i];
  for (int i = threadIdx.x; i < I; i += blockDim.x) a.s.phi_hybrid[i] = g.phi_hybrid[i];
  __syncthreads();
  LP(1);
  low_order_update_body(a);
  __syncthreads();
  LP(9);
  if (a.mode == 0) {  // the filtered inputs persist for the step's mid-step solves
    for (int i = threadIdx.x; i < I + 2; i += blockDim.x) {
      g.phi_prev[i] = a.s.phi_prev[i];
      g.F_prev[i] = a.s.F_prev[i];
    }
    for (int i = threadIdx.x; i < I + 1; i += blockDim.x) g.J_prev[i] = a.s.J_prev[i];
  }
  for (int i = threadIdx.x; i < I; i += blockDim.x) g.phi_hybrid[i] = a.s.phi_hybrid[i];
  __syncthreads();
  LP(10);
  if (a.debug && threadIdx.x == 0) {
    printf("[losm] mode %d cycles: load %llu prep %llu finite %llu assemble %llu solve %llu "
           "status %llu centers %llu tail %llu store %llu total %llu\n", a.mode,
           g_lp[1] - g_lp[0], g_lp[3] - g_lp[1], g_lp[4] - g_lp[3], g_lp[5] - g_lp[4],
           g_lp[6] - g_lp[5], g_lp[7] - g_lp[6], g_lp[8] - g_lp[7], g_lp[9] - g_lp[8],
           g_lp[10] - g_lp[9], g_lp[10] - g_lp[0]);
  }
}

__device__ __noinline__ void low_order_update_body(const LowOrderArgs& a) {
  __shared__ double red[32];
  const LowOrderState& s = a.s;
  const int I = a.I;
  double* tmp = s.sys;  // MA scratch (before assembly)
  if (a.mode == 0) {
    if (a.analytic) {  // analytic_pulse_inputs, driver.cpp:51-61
      for (int i = threadIdx.x; i < I + 2; i += blockDim.x) {
        s.phi_prev[i] = (i == a.pulse_cell + 1) ? a.pulse_value : 0.0;
        s.F_prev[i] = 0.0;
      }
      for (int i = threadIdx.x; i < I + 1; i += blockDim.x) s.J_prev[i] = 0.0;
      if (threadIdx.x == 0) {
        s.PLPR_prev[0] = 0.0;
        s.PLPR_prev[1] = 0.0;
      }
    } else {  // hybrid_inputs_from_report, driver.cpp:41-49; losm.cpp:12-32
      for (int i = threadIdx.x; i < I + 2; i += blockDim.x) {
        const int j = i == 0 ? 0 : (i == I + 1 ? I - 1 : i - 1);
        s.phi_prev[i] = s.rep_phi_census[j];
        s.F_prev[i] = s.rep_closure[j];
      }
      for (int e = threadIdx.x; e < I + 1; e += blockDim.x) {
        double v;
        if (e == 0) v = s.rep_current[0];
        else if (e == I) v = s.rep_current[I - 1];
        else {
          const double xl = 0.5 * (a.edges[e - 1] + a.edges[e]);
          const double xr = 0.5 * (a.edges[e] + a.edges[e + 1]);
          const double t = (a.edges[e] - xl) / (xr - xl);
          v = (1.0 - t) * s.rep_current[e - 1] + t * s.rep_current[e];
        }
        s.J_prev[e] = v;
      }
      if (threadIdx.x == 0) {
        s.PLPR_prev[0] = s.rep_PLPR[0];
        s.PLPR_prev[1] = s.rep_PLPR[1];
      }
    }
    __syncthreads();
    // apply_filter_pipeline(nullptr, F_prev, phi_prev, J_prev), filters.cpp:76-84
    filter_any(s.F_prev, I + 2, 1, a, tmp);
    filter_any(s.phi_prev, I + 2, 1, a, tmp);
    filter_any(s.J_prev, I + 1, 0, a, tmp);
    solve_and_center(a, s.F_prev, s.PLPR_prev[0], s.PLPR_prev[1], false, red);
  } else {
    // partial_snapshot (tally.cpp:116-128) -> with_boundary_extrapolated -> filter
    double* F = s.F_now;
    for (int i = threadIdx.x; i < I + 2; i += blockDim.x) {
      const int j = i == 0 ? 0 : (i == I + 1 ? I - 1 : i - 1);
      F[i] = a.closure_tally[j] * a.snapshot_inv_norm;
    }
    __syncthreads();
    filter_any(F, I + 2, 1, a, tmp);
    const double PL = a.bclosure_tally[0] * a.snapshot_inv_norm;
    const double PR = a.bclosure_tally[1] * a.snapshot_inv_norm;
    solve_and_center(a, F, PL, PR, true, red);
  }
}

// Mid-step window update of the throughput mode through the cached
// factorization, latency-first (the general kernel took ~11 us of
// in-kernel time per update at I = 400, ~30 us with its launch, on the
// critical path between segments). One row per thread; every global value the
// row needs — its cached factorization coefficients, the lagged state, the
// live closure tallies of the partial snapshot around it and q — is loaded up
// front in one round trip; the moving-average filter is evaluated per row
// from those loads; shared memory carries only the Schur right-hand side
// exchange and the PCR levels (one barrier each); the currents are not formed
// (the update keeps only phi_hybrid and the centres). Same arithmetic as
// low_order_update_body -> solve_and_center -> solve_cached on the same values.
__device__ __forceinline__ double snap_filtered(const LowOrderArgs& a, int m) {
  // partial_snapshot (tally.cpp:116-128) -> with_boundary_extrapolated ->
  // filter_cell_avg_with_boundary (filters.cpp:11-24, 63-70): element m of F
  const int I = a.I;
  if (m == 0) return a.closure_tally[0] * a.snapshot_inv_norm;
  if (m == I + 1) return a.closure_tally[I - 1] * a.snapshot_inv_norm;
  if (a.ma_k <= 0 || I <= 0) return a.closure_tally[m - 1] * a.snapshot_inv_norm;
  const int mi = m - 1;  // index in the interior g = F[1..I], g[j] = closure[j] * norm
  int km = a.ma_k;
  if (mi < km) km = mi;
  if (I - 1 - mi < km) km = I - 1 - mi;
  double sum = 0.0;
  for (int l = -km; l <= km; ++l) sum += a.closure_tally[mi + l] * a.snapshot_inv_norm;
  return sum / (2 * km + 1);
}

__global__ void __launch_bounds__(kCtaThreads) k_losm_mid_fast(LowOrderArgs a) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent launch
  // the next segment's transport grid may start its block-private setup now
  // (it waits for this kernel's completion before reading anything it writes)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ double P[kCtaThreads + 1], R0[kCtaThreads], R1[kCtaThreads], red[32];
  __shared__ int s_flags[2];
  if (a.pool_ctl && threadIdx.x == 0) fast_pool_reset(a.pool_ctl, a.pool_src_head, a.pool_span);
  const LowOrderState& st = a.s;
  const int I = a.I, N = I + 2, i = threadIdx.x;
  const FacView F = fac_view(st.fac, I);
  // ---- every global load of row i, issued before any is used
  double al[kFacLevels], ga[kFacLevels];
#pragma unroll
  for (int l = 0; l < kFacLevels; ++l) {
    al[l] = i < N ? F.al[(size_t)l * N + i] : 0.0;
    ga[l] = i < N ? F.ga[(size_t)l * N + i] : 0.0;
  }
  const bool row = i < N, mrow = i <= I;
  const double tau_b = row ? F.tau_b[i] : 0.0, remdx_b = row ? F.remdx_b[i] : 0.0;
  const double lo_b = row ? F.lo_b[i] : 0.0, up_b = row ? F.up_b[i] : 0.0;
  const double dfin = row ? F.dfin[i] : 1.0;
  const double tau_m = mrow ? F.tau_m[i] : 0.0, sdx_m = mrow ? F.sdx_m[i] : 0.0;
  const double inv_m = mrow ? F.inv_m[i] : 0.0;
  const double phi_i = row ? st.phi_prev[i] : 0.0, phi_n = mrow ? st.phi_prev[i + 1] : 0.0;
  const double J_i = mrow ? st.J_prev[i] : 0.0;
  const double J_p = (row && i >= 1 && i <= I) ? st.J_prev[i - 1] : 0.0;
  const double Fp_i = row ? st.F_prev[i] : 0.0, Fp_n = mrow ? st.F_prev[i + 1] : 0.0;
  const double qi = (a.q && i >= 1 && i <= I) ? a.q[i - 1] : 0.0;
  const double Fs_i = mrow ? snap_filtered(a, i) : 0.0, Fs_n = mrow ? snap_filtered(a, i + 1) : 0.0;
  const double PLs = a.bclosure_tally[0] * a.snapshot_inv_norm;
  const double PRs = a.bclosure_tally[1] * a.snapshot_inv_norm;
  const double fac_bad = *F.bad;
  // check_inputs (losm.cpp:43-66): finite lagged state and closures
  bool bad_in = false;
  if (row && (!isfinite(phi_i) || !isfinite(Fp_i))) bad_in = true;
  if (i <= I && !isfinite(J_i)) bad_in = true;
  // ---- Schur right-hand side (solve_cached)
  double rb = 0.0, rm = 0.0;
  if (row) {
    if (i == 0) rb = 2.0 * 0.0 + PLs;
    else if (i == N - 1) rb = 2.0 * 0.0 - PRs;
    else
      rb = tau_b * phi_i + a.theta * qi +
           (a.theta - 1.0) * (J_i - J_p + remdx_b * phi_i - qi);
    if (mrow) {
      rm = tau_m * J_i + a.theta * (Fs_n - Fs_i) +
           (a.theta - 1.0) * ((phi_n - phi_i) / 3.0 + sdx_m * J_i - (Fp_n - Fp_i));
      P[i] = rm * inv_m;
    }
  }
  const int any_bad = __syncthreads_or(bad_in ? 1 : 0);
  const int status = any_bad ? 1 : (fac_bad == 2.0 ? 1 : (fac_bad != 0.0 ? 2 : 0));
  if (status == 0) {
    if (row) {
      double r = rb;
      if (i > 0) r -= lo_b * P[i - 1];
      if (i < N - 1) r -= up_b * P[i];
      R0[i] = r;
    }
    __syncthreads();
    double* Rc = R0;
    double* Rn = R1;
#pragma unroll
    for (int lv = 0; lv < kFacLevels; ++lv) {
      const int sft = 1 << lv;
      if (sft >= N) break;
      if (row) {
        double r = Rc[i];
        if (i - sft >= 0) r += al[lv] * Rc[i - sft];
        if (i + sft < N) r += ga[lv] * Rc[i + sft];
        Rn[i] = r;
      }
      __syncthreads();
      double* t = Rc;
      Rc = Rn;
      Rn = t;
    }
    // phi_hybrid = interior phi (driver.cpp:80), then build_centers (ww.cpp:8-32)
    const double phi = row ? Rc[i] / dfin : 0.0;
    const bool cell = i >= 1 && i <= I;
    const double mx = block_max(cell && phi > 0.0 ? phi : 0.0, red);
    const bool fallback = !(mx > 0.0) || !isfinite(mx);
    if (cell) {
      st.phi_hybrid[i - 1] = phi;
      const double cl = phi > 0.0 ? phi : 0.0;
      st.centers[i - 1] = fallback ? 1.0 : (cl / mx) * (1.0 - a.eps_min) + a.eps_min;
    }
    if (i == 0) {
      st.flags[0] = 1;
      st.flags[1] = 1;
      ++st.flags[2];
      st.flags[4] = 0;
    }
  } else {  // keep the previous windows (driver.cpp:84-94)
    if (i == 0) s_flags[0] = st.flags[0];
    __syncthreads();
    if (!s_flags[0])
      for (int c = i; c < I; c += blockDim.x) st.centers[c] = 1.0;
    if (i == 0) {
      st.flags[0] = 1;
      st.flags[3] = 1;
      st.flags[4] = status;
    }
  }
}

__global__ void __launch_bounds__(kCtaThreads) k_raw_losm(RawLosmArgs a) {
  const int I = a.I, n = 2 * I + 3;
  double* lo = a.sys;
  double* di = lo + n;
  double* up = di + n;
  double* rh = up + n;
  double* fill = rh + n;
  double* x = fill + n;
  const bool ok = all_finite(a.phi_prev, I + 2) && all_finite(a.J_prev, I + 1) &&
                  all_finite(a.F_prev, I + 2);
  if (!ok) {
    if (threadIdx.x == 0) *a.status = 1;
    return;
  }
  assemble_rows(I, a.edges, a.cells, a.phi_prev, a.J_prev, a.J_L, a.J_R,
                a.implicit ? a.F_now : a.F_prev, a.implicit ? a.PL_now : a.PL_prev,
                a.implicit ? a.PR_now : a.PR_prev, a.F_prev, a.theta, a.dt, a.q, lo, di, up, rh);
  __syncthreads();
  __shared__ int st;
  if (threadIdx.x == 0) st = solve_pivoted_serial(n, lo, di, up, rh, fill, x);
  __syncthreads();
  if (st) {
    if (threadIdx.x == 0) *a.status = 1 + st;
    return;
  }
  for (int i = threadIdx.x; i <= I + 1; i += blockDim.x) a.phi_out[i] = x[2 * i];
  for (int i = threadIdx.x; i <= I; i += blockDim.x) a.J_out[i] = x[2 * i + 1];
  if (threadIdx.x == 0) *a.status = 0;
}

// tally.cpp:43-48
__device__ __forceinline__ uint64_t batch_size(uint64_t H, int B, int b) {
  const uint64_t lo = ((uint64_t)b * H + (uint64_t)B - 1) / (uint64_t)B;
  const uint64_t hi = ((uint64_t)(b + 1) * H + (uint64_t)B - 1) / (uint64_t)B;
  return hi - lo;
}

// tally.cpp:68-114
constexpr int kMaxFinalizeBatches = 1024;
__global__ void k_finalize(FinalizeArgs a) {
  const int I = a.I, B = a.B;
  const double inv_h = 1.0 / a.normalization;
  const bool sigma_valid = B >= 2 && a.histories >= (uint64_t)B;
  const double scale = (double)a.histories / a.normalization;
  const double ih = 1.0 / (double)a.histories;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  // 1/batch size, once per block (64-bit divisions per cell and batch made
  // this kernel ~20 us)
  __shared__ double inv_nb_s[kMaxFinalizeBatches];
  const bool cached = B <= kMaxFinalizeBatches;
  if (cached)
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
      const uint64_t nb = batch_size(a.histories, B, b);
      inv_nb_s[b] = nb ? 1.0 / (double)nb : 0.0;
    }
  __syncthreads();
  auto inv_nb_of = [&](int b) {
    if (cached) return inv_nb_s[b];
    const uint64_t nb = batch_size(a.histories, B, b);
    return nb ? 1.0 / (double)nb : 0.0;
  };
  if (i < I && a.track_from_batches) {
    double s = 0.0;
    for (int b = 0; b < B; ++b) s += a.t.track_flux_batch[(size_t)b * I + i];
    a.t.track_flux[i] = s;  // read back below by this thread only
  }
  if (i < I) {
    a.phi_track[i] = a.t.track_flux[i] * inv_h;
    a.phi_census[i] = a.t.census_phi[i] * inv_h;
    a.current[i] = a.t.census_current[i] * inv_h;
    a.closure[i] = a.t.census_closure[i] * inv_h;
    double sg = 0.0;
    if (sigma_valid) {
      const double mean = a.t.track_flux[i] * ih;
      double ss = 0.0;
      for (int b = 0; b < B; ++b) {
        const double bm = a.t.track_flux_batch[(size_t)b * I + i] * inv_nb_of(b);
        const double d = bm - mean;
        ss += d * d;
      }
      sg = scale * sqrt(ss / ((double)B * (B - 1)));
    }
    a.sigma[i] = sg;
  }
  if (i <= I) a.edge[i] = a.t.edge_current[i] * inv_h;
  if (i == 0) {
    a.scalars[0] = a.t.boundary_closure[0] * inv_h;
    a.scalars[1] = a.t.boundary_closure[1] * inv_h;
    double cw = 0.0;
    for (int b = 0; b < B; ++b) cw += a.t.census_weight_batch[b];
    a.scalars[2] = cw * inv_h;
    double cws = 0.0;
    if (sigma_valid) {
      const double wmean = cw * ih;
      double ss = 0.0;
      for (int b = 0; b < B; ++b) {
        const double bm = a.t.census_weight_batch[b] * inv_nb_of(b);
        const double d = bm - wmean;
        ss += d * d;
      }
      cws = scale * sqrt(ss / ((double)B * (B - 1)));
    }
    a.scalars[3] = cws;
    a.scalars[4] = sigma_valid ? 1.0 : 0.0;
  }
}

// popctrl.cpp:15-30 — the cumulative-weight walk s_k = fl(s_{k-1} + w_k),
// sequential in bank order, computed in parallel and bit for bit.
//
// While s stays in one binade [2^e, 2^{e+1}) every s_k is an integer multiple
// S_k of u = ulp = 2^{e-52}, and with q = w_k / u = a + r (a integer, r in
// [0, 1), both exact) round-to-nearest-even gives
//   S_k = S_{k-1} + a + [r > 1/2] + [r == 1/2 and S_{k-1} + a odd]
// as long as S_{k-1} + a < 2^53. Each weight is then a map S -> S + inc(S mod
// 2); maps compose associatively (an increment per input parity), so a run of
// weights inside one binade is an integer scan. s only grows, so it changes
// binade ~log2(n) times; the weight that leaves a binade (or any weight the
// rule does not cover: zero sum, negative, non-finite, huge) is added with a
// real fp64 add and the scan restarts after it.
//
// Across the bank (4096-weight tiles): an approximate parallel prefix of tile
// sums predicts each tile's binade; a tile whose predicted range stays well
// inside one binade gets its composed map (all tiles in parallel); one CTA
// then walks the tiles in order, applying maps where the exact running sum
// confirms the prediction and running the in-tile restart scan on the rest
// (the first tiles and the ~log2(n) binade crossings); all tiles then write
// their prefix values in parallel.
namespace combscan {
constexpr int kThreads = 512, kItems = 8, kTile = kThreads * kItems;
constexpr uint64_t kTop = 1ULL << 53;
constexpr uint64_t kSat = 1ULL << 62;
constexpr int kDirty = -100000;

struct Map {  // S -> S + inc[S & 1]
  uint64_t i0, i1;
};
__device__ __forceinline__ uint64_t sat_add(uint64_t x, uint64_t y) {
  const uint64_t z = x + y;
  return (z < x || z > kSat) ? kSat : z;
}
// f then g (saturating: a saturated map only ever lands at or past 2^53)
__device__ __forceinline__ Map compose(const Map& f, const Map& g) {
  return Map{sat_add(f.i0, (f.i0 & 1) ? g.i1 : g.i0),
             sat_add(f.i1, ((1 + f.i1) & 1) ? g.i1 : g.i0)};
}
__device__ __forceinline__ uint64_t apply(const Map& f, uint64_t S) {
  return sat_add(S, (S & 1) ? f.i1 : f.i0);
}
__device__ __forceinline__ bool in_rule(double s) { return s >= 0x1p-1000 && s < 0x1p1000; }
__device__ __forceinline__ int binade(double s) {  // s in [2^e, 2^{e+1})
  int e;
  frexp(s, &e);
  return e - 1;
}

// floor(w / u) (saturated at 2^53) and the rounding class of the remainder
__device__ __forceinline__ void split(double w, int e, uint64_t& a, int& cls) {
  if (!(w >= 0.0) || w >= ldexp(1.0, e + 1)) {  // off the rule: negative, NaN, inf, huge
    a = kTop;
    cls = 0;
    return;
  }
  const double q = ldexp(w, 52 - e);  // exact power-of-two scaling
  const double fa = floor(q);
  const double r = q - fa;  // exact
  a = (uint64_t)fa;
  cls = r > 0.5 ? 2 : (r == 0.5 ? 1 : 0);
}
__device__ __forceinline__ Map elem_map(uint64_t a, int cls) {
  const uint64_t b = a + (cls == 2 ? 1 : 0);
  const int tie = cls == 1;
  // input parity p: a tie rounds up when S + a is odd
  return Map{b + (uint64_t)(tie && (b & 1)), b + (uint64_t)(tie && !(b & 1))};
}

// Block-wide exclusive scan of one map per thread (thread order); also returns
// the block aggregate. Uses smem[kThreads / 32].
__device__ __forceinline__ Map block_exclusive(Map v, Map* smem, Map& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  Map inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Map p;
    p.i0 = __shfl_up_sync(0xffffffffu, inc.i0, o);
    p.i1 = __shfl_up_sync(0xffffffffu, inc.i1, o);
    if (lane >= o) inc = compose(p, inc);
  }
  if (lane == 31) smem[wid] = inc;
  __syncthreads();
  Map before{0, 0};
  for (int w = 0; w < wid; ++w) before = compose(before, smem[w]);
  total = before;
  for (int w = wid; w < kThreads / 32; ++w) total = compose(total, smem[w]);
  Map ex;
  ex.i0 = __shfl_up_sync(0xffffffffu, inc.i0, 1);
  ex.i1 = __shfl_up_sync(0xffffffffu, inc.i1, 1);
  if (lane > 0) before = compose(before, ex);
  __syncthreads();
  return before;
}

// The sequential walk over weights [k0, k1) from running sum s (one CTA, all
// threads; every thread returns the final sum); prefix (optional) receives
// s_k at index k. wt: kTile doubles of shared memory.
template <class WF>
__device__ double walk(WF W, uint64_t k0, uint64_t k1, double s, double* prefix, double* wt) {
  __shared__ Map wagg[kThreads / 32];
  __shared__ unsigned long long cross;
  __shared__ double s_sh;
  __shared__ unsigned long long k_sh;
  const int tid = threadIdx.x;
  uint64_t k = k0;
  while (k < k1) {
    if (!in_rule(s)) {  // one thread until s is a normal, finite, positive sum
      if (tid == 0) {
        while (k < k1 && !in_rule(s)) {
          s += W(k);
          if (prefix) prefix[k] = s;
          ++k;
        }
        s_sh = s;
        k_sh = k;
      }
      __syncthreads();
      s = s_sh;
      k = k_sh;
      __syncthreads();
      continue;
    }
    const int e = binade(s);
    const double u = ldexp(1.0, e - 52);
    const uint64_t S0 = (uint64_t)ldexp(s, 52 - e);
    const uint64_t m = k1 - k < (uint64_t)kTile ? k1 - k : (uint64_t)kTile;
    for (int j = tid; j < kTile; j += kThreads) wt[j] = (uint64_t)j < m ? W(k + j) : 0.0;
    if (tid == 0) cross = ~0ULL;
    __syncthreads();
    uint64_t a[kItems];
    int cls[kItems];
    Map agg{0, 0};
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      split(wt[tid * kItems + i], e, a[i], cls[i]);
      agg = compose(agg, elem_map(a[i], cls[i]));
    }
    Map total;
    const Map before = block_exclusive(agg, wagg, total);
    uint64_t S = apply(before, S0);
    unsigned long long first = ~0ULL;
    double out[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const uint64_t j = (uint64_t)tid * kItems + i;
      if (j < m && first == ~0ULL && S + a[i] >= kTop) first = j;
      S = apply(elem_map(a[i], cls[i]), S);
      out[i] = (double)S * u;
    }
    if (first != ~0ULL) atomicMin(&cross, first);
    __syncthreads();
    const uint64_t valid = cross < m ? cross : m;
    if (prefix) {
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        const uint64_t j = (uint64_t)tid * kItems + i;
        if (j < valid) prefix[k + j] = out[i];
      }
    }
#pragma unroll
    for (int i = 0; i < kItems; ++i)
      if (valid > 0 && (uint64_t)tid * kItems + i == valid - 1) s_sh = out[i];
    __syncthreads();
    if (valid > 0) s = s_sh;
    __syncthreads();
    if (valid < m && tid == 0) {  // the binade-leaving weight, added for real
      s += wt[valid];
      if (prefix) prefix[k + valid] = s;
      s_sh = s;
    }
    k += valid < m ? valid + 1 : m;
    __syncthreads();
    s = s_sh;
    __syncthreads();
  }
  return s;
}

// Sum of `count` copies of v, sequentially (total_weight of the combed bank):
// inside a binade the m-fold map is found by binary powering.
__device__ double const_walk(double v, uint64_t count) {
  double s = 0.0;
  uint64_t k = 0;
  while (k < count) {
    if (!in_rule(s)) {
      s += v;
      ++k;
      continue;
    }
    const int e = binade(s);
    uint64_t a;
    int cls;
    split(v, e, a, cls);
    if (a >= kTop) {
      s += v;
      ++k;
      continue;
    }
    const uint64_t S = (uint64_t)ldexp(s, 52 - e);
    Map pw[64];
    pw[0] = elem_map(a, cls);
    for (int b = 1; b < 64; ++b) pw[b] = compose(pw[b - 1], pw[b - 1]);
    Map acc{0, 0};
    uint64_t m = 0;
    for (int b = 63; b >= 0; --b) {
      const uint64_t step = 1ULL << b;
      if (step > count - k - m) continue;
      const Map t = compose(acc, pw[b]);
      if (apply(t, S) < kTop) {
        acc = t;
        m += step;
      }
    }
    s = (double)apply(acc, S) * ldexp(1.0, e - 52);
    k += m;
    if (k < count) {  // the binade-leaving add
      s += v;
      ++k;
    }
  }
  return s;
}

struct BankW {
  const hwwg_particle* b;
  __device__ double operator()(uint64_t k) const { return b[k].w; }
};

// tile scratch layout (doubles): [0, nt) approximate tile sums, [nt, 2nt)
// approximate tile starts, [2nt, 3nt) map i0, [3nt, 4nt) map i1, [4nt, 5nt)
// predicted binade (kDirty: walk the tile), [5nt, 6nt) exact tile start (NaN:
// the walk wrote the tile)
struct Tiles {
  double* base;
  uint64_t nt;
  __device__ double* sum() const { return base; }
  __device__ double* start() const { return base + nt; }
  __device__ uint64_t* i0() const { return reinterpret_cast<uint64_t*>(base + 2 * nt); }
  __device__ uint64_t* i1() const { return reinterpret_cast<uint64_t*>(base + 3 * nt); }
  __device__ int64_t* ebin() const { return reinterpret_cast<int64_t*>(base + 4 * nt); }
  __device__ double* exact() const { return base + 5 * nt; }
};
}  // namespace combscan

__global__ void __launch_bounds__(256) k_comb_tile_sums(CombArgs a) {
  using namespace combscan;
  __shared__ double red[8];
  const Tiles T{a.tiles, (a.n + kTile - 1) / kTile};
  const uint64_t k0 = (uint64_t)blockIdx.x * kTile;
  const uint64_t k1 = k0 + kTile < a.n ? k0 + kTile : a.n;
  double v = 0.0;
  for (uint64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) v += a.bank[k].w;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    T.sum()[blockIdx.x] = t;
  }
}

// approximate exclusive prefix of the tile sums (one CTA)
__global__ void __launch_bounds__(1024) k_comb_tile_starts(CombArgs a) {
  using namespace combscan;
  __shared__ double part[1024];
  const Tiles T{a.tiles, (a.n + kTile - 1) / kTile};
  const uint64_t per = (T.nt + 1023) / 1024;
  const uint64_t lo = threadIdx.x * per, hi = lo + per < T.nt ? lo + per : T.nt;
  double v = 0.0;
  for (uint64_t t = lo; t < hi; ++t) v += T.sum()[t];
  part[threadIdx.x] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int i = 0; i < 1024; ++i) {
      const double x = part[i];
      part[i] = r;
      r += x;
    }
  }
  __syncthreads();
  double r = part[threadIdx.x];
  for (uint64_t t = lo; t < hi; ++t) {
    T.start()[t] = r;
    r += T.sum()[t];
  }
}

// per tile: the predicted binade and, when the prediction has margin, the
// tile's composed map
__global__ void __launch_bounds__(combscan::kThreads) k_comb_tile_maps(CombArgs a) {
  using namespace combscan;
  __shared__ Map wagg[kThreads / 32];
  const Tiles T{a.tiles, (a.n + kTile - 1) / kTile};
  const uint64_t t = blockIdx.x;
  const double lo = T.start()[t] * (1.0 - 0x1p-16);
  const double hi = (T.start()[t] + T.sum()[t]) * (1.0 + 0x1p-16);
  const bool ok = in_rule(lo) && in_rule(hi) && binade(lo) == binade(hi);
  if (!ok) {
    if (threadIdx.x == 0) T.ebin()[t] = kDirty;
    return;
  }
  const int e = binade(lo);
  const uint64_t k0 = t * kTile;
  Map agg{0, 0};
  bool off = false;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t k = k0 + threadIdx.x * kItems + i;
    if (k < a.n) {
      uint64_t q;
      int cls;
      split(a.bank[k].w, e, q, cls);
      off |= q >= kTop;
      agg = compose(agg, elem_map(q, cls));
    }
  }
  Map total;
  block_exclusive(agg, wagg, total);
  off = __syncthreads_or(off);
  if (threadIdx.x == 0) {
    T.ebin()[t] = off ? kDirty : e;
    T.i0()[t] = total.i0;
    T.i1()[t] = total.i1;
  }
}

// One CTA, tiles in order: warp 0 applies maps (32 tiles' maps loaded per
// round) while the exact running sum confirms each tile's predicted binade and
// stays inside it; everything else goes through the in-tile walk.
__global__ void __launch_bounds__(combscan::kThreads) k_comb_tile_walk(CombArgs a) {
  using namespace combscan;
  __shared__ double wt[kTile];
  __shared__ double s_sh;
  __shared__ unsigned long long t_sh;
  const Tiles T{a.tiles, (a.n + kTile - 1) / kTile};
  double s = 0.0;
  uint64_t t = 0;
  while (t < T.nt) {
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      bool stop = false;
      while (!stop && t < T.nt) {
        const uint64_t tl = t + lane;
        int64_t e = kDirty;
        uint64_t i0 = 0, i1 = 0;
        if (tl < T.nt) {
          e = T.ebin()[tl];
          i0 = T.i0()[tl];
          i1 = T.i1()[tl];
        }
        const int cnt = T.nt - t < 32 ? (int)(T.nt - t) : 32;
        // fast path: the group's tiles predicted in the binade s is in — one warp
        // scan of their maps, valid up to the first tile that would end at 2^53
        if (in_rule(s)) {
          const int es = binade(s);
          const unsigned same = __ballot_sync(0xffffffffu, lane < cnt && e == es);
          const int run = same == 0xffffffffu ? 32 : __ffs(~same) - 1;  // leading lanes
          if (run > 1) {
            Map inc{i0, i1};
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              Map p;
              p.i0 = __shfl_up_sync(0xffffffffu, inc.i0, o);
              p.i1 = __shfl_up_sync(0xffffffffu, inc.i1, o);
              if (lane >= o) inc = compose(p, inc);
            }
            const uint64_t S = (uint64_t)ldexp(s, 52 - es);
            const uint64_t Se = apply(inc, S);
            const unsigned good = __ballot_sync(0xffffffffu, lane < run && Se < kTop);
            const int n_ok = good == 0xffffffffu ? 32 : __ffs(~good) - 1;
            if (n_ok > 0) {
              const double u = ldexp(1.0, es - 52);
              const double s_end = (double)Se * u;
              const double s_before = __shfl_up_sync(0xffffffffu, s_end, 1);
              if (lane < n_ok) T.exact()[tl] = lane == 0 ? s : s_before;
              s = __shfl_sync(0xffffffffu, s_end, n_ok - 1);
              t += n_ok;
              if (n_ok < run) stop = true;  // the next tile leaves the binade
              continue;
            }
          }
        }
        for (int j = 0; j < cnt; ++j) {  // serial in lane order, every lane in step
          const int64_t ej = __shfl_sync(0xffffffffu, e, j);
          const Map f{__shfl_sync(0xffffffffu, i0, j), __shfl_sync(0xffffffffu, i1, j)};
          if (ej == kDirty || !in_rule(s) || binade(s) != (int)ej) {
            stop = true;
            break;
          }
          const uint64_t S = (uint64_t)ldexp(s, 52 - (int)ej);
          const uint64_t Se = apply(f, S);
          if (Se >= kTop) {
            stop = true;
            break;
          }
          if (lane == 0) T.exact()[t] = s;
          s = (double)Se * ldexp(1.0, (int)ej - 52);
          ++t;
        }
      }
      if (lane == 0) {
        s_sh = s;
        t_sh = t;
      }
    }
    __syncthreads();
    s = s_sh;
    t = t_sh;
    __syncthreads();
    if (t >= T.nt) break;
    // tile t by the in-tile walk, which writes its prefix values
    const uint64_t k0 = t * kTile;
    const uint64_t k1 = k0 + kTile < a.n ? k0 + kTile : a.n;
    s = walk(BankW{a.bank}, k0, k1, s, a.prefix, wt);
    if (threadIdx.x == 0) T.exact()[t] = __longlong_as_double(0x7ff8000000000001LL);
    ++t;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    // total_weight(bank) (particle.hpp:18-22) is the same sequential sum
    const double W = s;
    const double spacing = W / (double)a.target;
    // total_weight(result.bank): every tooth carries `spacing`
    const double ow = a.exact_out_weight ? const_walk(spacing, a.target) : spacing * (double)a.target;
    Xoshiro r;
    r.seed(a.seed, a.stream);
    const double offset = r.uniform() * spacing;
    a.scalars[0] = W;
    a.scalars[1] = spacing;
    a.scalars[2] = offset;
    a.scalars[3] = ow;
  }
}

// the mapped tiles' prefix values, from their exact starts (all tiles in parallel)
__global__ void __launch_bounds__(combscan::kThreads) k_comb_tile_prefix(CombArgs a) {
  using namespace combscan;
  __shared__ Map wagg[kThreads / 32];
  const Tiles T{a.tiles, (a.n + kTile - 1) / kTile};
  const uint64_t t = blockIdx.x;
  const double s = T.exact()[t];
  if (s != s) return;  // walked (NaN marker)
  const int e = (int)T.ebin()[t];
  const double u = ldexp(1.0, e - 52);
  const uint64_t k0 = t * kTile + (uint64_t)threadIdx.x * kItems;
  uint64_t q[kItems];
  int cls[kItems];
  Map agg{0, 0};
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    q[i] = 0;
    cls[i] = 0;
    if (k0 + i < a.n) split(a.bank[k0 + i].w, e, q[i], cls[i]);
    agg = compose(agg, elem_map(q[i], cls[i]));
  }
  Map total;
  const Map before = block_exclusive(agg, wagg, total);
  uint64_t S = apply(before, (uint64_t)ldexp(s, 52 - e));
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    S = apply(elem_map(q[i], cls[i]), S);
    if (k0 + i < a.n) a.prefix[k0 + i] = (double)S * u;
  }
}

// Tooth k lands on the first particle whose cumulative weight exceeds
// offset + k * spacing (the while loop of popctrl.cpp:24-29 is exactly this
// because teeth and the prefix are both non-decreasing); stranded teeth copy
// bank.back() (popctrl.cpp:31-37).
__global__ void k_comb_teeth(CombArgs a) {
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
  const uint64_t src = lo < a.n ? lo : a.n - 1;
  const double2* s = reinterpret_cast<const double2*>(a.bank) + 2 * src;
  double2* d = reinterpret_cast<double2*>(a.out) + 2 * k;
  const double2 s1 = s[1];
  d[0] = s[0];
  d[1] = make_double2(spacing, s1.y);
}

__global__ void __launch_bounds__(kCtaThreads) k_build_centers(const double* phi, int n,
                                                               double eps_min, double* centers,
                                                               int* fallback) {
  __shared__ double red[32];
  const bool fb = build_centers_cta(phi, n, eps_min, centers, red);
  if (threadIdx.x == 0) *fallback = fb ? 1 : 0;
}

__global__ void __launch_bounds__(kCtaThreads) k_moving_average(const double* g, int n, int k,
                                                                double* out) {
  if (k == 0) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = g[i];
    return;
  }
  moving_average_cta(g, n, k, out);
}

__global__ void k_device_log(const double* x, uint64_t n, double* out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = hwwg_libm_log(x[i]);
}

}  // namespace

size_t lo_fac_words(int I) { return I + 2 <= 512 ? fac_words_for(I) : 0; }

void launch_low_order_update(const LowOrderArgs& a_in, cudaStream_t st) {
  LowOrderArgs a = a_in;
  static const bool dbg = std::getenv("HWWG_LOSM_DEBUG") != nullptr;
  static const bool general = std::getenv("HWWG_LOSM_GENERAL") != nullptr;  // tests
  a.debug = dbg ? 1 : 0;
  if (a.mode == 1 && a.fast_solve && a.s.fac && !a.refactor && !a.fourier_tab_cell &&
      a.I + 2 <= kCtaThreads && a.I + 2 <= (1 << kFacLevels) && !dbg && !general) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(kCtaThreads);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = a.pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    HWWG_CUDA(cudaLaunchKernelEx(&cfg, k_losm_mid_fast, a));
    return;
  }
  size_t smem = a.fast_solve ? (size_t)4 * (a.I + 2) * sizeof(double) : 0;
  a.smem_state = a.I <= kSmemStateMaxI ? 1 : 0;
  if (a.smem_state)
    smem += ((size_t)6 * (2 * a.I + 3) + (size_t)3 * (a.I + 2) + (a.I + 1) + a.I) * sizeof(double);
  static DynSmemCache configured;
  ensure_dyn_smem(k_low_order_update, smem, configured);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(kCtaThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = a.pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  HWWG_CUDA(cudaLaunchKernelEx(&cfg, k_low_order_update, a));
}

void launch_finalize(const FinalizeArgs& a, cudaStream_t st) {
  const int blocks = (a.I + 1 + 255) / 256;
  k_finalize<<<blocks, 256, 0, st>>>(a);
  HWWG_CUDA(cudaGetLastError());
}

size_t comb_tile_words(uint64_t n) { return 6 * ((n + combscan::kTile - 1) / combscan::kTile) + 1; }

void launch_comb(const CombArgs& a, cudaStream_t st) {
  const unsigned nt = (unsigned)((a.n + combscan::kTile - 1) / combscan::kTile);
  k_comb_tile_sums<<<nt, 256, 0, st>>>(a);
  k_comb_tile_starts<<<1, 1024, 0, st>>>(a);
  k_comb_tile_maps<<<nt, combscan::kThreads, 0, st>>>(a);
  k_comb_tile_walk<<<1, combscan::kThreads, 0, st>>>(a);
  k_comb_tile_prefix<<<nt, combscan::kThreads, 0, st>>>(a);
  const unsigned blocks = (unsigned)((a.target + 255) / 256);
  k_comb_teeth<<<blocks, 256, 0, st>>>(a);
  HWWG_CUDA(cudaGetLastError());
}

void launch_build_centers(const double* phi, int n, double eps_min, double rho, double* centers,
                          int* fallback, cudaStream_t st) {
  (void)rho;
  k_build_centers<<<1, kCtaThreads, 0, st>>>(phi, n, eps_min, centers, fallback);
  HWWG_CUDA(cudaGetLastError());
}

// Host: the reference's twiddles for an M-point transform (filters.cpp:33-47):
// w0 = 2 pi / M, forward angle (-w0 * j) * m, inverse (w0 * j) * m, through the
// host libm cos/sin (std::polar(1, a) = (cos a, sin a)). Layout: forward
// [m][j], inverse [j][m].
std::vector<double> fourier_tables(int M) {
  const size_t MM = (size_t)M * M;
  std::vector<double> t(4 * MM);
  const double w0 = 2.0 * 3.141592653589793 / M;  // std::numbers::pi
  for (int j = 0; j < M; ++j)
    for (int m = 0; m < M; ++m) {
      const double af = -w0 * j * m;
      const double ai = w0 * j * m;
      t[(size_t)m * M + j] = std::cos(af);
      t[MM + (size_t)m * M + j] = std::sin(af);
      t[2 * MM + (size_t)j * M + m] = std::cos(ai);
      t[3 * MM + (size_t)j * M + m] = std::sin(ai);
    }
  return t;
}

__global__ void __launch_bounds__(kCtaThreads) k_fourier(double* g, int n, int cutoff,
                                                          const double* tab, double* tmp) {
  fourier_cta(g, n, cutoff, tab, tmp);
}

void launch_fourier_lowpass(double* g, int n, int cutoff, const double* tab, double* tmp,
                            cudaStream_t st) {
  k_fourier<<<1, kCtaThreads, 0, st>>>(g, n, cutoff, tab, tmp);
  HWWG_CUDA(cudaGetLastError());
}

void launch_moving_average(const double* g, int n, int k, double* out, cudaStream_t st) {
  k_moving_average<<<1, kCtaThreads, 0, st>>>(g, n, k, out);
  HWWG_CUDA(cudaGetLastError());
}

void launch_raw_losm(const RawLosmArgs& a, cudaStream_t st) {
  k_raw_losm<<<1, kCtaThreads, 0, st>>>(a);
  HWWG_CUDA(cudaGetLastError());
}

void launch_device_log(const double* x, uint64_t n, double* out, cudaStream_t st) {
  if (!n) return;
  k_device_log<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(x, n, out);
  HWWG_CUDA(cudaGetLastError());
}

}  // namespace hwwg
