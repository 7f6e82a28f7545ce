// Between-segment pipeline on the device:
// partial snapshot -> boundary extrapolation -> moving-average filter ->
// LOSM assembly -> tridiagonal solve -> weight-window centres, all in ONE
// single-CTA kernel launch per window update, plus the step-end finalize and
// the comb.  Compiled with -fmad=false: every value is bit-identical to the
// reference given identical inputs (tests/test_gpu_components.py).
#pragma once

#include <vector>

#include "common.cuh"

namespace hwwg {

// Persistent per-run low-order state on the device.
struct LowOrderState {
  // filtered HybridInputs of the current step (driver.hpp:15-21)
  double* phi_prev;  // I+2
  double* J_prev;    // I+1
  double* F_prev;    // I+2
  double* PLPR_prev; // 2
  // previous step's report (census moments, tally.cpp means) feeding the next step
  double* rep_phi_census;  // I
  double* rep_current;     // I
  double* rep_closure;     // I
  double* rep_PLPR;        // 2
  // windows (WeightWindowGrid) and the last hybrid solution
  double* centers;    // I
  double* phi_hybrid; // I
  int* flags;         // [0] windows active, [1] has_hybrid, [2] updates_applied, [3] failed,
                      // [4] last solve status (0 ok, 1 invalid, 2 singular)
  // scratch for the n = 2I+3 system (lower, diag, upper, rhs, fill, x) and F_now
  double* sys;   // 6 * (2I+3)
  double* F_now; // I+2
  // throughput mode: the Schur + PCR factorization of the LOSM matrix, which
  // depends only on mesh, materials, theta and dt (lo_fac_words(I) doubles;
  // null = refactor every solve)
  double* fac;
};
// doubles of LowOrderState::fac for I cells (0 when the cached path does not apply)
size_t lo_fac_words(int I);

struct LowOrderArgs {
  int I;
  int smem_state;  // set by launch_low_order_update: state + system in shared memory
  int debug;       // HWWG_LOSM_DEBUG: printf per-phase cycle counts
  const double* edges;
  const CellInfo* cells;
  double theta, dt;
  double eps_min, rho;
  int ma_k;  // moving-average half-width, 0 = no filter
  // hww_fourier: fourier_tables(I) / fourier_tables(I + 1) on the device (null
  // = no Fourier filter) and the retained-mode bound
  const double* fourier_tab_cell;
  const double* fourier_tab_edge;
  int fourier_cutoff;
  const double* q;  // config-3 volumetric source per cell (I, device) or null (losm.cpp:101-103)
  // mode 0: start-of-step lagged solve; inputs from analytic pulse (step 1) or
  //         from the previous report.  mode 1: mid-step implicit solve from the
  //         partial snapshot of the live tallies.
  int mode;
  int fast_solve;  // throughput mode: Schur complement + parallel cyclic reduction
  int refactor;    // fast_solve with s.fac: 1 = (re)build the cached factorization
  int analytic;        // mode 0: step 1 cold start
  int pulse_cell;      // analytic: cell of the source point
  double pulse_value;  // analytic: speed * strength / dx
  const double* closure_tally;  // mode 1: census_closure accumulator (I)
  const double* bclosure_tally; // mode 1: boundary closure accumulators (2)
  double snapshot_inv_norm;     // mode 1: 1 / (H_cfg * h_done / H)
  // throughput mode: reset the transport pool counters for the next segment
  // (fast_pool_reset) so that launch needs no reset kernel of its own
  unsigned long long* pool_ctl;
  unsigned long long* pool_src_head;
  unsigned long long* pool_span;  // the next segment's launch span (FastArgs::span)
  int pdl;  // 1: programmatic dependent launch after the previous kernel
  // mode 0 at a step start (nullable): copy the incoming centres (I) and
  // flags (8) here first (the replay backup), then zero the record flags 1..4
  double* backup_centers;
  int* backup_flags;
  LowOrderState s;
};

void launch_low_order_update(const LowOrderArgs& a, cudaStream_t st);

// tally.cpp:68-128 finalize on the device (one CTA per 256 cells).
struct FinalizeArgs {
  int I, B;
  TallyPtrs t;
  uint64_t histories;
  double normalization;
  // outputs (device)
  double *phi_track, *sigma, *phi_census, *current, *closure, *edge;  // I / I+1
  double* scalars;  // PL, PR, census_weight, census_weight_sigma, sigma_valid
  // throughput mode scores the batch table only: track_flux[i] = sum over b of
  // track_flux_batch[b][i] (b ascending) is formed here first
  int track_from_batches;
};
void launch_finalize(const FinalizeArgs& a, cudaStream_t st);

// popctrl.cpp:7-42 on the device.  Exact mode: the cumulative weight walk is
// evaluated sequentially (the reference's fp64 summation order), teeth are
// then placed in parallel by binary search over the exact prefix.
struct CombArgs {
  const hwwg_particle* bank;
  uint64_t n;
  uint64_t target;
  uint64_t seed, stream;
  double* prefix;    // n scratch
  double* scalars;   // [0] W, [1] spacing, [2] offset, [3] output weight
  hwwg_particle* out;
  int exact_out_weight;
  double* tiles;     // comb_tile_words(n) scratch
};
size_t comb_tile_words(uint64_t n);
void launch_comb(const CombArgs& a, cudaStream_t st);

// Component entry points used by the C ABI (hwwg_build_centers etc.).
void launch_build_centers(const double* phi, int n, double eps_min, double rho,
                          double* centers, int* fallback, cudaStream_t st);
void launch_moving_average(const double* g, int n, int k, double* out, cudaStream_t st);
// filters.cpp:26-52 on the device with host twiddles (fourier_tables(n));
// tmp: 3n doubles of device scratch; g is filtered in place
std::vector<double> fourier_tables(int M);
void launch_fourier_lowpass(double* g, int n, int cutoff, const double* tab, double* tmp,
                            cudaStream_t st);
struct RawLosmArgs {
  int I;
  const double* edges;
  const CellInfo* cells;
  const double *phi_prev, *J_prev;
  double J_L, J_R;
  int implicit;
  const double* F_now;
  double PL_now, PR_now;
  const double* F_prev;
  double PL_prev, PR_prev, theta, dt;
  const double* q;  // may be null
  double* sys;      // 6*(2I+3) scratch
  double *phi_out, *J_out;
  int* status;
};
void launch_raw_losm(const RawLosmArgs& a, cudaStream_t st);
void launch_device_log(const double* x, uint64_t n, double* out, cudaStream_t st);

}  // namespace hwwg
