/*
 * TEST INFRASTRUCTURE — CPU oracle for the hybrid weight-window history loop.
 *
 * A plain-C restatement of the reference algorithm (arxiv 2512.19925,
 * /root/reference/proj) used ONLY by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py, as the checker. The product path never links
 * or calls anything in oracle/.
 *
 * Parity pin: every function here is checked bit-for-bit against the real
 * reference compiled by oracle/Makefile into oracle/_ref/libhww_ref.so and
 * against the golden vectors in tests/golden/ (tests/test_oracle_pin.py).
 * Tally summation follows the reference's 256-history chunk merge order
 * (proj/src/transport.cpp:209-237), so oracle tallies are bit-identical to the
 * reference's run_segment_parallel, not just within 1e-12.
 */
#ifndef HWW_ORACLE_H
#define HWW_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { double x, mu, w, t; } orc_particle;
typedef struct { double sigma_t, sigma_s, sigma_f, nu_f, speed; } orc_material;

typedef struct {
  uint64_t collisions, splits, split_daughters, capped_splits, roulette_kills,
      roulette_survivals, census_count, event_cap_aborts, nan_aborts;
  double leakage_weight, aborted_weight;
} orc_counters;

typedef struct {
  double* track_flux;           /* I   */
  double* track_flux_batch;     /* B*I */
  double* census_phi;           /* I   */
  double* census_current;       /* I   */
  double* census_closure;       /* I   */
  double* census_weight_batch;  /* B   */
  double* edge_current;         /* I+1 */
  double boundary_closure_left;
  double boundary_closure_right;
  uint64_t histories_scored;
  uint64_t grazing_discarded;
} orc_tallies;

typedef struct {
  orc_particle* data;
  uint64_t n, cap;
} orc_bank;

/* Same field order as the reference shim's hwwref_config. */
typedef struct {
  int32_t mode; /* 0 analog, 1 lww, 2 hww, 3 hww_ma, 4 hww_fourier */
  int32_t u_ww;
  uint64_t histories_per_step;
  double theta, rho, eps_min;
  int32_t n_fractions;
  int32_t ma_base_k;
  double fractions[8];
  int32_t fourier_cutoff;
  int32_t batches;
  uint64_t seed;
  uint64_t target_population;
  double comb_overflow_factor;
  double x0, t0, strength;
  double sigma_t, sigma_s, sigma_f, nu_f, speed;
  double x_min, x_max;
  int32_t cells;
  int32_t time_steps;
  double t_end;
  int32_t threads;
  int32_t pad_;
  /* Config-3 extensions (absent from the reference driver,
   * DESIGN.md "Config-3 features"): */
  int32_t n_regions;         /* 0: every cell takes the material above */
  int32_t no_pulse;          /* 1: no point pulse at t = 0 */
  double region_x_hi[8];     /* cell i takes the first region with centre < x_hi */
  double region_mat[8][5];   /* sigma_t, sigma_s, sigma_f, nu_f, speed per region */
  double vol_x_lo, vol_x_hi; /* isotropic volumetric source box in x ... */
  double vol_t_lo, vol_t_hi; /* ... and in t */
  double vol_rate;           /* emitted weight per unit time (same normalisation as strength) */
  uint64_t vol_histories;    /* particles sampled in every step the box overlaps */
} orc_config;

typedef struct {
  int32_t step;
  int32_t updates_applied;
  int32_t hybrid_solve_failed;
  int32_t n_thresholds;
  uint64_t thresholds[8];
  double t_begin, t_end, tau;
  uint64_t histories;
  uint64_t comb_in, comb_out;
  double comb_in_weight, comb_out_weight;
  orc_counters counters;
  uint64_t segments;
  uint64_t census_size;
  double census_weight, census_weight_sigma;
  double boundary_closure_left, boundary_closure_right;
  double fom_sigma_l2;
  int32_t sigma_valid;
  int32_t has_windows;
  int32_t has_hybrid;
  int32_t pad_;
} orc_step_out;

const char* orc_last_error(void);

/* rng.hpp:10-59 */
void orc_stream_uniforms(uint64_t seed, uint64_t stream_id, uint64_t n, double* out);
void orc_stream_u64(uint64_t seed, uint64_t stream_id, uint64_t n, uint64_t* out);
uint64_t orc_stream_id(uint64_t step, uint64_t history, uint64_t purpose);

/* std::log as the reference calls it (transport.cpp:26) */
void orc_log_array(const double* x, uint64_t n, double* out);

/* mesh.cpp:26-50 */
void orc_uniform_edges(double x_min, double x_max, int32_t cells, double* out);
int32_t orc_locate(const double* edges, int32_t cells, double x);

/* transport.cpp:13-22 with the driver's source stream (driver.cpp:309-316) */
void orc_pulse_source(uint64_t seed, uint64_t histories, double x0, double strength,
                      orc_particle* out);

/* transport.cpp:194-237: one segment of histories [h_begin, h_begin+n).
 * chunk <= 0 selects the serial path; otherwise the reference's chunked
 * merge order (run_segment_parallel) is reproduced. census may be NULL. */
int orc_run_segment(const double* edges, int32_t cells, const orc_material* mats,
                    double t_begin, double t_end, uint64_t seed, int32_t step,
                    uint64_t histories_total, int32_t batches, const orc_particle* source,
                    uint64_t n, uint64_t h_begin, const double* centers, double rho,
                    int32_t chunk, orc_tallies* t, orc_counters* counters,
                    uint64_t* tracks_per_cell, orc_bank* census,
                    uint32_t* max_stack_runs);

void orc_bank_free(orc_bank* b);

/* tally.cpp:68-128 (scalars: PL, PR, census_weight, census_weight_sigma, sigma_valid) */
int orc_report(int32_t cells, int32_t batches, const orc_tallies* t, uint64_t histories,
               uint64_t histories_total, double normalization, int32_t snapshot,
               double* phi_track, double* sigma, double* phi_census, double* current,
               double* closure, double* edge, double* scalars);

/* banded.cpp:8-38; returns 0 or -1-row */
int orc_solve_tridiagonal(int32_t n, const double* lower, const double* diag,
                          const double* upper, const double* rhs, double* x);

/* losm.cpp:143-165 */
int orc_assemble_solve(int32_t cells, const double* edges, const orc_material* mats,
                       const double* phi_prev, const double* J_prev, double J_L, double J_R,
                       int32_t implicit, const double* F_now, double PL_now, double PR_now,
                       const double* F_prev, double PL_prev, double PR_prev, double theta,
                       double dt, const double* q, double* phi_out, double* J_out);

/* losm.cpp:12-32 */
int orc_edge_currents(const double* census_current, int32_t cells, const double* edges,
                      double* out);
/* filters.cpp:11-24 */
int orc_moving_average(const double* g, int32_t n, int32_t k, double* out);
int orc_fourier_lowpass(const double* g, int32_t n, int32_t cutoff, double* out);
void orc_volume_source(uint64_t seed, int step, uint64_t n, double x_lo, double x_hi, double ta,
                       double tb, double rate, uint64_t h_cfg, orc_particle* out);
void orc_volume_q(const double* edges, int I, double x_lo, double x_hi, double ta, double tb,
                  double dt, double rate, double* q);
/* ww.cpp:8-32; returns 1 on uniform fallback */
int orc_build_centers(const double* phi, int32_t n, double eps_min, double rho,
                      double* centers);
/* ww.cpp:74-87 */
int orc_update_thresholds(uint64_t histories, const double* f, int32_t n, uint64_t* out);
/* popctrl.cpp:7-42 */
int orc_uniform_comb(const orc_particle* bank, uint64_t n, uint64_t target, uint64_t seed,
                     uint64_t stream_id, orc_particle* out, double* in_w, double* out_w);

/* driver.cpp:99-342, stepwise */
void* orc_driver_create(const orc_config* c);
void orc_driver_destroy(void* h);
int orc_driver_step(void* h, orc_step_out* out);
void orc_driver_arrays(void* h, double* phi_track, double* phi_sigma, double* phi_census,
                       double* current_census, double* closure_census, double* edge_current,
                       double* ww_centers, double* phi_hybrid, uint64_t* tracks_per_cell);
uint64_t orc_driver_bank(void* h, orc_particle* out, uint64_t cap);

#ifdef __cplusplus
}
#endif
#endif
