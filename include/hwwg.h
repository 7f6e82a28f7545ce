/*
 * hwwg — B200-native engine for the hybrid weight-window time-dependent Monte
 * Carlo history loop (arxiv 2512.19925).  C ABI: plain pointers and sizes, no
 * exceptions, no C++ or torch types.  Every entry point returns an int status
 * (HWWG_OK == 0, negative on error; hwwg_last_error() holds the message) unless
 * stated otherwise.  All host pointers are caller-owned and never retained.
 *
 * Boundary:
 *   hwwg_run_segment_parallel  replaces  hww::run_segment_parallel
 *       proj/include/hww/transport.hpp:117-120 / proj/src/transport.cpp:209-237
 *       (and its serial twin transport.hpp:109-111) — same inputs (StepContext,
 *       source span, h_begin, nullable window grid) and the same accumulate-into-
 *       caller semantics for TallySet / StepOutcome; std::invalid_argument
 *       becomes HWWG_EINVAL.
 *   hwwg_driver_*              replaces  hww::run / hww::run_step
 *       proj/include/hww/driver.hpp:80-88 (device-resident time-step loop:
 *       comb -> LOSM windows -> segments with mid-step updates -> finalize).
 *   hwwg_losm_assemble_solve   replaces  hww::assemble_solve
 *       proj/include/hww/losm.hpp:77-80 (single-CTA device solve).
 *   hwwg_build_centers         replaces  hww::build_centers  proj/include/hww/ww.hpp:34-35
 *   hwwg_moving_average        replaces  hww::moving_average proj/include/hww/filters.hpp:30
 *   hwwg_fourier_lowpass       replaces  hww::fourier_lowpass proj/include/hww/filters.hpp:36
 *   hwwg_uniform_comb          replaces  hww::uniform_comb   proj/include/hww/popctrl.hpp:22
 *
 * Calls on one context are single-threaded; device work runs on the context's
 * own CUDA stream; calls that return host data synchronise that stream.
 */
#ifndef HWWG_H
#define HWWG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HWWG_OK 0
#define HWWG_EINVAL (-1)    /* invalid argument (reference: std::invalid_argument) */
#define HWWG_ECUDA (-2)     /* CUDA runtime failure or no device */
#define HWWG_ENOMEM (-3)    /* device allocation failed */
#define HWWG_ESTATE (-4)    /* call out of order */
#define HWWG_ESINGULAR (-5) /* LOSM system singular (reference: std::runtime_error) */
#define HWWG_ENOSPC (-6)    /* caller buffer too small; *needed is set */
#define HWWG_ESTACK (-7)    /* exact-mode daughter stack exceeded its run capacity */
#define HWWG_EFORMAT (-8)   /* reference file missing, malformed or of the wrong shape
                               (reference: std::runtime_error from load_reference) */

#define HWWG_RNG_EXACT 0  /* replay the reference's xoshiro256** streams bit-for-bit */
#define HWWG_RNG_PHILOX 1 /* event-based throughput mode, counter-based Philox4x32-10 */

typedef struct hwwg_ctx hwwg_ctx;
typedef struct hwwg_driver hwwg_driver;
typedef struct hwwg_loopback hwwg_loopback;

/* == hww::Particle (proj/include/hww/particle.hpp:9-14), 32 bytes. */
typedef struct { double x, mu, w, t; } hwwg_particle;

/* == hww::Material (proj/include/hww/material.hpp:9-18). */
typedef struct { double sigma_t, sigma_s, sigma_f, nu_f, speed; } hwwg_material;

/* == hww::StepCounters (proj/include/hww/transport.hpp:37-63). */
typedef struct {
  uint64_t collisions, splits, split_daughters, capped_splits, roulette_kills,
      roulette_survivals, census_count, event_cap_aborts, nan_aborts;
  double leakage_weight, aborted_weight;
} hwwg_counters;

/* == hww::StepContext (proj/include/hww/transport.hpp:83-94); the mesh is given
 * by its I+1 strictly increasing edges, materials per cell. */
typedef struct {
  const double* edges;
  int32_t cells;
  int32_t batches;
  const hwwg_material* materials;
  double t_begin, t_end;
  uint64_t seed;
  int32_t step_index;
  int32_t pad_;
  uint64_t histories_total;
} hwwg_step_context;

/* == hww::WeightWindowGrid (proj/include/hww/ww.hpp:13-27); NULL grid = analog. */
typedef struct {
  const double* centers; /* I */
  double rho;
  double eps_min;
} hwwg_window_grid;

/* == hww::TallySet (proj/include/hww/tally.hpp:16-45), caller-owned arrays that
 * the engine ACCUMULATES into (any array pointer may be NULL to skip it). */
typedef struct {
  double* track_flux;          /* I   */
  double* track_flux_batch;    /* B*I */
  double* census_phi;          /* I   */
  double* census_current;      /* I   */
  double* census_closure;      /* I   */
  double* census_weight_batch; /* B   */
  double* edge_current;        /* I+1 */
  double boundary_closure_left;
  double boundary_closure_right;
  uint64_t histories_scored;
  uint64_t grazing_discarded;
} hwwg_tally_set;

/* == hww::StepOutcome (proj/include/hww/transport.hpp:67-80): the census is
 * APPENDED at census[census_size...] (reference emission order), counters and
 * tracks_per_cell are summed.  If census_capacity is too small the call fails
 * with HWWG_ENOSPC, sets census_needed and leaves every output untouched. */
typedef struct {
  hwwg_particle* census;
  uint64_t census_size;
  uint64_t census_capacity;
  uint64_t census_needed;
  hwwg_counters counters;
  uint64_t* tracks_per_cell; /* I */
} hwwg_step_outcome;

/* Engine construction: the problem that stays resident on the device. */
typedef struct {
  int32_t device;        /* CUDA ordinal */
  int32_t rng_mode;      /* HWWG_RNG_EXACT or HWWG_RNG_PHILOX */
  uint64_t bank_capacity;/* initial particle capacity of each device bank (grows) */
  /* Multi-GPU driver (one process per GPU); world <= 1 means
   * single GPU. nccl_id: the bytes of an ncclUniqueId made by rank 0 with
   * hwwg_nccl_unique_id and broadcast by the caller (torch.distributed). */
  int32_t rank;
  int32_t world;
  uint8_t nccl_id[128];
  /* Non-NULL: the ranks are host threads of THIS process on one device and
   * exchange through this in-process hub instead of NCCL (tests of the
   * multi-rank driver on one GPU; world must equal the hub's). */
  hwwg_loopback* loopback;
} hwwg_options;

/* ncclGetUniqueId for the multi-GPU driver (out: 128 bytes). */
int hwwg_nccl_unique_id(uint8_t* out);
/* The driver's NCCL calls (run-time load, unique id, CommInitRank, sum/max
 * all-reduce, all-gather, grouped send/recv) on a one-rank communicator on
 * `device`, results checked; report (nullable) gets "ok" or the mismatches. */
int hwwg_nccl_selftest(int32_t device, uint8_t* report, uint64_t report_bytes);
/* In-process collective hub for `world` driver ranks on `device`: the drivers
 * share one CUDA stream and meet at a host barrier in every collective (each
 * rank's hwwg_driver_step must run on its own host thread). */
int hwwg_loopback_create(int32_t world, int32_t device, hwwg_loopback** out);
void hwwg_loopback_destroy(hwwg_loopback* hub);

/* Host-side sharding plan shared by every rank (pure functions):
 * shard(rank) = [H*rank/world, H*(rank+1)/world). */
void hwwg_shard_range(uint64_t H, int32_t rank, int32_t world, uint64_t* lo, uint64_t* hi);
/* Global comb across ranks (popctrl.cpp:7-42 over the rank-ordered concatenated
 * census): from every rank's census weight total, this rank's tooth range
 * [k_lo, k_hi), the spacing, the offset (offset_frac * spacing) and the rank's
 * origin on the cumulative-weight axis. */
int hwwg_comb_plan(const double* rank_weights, int32_t world, int32_t rank, uint64_t target,
                   double offset_frac, double* spacing, double* offset, double* rank_origin,
                   uint64_t* k_lo, uint64_t* k_hi);
/* Census rebalance after the comb: per peer, teeth to send (count, first
 * tooth) and teeth to receive so each rank holds its next-step shard. */
void hwwg_rebalance_plan(const uint64_t* k_lo_all, const uint64_t* k_hi_all, int32_t world,
                         int32_t rank, uint64_t H, uint64_t* send, uint64_t* send_first,
                         uint64_t* recv);

const char* hwwg_last_error(void);
const char* hwwg_version(void);

int hwwg_create(const hwwg_options* opts, hwwg_ctx** out);
void hwwg_destroy(hwwg_ctx* ctx);

/* Drop-in for hww::run_segment_parallel (transport.hpp:117-120): histories
 * [h_begin, h_begin + n) of step ctx->step_index, source[0..n) on the HOST.
 * Copies the source to the device, runs the history loop, accumulates the
 * tallies/counters/tracks and appends the census in reference order. */
int hwwg_run_segment_parallel(hwwg_ctx* ctx, const hwwg_step_context* step,
                              const hwwg_particle* source, uint64_t n, uint64_t h_begin,
                              const hwwg_window_grid* ww, hwwg_tally_set* tallies,
                              hwwg_step_outcome* outcome);

/* ------------------------------------------------------------------ driver */
/* == hww::RunConfig (proj/include/hww/config.hpp:33-66) plus engine options. */
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
  int32_t threads; /* accepted for config-file parity; unused */
  int32_t host_bank; /* 1: bank round-trips through host memory each step (e2e) */
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
  /* RunConfig::reference (config.hpp:64): "auto" | reference file path | "" (none).
   * Carried for the tools and run.json; the driver takes the reference itself
   * through hwwg_driver_set_reference / hwwg_driver_load_reference, as hww::run
   * takes a ReferenceSolution* (driver.hpp:88). */
  char reference[256];
} hwwg_run_config;

/* == hww::StepRecord scalars (proj/include/hww/driver.hpp:41-56). */
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
  hwwg_counters counters;
  uint64_t segments; /* sum of tracks_per_cell: the throughput unit */
  uint64_t census_size;
  double census_weight, census_weight_sigma;
  double boundary_closure_left, boundary_closure_right;
  double fom_sigma_l2;
  int32_t sigma_valid;
  int32_t has_windows;
  int32_t has_hybrid;
  /* 1: the step's census was thinned on the fly (throughput mode): the bank the
   * next comb reads holds ~k x target records of weight n * s0 (an unbiased
   * equal-quantum restatement of the census), not census_size */
  int32_t thinned;
  double device_ms;    /* CUDA-event time of the whole step on the engine stream */
  double transport_ms; /* CUDA-event time of the transport (history) kernels only */
  uint64_t transport_launches; /* transport kernel launches in the step */
  uint64_t kernel_launches;    /* all engine kernel launches in the step */
  uint64_t h2d_bytes, d2h_bytes; /* host<->device bytes moved by the step (host_bank mode) */
  /* StepMetrics against a deterministic reference (metrics.hpp:41-51; driver.cpp:231-271);
   * NaN without one (fom_sigma_l2 above is set either way). */
  double rel_l2_error, rel_mod_l2_error, hybrid_rel_l2_error;
  double fom_err_l2, fom_err_mod, fom_sigma_mod, alpha;
} hwwg_step_record;

int hwwg_driver_create(const hwwg_run_config* cfg, const hwwg_options* opts,
                       hwwg_driver** out);
void hwwg_driver_destroy(hwwg_driver* d);
/* Runs the next time step (driver.cpp:99-284); fills *rec. */
int hwwg_driver_step(hwwg_driver* d, hwwg_step_record* rec);
/* Per-cell arrays of the last step (any pointer may be NULL). */
int hwwg_driver_arrays(hwwg_driver* d, double* phi_track, double* phi_sigma,
                       double* phi_census, double* current_census, double* closure_census,
                       double* edge_current, double* ww_centers, double* phi_hybrid,
                       uint64_t* tracks_per_cell);
/* Census bank after the last step (the next step's comb input): reference
 * order in exact mode; in Philox mode the banked particles in completion order
 * (after a thinned step, rec.thinned, the ~k x target equal-quantum records the
 * next comb reads), or with host_bank the next step's combed source.  Waits for
 * a pipelined host-bank download still in flight.  Returns HWWG_ENOSPC with
 * *n = size when cap is too small. */
int hwwg_driver_bank(hwwg_driver* d, hwwg_particle* out, uint64_t cap, uint64_t* n);
/* The deterministic reference for the step diagnostics (hww::run's
 * ReferenceSolution*, driver.hpp:88): phi_layer[(steps+1)*cells] layer values,
 * phi_interval[steps*cells] interval averages of steps 1..N (ReferenceSolution,
 * reference.hpp:76-85).  name goes to run.json's "reference" (NULL keeps
 * cfg.reference).  After this every step fills the record's metric fields. */
int hwwg_driver_set_reference(hwwg_driver* d, const double* phi_layer,
                              const double* phi_interval, const char* name);
/* hww::load_reference on the driver's own mesh and time grid, then
 * hwwg_driver_set_reference(d, ..., path) (hww_main.cpp:250-252). */
int hwwg_driver_load_reference(hwwg_driver* d, const char* path);
/* reference = "auto" (hww_main.cpp:240-249): hww::compute_reference on the driver's
 * device (hwwg_compute_reference), then hwwg_driver_set_reference(d, ..., "auto"). */
int hwwg_driver_compute_reference(hwwg_driver* d, int32_t space_refine, int32_t time_refine,
                                  int32_t sn_order);
/* Key = value config file (proj/tools/hww_main.cpp:20-92 key names). */
int hwwg_load_config_file(const char* path, hwwg_run_config* cfg);
/* Reference defaults (config.hpp:33-66). */
void hwwg_default_config(hwwg_run_config* cfg);
/* validate_config (proj/src/config.cpp:27-69): number of violations, messages
 * joined with '\n' into buf. */
int hwwg_validate_config(const hwwg_run_config* cfg, char* buf, uint64_t buf_len);

/* ---------------------------------------------------------- output files */
/* The reference's run outputs (proj/src/driver.cpp:355-438), same bytes for
 * equal records: step_<n>.csv (write_step_csv; ww_centers / phi_hybrid NULL
 * print as nan, sigma prints as nan unless rec->sigma_valid), summary.csv over
 * recs[0..n) (write_summary_csv; the metric fields as the records carry them, NaN
 * without a reference), run.json (write_run_json; "reference" = cfg->reference).
 * dir is created if missing. */
int hwwg_write_step_csv(const char* dir, const hwwg_step_record* rec, int32_t cells,
                        const double* edges, const double* phi_track, const double* sigma,
                        const double* phi_census, const double* current, const double* closure,
                        const double* ww_centers, const double* phi_hybrid,
                        const uint64_t* tracks, double normalization);
int hwwg_write_summary_csv(const char* dir, const hwwg_step_record* recs, uint64_t n);
int hwwg_write_run_json(const char* dir, const hwwg_run_config* cfg, double total_seconds,
                        uint64_t steps_completed);
/* hww::run's per-step writing (driver.cpp:318-321): step_<last>.csv and
 * summary.csv of every step so far; final != 0 also writes run.json with
 * total_seconds. */
int hwwg_driver_write(hwwg_driver* d, const char* dir, int32_t final, double total_seconds);

/* ------------------------------------------------- reference solution */
/* hww::save_reference (proj/src/reference.cpp:374-393), same bytes: one row per
 * (layer, cell) "t_layer, cell_index, x_center, phi_layer, phi_interval_avg",
 * precision 17, layer 0's interval as nan.  edges[cells+1], layers[steps+1],
 * phi_layer[(steps+1)*cells], phi_interval[steps*cells]. */
int hwwg_save_reference_csv(const char* path, int32_t cells, const double* edges,
                            int32_t steps, const double* layers, const double* phi_layer,
                            const double* phi_interval);
/* hww::load_reference (reference.cpp:395-456): same parse and shape checks (cell
 * index, layer time within 1e-9, centre within 1e-9 of the mesh span, row count),
 * failing with HWWG_EFORMAT and the reference's message; outputs untouched on
 * failure.  phi_interval may be NULL. */
int hwwg_load_reference_csv(const char* path, int32_t cells, const double* edges,
                            int32_t steps, const double* layers, double* phi_layer,
                            double* phi_interval);
/* RunConfig::make_time_grid layers (config.hpp:88; time_grid.hpp:22-29): steps+1 values. */
int hwwg_time_layers(const hwwg_run_config* cfg, double* layers);
/* hww::run_step's diagnostics (driver.cpp:231-275; metrics.cpp:8-66) from a step's
 * arrays: reads rec->tau and rec->sigma_valid, writes rec's fom_sigma_l2 and metric
 * fields.  ref_interval == NULL: no reference (fom_sigma_l2 only); otherwise
 * ref_layer / ref_layer_prev are the reference's layers n and n-1.  phi_hybrid NULL:
 * no hybrid solve.  HWWG_EINVAL when the reference layer is all zero (relative_change). */
int hwwg_step_metrics(int32_t cells, const double* edges, const double* phi_track,
                      const double* phi_sigma, const double* phi_hybrid,
                      const double* ref_interval, const double* ref_layer,
                      const double* ref_layer_prev, hwwg_step_record* rec);

/* ------------------------------------------------------ S_N reference */
/* GaussLegendre::order (reference.cpp:14-42): same nodes and weights. */
int hwwg_gauss_legendre(int32_t n, double* mu, double* weight);
/* hww::sn_solve (reference.cpp:151-233) on the device: diamond difference in space,
 * backward Euler in time, source iteration to `tolerance` (max-norm, relative) on the
 * isotropic scatter + fission source.  psi0[order*cells] ([k*cells + i]); inc_left /
 * inc_right[order] (NULL = vacuum); q[cells] source density constant in time (NULL =
 * none).  Outputs (NULL to skip): phi_layers[(steps+1)*cells] scalar flux per layer,
 * iterations[steps+1].  Non-convergence is HWWG_ESINGULAR with the reference's
 * message.  One persistent cooperative launch, one CTA per direction (order <= 256). */
int hwwg_sn_solve(hwwg_ctx* ctx, int32_t cells, const double* edges,
                  const hwwg_material* materials, int32_t steps, const double* layers,
                  int32_t order, const double* psi0, const double* inc_left,
                  const double* inc_right, const double* q, double tolerance,
                  int32_t max_iterations, double* phi_layers, int32_t* iterations);
/* hww::compute_reference (reference.cpp:302-372) on the device: the pulse problem on
 * a mesh refined space_refine times per cell and time_refine layers per step, S_N of
 * sn_order, projected onto cfg's tally grids (phi_layer[(N+1)*I], phi_interval[N*I],
 * the ReferenceSolution layout).  Config-3 extensions: material regions per tally
 * cell, no_pulse, and the volumetric source as a time-boxed q. */
int hwwg_compute_reference(hwwg_ctx* ctx, const hwwg_run_config* cfg, int32_t space_refine,
                           int32_t time_refine, int32_t sn_order, double* phi_layer,
                           double* phi_interval);

/* ----------------------------------------------------- device components */
/* hww::assemble_solve (losm.cpp:143-165) on the device, single CTA.
 * phi_prev/F_* are I+2 long, J_prev I+1, q I (NULL = zero).  implicit != 0
 * selects ClosureInput::implicit. */
int hwwg_losm_assemble_solve(hwwg_ctx* ctx, int32_t cells, const double* edges,
                             const hwwg_material* materials, const double* phi_prev,
                             const double* J_prev, double J_L, double J_R, int32_t implicit,
                             const double* F_now, double PL_now, double PR_now,
                             const double* F_prev, double PL_prev, double PR_prev,
                             double theta, double dt, const double* q, double* phi_out,
                             double* J_out);
/* hww::build_centers (ww.cpp:8-32); returns 1 on uniform fallback, 0 otherwise. */
int hwwg_build_centers(hwwg_ctx* ctx, const double* phi, int32_t n, double eps_min,
                       double rho, double* centers);
/* hww::moving_average (filters.cpp:11-24). */
int hwwg_moving_average(hwwg_ctx* ctx, const double* g, int32_t n, int32_t k, double* out);
/* hww::fourier_lowpass (filters.cpp:26-52; filters.hpp:36): the hww_fourier
 * filter, bit-identical to the reference (host-libm twiddles, reference order). */
int hwwg_fourier_lowpass(hwwg_ctx* ctx, const double* g, int32_t n, int32_t cutoff, double* out);
/* hww::uniform_comb (popctrl.cpp:7-42) with stream (seed, stream_id). */
int hwwg_uniform_comb(hwwg_ctx* ctx, const hwwg_particle* bank, uint64_t n, uint64_t target,
                      uint64_t seed, uint64_t stream_id, hwwg_particle* out,
                      double* in_weight, double* out_weight);
/* Bit-exact device replay of the host libm log (csrc/libm_log.h) on n inputs. */
int hwwg_device_log(hwwg_ctx* ctx, const double* x, uint64_t n, double* out);

#ifdef __cplusplus
}
#endif
#endif /* HWWG_H */
