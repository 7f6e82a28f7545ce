// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libhww_ref.so).
// It exposes the reference's own public API (driver run_step, the segment
// transport, LOSM assemble/solve, filters, centres, comb, tallies) to ctypes so
// the tests can (1) pin the C restatement in oracle/hww_oracle.c against the
// real reference and (2) generate golden vectors under tests/golden/, and so
// bench.py --impl reference can time the reference's CPU path.
//
// Every function forwards to the reference symbol named in its comment;
// nothing here re-implements reference arithmetic.

#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <filesystem>
#include <memory>
#include <optional>
#include <span>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "hww/banded.hpp"
#include "hww/config.hpp"
#include "hww/driver.hpp"
#include "hww/filters.hpp"
#include "hww/losm.hpp"
#include "hww/popctrl.hpp"
#include "hww/reference.hpp"
#include "hww/tally.hpp"
#include "hww/transport.hpp"
#include "hww/ww.hpp"

extern "C" {

typedef struct {
  double x, mu, w, t;
} hwwref_particle;

typedef struct {
  double sigma_t, sigma_s, sigma_f, nu_f, speed;
} hwwref_material;

typedef struct {
  uint64_t collisions, splits, split_daughters, capped_splits, roulette_kills,
      roulette_survivals, census_count, event_cap_aborts, nan_aborts;
  double leakage_weight, aborted_weight;
} hwwref_counters;

typedef struct {
  int32_t mode;  // 0 analog, 1 lww, 2 hww, 3 hww_ma, 4 hww_fourier
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
} hwwref_config;

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
  hwwref_counters counters;
  uint64_t segments;        // sum of tracks_per_cell (SURVEY §8(d) unit)
  uint64_t census_size;     // state.bank size after the step
  double census_weight, census_weight_sigma;
  double boundary_closure_left, boundary_closure_right;
  double fom_sigma_l2;
  int32_t sigma_valid;
  int32_t has_windows;
  int32_t has_hybrid;
  int32_t pad_;
} hwwref_step_out;

typedef struct {
  double* track_flux;           // I
  double* track_flux_batch;     // B*I
  double* census_phi;           // I
  double* census_current;       // I
  double* census_closure;       // I
  double* census_weight_batch;  // B
  double* edge_current;         // I+1
  double boundary_closure_left;
  double boundary_closure_right;
  uint64_t histories_scored;
  uint64_t grazing_discarded;
} hwwref_tallies;

static thread_local std::string g_err;
const char* hwwref_last_error(void) { return g_err.c_str(); }

int hwwref_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
void hwwref_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

}  // extern "C"

namespace {

hww::RunConfig to_config(const hwwref_config& c) {
  hww::RunConfig r;
  r.mode = static_cast<hww::Mode>(c.mode);
  r.histories_per_step = c.histories_per_step;
  r.theta = c.theta;
  r.rho = c.rho;
  r.eps_min = c.eps_min;
  r.u_ww = c.u_ww;
  r.update_fractions.assign(c.fractions, c.fractions + c.n_fractions);
  r.ma_base_k = c.ma_base_k;
  r.fourier_cutoff = c.fourier_cutoff;
  r.batches = c.batches;
  r.seed = c.seed;
  r.target_population = c.target_population;
  r.comb_overflow_factor = c.comb_overflow_factor;
  r.source = {c.x0, c.t0, c.strength};
  r.material = {c.sigma_t, c.sigma_s, c.sigma_f, c.nu_f, c.speed};
  r.x_min = c.x_min;
  r.x_max = c.x_max;
  r.cells = c.cells;
  r.t_end = c.t_end;
  r.time_steps = c.time_steps;
  r.reference = "";
  r.threads = c.threads;
  return r;
}

void put_counters(const hww::StepCounters& s, hwwref_counters* o) {
  o->collisions = s.collisions;
  o->splits = s.splits;
  o->split_daughters = s.split_daughters;
  o->capped_splits = s.capped_splits;
  o->roulette_kills = s.roulette_kills;
  o->roulette_survivals = s.roulette_survivals;
  o->census_count = s.census_count;
  o->event_cap_aborts = s.event_cap_aborts;
  o->nan_aborts = s.nan_aborts;
  o->leakage_weight = s.leakage_weight;
  o->aborted_weight = s.aborted_weight;
}

hww::StepCounters get_counters(const hwwref_counters* o) {
  hww::StepCounters s;
  s.collisions = o->collisions;
  s.splits = o->splits;
  s.split_daughters = o->split_daughters;
  s.capped_splits = o->capped_splits;
  s.roulette_kills = o->roulette_kills;
  s.roulette_survivals = o->roulette_survivals;
  s.census_count = o->census_count;
  s.event_cap_aborts = o->event_cap_aborts;
  s.nan_aborts = o->nan_aborts;
  s.leakage_weight = o->leakage_weight;
  s.aborted_weight = o->aborted_weight;
  return s;
}

// Stepwise replica of hww::run (proj/src/driver.cpp:286-342) built only from
// the reference's public API: same mesh/time grid/materials/source sampling,
// then one hww::run_step per call.
struct Driver {
  hww::RunConfig config;
  hww::Mesh1D mesh;
  hww::TimeGrid tgrid;
  std::vector<hww::Material> materials;
  hww::RunState state;
  int next_step = 1;
  hww::StepRecord last;
  std::optional<hww::ReferenceSolution> reference;  // hww::run's ReferenceSolution*
};

}  // namespace

extern "C" {

void* hwwref_driver_create(const hwwref_config* c) {
  try {
    auto d = std::make_unique<Driver>();
    d->config = to_config(*c);
    if (const auto v = hww::validate_config(d->config); !v.empty()) {
      g_err = "invalid configuration:";
      for (const auto& s : v) g_err += " " + s + ";";
      return nullptr;
    }
#ifdef _OPENMP
    if (d->config.threads > 0) omp_set_num_threads(d->config.threads);
#endif
    d->mesh = d->config.make_mesh();
    d->tgrid = d->config.make_time_grid();
    d->materials.assign(d->mesh.cells(), d->config.material);
    hww::RngStream source_rng = hww::spawn_stream(
        d->config.seed, hww::stream_id(0, 0, hww::StreamPurpose::source));
    const double total_weight =
        d->config.source.strength * static_cast<double>(d->config.histories_per_step);
    d->state.bank = hww::sample_pulse_source(d->config.histories_per_step,
                                             d->config.source.x0, total_weight, 0.0,
                                             source_rng);
    return d.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void hwwref_driver_destroy(void* h) { delete static_cast<Driver*>(h); }

int hwwref_driver_step(void* h, hwwref_step_out* out) {
  auto* d = static_cast<Driver*>(h);
  try {
    if (d->next_step > d->tgrid.steps()) {
      g_err = "run already complete";
      return -1;
    }
    d->last = hww::run_step(d->next_step, d->state, d->config, d->mesh, d->tgrid,
                            d->materials, d->reference ? &*d->reference : nullptr);
    ++d->next_step;
    const auto& r = d->last;
    std::memset(out, 0, sizeof(*out));
    out->step = r.step;
    out->updates_applied = r.updates_applied;
    out->hybrid_solve_failed = r.hybrid_solve_failed ? 1 : 0;
    out->n_thresholds = static_cast<int32_t>(r.update_thresholds.size());
    for (std::size_t i = 0; i < r.update_thresholds.size() && i < 8; ++i)
      out->thresholds[i] = r.update_thresholds[i];
    out->t_begin = r.t_begin;
    out->t_end = r.t_end;
    out->tau = r.metrics.tau;
    out->histories = r.report.histories;
    out->comb_in = r.comb.input_count;
    out->comb_out = r.comb.output_count;
    out->comb_in_weight = r.comb.input_weight;
    out->comb_out_weight = r.comb.output_weight;
    put_counters(r.counters, &out->counters);
    uint64_t seg = 0;
    for (auto t : r.tracks_per_cell) seg += t;
    out->segments = seg;
    out->census_size = d->state.bank.size();
    out->census_weight = r.report.census_weight;
    out->census_weight_sigma = r.report.census_weight_sigma;
    out->boundary_closure_left = r.report.boundary_closure_left;
    out->boundary_closure_right = r.report.boundary_closure_right;
    out->fom_sigma_l2 = r.metrics.fom_sigma_l2;
    out->sigma_valid = r.report.sigma_valid ? 1 : 0;
    out->has_windows = r.ww_centers.empty() ? 0 : 1;
    out->has_hybrid = r.phi_hybrid.empty() ? 0 : 1;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Per-cell arrays of the last step (any pointer may be NULL).
void hwwref_driver_arrays(void* h, double* phi_track, double* phi_sigma,
                          double* phi_census, double* current_census,
                          double* closure_census, double* edge_current,
                          double* ww_centers, double* phi_hybrid,
                          uint64_t* tracks_per_cell) {
  auto* d = static_cast<Driver*>(h);
  const auto& r = d->last;
  const int I = d->mesh.cells();
  auto cp = [](double* dst, const std::vector<double>& src) {
    if (dst && !src.empty()) std::memcpy(dst, src.data(), src.size() * sizeof(double));
  };
  cp(phi_track, r.report.phi_track);
  cp(phi_sigma, r.report.phi_track_sigma);
  cp(phi_census, r.report.phi_census);
  cp(current_census, r.report.current_census);
  cp(closure_census, r.report.closure_census);
  cp(edge_current, r.report.edge_current);
  cp(ww_centers, r.ww_centers);
  cp(phi_hybrid, r.phi_hybrid);
  if (tracks_per_cell)
    for (int i = 0; i < I; ++i) tracks_per_cell[i] = r.tracks_per_cell[i];
}

uint64_t hwwref_driver_bank(void* h, hwwref_particle* out, uint64_t cap) {
  auto* d = static_cast<Driver*>(h);
  const auto& b = d->state.bank;
  if (out) {
    const uint64_t n = b.size() < cap ? b.size() : cap;
    std::memcpy(out, b.data(), n * sizeof(hwwref_particle));
  }
  return b.size();
}

// hww::run_segment_serial / run_segment_parallel
// (proj/src/transport.cpp:194-237). Tallies and counters accumulate into the
// caller's buffers; the census is appended to an internal buffer read with
// hwwref_take_census.
static thread_local std::vector<hww::Particle> g_census;
static thread_local std::vector<uint64_t> g_tracks;

int hwwref_run_segment(const double* edges, int32_t cells, const hwwref_material* mats,
                       double t_begin, double t_end, uint64_t seed, int32_t step,
                       uint64_t histories_total, int32_t batches,
                       const hwwref_particle* source, uint64_t n, uint64_t h_begin,
                       const double* centers, double rho, double eps_min,
                       int32_t parallel, int32_t chunk, hwwref_tallies* t,
                       hwwref_counters* counters, uint64_t* tracks_per_cell) {
  try {
    const hww::Mesh1D mesh =
        hww::Mesh1D::from_edges(std::vector<double>(edges, edges + cells + 1));
    std::vector<hww::Material> m(cells);
    for (int i = 0; i < cells; ++i)
      m[i] = {mats[i].sigma_t, mats[i].sigma_s, mats[i].sigma_f, mats[i].nu_f,
              mats[i].speed};
    hww::StepContext ctx;
    ctx.mesh = &mesh;
    ctx.materials = &m;
    ctx.t_begin = t_begin;
    ctx.t_end = t_end;
    ctx.seed = seed;
    ctx.step_index = step;
    ctx.histories_total = histories_total;
    ctx.batches = batches;
    hww::WeightWindowGrid ww;
    if (centers) {
      ww.centers.assign(centers, centers + cells);
      ww.rho = rho;
      ww.eps_min = eps_min;
    }
    hww::TallySet ts(cells, batches);
    auto load = [](std::vector<double>& v, const double* p) {
      if (p) std::memcpy(v.data(), p, v.size() * sizeof(double));
    };
    load(ts.track_flux, t->track_flux);
    load(ts.track_flux_batch, t->track_flux_batch);
    load(ts.census_phi, t->census_phi);
    load(ts.census_current, t->census_current);
    load(ts.census_closure, t->census_closure);
    load(ts.census_weight_batch, t->census_weight_batch);
    load(ts.edge_current, t->edge_current);
    ts.boundary_closure_left = t->boundary_closure_left;
    ts.boundary_closure_right = t->boundary_closure_right;
    ts.histories_scored = t->histories_scored;
    ts.grazing_discarded = t->grazing_discarded;

    hww::StepOutcome outcome(cells);
    outcome.counters = get_counters(counters);
    if (tracks_per_cell)
      for (int i = 0; i < cells; ++i) outcome.tracks_per_cell[i] = tracks_per_cell[i];
    std::span<const hww::Particle> src(reinterpret_cast<const hww::Particle*>(source), n);
    if (parallel)
      hww::run_segment_parallel(ctx, src, h_begin, centers ? &ww : nullptr, ts, outcome,
                                chunk > 0 ? chunk : 256);
    else
      hww::run_segment_serial(ctx, src, h_begin, centers ? &ww : nullptr, ts, outcome);

    auto store = [](double* p, const std::vector<double>& v) {
      if (p) std::memcpy(p, v.data(), v.size() * sizeof(double));
    };
    store(t->track_flux, ts.track_flux);
    store(t->track_flux_batch, ts.track_flux_batch);
    store(t->census_phi, ts.census_phi);
    store(t->census_current, ts.census_current);
    store(t->census_closure, ts.census_closure);
    store(t->census_weight_batch, ts.census_weight_batch);
    store(t->edge_current, ts.edge_current);
    t->boundary_closure_left = ts.boundary_closure_left;
    t->boundary_closure_right = ts.boundary_closure_right;
    t->histories_scored = ts.histories_scored;
    t->grazing_discarded = ts.grazing_discarded;
    put_counters(outcome.counters, counters);
    if (tracks_per_cell)
      for (int i = 0; i < cells; ++i) tracks_per_cell[i] = outcome.tracks_per_cell[i];
    g_census = std::move(outcome.census);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

uint64_t hwwref_take_census(hwwref_particle* out, uint64_t cap) {
  const uint64_t n = g_census.size();
  if (out) std::memcpy(out, g_census.data(), (n < cap ? n : cap) * sizeof(hwwref_particle));
  return n;
}

// hww::assemble_solve (proj/src/losm.cpp:143-165). q may be NULL (zero).
int hwwref_assemble_solve(int32_t cells, const double* edges, const hwwref_material* mats,
                          const double* phi_prev, const double* J_prev, double J_L,
                          double J_R, int32_t implicit, const double* F_now,
                          double PL_now, double PR_now, const double* F_prev,
                          double PL_prev, double PR_prev, double theta, double dt,
                          const double* q, double* phi_out, double* J_out) {
  try {
    const hww::Mesh1D mesh =
        hww::Mesh1D::from_edges(std::vector<double>(edges, edges + cells + 1));
    std::vector<hww::Material> m(cells);
    for (int i = 0; i < cells; ++i)
      m[i] = {mats[i].sigma_t, mats[i].sigma_s, mats[i].sigma_f, mats[i].nu_f,
              mats[i].speed};
    hww::LOSMState prev = hww::LOSMState::zero(cells);
    prev.phi.values.assign(phi_prev, phi_prev + cells + 2);
    prev.current.values.assign(J_prev, J_prev + cells + 1);
    prev.incoming_left = J_L;
    prev.incoming_right = J_R;
    hww::GridFunction Fp = hww::GridFunction::cell_with_boundary(cells);
    Fp.values.assign(F_prev, F_prev + cells + 2);
    hww::ClosureInput cl;
    if (implicit) {
      hww::GridFunction Fn = hww::GridFunction::cell_with_boundary(cells);
      Fn.values.assign(F_now, F_now + cells + 2);
      cl = hww::ClosureInput::implicit(std::move(Fn), PL_now, PR_now, std::move(Fp),
                                       PL_prev, PR_prev);
    } else {
      cl = hww::ClosureInput::lagged(std::move(Fp), PL_prev, PR_prev);
    }
    hww::GridFunction qq = hww::GridFunction::cell(cells);
    if (q) qq.values.assign(q, q + cells);
    const hww::LOSMState s = hww::assemble_solve(prev, cl, theta, dt, m, mesh, qq);
    std::memcpy(phi_out, s.phi.values.data(), (cells + 2) * sizeof(double));
    std::memcpy(J_out, s.current.values.data(), (cells + 1) * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// hww::solve_tridiagonal_pivoted (proj/src/banded.cpp:8-38).
int hwwref_solve_tridiagonal(int32_t n, const double* lower, const double* diag,
                             const double* upper, const double* rhs, double* x) {
  hww::TridiagonalSystem s(n);
  s.lower.assign(lower, lower + n);
  s.diag.assign(diag, diag + n);
  s.upper.assign(upper, upper + n);
  s.rhs.assign(rhs, rhs + n);
  try {
    const auto u = hww::solve_tridiagonal_pivoted(std::move(s));
    std::memcpy(x, u.data(), n * sizeof(double));
    return 0;
  } catch (const hww::SingularSystemError& e) {
    g_err = "singular at row " + std::to_string(e.row);
    return -1 - e.row;
  }
}

// hww::build_centers (proj/src/ww.cpp:8-32).
int hwwref_build_centers(const double* phi, int32_t n, double eps_min, double rho,
                         double* centers) {
  try {
    const auto g = hww::build_centers(std::vector<double>(phi, phi + n), eps_min, rho);
    std::memcpy(centers, g.centers.data(), n * sizeof(double));
    return g.uniform_fallback ? 1 : 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// hww::moving_average (proj/src/filters.cpp:11-24).
int hwwref_moving_average(const double* g, int32_t n, int32_t k, double* out) {
  try {
    const auto r = hww::moving_average(std::vector<double>(g, g + n), k);
    std::memcpy(out, r.data(), n * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// hww::fourier_lowpass (proj/src/filters.cpp:26-52).
int hwwref_fourier_lowpass(const double* g, int32_t n, int32_t cutoff, double* out) {
  try {
    const auto r = hww::fourier_lowpass(std::vector<double>(g, g + n), cutoff);
    std::memcpy(out, r.data(), n * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// hww::edge_currents_from_census (proj/src/losm.cpp:12-32).
int hwwref_edge_currents(const double* census_current, int32_t cells, const double* edges,
                         double* out) {
  try {
    const hww::Mesh1D mesh =
        hww::Mesh1D::from_edges(std::vector<double>(edges, edges + cells + 1));
    const auto g = hww::edge_currents_from_census(
        std::vector<double>(census_current, census_current + cells), mesh);
    std::memcpy(out, g.values.data(), (cells + 1) * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// hww::uniform_comb (proj/src/popctrl.cpp:7-42) with the driver's comb stream
// spawn_stream(seed, stream_id(step, 0, comb)) (proj/src/driver.cpp:119-121).
int hwwref_uniform_comb(const hwwref_particle* bank, uint64_t n, uint64_t target,
                        uint64_t seed, uint64_t stream_id, hwwref_particle* out,
                        double* in_w, double* out_w) {
  try {
    hww::ParticleBank b(reinterpret_cast<const hww::Particle*>(bank),
                        reinterpret_cast<const hww::Particle*>(bank) + n);
    hww::RngStream rng(seed, stream_id);
    const auto r = hww::uniform_comb(b, target, rng);
    std::memcpy(out, r.bank.data(), r.bank.size() * sizeof(hwwref_particle));
    *in_w = r.input_weight;
    *out_w = r.output_weight;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// hww::finalize / hww::partial_snapshot (proj/src/tally.cpp:68-128).
// Outputs: phi_track, sigma (finalize only), phi_census, current, closure (I),
// edge (I+1), scalars[0..4] = PL, PR, census_weight, census_weight_sigma,
// sigma_valid.
int hwwref_report(int32_t cells, int32_t batches, const hwwref_tallies* t,
                  uint64_t histories, uint64_t histories_total, double normalization,
                  int32_t snapshot, double* phi_track, double* sigma, double* phi_census,
                  double* current, double* closure, double* edge, double* scalars) {
  try {
    hww::TallySet ts(cells, batches);
    std::memcpy(ts.track_flux.data(), t->track_flux, cells * sizeof(double));
    std::memcpy(ts.track_flux_batch.data(), t->track_flux_batch,
                static_cast<std::size_t>(cells) * batches * sizeof(double));
    std::memcpy(ts.census_phi.data(), t->census_phi, cells * sizeof(double));
    std::memcpy(ts.census_current.data(), t->census_current, cells * sizeof(double));
    std::memcpy(ts.census_closure.data(), t->census_closure, cells * sizeof(double));
    std::memcpy(ts.census_weight_batch.data(), t->census_weight_batch,
                batches * sizeof(double));
    std::memcpy(ts.edge_current.data(), t->edge_current, (cells + 1) * sizeof(double));
    ts.boundary_closure_left = t->boundary_closure_left;
    ts.boundary_closure_right = t->boundary_closure_right;
    ts.histories_scored = t->histories_scored;
    ts.grazing_discarded = t->grazing_discarded;
    const hww::TallyReport r =
        snapshot ? hww::partial_snapshot(ts, histories, histories_total, normalization)
                 : hww::finalize(ts, histories, normalization);
    std::memcpy(phi_track, r.phi_track.data(), cells * sizeof(double));
    if (sigma && !r.phi_track_sigma.empty())
      std::memcpy(sigma, r.phi_track_sigma.data(), cells * sizeof(double));
    std::memcpy(phi_census, r.phi_census.data(), cells * sizeof(double));
    std::memcpy(current, r.current_census.data(), cells * sizeof(double));
    std::memcpy(closure, r.closure_census.data(), cells * sizeof(double));
    std::memcpy(edge, r.edge_current.data(), (cells + 1) * sizeof(double));
    scalars[0] = r.boundary_closure_left;
    scalars[1] = r.boundary_closure_right;
    scalars[2] = r.census_weight;
    scalars[3] = r.census_weight_sigma;
    scalars[4] = r.sigma_valid ? 1.0 : 0.0;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// hww::update_thresholds (proj/src/ww.cpp:74-87).
int hwwref_update_thresholds(uint64_t histories, const double* f, int32_t n,
                             uint64_t* out) {
  try {
    const auto r = hww::update_thresholds(histories, std::vector<double>(f, f + n));
    for (int i = 0; i < n; ++i) out[i] = r[i];
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// hww::RngStream::uniform (proj/include/hww/rng.hpp:51-53) and next_u64.
void hwwref_stream_uniforms(uint64_t seed, uint64_t stream_id, uint64_t n, double* out) {
  hww::RngStream r(seed, stream_id);
  for (uint64_t i = 0; i < n; ++i) out[i] = r.uniform();
}
void hwwref_stream_u64(uint64_t seed, uint64_t stream_id, uint64_t n, uint64_t* out) {
  hww::RngStream r(seed, stream_id);
  for (uint64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}

// hww::sample_pulse_source with the driver's source stream
// (proj/src/driver.cpp:309-316).
void hwwref_pulse_source(uint64_t seed, uint64_t histories, double x0, double strength,
                         hwwref_particle* out) {
  hww::RngStream rng = hww::spawn_stream(seed, hww::stream_id(0, 0, hww::StreamPurpose::source));
  const auto b = hww::sample_pulse_source(histories, x0,
                                          strength * static_cast<double>(histories), 0.0, rng);
  std::memcpy(out, b.data(), b.size() * sizeof(hwwref_particle));
}

// hww::Mesh1D::locate (proj/src/mesh.cpp:26-40); -1 when outside.
int32_t hwwref_locate(const double* edges, int32_t cells, double x) {
  const hww::Mesh1D mesh =
      hww::Mesh1D::from_edges(std::vector<double>(edges, edges + cells + 1));
  const auto c = mesh.locate(x);
  return c ? *c : -1;
}

// hww::load_reference (reference.cpp:395-456) on the driver's grids; the
// following steps run against it (driver.cpp:231-271).
int hwwref_driver_load_reference(void* h, const char* path) {
  auto* d = static_cast<Driver*>(h);
  try {
    d->reference = hww::load_reference(path, d->mesh, d->tgrid);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// StepMetrics of the last step (metrics.hpp:41-51): rel_l2_error,
// rel_mod_l2_error, hybrid_rel_l2_error, fom_err_l2, fom_err_mod, fom_sigma_l2,
// fom_sigma_mod, alpha, tau.
void hwwref_driver_metrics(void* h, double* out) {
  const auto& m = static_cast<Driver*>(h)->last.metrics;
  const double v[9] = {m.rel_l2_error, m.rel_mod_l2_error, m.hybrid_rel_l2_error,
                       m.fom_err_l2,   m.fom_err_mod,      m.fom_sigma_l2,
                       m.fom_sigma_mod, m.alpha,           m.tau};
  std::memcpy(out, v, sizeof v);
}

// hww::compute_reference (reference.cpp:364-372): the S_N oracle projected onto
// the config's tally grids; phi_layer (N+1)*I, phi_interval N*I.
int hwwref_compute_reference(const hwwref_config* c, int32_t space_refine, int32_t time_refine,
                             int32_t sn_order, double* phi_layer, double* phi_interval) {
  try {
    const auto ref =
        hww::compute_reference(to_config(*c), space_refine, time_refine, sn_order);
    const size_t I = ref.mesh.cells();
    for (size_t n = 0; n < ref.phi_layer.size(); ++n)
      std::memcpy(phi_layer + n * I, ref.phi_layer[n].data(), I * sizeof(double));
    for (size_t n = 0; n < ref.phi_interval.size(); ++n)
      std::memcpy(phi_interval + n * I, ref.phi_interval[n].data(), I * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// hww::save_reference (reference.cpp:374-393) of arrays on the config's grids.
int hwwref_save_reference(const hwwref_config* c, const char* path, const double* phi_layer,
                          const double* phi_interval) {
  try {
    const hww::RunConfig config = to_config(*c);
    hww::ReferenceSolution ref;
    ref.mesh = config.make_mesh();
    ref.tgrid = config.make_time_grid();
    const int I = ref.mesh.cells(), N = ref.tgrid.steps();
    for (int n = 0; n <= N; ++n)
      ref.phi_layer.emplace_back(phi_layer + (size_t)n * I, phi_layer + (size_t)(n + 1) * I);
    for (int n = 0; n < N; ++n)
      ref.phi_interval.emplace_back(phi_interval + (size_t)n * I,
                                    phi_interval + (size_t)(n + 1) * I);
    hww::save_reference(ref, path);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// hww::load_reference (reference.cpp:395-456) on the config's grids.
int hwwref_load_reference(const hwwref_config* c, const char* path, double* phi_layer,
                          double* phi_interval) {
  try {
    const hww::RunConfig config = to_config(*c);
    const auto ref = hww::load_reference(path, config.make_mesh(), config.make_time_grid());
    const size_t I = ref.mesh.cells();
    for (size_t n = 0; n < ref.phi_layer.size(); ++n)
      std::memcpy(phi_layer + n * I, ref.phi_layer[n].data(), I * sizeof(double));
    for (size_t n = 0; n < ref.phi_interval.size(); ++n)
      std::memcpy(phi_interval + n * I, ref.phi_interval[n].data(), I * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// GaussLegendre::order (reference.cpp:14-42).
int hwwref_gauss_legendre(int32_t n, double* mu, double* w) {
  try {
    const auto q = hww::GaussLegendre::order(n);
    std::memcpy(mu, q.mu.data(), n * sizeof(double));
    std::memcpy(w, q.weight.data(), n * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// hww::sn_solve (reference.cpp:151-233) on a problem given as arrays; writes the
// scalar flux of every layer and the source-iteration count of every step.
int hwwref_sn_solve(int32_t cells, const double* edges, const hwwref_material* mats,
                    int32_t steps, const double* layers, int32_t order, const double* psi0,
                    const double* inc_left, const double* inc_right, const double* q,
                    double tolerance, int32_t max_iterations, double* phi_layers,
                    int32_t* iterations) {
  try {
    hww::SnProblem prob;
    prob.mesh = hww::Mesh1D::from_edges(std::vector<double>(edges, edges + cells + 1));
    for (int i = 0; i < cells; ++i)
      prob.materials.push_back(
          {mats[i].sigma_t, mats[i].sigma_s, mats[i].sigma_f, mats[i].nu_f, mats[i].speed});
    prob.tgrid = hww::TimeGrid::from_layers(std::vector<double>(layers, layers + steps + 1));
    prob.psi0.assign(psi0, psi0 + (size_t)order * cells);
    prob.inc_left.assign(inc_left, inc_left + order);
    prob.inc_right.assign(inc_right, inc_right + order);
    prob.q.assign(q, q + cells);
    hww::SnConfig sn;
    sn.quadrature_order = order;
    sn.tolerance = tolerance;
    sn.max_iterations = max_iterations;
    const hww::SnSolution sol = hww::sn_solve(prob, sn);
    for (int n = 0; n <= steps; ++n) {
      std::memcpy(phi_layers + (size_t)n * cells, sol.layers[n].phi.data(), cells * sizeof(double));
      iterations[n] = sol.iterations[n];
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// hww::build_uniform_mesh edges (proj/src/mesh.cpp:42-50).
// hww::run with out_dir (proj/src/driver.cpp:286-342): the reference's own
// writers produce step_<n>.csv, summary.csv and run.json in dir.
int hwwref_run_to_dir(const hwwref_config* c, const char* dir, const char* reference) {
  try {
    hww::RunConfig config = to_config(*c);
    config.out_dir = dir;
    if (reference && *reference) {
      // hww_main.cpp:250-256: config.reference holds the path, the run gets the file
      config.reference = reference;
      const auto ref =
          hww::load_reference(reference, config.make_mesh(), config.make_time_grid());
      hww::run(config, &ref);
      return 0;
    }
    hww::run(config);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// The reference writers (driver.cpp:355-438) on records built from arrays:
// step k of n has cells values per field at phi_track + k*cells etc.;
// scalars[k*8 + ...] = {t_end, tau, fom_sigma_l2, census_weight,
// census_weight_sigma, normalization, sigma_valid, hybrid_solve_failed};
// ints[k*6 + ...] = {step, histories, comb_in, comb_out, updates_applied,
// has_centers | has_hybrid << 1}; metrics[k*7 + ...] (NULL: NaN) = {rel_l2_error,
// rel_mod_l2_error, hybrid_rel_l2_error, fom_err_l2, fom_err_mod, fom_sigma_mod,
// alpha}. Writes every step_<n>.csv, summary.csv and run.json (total_seconds) to dir.
int hwwref_write_outputs(const char* dir, const hwwref_config* c, int32_t n, int32_t cells,
                         const double* phi_track, const double* sigma, const double* phi_census,
                         const double* current, const double* closure, const double* centers,
                         const double* hybrid, const uint64_t* tracks, const double* scalars,
                         const uint64_t* ints, const hwwref_counters* counters,
                         const double* metrics, double total_seconds) {
  try {
    std::filesystem::create_directories(dir);  // as hww::run does (driver.cpp:301)
    hww::RunRecord run;
    run.config = to_config(*c);
    run.total_seconds = total_seconds;
    const hww::Mesh1D mesh = run.config.make_mesh();
    for (int k = 0; k < n; ++k) {
      const size_t o = (size_t)k * cells;
      hww::StepRecord r;
      r.step = (int)ints[6 * k + 0];
      r.t_end = scalars[8 * k + 0];
      r.metrics.tau = scalars[8 * k + 1];
      r.metrics.fom_sigma_l2 = scalars[8 * k + 2];
      r.report.census_weight = scalars[8 * k + 3];
      r.report.census_weight_sigma = scalars[8 * k + 4];
      r.report.normalization = scalars[8 * k + 5];
      r.report.sigma_valid = scalars[8 * k + 6] != 0.0;
      r.hybrid_solve_failed = scalars[8 * k + 7] != 0.0;
      r.report.histories = ints[6 * k + 1];
      r.comb.input_count = ints[6 * k + 2];
      r.comb.output_count = ints[6 * k + 3];
      r.updates_applied = (int)ints[6 * k + 4];
      r.report.phi_track.assign(phi_track + o, phi_track + o + cells);
      r.report.phi_track_sigma.assign(sigma + o, sigma + o + cells);
      r.report.phi_census.assign(phi_census + o, phi_census + o + cells);
      r.report.current_census.assign(current + o, current + o + cells);
      r.report.closure_census.assign(closure + o, closure + o + cells);
      if (ints[6 * k + 5] & 1) r.ww_centers.assign(centers + o, centers + o + cells);
      if (ints[6 * k + 5] & 2) r.phi_hybrid.assign(hybrid + o, hybrid + o + cells);
      r.tracks_per_cell.assign(tracks + o, tracks + o + cells);
      r.counters = get_counters(&counters[k]);
      if (metrics) {  // metrics[k*7 + ...] = StepMetrics' reference diagnostics
        const double* m = metrics + 7 * k;
        r.metrics.rel_l2_error = m[0];
        r.metrics.rel_mod_l2_error = m[1];
        r.metrics.hybrid_rel_l2_error = m[2];
        r.metrics.fom_err_l2 = m[3];
        r.metrics.fom_err_mod = m[4];
        r.metrics.fom_sigma_mod = m[5];
        r.metrics.alpha = m[6];
      }
      run.steps.push_back(r);
      hww::write_step_csv(dir, run.steps.back(), mesh);
    }
    hww::write_summary_csv(dir, run);
    hww::write_run_json(dir, run);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

void hwwref_uniform_edges(double x_min, double x_max, int32_t cells, double* out) {
  const auto m = hww::build_uniform_mesh(x_min, x_max, cells);
  std::memcpy(out, m.edges().data(), (cells + 1) * sizeof(double));
}

}  // extern "C"
