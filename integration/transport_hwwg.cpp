// Reference-side drop-in: hww::run_segment_parallel
// (proj/include/hww/transport.hpp:117-120) forwarded to the B200 engine through
// the C ABI (include/hwwg.h).  This translation unit belongs to the
// REFERENCE's build: it is compiled against the reference headers and linked
// with the reference's own driver.cpp, whose run_step calls
// run_segment_parallel through its run_to lambda (proj/src/driver.cpp:195-202).
// The reference's CPU definition (proj/src/transport.cpp:209-237) is renamed
// out of the way at compile time (oracle/Makefile `dropin`), nothing else of
// the reference changes.
//
// Exact mode (HWWG_RNG_EXACT) replays the reference bit for bit: the census is
// appended in the reference order, tallies are accumulated in its chunk-merge
// order, and the running StepCounters are handed to the engine (not zeroed and
// merged afterwards), so the fp64 leakage / aborted weights take the same
// ((out + c0) + c1) + ... sequence as StepOutcome::merge_from in chunk order
// (transport.cpp:233-236, transport.hpp:74-79).
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>

#include "hww/transport.hpp"
#include "hwwg.h"

namespace hww {

namespace {

hwwg_ctx* engine() {  // one engine per host thread (driver.cpp calls from one)
  thread_local hwwg_ctx* ctx = [] {
    hwwg_options o{};
    o.device = 0;
    o.rng_mode = HWWG_RNG_EXACT;
    o.world = 1;
    hwwg_ctx* c = nullptr;
    if (hwwg_create(&o, &c) != HWWG_OK) throw std::runtime_error(hwwg_last_error());
    return c;
  }();
  return ctx;
}

static_assert(sizeof(Particle) == sizeof(hwwg_particle), "Particle is {x, mu, w, t}");
static_assert(sizeof(Material) == sizeof(hwwg_material), "Material field order");
static_assert(sizeof(StepCounters) == sizeof(hwwg_counters), "StepCounters field order");

}  // namespace

void run_segment_parallel(const StepContext& ctx, std::span<const Particle> source,
                          std::uint64_t h_begin, const WeightWindowGrid* ww, TallySet& t,
                          StepOutcome& out, int chunk_size) {
  if (chunk_size != 256)  // the engine's chunk-merge order is the driver's default
    throw std::invalid_argument("hwwg drop-in: chunk_size must be 256, got " +
                                std::to_string(chunk_size));
  hwwg_step_context sc{};
  sc.edges = ctx.mesh->edges().data();
  sc.cells = ctx.mesh->cells();
  sc.batches = ctx.batches;
  sc.materials = reinterpret_cast<const hwwg_material*>(ctx.materials->data());
  sc.t_begin = ctx.t_begin;
  sc.t_end = ctx.t_end;
  sc.seed = ctx.seed;
  sc.step_index = ctx.step_index;
  sc.histories_total = ctx.histories_total;

  hwwg_window_grid g{};
  if (ww) {
    g.centers = ww->centers.data();
    g.rho = ww->rho;
    g.eps_min = ww->eps_min;
  }
  hwwg_tally_set ts{t.track_flux.data(),        t.track_flux_batch.data(),
                    t.census_phi.data(),         t.census_current.data(),
                    t.census_closure.data(),     t.census_weight_batch.data(),
                    t.edge_current.data(),       t.boundary_closure_left,
                    t.boundary_closure_right,    t.histories_scored,
                    t.grazing_discarded};

  const std::size_t base = out.census.size();
  for (std::uint64_t cap = base + 2 * source.size() + 1024;;) {
    out.census.resize(cap);
    hwwg_step_outcome o{};
    o.census = reinterpret_cast<hwwg_particle*>(out.census.data());
    o.census_size = base;
    o.census_capacity = cap;
    std::memcpy(&o.counters, &out.counters, sizeof o.counters);  // the RUNNING counters
    o.tracks_per_cell = out.tracks_per_cell.data();
    const int rc = hwwg_run_segment_parallel(
        engine(), &sc, reinterpret_cast<const hwwg_particle*>(source.data()), source.size(),
        h_begin, ww ? &g : nullptr, &ts, &o);
    if (rc == HWWG_ENOSPC) {  // nothing was touched: make room and run again
      cap = o.census_needed;
      continue;
    }
    if (rc != HWWG_OK) {
      out.census.resize(base);
      if (rc == HWWG_EINVAL) throw std::invalid_argument(hwwg_last_error());
      throw std::runtime_error(hwwg_last_error());
    }
    out.census.resize(o.census_size);
    std::memcpy(&out.counters, &o.counters, sizeof o.counters);
    break;
  }
  t.boundary_closure_left = ts.boundary_closure_left;
  t.boundary_closure_right = ts.boundary_closure_right;
  t.histories_scored = ts.histories_scored;
  t.grazing_discarded = ts.grazing_discarded;
}

}  // namespace hww
