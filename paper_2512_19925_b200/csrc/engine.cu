// hwwg_ctx: the drop-in segment boundary (hww::run_segment_parallel) and the
// device component entry points of the C ABI (include/hwwg.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "capi_util.h"
#include "common.cuh"
#include "device_state.cuh"
#include "engine.cuh"
#include "low_order.cuh"
#include "sn.cuh"
#include "transport.cuh"

namespace hwwg {

std::string& last_error_slot() {
  static thread_local std::string s;
  return s;
}

int bit_length(unsigned long long v) {
  int b = 0;
  while (v) {
    ++b;
    v >>= 1;
  }
  return b;
}

void CensusStage::ensure(uint64_t cap) {
  if (cap <= records.n) return;
  const uint64_t c = std::max<uint64_t>(cap, 1024);
  records.reserve(c);
  keys.reserve(c);
  keys_alt.reserve(c);
  idx.reserve(c);
  idx_alt.reserve(c);
  const size_t tb = census_sort_temp_bytes(c);
  temp.reserve(tb);
  temp_bytes = tb;
}

void CensusStage::sort_into(hwwg_particle* out, uint64_t n, unsigned long long max_key,
                            cudaStream_t s) {
  CensusSortArgs a{};
  a.records = records.p;
  a.keys_in = keys.p;
  a.keys_out = keys_alt.p;
  a.idx_in = idx.p;
  a.idx_out = idx_alt.p;
  a.out = out;
  a.n = n;
  a.begin_bit = 0;
  a.end_bit = std::max(1, bit_length(max_key));
  a.temp = temp.p;
  a.temp_bytes = temp_bytes;
  sort_census(a, s);
}

}  // namespace hwwg

using namespace hwwg;

struct hwwg_ctx {
  int device = 0;
  int rng_mode = HWWG_RNG_EXACT;
  cudaStream_t stream = nullptr;
  DeviceProblem prob;
  DeviceTallies tal;
  HostTallies host_tal;
  DevBuf<hwwg_particle> src, sorted;
  CensusStage stage;
  DevBuf<double> centers, scratch;
  DevBuf<unsigned long long> counter;
  DevBuf<DevError> err;
  DevBuf<int> iscratch;
  DevBuf<hwwg_particle> comb_in, comb_out;
  DevBuf<CellInfo> comp_cells;
  DevBuf<double> chunk_mem;
  ExactLogBuf xlog;

  ~hwwg_ctx() {
    if (stream) cudaStreamDestroy(stream);
  }
};

extern "C" {

const char* hwwg_last_error(void) { return last_error_slot().c_str(); }
const char* hwwg_version(void) { return "hwwg 0.1 (sm_100a)"; }

int hwwg_create(const hwwg_options* opts, hwwg_ctx** out) {
  HWWG_API_BEGIN
  if (!out) return fail(HWWG_EINVAL, "hwwg_create: out is NULL");
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(HWWG_ECUDA, "no CUDA device available");
  }
  auto c = new hwwg_ctx();
  c->device = opts ? opts->device : 0;
  c->rng_mode = opts ? opts->rng_mode : HWWG_RNG_EXACT;
  if (c->rng_mode != HWWG_RNG_EXACT && c->rng_mode != HWWG_RNG_PHILOX) {
    delete c;
    return fail(HWWG_EINVAL, "unknown rng_mode");
  }
  HWWG_CUDA(cudaSetDevice(c->device));
  HWWG_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  c->counter.reserve(1);
  c->err.reserve(1);
  c->iscratch.reserve(4);
  if (opts && opts->bank_capacity) c->stage.ensure(opts->bank_capacity);
  *out = c;
  return HWWG_OK;
  HWWG_API_END
}

void hwwg_destroy(hwwg_ctx* ctx) { delete ctx; }

int hwwg_run_segment_parallel(hwwg_ctx* c, const hwwg_step_context* st,
                              const hwwg_particle* source, uint64_t n, uint64_t h_begin,
                              const hwwg_window_grid* ww, hwwg_tally_set* tallies,
                              hwwg_step_outcome* outcome) {
  HWWG_API_BEGIN
  if (!c || !st || !tallies || !outcome) return fail(HWWG_EINVAL, "NULL argument");
  if (n && !source) return fail(HWWG_EINVAL, "source is NULL");
  HWWG_CUDA(cudaSetDevice(c->device));
  std::string why;
  if (!c->prob.set(st->edges, st->cells, st->materials, c->stream, why))
    return fail(HWWG_EINVAL, why);
  if (st->batches < 1) return fail(HWWG_EINVAL, "batches must be >= 1");
  if (!(st->t_end > st->t_begin)) return fail(HWWG_EINVAL, "t_end must exceed t_begin");
  if (ww && (!ww->centers || !(ww->rho >= 1.0)))
    return fail(HWWG_EINVAL, "window grid needs centers and rho >= 1");
  // run_segment_parallel with an empty span does nothing (transport.cpp:212-217)
  if (n == 0) return HWWG_OK;
  if (c->rng_mode != HWWG_RNG_EXACT)
    return fail(HWWG_EINVAL, "hwwg_run_segment_parallel replays the reference streams: "
                             "create the context with HWWG_RNG_EXACT");
  const int I = st->cells, B = st->batches;
  cudaStream_t s = c->stream;
  c->tal.shape(I, B);
  c->src.reserve(n);
  HWWG_CUDA(cudaMemcpyAsync(c->src.p, source, n * sizeof(hwwg_particle), cudaMemcpyHostToDevice, s));
  if (ww) {
    c->centers.reserve(I);
    HWWG_CUDA(cudaMemcpyAsync(c->centers.p, ww->centers, I * sizeof(double),
                              cudaMemcpyHostToDevice, s));
  }
  c->stage.ensure(std::max<uint64_t>(2 * n + 1024, c->stage.records.n));

  ExactArgs a{};
  a.src = c->src.p;
  a.n = n;
  a.h_begin = h_begin;
  a.mesh = c->prob.view;
  a.t_begin = st->t_begin;
  a.t_end = st->t_end;
  a.inv_dt = 1.0 / (st->t_end - st->t_begin);
  a.seed = st->seed;
  a.step = (uint64_t)st->step_index;
  a.H = st->histories_total;
  a.B = B;
  a.centers = ww ? c->centers.p : nullptr;
  a.active = nullptr;
  a.rho = ww ? ww->rho : 1.0;
  a.err = c->err.p;
  a.census_count = c->counter.p;

  // the running TallySet / counters (reference: accumulated in place, chunk sums
  // merged in order), uploaded so the device adds in the reference's order
  const ChunkLayout L0 = chunk_layout(n, h_begin, st->histories_total, I, B);
  c->chunk_mem.reserve(std::max<size_t>((size_t)L0.count * L0.stride, 1));
  std::vector<double> up(c->tal.words(), 0.0);
  {
    double* q = up.data();
    auto put = [&](const double* srcv, size_t len) {
      if (srcv) std::memcpy(q, srcv, len * 8);
      q += len;
    };
    put(tallies->track_flux, I);
    put(tallies->track_flux_batch, (size_t)B * I);
    put(tallies->census_phi, I);
    put(tallies->census_current, I);
    put(tallies->census_closure, I);
    put(tallies->census_weight_batch, B);
    put(tallies->edge_current, I + 1);
    q[0] = tallies->boundary_closure_left;
    q[1] = tallies->boundary_closure_right;
    q[2] = outcome->counters.leakage_weight;
    q[3] = outcome->counters.aborted_weight;
  }
  unsigned long long count = 0;
  DevError derr{};
  for (int attempt = 0; attempt < 4; ++attempt) {
    HWWG_CUDA(cudaMemcpyAsync(c->tal.slab.p, up.data(), up.size() * 8, cudaMemcpyHostToDevice, s));
    HWWG_CUDA(cudaMemsetAsync(c->counter.p, 0, sizeof(unsigned long long), s));
    HWWG_CUDA(cudaMemsetAsync(c->err.p, 0, sizeof(DevError), s));
    a.t = c->tal.p;
    a.chunks = L0;
    a.chunks.base = c->chunk_mem.p;
    a.census = c->stage.records.p;
    a.census_keys = c->stage.keys.p;
    a.census_cap = c->stage.records.n;
    a.log = c->xlog.view(n);
    if (a.log.slot) c->xlog.reset_need(s);
    launch_exact_segment(a, s);
    HWWG_CUDA(cudaMemcpyAsync(&count, c->counter.p, sizeof(count), cudaMemcpyDeviceToHost, s));
    HWWG_CUDA(cudaMemcpyAsync(&derr, c->err.p, sizeof(derr), cudaMemcpyDeviceToHost, s));
    HWWG_CUDA(cudaStreamSynchronize(s));
    // deterministic replay with room: the log arena the overflowing histories
    // counted and/or the census stage, both at once
    bool again = false;
    if (derr.code == kLogOverflow) {
      const unsigned long long need = c->xlog.need(s);
      c->xlog.ensure_blocks(need + need / 4 + 1024);
      again = true;
    }
    if ((derr.code == 0 || again) && count > a.census_cap) {
      c->stage.ensure(count + count / 4 + 1024);
      again = true;
    }
    if (!again) break;
  }
  if (derr.code == kLogOverflow) return fail(HWWG_ENOMEM, "exact tally log exceeds 2^32 blocks");
  if (derr.code == HWWG_EINVAL)
    return fail(HWWG_EINVAL, "history " + std::to_string(derr.history) +
                                 " starts outside the mesh or the time step");
  if (derr.code == HWWG_ESTACK)
    return fail(HWWG_ESTACK, "history " + std::to_string(derr.history) +
                                 " exceeded the daughter-stack run capacity");
  if (outcome->census_size + count > outcome->census_capacity) {
    outcome->census_needed = outcome->census_size + count;
    return fail(HWWG_ENOSPC, "census buffer too small");
  }
  c->sorted.reserve(std::max<uint64_t>(count, 1));
  c->stage.sort_into(c->sorted.p, count, ((unsigned long long)(h_begin + n) << 24) | 0xffffffULL, s);
  if (count)
    HWWG_CUDA(cudaMemcpyAsync(outcome->census + outcome->census_size, c->sorted.p,
                              count * sizeof(hwwg_particle), cudaMemcpyDeviceToHost, s));
  c->host_tal.fetch(c->tal, s);  // synchronises
  const HostTallies& h = c->host_tal;
  auto put_back = [](double* dst, const double* srcv, size_t len) {
    if (dst) std::memcpy(dst, srcv, len * 8);
  };
  put_back(tallies->track_flux, h.track_flux(), I);
  put_back(tallies->track_flux_batch, h.track_flux_batch(), (size_t)B * I);
  put_back(tallies->census_phi, h.census_phi(), I);
  put_back(tallies->census_current, h.census_current(), I);
  put_back(tallies->census_closure, h.census_closure(), I);
  put_back(tallies->census_weight_batch, h.census_weight_batch(), B);
  put_back(tallies->edge_current, h.edge_current(), I + 1);
  tallies->boundary_closure_left = h.boundary_closure()[0];
  tallies->boundary_closure_right = h.boundary_closure()[1];
  tallies->histories_scored += h.ucount()[kHistoriesScored];
  tallies->grazing_discarded += h.ucount()[kGrazingDiscarded];
  hwwg_counters& k = outcome->counters;
  const unsigned long long* u = h.ucount();
  k.collisions += u[kCollisions];
  k.splits += u[kSplits];
  k.split_daughters += u[kSplitDaughters];
  k.capped_splits += u[kCappedSplits];
  k.roulette_kills += u[kRouletteKills];
  k.roulette_survivals += u[kRouletteSurvivals];
  k.census_count += u[kCensusCount];
  k.event_cap_aborts += u[kEventCapAborts];
  k.nan_aborts += u[kNanAborts];
  k.leakage_weight = h.dcount()[0];
  k.aborted_weight = h.dcount()[1];
  if (outcome->tracks_per_cell)
    for (int i = 0; i < I; ++i) outcome->tracks_per_cell[i] += h.tracks()[i];
  outcome->census_size += count;
  outcome->census_needed = outcome->census_size;
  return HWWG_OK;
  HWWG_API_END
}

int hwwg_losm_assemble_solve(hwwg_ctx* c, int32_t I, const double* edges,
                             const hwwg_material* mats, const double* phi_prev,
                             const double* J_prev, double J_L, double J_R, int32_t implicit,
                             const double* F_now, double PL_now, double PR_now,
                             const double* F_prev, double PL_prev, double PR_prev, double theta,
                             double dt, const double* q, double* phi_out, double* J_out) {
  HWWG_API_BEGIN
  if (!c || !phi_prev || !J_prev || !F_prev || !phi_out || !J_out || (implicit && !F_now))
    return fail(HWWG_EINVAL, "NULL argument");
  // check_inputs (losm.cpp:43-53) scalar preconditions
  if (!(theta >= 0.5 && theta <= 1.0)) return fail(HWWG_EINVAL, "theta must lie in [1/2, 1]");
  if (!(dt > 0.0)) return fail(HWWG_EINVAL, "dt must be > 0");
  HWWG_CUDA(cudaSetDevice(c->device));
  std::string why;
  if (!c->prob.set(edges, I, mats, c->stream, why)) return fail(HWWG_EINVAL, why);
  cudaStream_t s = c->stream;
  const int n = 2 * I + 3;
  // layout: phi_prev I+2 | J_prev I+1 | F_now I+2 | F_prev I+2 | q I | phi I+2 | J I+1 | sys 6n
  const size_t need = (size_t)(I + 2) * 4 + (size_t)(I + 1) * 2 + I + 6 * (size_t)n;
  c->scratch.reserve(need);
  double* b = c->scratch.p;
  double* d_phi = b; b += I + 2;
  double* d_J = b; b += I + 1;
  double* d_Fn = b; b += I + 2;
  double* d_Fp = b; b += I + 2;
  double* d_q = b; b += I;
  double* d_po = b; b += I + 2;
  double* d_Jo = b; b += I + 1;
  double* d_sys = b;
  auto up = [&](double* dst, const double* srcv, size_t len) {
    HWWG_CUDA(cudaMemcpyAsync(dst, srcv, len * 8, cudaMemcpyHostToDevice, s));
  };
  up(d_phi, phi_prev, I + 2);
  up(d_J, J_prev, I + 1);
  if (implicit) up(d_Fn, F_now, I + 2);
  up(d_Fp, F_prev, I + 2);
  if (q) up(d_q, q, I);
  RawLosmArgs a{};
  a.I = I;
  a.edges = c->prob.view.edges;
  a.cells = c->prob.view.cells;
  a.phi_prev = d_phi;
  a.J_prev = d_J;
  a.J_L = J_L;
  a.J_R = J_R;
  a.implicit = implicit;
  a.F_now = d_Fn;
  a.PL_now = PL_now;
  a.PR_now = PR_now;
  a.F_prev = d_Fp;
  a.PL_prev = PL_prev;
  a.PR_prev = PR_prev;
  a.theta = theta;
  a.dt = dt;
  a.q = q ? d_q : nullptr;
  a.sys = d_sys;
  a.phi_out = d_po;
  a.J_out = d_Jo;
  a.status = c->iscratch.p;
  launch_raw_losm(a, s);
  int status = 0;
  HWWG_CUDA(cudaMemcpyAsync(&status, c->iscratch.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  HWWG_CUDA(cudaStreamSynchronize(s));
  if (status == 1) return fail(HWWG_EINVAL, "non-finite low-order inputs");
  if (status > 1)
    return fail(HWWG_ESINGULAR,
                "singular low-order system at pivot row " + std::to_string(status - 2));
  HWWG_CUDA(cudaMemcpyAsync(phi_out, d_po, (I + 2) * 8, cudaMemcpyDeviceToHost, s));
  HWWG_CUDA(cudaMemcpyAsync(J_out, d_Jo, (I + 1) * 8, cudaMemcpyDeviceToHost, s));
  HWWG_CUDA(cudaStreamSynchronize(s));
  return HWWG_OK;
  HWWG_API_END
}

int hwwg_build_centers(hwwg_ctx* c, const double* phi, int32_t n, double eps_min, double rho,
                       double* centers) {
  HWWG_API_BEGIN
  if (!c || (n && (!phi || !centers))) return fail(HWWG_EINVAL, "NULL argument");
  if (!(eps_min > 0.0 && eps_min < 1.0)) return fail(HWWG_EINVAL, "eps_min must lie in (0,1)");
  if (!(rho >= 1.0)) return fail(HWWG_EINVAL, "rho must be >= 1");
  if (n == 0) return 1;  // empty flux: uniform fallback with no cells
  HWWG_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  c->scratch.reserve(2 * (size_t)n);
  HWWG_CUDA(cudaMemcpyAsync(c->scratch.p, phi, n * 8, cudaMemcpyHostToDevice, s));
  launch_build_centers(c->scratch.p, n, eps_min, rho, c->scratch.p + n, c->iscratch.p, s);
  int fb = 0;
  HWWG_CUDA(cudaMemcpyAsync(centers, c->scratch.p + n, n * 8, cudaMemcpyDeviceToHost, s));
  HWWG_CUDA(cudaMemcpyAsync(&fb, c->iscratch.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  HWWG_CUDA(cudaStreamSynchronize(s));
  return fb ? 1 : 0;
  HWWG_API_END
}

int hwwg_moving_average(hwwg_ctx* c, const double* g, int32_t n, int32_t k, double* out) {
  HWWG_API_BEGIN
  if (!c || (n && (!g || !out))) return fail(HWWG_EINVAL, "NULL argument");
  if (k < 0) return fail(HWWG_EINVAL, "moving average half-width must be >= 0");
  if (n == 0) return HWWG_OK;
  HWWG_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  c->scratch.reserve(2 * (size_t)n);
  HWWG_CUDA(cudaMemcpyAsync(c->scratch.p, g, n * 8, cudaMemcpyHostToDevice, s));
  launch_moving_average(c->scratch.p, n, k, c->scratch.p + n, s);
  HWWG_CUDA(cudaMemcpyAsync(out, c->scratch.p + n, n * 8, cudaMemcpyDeviceToHost, s));
  HWWG_CUDA(cudaStreamSynchronize(s));
  return HWWG_OK;
  HWWG_API_END
}

int hwwg_fourier_lowpass(hwwg_ctx* c, const double* g, int32_t n, int32_t cutoff, double* out) {
  HWWG_API_BEGIN
  if (!c || (n && (!g || !out))) return fail(HWWG_EINVAL, "NULL argument");
  if (cutoff < 0) return fail(HWWG_EINVAL, "fourier cutoff must be >= 0");
  if (n == 0) return HWWG_OK;
  if (n == 1) {
    out[0] = g[0];
    return HWWG_OK;
  }
  HWWG_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  const std::vector<double> tab = fourier_tables(n);
  c->scratch.reserve(4 * (size_t)n + tab.size());
  double* d_g = c->scratch.p;
  double* d_tmp = d_g + n;
  double* d_tab = d_tmp + 3 * (size_t)n;
  HWWG_CUDA(cudaMemcpyAsync(d_g, g, n * 8, cudaMemcpyHostToDevice, s));
  HWWG_CUDA(cudaMemcpyAsync(d_tab, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, s));
  launch_fourier_lowpass(d_g, n, cutoff, d_tab, d_tmp, s);
  HWWG_CUDA(cudaMemcpyAsync(out, d_g, n * 8, cudaMemcpyDeviceToHost, s));
  HWWG_CUDA(cudaStreamSynchronize(s));
  return HWWG_OK;
  HWWG_API_END
}

int hwwg_uniform_comb(hwwg_ctx* c, const hwwg_particle* bank, uint64_t n, uint64_t target,
                      uint64_t seed, uint64_t stream_id, hwwg_particle* out, double* in_weight,
                      double* out_weight) {
  HWWG_API_BEGIN
  if (!c || !out) return fail(HWWG_EINVAL, "NULL argument");
  if (n == 0 || !bank) return fail(HWWG_EINVAL, "cannot comb an empty bank");
  if (target < 1) return fail(HWWG_EINVAL, "comb target must be positive");
  HWWG_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  c->comb_in.reserve(n);
  c->comb_out.reserve(target);
  c->scratch.reserve(n + 4 + comb_tile_words(n));
  HWWG_CUDA(cudaMemcpyAsync(c->comb_in.p, bank, n * sizeof(hwwg_particle), cudaMemcpyHostToDevice, s));
  CombArgs a{};
  a.bank = c->comb_in.p;
  a.n = n;
  a.target = target;
  a.seed = seed;
  a.stream = stream_id;
  a.prefix = c->scratch.p + 4;
  a.scalars = c->scratch.p;
  a.out = c->comb_out.p;
  a.exact_out_weight = 1;
  a.tiles = c->scratch.p + 4 + n;
  launch_comb(a, s);
  double sc[4];
  HWWG_CUDA(cudaMemcpyAsync(sc, c->scratch.p, sizeof sc, cudaMemcpyDeviceToHost, s));
  HWWG_CUDA(cudaMemcpyAsync(out, c->comb_out.p, target * sizeof(hwwg_particle), cudaMemcpyDeviceToHost, s));
  HWWG_CUDA(cudaStreamSynchronize(s));
  if (in_weight) *in_weight = sc[0];
  if (out_weight) *out_weight = sc[3];
  return HWWG_OK;
  HWWG_API_END
}

// Test hook (not part of include/hwwg.h): the throughput-mode window update
// solved through the cached factorization must give bit-identical centres and
// hybrid flux to the same update rebuilding the factorization. Synthetic
// smooth inputs on a uniform I-cell slab; returns the number of differing
// values (or a negative status), *max_abs_diff their largest difference.
int hwwg_internal_losm_cache_check(hwwg_ctx* c, int32_t I, uint32_t seed, double* max_abs_diff) {
  HWWG_API_BEGIN
  if (!c || I < 2 || !max_abs_diff) return fail(HWWG_EINVAL, "bad argument");
  if (!lo_fac_words(I)) return fail(HWWG_EINVAL, "I too large for the cached factorization");
  HWWG_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  std::vector<double> edges(I + 1);
  for (int e = 0; e <= I; ++e) edges[e] = -20.0 + 40.0 * e / I;
  std::vector<hwwg_material> mats(I, hwwg_material{1.0, 0.9, 0.0, 0.0, 1.0});
  std::string why;
  if (!c->prob.set(edges.data(), I, mats.data(), s, why)) return fail(HWWG_EINVAL, why);
  uint64_t z = seed * 0x9E3779B97F4A7C15ULL + 1;
  auto rnd = [&]() {  // splitmix64 -> [0, 1)
    z += 0x9E3779B97F4A7C15ULL;
    uint64_t t = z;
    t = (t ^ (t >> 30)) * 0xBF58476D1CE4E5B9ULL;
    t = (t ^ (t >> 27)) * 0x94D049BB133111EBULL;
    return (double)((t ^ (t >> 31)) >> 11) * 0x1.0p-53;
  };
  const int n = 2 * I + 3;
  const size_t fw = lo_fac_words(I);
  // phi_prev I+2 | J_prev I+1 | F_prev I+2 | PLPR 2 | centers I | hybrid I | sys 6n | F_now I+2 |
  // closure I | bclosure 2 | fac
  const size_t words = (size_t)(I + 2) * 3 + (I + 1) + 2 + 2 * (size_t)I + 6 * (size_t)n + I + 2 + fw;
  c->scratch.reserve(words);
  c->iscratch.reserve(8);
  std::vector<double> h(words, 0.0);
  double* q = h.data();
  for (int i = 0; i < I + 2; ++i) q[i] = std::exp(-0.01 * (i - I / 2) * (i - I / 2)) + 0.01 * rnd();
  q += I + 2;
  for (int i = 0; i < I + 1; ++i) q[i] = 0.1 * (rnd() - 0.5);
  q += I + 1;
  for (int i = 0; i < I + 2; ++i) q[i] = 0.05 * (rnd() - 0.5);
  q += I + 2 + 2 + 2 * (size_t)I + 6 * (size_t)n + I + 2;
  for (int i = 0; i < I; ++i) q[i] = 1e6 * 0.05 * (rnd() - 0.5);  // closure tally
  q[I] = 1e6 * 0.01;
  q[I + 1] = -1e6 * 0.01;
  h[words - 1] = 2.0;  // factorization not built
  HWWG_CUDA(cudaMemcpyAsync(c->scratch.p, h.data(), words * 8, cudaMemcpyHostToDevice, s));
  HWWG_CUDA(cudaMemsetAsync(c->iscratch.p, 0, 8 * sizeof(int), s));
  double* d = c->scratch.p;
  LowOrderArgs a{};
  a.I = I;
  a.edges = c->prob.view.edges;
  a.cells = c->prob.view.cells;
  a.theta = 0.5;
  a.dt = 0.5;
  a.eps_min = 1e-3;
  a.rho = 5.0;
  a.ma_k = 1;
  a.mode = 1;
  a.fast_solve = 1;
  a.s.phi_prev = d; d += I + 2;
  a.s.J_prev = d; d += I + 1;
  a.s.F_prev = d; d += I + 2;
  a.s.PLPR_prev = d; d += 2;
  a.s.centers = d; d += I;
  a.s.phi_hybrid = d; d += I;
  a.s.sys = d; d += 6 * (size_t)n;
  a.s.F_now = d; d += I + 2;
  a.closure_tally = d; d += I;
  a.bclosure_tally = d; d += 2;
  a.s.fac = d;
  a.s.flags = c->iscratch.p;
  a.snapshot_inv_norm = 1e-6;
  std::vector<double> r1(2 * (size_t)I), r2(2 * (size_t)I);
  for (int pass = 0; pass < 2; ++pass) {
    a.refactor = pass == 0 ? 1 : 0;
    launch_low_order_update(a, s);
    std::vector<double>& r = pass == 0 ? r1 : r2;
    HWWG_CUDA(cudaMemcpyAsync(r.data(), a.s.centers, 2 * (size_t)I * 8, cudaMemcpyDeviceToHost, s));
    HWWG_CUDA(cudaStreamSynchronize(s));
  }
  int fl[8];
  HWWG_CUDA(cudaMemcpy(fl, c->iscratch.p, sizeof fl, cudaMemcpyDeviceToHost));
  if (fl[4] != 0) return fail(HWWG_ESINGULAR, "synthetic LOSM solve failed");
  int diff = 0;
  double mx = 0.0;
  for (size_t i = 0; i < r1.size(); ++i) {
    if (std::memcmp(&r1[i], &r2[i], 8) != 0) {
      ++diff;
      mx = std::max(mx, std::fabs(r1[i] - r2[i]));
    }
  }
  *max_abs_diff = mx;
  return diff;
  HWWG_API_END
}

int hwwg_gauss_legendre(int32_t n, double* mu, double* weight) {
  HWWG_API_BEGIN
  if (!mu || !weight) return fail(HWWG_EINVAL, "NULL argument");
  gauss_legendre(n, mu, weight);
  return HWWG_OK;
  HWWG_API_END
}

int hwwg_sn_solve(hwwg_ctx* c, int32_t cells, const double* edges,
                  const hwwg_material* materials, int32_t steps, const double* layers,
                  int32_t order, const double* psi0, const double* inc_left,
                  const double* inc_right, const double* q, double tolerance,
                  int32_t max_iterations, double* phi_layers, int32_t* iterations) {
  HWWG_API_BEGIN
  if (!c || !edges || !materials || !layers || !psi0 || cells < 1 || steps < 1 || order < 1)
    return fail(HWWG_EINVAL, "NULL argument");
  SnHostProblem p;
  p.edges.assign(edges, edges + cells + 1);
  p.materials.assign(materials, materials + cells);
  p.layers.assign(layers, layers + steps + 1);
  p.order = order;
  p.psi0.assign(psi0, psi0 + (size_t)order * cells);
  p.inc_left = inc_left ? std::vector<double>(inc_left, inc_left + order)
                        : std::vector<double>(order, 0.0);
  p.inc_right = inc_right ? std::vector<double>(inc_right, inc_right + order)
                          : std::vector<double>(order, 0.0);
  if (q) {  // constant in time (SnProblem::q): one row for every step
    p.q_rows.assign(q, q + cells);
    p.q_index.assign(steps + 1, 0);
  }
  p.tolerance = tolerance;
  p.max_iterations = max_iterations;
  sn_solve_device(p, c->device, c->stream, phi_layers, iterations, nullptr, nullptr);
  return HWWG_OK;
  HWWG_API_END
}

int hwwg_compute_reference(hwwg_ctx* c, const hwwg_run_config* cfg, int32_t space_refine,
                           int32_t time_refine, int32_t sn_order, double* phi_layer,
                           double* phi_interval) {
  HWWG_API_BEGIN
  if (!c || !cfg || !phi_layer || !phi_interval) return fail(HWWG_EINVAL, "NULL argument");
  const SnHostProblem p = reference_problem(*cfg, space_refine, time_refine, sn_order);
  sn_solve_device(p, c->device, c->stream, nullptr, nullptr, phi_layer, phi_interval);
  return HWWG_OK;
  HWWG_API_END
}

int hwwg_device_log(hwwg_ctx* c, const double* x, uint64_t n, double* out) {
  HWWG_API_BEGIN
  if (!c || (n && (!x || !out))) return fail(HWWG_EINVAL, "NULL argument");
  if (!n) return HWWG_OK;
  HWWG_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  c->scratch.reserve(2 * n);
  HWWG_CUDA(cudaMemcpyAsync(c->scratch.p, x, n * 8, cudaMemcpyHostToDevice, s));
  launch_device_log(c->scratch.p, n, c->scratch.p + n, s);
  HWWG_CUDA(cudaMemcpyAsync(out, c->scratch.p + n, n * 8, cudaMemcpyDeviceToHost, s));
  HWWG_CUDA(cudaStreamSynchronize(s));
  return HWWG_OK;
  HWWG_API_END
}

}  // extern "C"
