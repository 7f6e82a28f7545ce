// hwwg_driver: the reference's time-step loop (hww::run / hww::run_step,
// proj/src/driver.cpp:99-342) with every per-step array resident on the GPU.
//
// One step = comb -> start-of-step LOSM windows -> u_ww+1 transport segments
// with a single-CTA snapshot/filter/solve/centres kernel at each update
// barrier -> finalize -> census sort.  The host only computes the update
// thresholds (driver.cpp:170-177) and reads the step record back once, at the
// end of the step.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "capi_util.h"
#include "comm.h"
#include "common.cuh"
#include "device_state.cuh"
#include "driver_host.h"
#include "engine.cuh"
#include "low_order.cuh"
#include "reference_io.h"
#include "sn.cuh"
#include "rng.cuh"
#include "fast.cuh"
#include "transport.cuh"

using namespace hwwg;

namespace {

__global__ void k_bank_weight(const hwwg_particle* bank, uint64_t n, double* out) {
  double w = 0.0;  // total_weight (particle.hpp:18-22), sequential
  for (uint64_t i = 0; i < n; ++i) w += bank[i].w;
  *out = w;
}

__global__ void k_active_from_fallback(int* flags) { flags[0] = flags[5] ? 0 : 1; }

}  // namespace

namespace hwwg {
void set_active_from_fallback(int* flags, cudaStream_t s) {
  k_active_from_fallback<<<1, 1, 0, s>>>(flags);
  HWWG_CUDA(cudaGetLastError());
}

// Owner of a SoA particle bank (fast mode).
struct FastBankBuf {
  DevBuf<double2> xm, wt;
  DevBuf<uint4> meta;
  void reserve(uint64_t n) {
    n = n ? n : 1;
    xm.reserve(n);
    wt.reserve(n);
    meta.reserve(n);
  }
  uint64_t cap() const { return std::min(xm.n, std::min(wt.n, meta.n)); }
  void release() {
    for (void* p : {(void*)xm.p, (void*)wt.p, (void*)meta.p})
      if (p) cudaFree(p);
    xm.p = wt.p = nullptr;
    meta.p = nullptr;
    xm.n = wt.n = meta.n = 0;
  }
  FastBank view() { return FastBank{xm.p, wt.p, meta.p}; }
  void swap(FastBankBuf& o) {
    std::swap(xm.p, o.xm.p);
    std::swap(xm.n, o.xm.n);
    std::swap(wt.p, o.wt.p);
    std::swap(wt.n, o.wt.n);
    std::swap(meta.p, o.meta.p);
    std::swap(meta.n, o.meta.n);
  }
};
// Owner of a census bank (fast mode; fast.cuh CensusBank, 24 B per particle).
struct CensusBankBuf {
  DevBuf<double2> xm;
  DevBuf<double> w;
  void reserve(uint64_t n) {
    n = n ? n : 1;
    xm.reserve(n);
    w.reserve(n);
  }
  uint64_t cap() const { return std::min(xm.n, w.n); }
  void release() {
    if (xm.p) cudaFree(xm.p);
    if (w.p) cudaFree(w.p);
    xm.p = nullptr;
    w.p = nullptr;
    xm.n = w.n = 0;
  }
  CensusBank view() { return CensusBank{xm.p, w.p}; }
  void swap(CensusBankBuf& o) {
    std::swap(xm.p, o.xm.p);
    std::swap(xm.n, o.xm.n);
    std::swap(w.p, o.w.p);
    std::swap(w.n, o.w.n);
  }
};
}  // namespace hwwg

// e2e transfer pieces per step at most (xfer_chunks)
constexpr size_t kMaxXferChunks = 48;

struct hwwg_driver {
  hwwg_run_config cfg{};
  hwwg_options opt{};
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  DeviceProblem prob;
  DeviceTallies tal;
  HostTallies host_tal;
  std::vector<double> layers;
  // deterministic reference for the step diagnostics (hwwg_driver_set_reference)
  std::vector<double> ref_layer, ref_interval;
  int I = 0, B = 0;
  uint64_t target = 0;
  int next_step = 1;

  // particle banks: `bank` holds the previous census (reference order)
  DevBuf<hwwg_particle> bank, source;
  uint64_t bank_n = 0;
  // host_bank mode (e2e): the bank round-trips through pinned host memory
  hwwg_particle* host_bank = nullptr;
  uint64_t host_bank_n = 0, host_bank_cap = 0;
  std::vector<cudaEvent_t> seg_ev;  // transport-kernel timing (2 per segment)
  uint64_t launches = 0;
  CensusStage stage;
  DevBuf<double> comb_mem;  // scalars[4] + prefix
  DevBuf<unsigned long long> counter;
  DevBuf<DevError> err;
  DevBuf<double> chunk_mem;
  ExactLogBuf xlog;  // history-parallel exact path

  // throughput (Philox) mode: SoA banks, warp split stacks, refill cursor
  bool fast = false;
  uint64_t census_hwm = 0;  // census capacity high-water mark (banks swap each step)
  uint64_t census_floor = 0;  // the creation-time capacity (64 x H)
  // fbank: the bank the next comb reads (the last census, or the pulse), all
  // at time bank_t; fcensus: the census being written; fsrc: the step's source
  CensusBankBuf fbank, fcensus;
  FastBankBuf fsrc;
  double bank_t = 0.0;
  DevBuf<FastStackRec> stacks;
  int stack_cap = 1024;
  int sms = 148;
  DevBuf<unsigned long long> src_head;
  DevBuf<char> comb_temp;
  DevBuf<FastStackRec> pool_recs;
  DevBuf<unsigned long long> pool_ctl;
  int smem_mode = 1;  // fast tallies (FastArgs::smem_tallies) outside the cold start
  int scramble = 1;   // FastArgs::scramble outside the cold start
  // warp-aggregated tallies: step 1 always; later steps when the tally
  // histograms do not fit shared memory (-1, default), every step (1), or
  // step 1 only (0), never (2, tests) — HWWG_FAST_AGG
  int agg_all = -1;
  // fixed-point track/edge tallies (FastArgs::fix; HWWG_FAST_FIX=0 disables);
  // step_wref: the largest source weight the step is expected to carry (the
  // pulse strength, the volumetric source's particle weight)
  int fix_tallies = 1;
  int pdl = 1;  // programmatic dependent launches across segment boundaries (HWWG_PDL)
  int block_warps = 0;  // transport block shape: 0 per launch, else 12 or 24 (HWWG_FAST_BLOCK_WARPS)
  // transport_ms: exact mode times its segments with CUDA events; the
  // throughput mode with in-kernel launch spans (FastArgs::span), because
  // events between its segment kernels cost 4% (HWWG_SEG_EVENTS=1 restores them)
  int seg_events = 1;
  DevBuf<unsigned long long> span;  // 2 words per segment
  double step_wref = 1.0;
  // config-3 volumetric source: the step's LOSM q (device) and particle staging
  // q of every step the box overlaps, precomputed at creation (q_row[step]:
  // row of q_all, -1 when the step sees no emission)
  DevBuf<double> q_all;
  std::vector<int> q_row;
  const double* q_step = nullptr;
  // start-of-step window update overlapping the comb (auxiliary stream)
  cudaStream_t aux_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // e2e (host_bank): chunked source upload on its own stream (one event per chunk)
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> h2d_ev;
  // e2e round-trip pipeline (single GPU, packed): the combed source goes down to
  // the host in sub-chunks on d2h_stream right after the comb, and the next
  // step uploads sub-chunk i as soon as its download (d2h_ev[i]) landed, so the
  // two PCIe directions overlap each other and the transport of earlier
  // segments; xfer_end: the sub-chunks' ends (every segment end among them)
  cudaStream_t d2h_stream = nullptr;
  cudaEvent_t ev_pre = nullptr;
  std::vector<cudaEvent_t> d2h_ev;
  std::vector<uint64_t> xfer_end;
  bool d2h_pending = false;
  bool e2e_pipe = true;  // HWWG_E2E_PIPE=0: the download completes inside its step
  cudaEvent_t xt[8] = {};  // HWWG_HOST_PROF: d2h start/end, h2d start/end, d2h p0 end, h2d p0 end, seg0 start
  // e2e (host_bank) Philox runs: the bank in host memory is already combed
  bool host_pre_combed = false;
  uint64_t pre_comb_in = 0;
  uint64_t pre_Hc = 0, pre_nv = 0;  // multi-rank: combed / volumetric histories of the pre-combed step
  // packed wire format of a pre-combed host bank: (x, mu) per particle, then
  // (w, t) per particle only when they are not one shared pair (host_uniform)
  bool host_packed = false, host_uniform = false;
  bool host_pulse_mu = false;  // the host bank holds the pulse as directions only (step 1)
  double host_w0 = 0.0, host_t0 = 0.0;
  DevBuf<unsigned> uni_flag;
  DevBuf<double2> uni_first;
  unsigned* h_uni = nullptr;  // pinned: [0] flag, then (w0, t0) at byte 16
  int flush_replicas = 0;  // FastArgs::flush_replicas (HWWG_FAST_FLUSH_R; 0 = direct REDs, measured best)
  DevBuf<double> flush_scratch;
  bool timeline_on = false;
  // HWWG_PHASES=1: CUDA-event time of the step's non-transport phases (stderr)
  bool phases_on = false;
  std::vector<cudaEvent_t> ph_ev;
  std::vector<const char*> ph_name;
  size_t ph_n = 0;
  void ph_mark(const char* name, cudaStream_t s) {  // closes the previous phase, opens `name`
    if (!phases_on) return;
    if (ph_n >= ph_ev.size()) {
      cudaEvent_t e;
      HWWG_CUDA(cudaEventCreate(&e));
      ph_ev.push_back(e);
      ph_name.push_back(name);
    }
    ph_name[ph_n] = name;
    HWWG_CUDA(cudaEventRecord(ph_ev[ph_n++], s));
  }
  DevBuf<unsigned long long> timeline;
  unsigned timeline_warps = 0;
  DevBuf<unsigned long long> warp_cursor;  // per-warp census chunks
  int max_warps = 0;
  // census thinning (FastArgs::precomb): on in the cold start and whenever the
  // previous census held more than precomb_k x target particles; the thinned
  // census holds ~precomb_k x target records (HWWG_PRECOMB=0 disables it,
  // HWWG_PRECOMB_K sets k)
  int precomb = 1;
  double precomb_k = 8.0;
  DevBuf<double> pc_need;  // per-lane comb residuals (32 per warp)

  // multi-GPU: histories sharded by rank, tallies all-reduced
  // at every window-update barrier and at step end, census combed globally and
  // rebalanced with grouped send/recv
  int rank = 0, world = 1;
  uint64_t shard_lo = 0;    // first history of this rank's share of the step-1 pulse bank
  uint64_t fsrc_local = 0;  // combed histories this rank holds (the front of fsrc)
  // fsrc's first src_packed slots are single-GPU comb teeth stored as (x, mu)
  // only (FastCombArgs::packed_out; FastArgs::n_packed): weight comb_mem[1]
  // (the spacing, on the device), time src_t0
  uint64_t src_packed = 0;
  double src_t0 = 0.0;
  int packed_teeth = 1;  // HWWG_PACKED_TEETH=0: full 48 B teeth (A/B and tests)
  int tally_window = 1;  // HWWG_TALLY_WINDOW=0: no windowed shared tallies (config 4)
  int tally_window_max = 0;  // HWWG_TALLY_WINDOW_MAX=n: clip the window to n cells (tests of the fallback)
  Comm* comm = nullptr;      // NCCL or the in-process loopback (comm.h)
  bool own_stream = true;    // false: the loopback hub's shared stream
  DevBuf<double> nccl_buf;    // all-gathered census weights, snapshot slabs
  FastBankBuf fteeth;         // teeth this rank produced, before the rebalance
  FastBankBuf fperm;          // the rebalanced teeth before the local permutation

  // low-order state
  DevBuf<double> lo_mem;
  DevBuf<double> lo_fac;  // cached LOSM factorization (throughput mode)
  DevBuf<double> ftab_cell, ftab_edge;  // hww_fourier twiddles (fourier_tables)
  bool losm_cache = true;  // HWWG_LOSM_NOCACHE=1 disables it
  bool fac_valid = false;
  double fac_theta = 0.0, fac_dt = 0.0;
  // 1 when the cached factorization does not match (theta, dt): the next
  // update kernel rebuilds it (launches are stream-ordered)
  int need_refactor(double theta, double dt) {
    if (fac_valid && fac_theta == theta && fac_dt == dt) return 0;
    fac_valid = true;
    fac_theta = theta;
    fac_dt = dt;
    return 1;
  }
  DevBuf<int> lo_flags;
  LowOrderState lo{};
  DevBuf<double> centers_backup;
  DevBuf<int> flags_backup;
  // finalize outputs: two report buffers, current and previous
  DevBuf<double> rep_mem[2];
  int rep_cur = 0;
  bool has_prev_report = false;

  // host copies of the last StepRecord arrays
  std::vector<double> h_phi_track, h_sigma, h_phi_census, h_current, h_closure, h_edge,
      h_centers, h_hybrid;
  std::vector<unsigned long long> h_tracks;
  bool h_has_centers = false, h_has_hybrid = false;
  std::vector<hwwg_step_record> history;  // every step so far (summary.csv)

  ~hwwg_driver() {
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    for (auto e : seg_ev) cudaEventDestroy(e);
    for (auto e : ph_ev) cudaEventDestroy(e);
    for (auto e : h2d_ev) cudaEventDestroy(e);
    if (d2h_stream) cudaStreamSynchronize(d2h_stream);
    for (auto e : d2h_ev) cudaEventDestroy(e);
    for (auto e : xt)
      if (e) cudaEventDestroy(e);
    if (ev_pre) cudaEventDestroy(ev_pre);
    if (d2h_stream) cudaStreamDestroy(d2h_stream);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (aux_stream) cudaStreamDestroy(aux_stream);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (host_bank) cudaFreeHost(host_bank);
    if (h_uni) cudaFreeHost(h_uni);
    delete comm;
    if (stream && own_stream) cudaStreamDestroy(stream);
  }

  double* rep(int which, int field) {  // field: 0 phi_track,1 sigma,2 phi_census,3 current,
                                       // 4 closure,5 edge(I+1),6 scalars(8)
    return rep_mem[which].p + (size_t)field * (I + 1);
  }

  bool hybrid() const { return cfg.mode >= 2; }
};

namespace {

void init_driver(hwwg_driver* d) {
  const hwwg_run_config& c = d->cfg;
  d->I = c.cells;
  d->B = c.batches;
  d->target = c.target_population ? c.target_population : c.histories_per_step;
  HWWG_CUDA(cudaSetDevice(d->opt.device));
  if (d->world > 1) {  // communicator first: a loopback hub supplies the stream
    if (d->opt.loopback) d->comm = make_loopback_comm(d->opt.loopback, d->rank);
    else d->comm = make_nccl_comm(d->opt.nccl_id, d->rank, d->world);
  }
  if (d->comm && d->comm->shared_stream()) {
    d->stream = d->comm->shared_stream();
    d->own_stream = false;
  } else {
    HWWG_CUDA(cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking));
  }
  HWWG_CUDA(cudaEventCreate(&d->ev0));
  HWWG_CUDA(cudaEventCreate(&d->ev1));
  const int I = d->I;
  // mesh and time grid (config.hpp:87-88; mesh.cpp:42-50; time_grid.hpp:22-29)
  std::vector<double> edges(I + 1);
  const double w = (c.x_max - c.x_min) / I;
  for (int e = 0; e <= I; ++e) edges[e] = c.x_min + e * w;
  edges[I] = c.x_max;
  std::vector<hwwg_material> mats(I, hwwg_material{c.sigma_t, c.sigma_s, c.sigma_f, c.nu_f, c.speed});
  if (c.n_regions > 0)  // config-3 regions: the first whose upper bound exceeds the cell centre
    for (int i = 0; i < I; ++i) {
      const double xc = 0.5 * (edges[i] + edges[i + 1]);
      int r = 0;
      while (r < c.n_regions - 1 && !(xc < c.region_x_hi[r])) ++r;
      const double* m = c.region_mat[r];
      mats[i] = hwwg_material{m[0], m[1], m[2], m[3], m[4]};
    }
  std::string why;
  if (!d->prob.set(edges.data(), I, mats.data(), d->stream, why)) throw ApiError(HWWG_EINVAL, why);
  d->layers.resize(c.time_steps + 1);
  const double dt = (c.t_end - 0.0) / c.time_steps;
  for (int n = 0; n <= c.time_steps; ++n) d->layers[n] = 0.0 + n * dt;
  d->layers[c.time_steps] = c.t_end;
  d->tal.shape(I, d->B);

  // low-order state
  const int n = 2 * I + 3;
  const size_t lo_words = (size_t)(I + 2) * 3 + (I + 1) + 2 + 3 * (size_t)I + 2 + 2 * (size_t)I +
                          6 * (size_t)n + (I + 2);
  d->lo_mem.reserve(lo_words);
  HWWG_CUDA(cudaMemsetAsync(d->lo_mem.p, 0, lo_words * 8, d->stream));
  double* q = d->lo_mem.p;
  LowOrderState& s = d->lo;
  s.phi_prev = q; q += I + 2;
  s.J_prev = q; q += I + 1;
  s.F_prev = q; q += I + 2;
  s.PLPR_prev = q; q += 2;
  s.rep_phi_census = nullptr;  // bound per step to the previous report
  s.rep_current = nullptr;
  s.rep_closure = nullptr;
  s.rep_PLPR = nullptr;
  s.centers = q; q += I;
  s.phi_hybrid = q; q += I;
  s.sys = q; q += 6 * (size_t)n;
  s.F_now = q; q += I + 2;
  s.fac = nullptr;
  if (c.mode == 4) {  // hww_fourier: host-libm twiddles for the I- and (I+1)-point transforms
    const std::vector<double> tc = fourier_tables(I), te = fourier_tables(I + 1);
    d->ftab_cell.reserve(tc.size());
    d->ftab_edge.reserve(te.size());
    HWWG_CUDA(cudaMemcpy(d->ftab_cell.p, tc.data(), tc.size() * 8, cudaMemcpyHostToDevice));
    HWWG_CUDA(cudaMemcpy(d->ftab_edge.p, te.data(), te.size() * 8, cudaMemcpyHostToDevice));
  }
  if (d->fast && d->losm_cache && lo_fac_words(I)) {  // cached LOSM factorization
    d->lo_fac.reserve(lo_fac_words(I));
    s.fac = d->lo_fac.p;
    static const double kUnbuilt = 2.0;  // state word (last): not built yet
    HWWG_CUDA(cudaMemcpyAsync(d->lo_fac.p + lo_fac_words(I) - 1, &kUnbuilt, sizeof(double),
                              cudaMemcpyHostToDevice, d->stream));
  }
  d->lo_flags.reserve(8);
  HWWG_CUDA(cudaMemsetAsync(d->lo_flags.p, 0, 8 * sizeof(int), d->stream));
  s.flags = d->lo_flags.p;
  d->centers_backup.reserve(I);
  d->flags_backup.reserve(8);
  for (auto& r : d->rep_mem) {
    r.reserve((size_t)7 * (I + 1) + 8);
    HWWG_CUDA(cudaMemsetAsync(r.p, 0, ((size_t)7 * (I + 1) + 8) * 8, d->stream));
  }
  d->counter.reserve(1);
  d->err.reserve(1);
  d->comb_mem.reserve(4);
  if (c.vol_rate > 0.0) {  // config-3 LOSM q per step (volume_q_host), uploaded once
    d->q_row.assign(c.time_steps + 1, -1);
    std::vector<double> qh;
    for (int n = 1; n <= c.time_steps; ++n) {
      const double ta = std::max(d->layers[n - 1], c.vol_t_lo);
      const double tb = std::min(d->layers[n], c.vol_t_hi);
      if (!(tb > ta)) continue;
      d->q_row[n] = (int)(qh.size() / I);
      qh.resize(qh.size() + I);
      volume_q_host(d->prob.edges.data(), I, c.vol_x_lo, c.vol_x_hi, ta, tb,
                    d->layers[n] - d->layers[n - 1], c.vol_rate, qh.data() + qh.size() - I);
    }
    d->q_all.reserve(std::max<size_t>(qh.size(), 1));
    if (!qh.empty())
      HWWG_CUDA(cudaMemcpyAsync(d->q_all.p, qh.data(), qh.size() * 8, cudaMemcpyHostToDevice, d->stream));
  }

  // source sampling (driver.cpp:309-316) on the host: one sequential stream
  std::vector<hwwg_particle> src(c.no_pulse ? 0 : c.histories_per_step);
  if (!c.no_pulse)
    sample_pulse_source_host(c.seed, c.histories_per_step, c.x0,
                             c.strength * (double)c.histories_per_step, 0.0, src.data());
  if (d->world > 1) {  // this rank's shard of the step-1 histories
    uint64_t lo, hi;
    hwwg_shard_range(src.size(), d->rank, d->world, &lo, &hi);  // empty without a pulse
    src = std::vector<hwwg_particle>(src.begin() + lo, src.begin() + hi);
    d->shard_lo = lo;
  }
  d->bank.reserve(std::max<uint64_t>(src.size(), 1));
  HWWG_CUDA(cudaMemcpyAsync(d->bank.p, src.data(), src.size() * sizeof(hwwg_particle),
                            cudaMemcpyHostToDevice, d->stream));
  d->bank_n = src.size();
  if (c.host_bank) {
    // exact mode: room for the cold-start census (x60+ of H) so no step re-pins
    // host memory; Philox mode hands the host the combed bank (target
    // particles; multi-rank runs grow it on demand)
    d->host_bank_cap = std::max<uint64_t>(
        src.size(), (d->fast ? 1 : 64) * d->target + 4096);
    HWWG_CUDA(cudaMallocHost(&d->host_bank, d->host_bank_cap * sizeof(hwwg_particle)));
    d->host_bank_n = src.size();
    // Philox mode, one GPU: the pulse's particles share x0, w0 and t = 0, so the
    // host holds (and step 1 uploads) their directions alone, 8 B per particle
    d->host_pulse_mu = d->fast && d->world == 1 && !src.empty();
    if (d->host_pulse_mu) {
      double* hm = reinterpret_cast<double*>(d->host_bank);
      for (size_t i = 0; i < src.size(); ++i) hm[i] = src[i].mu;
      d->host_w0 = src[0].w;
      d->host_t0 = src[0].t;
    } else {
      std::memcpy(d->host_bank, src.data(), src.size() * sizeof(hwwg_particle));
    }
  }
  d->seg_ev.resize(32);
  for (auto& e : d->seg_ev) HWWG_CUDA(cudaEventCreate(&e));
  HWWG_CUDA(cudaStreamCreateWithFlags(&d->aux_stream, cudaStreamNonBlocking));
  HWWG_CUDA(cudaEventCreateWithFlags(&d->ev_fork, cudaEventDisableTiming));
  HWWG_CUDA(cudaEventCreateWithFlags(&d->ev_join, cudaEventDisableTiming));
  if (c.host_bank) {
    HWWG_CUDA(cudaStreamCreateWithFlags(&d->copy_stream, cudaStreamNonBlocking));
    d->h2d_ev.resize(kMaxXferChunks);
    for (auto& e : d->h2d_ev) HWWG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    HWWG_CUDA(cudaStreamCreateWithFlags(&d->d2h_stream, cudaStreamNonBlocking));
    HWWG_CUDA(cudaEventCreateWithFlags(&d->ev_pre, cudaEventDisableTiming));
    d->d2h_ev.resize(kMaxXferChunks);
    for (auto& e : d->d2h_ev) HWWG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    HWWG_CUDA(cudaMallocHost(&d->h_uni, 64));
    d->uni_flag.reserve(1);
    d->uni_first.reserve(1);
  }
  if (d->fast) {
    const uint64_t local_target = d->target / (uint64_t)d->world + 1;
    d->fbank.reserve(std::max<uint64_t>(d->bank_n, 64 * local_target + 4096));
    launch_aos_to_census(d->bank.p, d->bank_n, d->fbank.view(), d->stream);
    d->bank_t = 0.0;  // the pulse is emitted at t = 0 (driver.cpp:309-316)
    // Everything a step can grow into is allocated here, up front: a cudaMalloc
    // inside a step synchronises the device (the step-1 census is x60+ of H,
    // and it becomes step 2's comb input in the other bank of the swap pair).
    // (with census thinning the cold start banks ~precomb_k x H records, not the
    // x60-x150 raw census; a larger census replays its step with room)
    const uint64_t mult = d->precomb ? (uint64_t)(2.0 * d->precomb_k) : 64;
    d->census_hwm = d->census_floor = mult * local_target + 4096;
    d->fcensus.reserve(d->census_hwm);
    d->fbank.reserve(d->census_hwm);
    d->fsrc.reserve(std::max<uint64_t>(d->target + (c.vol_rate > 0.0 ? c.vol_histories : 0), 1));
    // comb scratch: O(n / 4096) words (single GPU); the multi-GPU local scan
    // keeps an n-sized prefix, sized per step
    d->comb_mem.reserve(4 + fast_comb_scratch_words(d->census_hwm));
    if (d->world > 1) {
      d->comb_temp.reserve(fast_comb_temp_bytes(d->census_hwm));
      d->comb_mem.reserve(4 + d->census_hwm);
    }
    if (c.host_bank) d->bank.reserve(d->census_hwm);
    if (d->world > 1) {
      d->nccl_buf.reserve(std::max<size_t>(4 * (size_t)d->world + 16, (size_t)I + 8));
      d->fperm.reserve(local_target + 4096);  // the rebalanced teeth before their permutation
    }
    HWWG_CUDA(cudaDeviceGetAttribute(&d->sms, cudaDevAttrMultiProcessorCount, d->opt.device));
    const int warps = d->sms * fast_max_warps_per_sm();
    d->max_warps = warps;
    d->warp_cursor.reserve((size_t)kWarpCursorWords * warps);
    d->pc_need.reserve((size_t)32 * warps);
    d->stacks.reserve((size_t)warps * d->stack_cap);
    d->src_head.reserve(1);
    d->pool_recs.reserve(1u << 20);  // 64 MB of donated split records per segment
    HWWG_CUDA(cudaMemsetAsync(d->pool_recs.p, 0, d->pool_recs.n * sizeof(FastStackRec), d->stream));
    d->pool_ctl.reserve(8);  // [0..3] pool control, [4] segment start (diagnostics)
    if (d->flush_replicas) {
      const size_t words = (size_t)d->flush_replicas * fast_flush_stride(I, d->B);
      d->flush_scratch.reserve(words);
      HWWG_CUDA(cudaMemsetAsync(d->flush_scratch.p, 0, words * 8, d->stream));
    }
  } else {
    d->stage.ensure(64 * d->target + 4096);
    // the tally log arena, up front: the cold-start step logs ~10 blocks per
    // history at config 2, and growing a multi-GB arena inside a step (free +
    // malloc + a replay) costs 0.1-0.7 s
    d->xlog.ensure_blocks(16 * (d->target + 1) + 65536);
  }
  HWWG_CUDA(cudaStreamSynchronize(d->stream));
}

// Diagnostics (HWWG_FAST_TIMELINE=1): per segment, the spread of warp exit
// times and work, to separate load imbalance from per-event cost.
void print_timeline(hwwg_driver* d, int nseg, int step) {
  constexpr int K = kTimelineWords;
  const size_t per = (size_t)d->timeline_warps * K;
  std::vector<unsigned long long> h(per * nseg);
  HWWG_CUDA(cudaMemcpy(h.data(), d->timeline.p, h.size() * 8, cudaMemcpyDeviceToHost));
  std::vector<unsigned long long> sp(2 * (size_t)nseg, 0);  // launch spans (block start / end)
  if (!d->seg_events)
    HWWG_CUDA(cudaMemcpy(sp.data(), d->span.p, sp.size() * 8, cudaMemcpyDeviceToHost));
  for (int s = 0; s < nseg; ++s) {
    const unsigned long long* t = h.data() + per * s;
    if (sp[2 * s + 1]) {  // the flush tail: last block end after the last warp's exit
      unsigned long long lastx = 0;
      for (unsigned w = 0; w < d->timeline_warps; ++w) lastx = std::max(lastx, t[K * w + 2]);
      std::fprintf(stderr, "[timeline] step %d seg %d: launch span %.1f us, flush tail %.1f us\n", step, s,
                   1e-3 * (double)(sp[2 * s + 1] - sp[2 * s]),
                   sp[2 * s + 1] > lastx ? 1e-3 * (double)(sp[2 * s + 1] - lastx) : 0.0);
    }
    unsigned long long t0 = ~0ULL, tmax = 0, evs = 0, evmax = 0;
    unsigned wmax = 0;  // the warp with the most loop trips
    std::vector<double> ex, sd;
    for (unsigned w = 0; w < d->timeline_warps; ++w) {
      if (!t[K * w]) continue;
      t0 = std::min(t0, t[K * w]);
      tmax = std::max(tmax, t[K * w + 2]);
      evs += t[K * w + 3];
      evmax = std::max(evmax, t[K * w + 3]);
      if (t[K * w + 1] > t[K * wmax + 1]) wmax = w;
    }
    for (unsigned w = 0; w < d->timeline_warps; ++w) {
      if (!t[K * w]) continue;
      ex.push_back(1e-3 * (double)(t[K * w + 2] - t0));
      sd.push_back((double)t[K * w + 1]);
    }
    std::sort(ex.begin(), ex.end());
    std::sort(sd.begin(), sd.end());
    auto q = [](const std::vector<double>& v, double f) {
      return v.empty() ? 0.0 : v[std::min(v.size() - 1, (size_t)(f * v.size()))];
    };
    const unsigned long long* m = t + (size_t)K * wmax;
    std::fprintf(stderr,
                 "[timeline] step %d seg %d: span %.1f us, loop trips p50 %.0f max %.0f, "
                 "exit p10 %.1f p50 %.1f p90 %.1f p99 %.1f max %.1f us, events %llu "
                 "(per warp mean %.0f max %llu) | busiest warp %u: start %.1f exit %.1f us, "
                 "events %llu, max pending %llu, shared %llu, donated %llu, taken %llu\n",
                 step, s, 1e-3 * (double)(tmax - t0), q(sd, 0.5), q(sd, 1.0), q(ex, 0.1),
                 q(ex, 0.5), q(ex, 0.9), q(ex, 0.99), q(ex, 1.0), evs,
                 (double)evs / std::max<size_t>(ex.size(), 1), evmax, wmax,
                 1e-3 * (double)(m[0] - t0), 1e-3 * (double)(m[2] - t0), m[3], m[4], m[5], m[6],
                 m[7]);
  }
}

// Update thresholds (driver.cpp:170-177; ww.cpp:74-87): ceil(f * H), deduped.
std::vector<uint64_t> step_thresholds(const hwwg_run_config& c, bool hybrid, uint64_t H) {
  std::vector<uint64_t> thr;
  if (hybrid && c.u_ww > 0)
    for (int i = 0; i < c.n_fractions; ++i) {
      const uint64_t h = (uint64_t)std::ceil(c.fractions[i] * (double)H);
      if (h >= H) continue;
      if (!thr.empty() && h <= thr.back()) continue;
      thr.push_back(h);
    }
  return thr;
}

// Which histories of a step each rank runs. The step's
// global history ids [0, H) — combed teeth [0, H_c), then the step's
// volumetric particles [H_c, H) — are cut into the window-update segments
// [seg[u], seg[u+1]), and every segment is split into W contiguous pieces:
// rank q runs piece q of EVERY segment, so all ranks work in every segment
// and meet at every barrier. A rank holds its histories in global-id order
// (local index = number of its ids below), so each of its pieces, its combed
// ids and its volumetric ids are contiguous locally.
struct StepLayout {
  std::vector<uint64_t> seg;  // 0 = seg[0] <= ... <= seg[S] = H
  int W = 1;
  uint64_t H = 0, Hc = 0;
  void piece(int q, size_t u, uint64_t& lo, uint64_t& hi) const {
    uint64_t a, b;
    hwwg_shard_range(seg[u + 1] - seg[u], q, W, &a, &b);
    lo = seg[u] + a;
    hi = seg[u] + b;
  }
  size_t segments() const { return seg.size() - 1; }
  uint64_t owned_before(int q, uint64_t g) const {  // rank q's ids below g
    uint64_t n = 0, lo, hi;
    for (size_t u = 0; u < segments(); ++u) {
      piece(q, u, lo, hi);
      n += std::min(std::max(g, lo), hi) - lo;
    }
    return n;
  }
  uint64_t global_of(int q, uint64_t l) const {  // rank q's l-th id (H past the end)
    uint64_t lo, hi;
    for (size_t u = 0; u < segments(); ++u) {
      piece(q, u, lo, hi);
      if (l < hi - lo) return lo + l;
      l -= hi - lo;
    }
    return H;
  }
};

StepLayout make_layout(const hwwg_run_config& c, bool hybrid, uint64_t Hc, uint64_t H, int W) {
  StepLayout L;
  L.W = W;
  L.H = H;
  L.Hc = Hc;
  L.seg.push_back(0);
  for (uint64_t t : step_thresholds(c, hybrid, H)) L.seg.push_back(t);
  L.seg.push_back(H);
  return L;
}

// The rank's combed histories as (first global id, count) ranges, in its local order.
PieceTable comb_pieces(const StepLayout& L, int R) {
  PieceTable t{};
  for (size_t u = 0; u < L.segments() && t.n < 9; ++u) {
    uint64_t lo, hi;
    L.piece(R, u, lo, hi);
    hi = std::min(hi, L.Hc);
    if (hi <= lo) continue;
    t.lo[t.n] = lo;
    t.cnt[t.n] = hi - lo;
    ++t.n;
  }
  return t;
}

// Global comb + census rebalance over `world` ranks:
// local weight scan -> all-gather of the rank totals -> the same host plan on
// every rank (hwwg_comb_plan) -> this rank's teeth -> grouped send/recv so that
// rank r ends up holding the teeth of its pieces of the step layout (tooth g =
// history g), then — after the cold start — a local permutation of them (see
// Perm). Returns the number of combed histories (the target, or 0 when the
// global census is empty: a volumetric-source run before its first census),
// and the step layout for H_c + nv histories.
uint64_t multi_gpu_comb(hwwg_driver* d, int step, uint64_t nv, StepLayout& L, cudaStream_t s) {
  const int W = d->world, R = d->rank;
  const uint64_t n = d->bank_n;
  d->comb_mem.reserve(4 + std::max<uint64_t>(n, 1));
  const size_t tb = fast_comb_temp_bytes(std::max<uint64_t>(n, 1));
  d->comb_temp.reserve(tb);
  FastCombArgs a{};
  a.bank = d->fbank.view();
  a.t_bank = d->bank_t;
  a.mesh = d->prob.view;
  a.n = n;
  a.prefix = d->comb_mem.p + 4;
  a.scalars = d->comb_mem.p;
  a.temp = d->comb_temp.p;
  a.temp_bytes = tb;
  launch_fast_comb_local_scan(a, s);  // scalars[0] = this rank's census weight
  d->comm->all_gather(d->comb_mem.p, d->nccl_buf.p, 1, DType::kF64, s);
  std::vector<double> wr(W);
  HWWG_CUDA(cudaMemcpyAsync(wr.data(), d->nccl_buf.p, W * 8, cudaMemcpyDeviceToHost, s));
  HWWG_CUDA(cudaStreamSynchronize(s));
  double total = 0.0;
  for (double w : wr) total += w;
  const uint64_t Hc = total > 0.0 ? d->target : 0;  // same decision on every rank
  L = make_layout(d->cfg, d->hybrid(), Hc, Hc + nv, W);
  d->fsrc_local = L.owned_before(R, Hc);
  if (Hc == 0) {
    HWWG_CUDA(cudaMemsetAsync(d->comb_mem.p, 0, 4 * sizeof(double), s));
    return 0;
  }
  Xoshiro rng;  // the comb stream of the step (driver.cpp:119-121), same on every rank
  rng.seed(d->cfg.seed, stream_id_host(step, 0, 3));
  const double frac = rng.uniform();
  std::vector<uint64_t> klo(W), khi(W);
  double spacing = 0, offset = 0, origin = 0;
  for (int q = 0; q < W; ++q) {
    double sp, off, org;
    if (hwwg_comb_plan(wr.data(), W, q, d->target, frac, &sp, &off, &org, &klo[q], &khi[q]) != 0)
      throw ApiError(HWWG_EINVAL, last_error_slot());
    if (q == R) {
      spacing = sp;
      offset = off;
      origin = org;
    }
  }
  const uint64_t nt = khi[R] - klo[R];
  d->fteeth.reserve(std::max<uint64_t>(nt, 1));
  if (nt) launch_fast_comb_teeth_range(a, spacing, offset, origin, klo[R], khi[R], d->fteeth.view(), s);
  const bool permute = step > 1;  // the cold-start bank is the i.i.d. pulse
  const uint64_t nloc = d->fsrc_local;
  FastBankBuf& dst_buf = permute ? d->fperm : d->fsrc;
  dst_buf.reserve(std::max<uint64_t>(nloc, 1));
  const FastBank dst = dst_buf.view(), th = d->fteeth.view();
  auto copy = [&](uint64_t to, uint64_t from, uint64_t m) {
    HWWG_CUDA(cudaMemcpyAsync(dst.xm + to, th.xm + from, m * 16, cudaMemcpyDeviceToDevice, s));
    HWWG_CUDA(cudaMemcpyAsync(dst.wt + to, th.wt + from, m * 16, cudaMemcpyDeviceToDevice, s));
    HWWG_CUDA(cudaMemcpyAsync(dst.meta + to, th.meta + from, m * 16, cudaMemcpyDeviceToDevice, s));
  };
  auto send = [&](uint64_t from, uint64_t m, int q) {
    d->comm->send(th.xm + from, 2 * m, DType::kF64, q, s);
    d->comm->send(th.wt + from, 2 * m, DType::kF64, q, s);
    d->comm->send(th.meta + from, 4 * m, DType::kU32, q, s);
  };
  auto recv = [&](uint64_t to, uint64_t m, int q) {
    d->comm->recv(dst.xm + to, 2 * m, DType::kF64, q, s);
    d->comm->recv(dst.wt + to, 2 * m, DType::kF64, q, s);
    d->comm->recv(dst.meta + to, 4 * m, DType::kU32, q, s);
  };
  d->comm->group_start();
  if (!permute) {
    // Cold start: the teeth with ids in rank q's pieces go to q, at q's local
    // index of the id (both sides walk q's pieces in order: sends and receives
    // match), so history g gets tooth g on any rank count — step 1 is the
    // single-GPU step (tests/test_gpu_multirank.py).
    auto cut = [&](int q, size_t u, uint64_t k_lo, uint64_t k_hi, uint64_t& lo, uint64_t& hi) {
      L.piece(q, u, lo, hi);
      lo = std::max(lo, k_lo);
      hi = std::min(std::min(hi, Hc), k_hi);
      return hi > lo;
    };
    for (int q = 0; q < W; ++q) {
      for (size_t u = 0; u < L.segments(); ++u) {
        uint64_t lo, hi;
        if (!cut(q, u, klo[R], khi[R], lo, hi)) continue;
        if (q == R) copy(L.owned_before(R, lo), lo - klo[R], hi - lo);
        else send(lo - klo[R], hi - lo, q);
      }
      if (q == R) continue;
      for (size_t u = 0; u < L.segments(); ++u) {
        uint64_t lo, hi;
        if (cut(R, u, klo[q], khi[q], lo, hi)) recv(L.owned_before(R, lo), hi - lo, q);
      }
    }
  } else {
    // Later steps: the rank's teeth are about its share already (a census
    // weight share of ~1/W, off by a few 1e-3 at 1e7 histories per rank), and
    // its histories are a permutation of its slots anyway, so a rank keeps
    // min(teeth, slots) of its own teeth and only the excess moves: excess
    // rank tails are matched to deficit ranks in rank order, identically on
    // every rank (round 2's first version moved (W-1)/W of all teeth).
    std::vector<uint64_t> own(W), have(W);
    for (int q = 0; q < W; ++q) {
      own[q] = L.owned_before(q, Hc);
      have[q] = khi[q] - klo[q];
    }
    const uint64_t keep = std::min(have[R], own[R]);
    if (keep) copy(0, 0, keep);
    int qe = 0, qd = 0;            // next excess / deficit rank
    uint64_t oe = 0, od = 0;       // consumed within them
    while (true) {
      while (qe < W && (have[qe] <= own[qe] || oe == have[qe] - own[qe])) ++qe, oe = 0;
      while (qd < W && (own[qd] <= have[qd] || od == own[qd] - have[qd])) ++qd, od = 0;
      if (qe >= W || qd >= W) break;
      const uint64_t m = std::min(have[qe] - own[qe] - oe, own[qd] - have[qd] - od);
      if (qe == R) send(own[R] + oe, m, qd);  // the excess is the tail of the rank's teeth
      if (qd == R) recv(have[R] + od, m, qe);
      oe += m;
      od += m;
    }
  }
  d->comm->group_end(s);
  d->launches += 3;
  if (permute) {  // out[c] = in[perm(c)], history = the global id of slot c
    const PieceTable t = comb_pieces(L, R);
    launch_fast_permute(d->fperm.view(), d->fsrc.view(), nloc, make_perm(nloc, d->cfg.seed, step),
                        t, s);
    ++d->launches;
  }
  // the step record's comb scalars: global input weight and combed weight
  // (pageable source: staged before the call returns)
  const double sc[4] = {total, spacing, offset, spacing * (double)d->target};
  HWWG_CUDA(cudaMemcpyAsync(d->comb_mem.p, sc, sizeof sc, cudaMemcpyHostToDevice, s));
  return d->target;
}

__global__ void k_stream_mark() {}

// e2e transfer pieces of a combed source of Hs histories in a step of Hs + nv
// (nv: the step's volumetric particles, sampled on the device after the teeth):
// the step's segment ranges [0, h_1), [h_1, h_2), ... (driver.cpp:170-177,
// make_layout) clipped to [0, Hs), each cut into pieces of about Hs / 32
// particles, so an upload can start as soon as its piece came down;
// *seg_last[u] = index of the last piece segment u needs.
std::vector<uint64_t> xfer_chunks(const hwwg_run_config& c, bool hybrid, uint64_t Hs, uint64_t nv,
                                  std::vector<size_t>* seg_last, uint64_t piece = 0) {
  std::vector<uint64_t> segs = step_thresholds(c, hybrid, Hs + nv);
  segs.push_back(Hs + nv);
  if (!piece) piece = std::max<uint64_t>(Hs / 32, 1 << 16);
  std::vector<uint64_t> ends;
  if (seg_last) seg_last->clear();
  uint64_t lo = 0;
  for (uint64_t e : segs) {
    const uint64_t hi = std::min(e, Hs);
    if (hi > lo) {
      const uint64_t n = std::max<uint64_t>(1, (hi - lo + piece - 1) / piece);
      for (uint64_t k = 1; k <= n; ++k) ends.push_back(k == n ? hi : lo + k * ((hi - lo) / n));
      lo = hi;
    }
    if (seg_last) seg_last->push_back(ends.empty() ? 0 : ends.size() - 1);
  }
  // many thresholds: one piece per segment
  if (ends.size() > kMaxXferChunks) return xfer_chunks(c, hybrid, Hs, nv, seg_last, Hs + 1);
  return ends;
}

// volumetric particles a step appends to its combed source (config 3)
uint64_t step_volume_histories(const hwwg_driver* d, int step);

uint64_t step_volume_histories(const hwwg_driver* d, int step) {
  const hwwg_run_config& c = d->cfg;
  if (!(c.vol_rate > 0.0) || step < 1 || step > c.time_steps) return 0;
  return d->q_row[step] >= 0 ? c.vol_histories : 0;
}

// One time step (driver.cpp:99-284).
void driver_step(hwwg_driver* d, hwwg_step_record* rec) {
  const hwwg_run_config& c = d->cfg;
  const int I = d->I, B = d->B;
  const int step = d->next_step;
  cudaStream_t s = d->stream;
  std::memset(rec, 0, sizeof(*rec));
  d->launches = 0;
  rec->step = step;
  rec->t_begin = d->layers[step - 1];
  rec->t_end = d->layers[step];
  const double dt = d->layers[step] - d->layers[step - 1];
  const auto t0 = std::chrono::steady_clock::now();
  const bool hprof = std::getenv("HWWG_HOST_PROF") != nullptr;  // host-side timestamps (stderr)
  auto hmark = [&](const char* what) {
    if (hprof)
      std::fprintf(stderr, "[host] step %d %s %.3f ms\n", step, what,
                   1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  };
  HWWG_CUDA(cudaEventRecord(d->ev0, s));
  const double theta_eff = step == 1 ? 1.0 : c.theta;
  const int ma_k = c.mode == 3 ? c.ma_base_k : 0;
  const int prev = d->rep_cur ^ 1;  // report of the previous step lives in the other buffer
  // config-3: the step's LOSM q (precomputed) and the volumetric particles' weight
  d->q_step = nullptr;
  d->step_wref = c.strength;
  uint64_t nv_step = 0;  // the step's volumetric particles
  if (c.vol_rate > 0.0 && d->q_row[step] >= 0) {
    nv_step = c.vol_histories;
    d->q_step = d->q_all.p + (size_t)d->q_row[step] * I;
    const double ta = std::max(rec->t_begin, c.vol_t_lo), tb = std::min(rec->t_end, c.vol_t_hi);
    if (c.vol_histories)
      d->step_wref = std::max(d->step_wref, c.vol_rate * (tb - ta) *
                                                (double)c.histories_per_step / (double)c.vol_histories);
  }

  // ---- the start-of-step windows (driver.cpp:136-167) on stream st: record
  // flags, then lww centres or the lagged hybrid solve
  // fold_backup: the hybrid solve kernel also takes the replay backup of the
  // incoming windows and zeroes the record flags (two copies and a memset less
  // ahead of the comb)
  auto enqueue_windows = [&](cudaStream_t st, bool fold_backup) {
    // per-step record flags: has_hybrid, updates_applied, failed, status
    if (!(fold_backup && d->hybrid()))
      HWWG_CUDA(cudaMemsetAsync(d->lo.flags + 1, 0, 4 * sizeof(int), st));
    if (c.mode == 1) {  // lww: lagged track-length flux of the previous step
      HWWG_CUDA(cudaMemsetAsync(d->lo.flags, 0, sizeof(int), st));
      if (d->has_prev_report) {
        launch_build_centers(d->rep(prev, 0), I, c.eps_min, c.rho, d->lo.centers,
                             d->lo.flags + 5, st);
        set_active_from_fallback(d->lo.flags, st);
        d->launches += 2;
      }
    } else if (d->hybrid()) {
      LowOrderArgs a{};
      a.I = I;
      a.edges = d->prob.view.edges;
      a.cells = d->prob.view.cells;
      a.theta = theta_eff;
      a.dt = dt;
      a.eps_min = c.eps_min;
      a.rho = c.rho;
      a.ma_k = ma_k;
      a.fourier_tab_cell = c.mode == 4 ? d->ftab_cell.p : nullptr;
      a.fourier_tab_edge = c.mode == 4 ? d->ftab_edge.p : nullptr;
      a.fourier_cutoff = c.fourier_cutoff;
      a.q = d->q_step;
      a.mode = 0;
      a.fast_solve = d->fast ? 1 : 0;
      a.refactor = d->need_refactor(theta_eff, dt);
      a.analytic = step == 1;
      if (step == 1 && !c.no_pulse) {
        const int cell = locate_host(d->prob.edges, c.x0);
        a.pulse_cell = cell;
        a.pulse_value = c.speed * c.strength / (d->prob.edges[cell + 1] - d->prob.edges[cell]);
      } else if (step == 1) {  // no pulse: the analytic initial state is zero
        a.pulse_cell = -2;
        a.pulse_value = 0.0;
      }
      a.s = d->lo;
      a.s.rep_phi_census = d->rep(prev, 2);
      a.s.rep_current = d->rep(prev, 3);
      a.s.rep_closure = d->rep(prev, 4);
      a.s.rep_PLPR = d->rep(prev, 6);
      if (fold_backup) {
        a.backup_centers = d->centers_backup.p;
        a.backup_flags = d->flags_backup.p;
      }
      d->ph_mark("losm0", st);
      launch_low_order_update(a, st);
      d->ph_mark("-", st);
      ++d->launches;
    }
  };
  // Single-GPU Philox steps without a volumetric source (whose q is known only
  // after the comb): the window update depends on the previous step alone, so
  // it runs on the auxiliary stream alongside the comb.
  const bool early_windows = d->fast && d->world == 1 && !d->phases_on;
  if (early_windows) {
    // backup of the windows so an overflowing step can be replayed exactly
    // (taken by the hybrid solve kernel itself when there is one)
    if (!d->hybrid()) {
      HWWG_CUDA(cudaMemcpyAsync(d->centers_backup.p, d->lo.centers, I * 8, cudaMemcpyDeviceToDevice, s));
      HWWG_CUDA(cudaMemcpyAsync(d->flags_backup.p, d->lo.flags, 8 * sizeof(int), cudaMemcpyDeviceToDevice, s));
    }
    HWWG_CUDA(cudaEventRecord(d->ev_fork, s));
    HWWG_CUDA(cudaStreamWaitEvent(d->aux_stream, d->ev_fork, 0));
    enqueue_windows(d->aux_stream, true);
    HWWG_CUDA(cudaEventRecord(d->ev_join, d->aux_stream));
  }

  // e2e with a pre-combed host bank: the source crosses PCIe in the chunks the
  // step's segments consume ([0, h_1), [h_1, h_2), ...) on a copy stream, and
  // segment u waits only for chunk u, so the later chunks overlap the earlier
  // segments' transport.
  std::vector<size_t> seg_wait;  // segment u waits for upload event h2d_ev[seg_wait[u]]
  std::vector<uint64_t> seg_range;  // packed uploads: segment u converts [seg_range[u], seg_range[u+1])
  d->src_packed = 0;  // set below where the step's source starts with packed comb teeth
  if (c.host_bank && d->fast && d->host_pre_combed && d->world == 1) {
    const uint64_t Hs = d->host_bank_n;
    const std::vector<uint64_t> bounds = xfer_chunks(c, d->hybrid(), Hs, nv_step, &seg_wait);
    const bool piped = d->d2h_pending && d->host_packed && bounds == d->xfer_end && d->e2e_pipe;
    if (d->d2h_pending && !piped) HWWG_CUDA(cudaStreamSynchronize(d->d2h_stream));
    d->d2h_pending = false;
    d->bank.reserve(std::max<uint64_t>(Hs, 1));
    const FastBank f = d->fsrc.view();
    const double2* hb = reinterpret_cast<const double2*>(d->host_bank);
    uint64_t lo = 0;
    if (hprof && d->xt[2]) HWWG_CUDA(cudaEventRecord(d->xt[2], d->copy_stream));
    for (size_t u = 0; u < bounds.size(); ++u) {
      const uint64_t hi = bounds[u];
      if (piped) HWWG_CUDA(cudaStreamWaitEvent(d->copy_stream, d->d2h_ev[u], 0));
      const FastBank fu{f.xm + lo, f.wt + lo, f.meta + lo};
      if (d->host_packed) {  // (x, mu) [+ (w, t)] straight into the SoA source
        HWWG_CUDA(cudaMemcpyAsync(fu.xm, hb + lo, (hi - lo) * sizeof(double2),
                                  cudaMemcpyHostToDevice, d->copy_stream));
        if (!d->host_uniform)
          HWWG_CUDA(cudaMemcpyAsync(fu.wt, hb + Hs + lo, (hi - lo) * sizeof(double2),
                                    cudaMemcpyHostToDevice, d->copy_stream));
        // (the conversion to SoA records runs on the step stream just before
        // the segment: a kernel on the copy stream would wait for SMs behind
        // the persistent transport grid and hold up the copies queued after it)
      } else {
        HWWG_CUDA(cudaMemcpyAsync(d->bank.p + lo, d->host_bank + lo, (hi - lo) * sizeof(hwwg_particle),
                                  cudaMemcpyHostToDevice, d->copy_stream));
        launch_aos_to_fast(d->bank.p + lo, hi - lo, d->prob.view, fu, lo, d->copy_stream);
      }
      HWWG_CUDA(cudaEventRecord(d->h2d_ev[u], d->copy_stream));
      if (hprof && d->xt[5] && u == 0) HWWG_CUDA(cudaEventRecord(d->xt[5], d->copy_stream));
      ++d->launches;
      lo = hi;
    }
    if (hprof && d->xt[3]) HWWG_CUDA(cudaEventRecord(d->xt[3], d->copy_stream));
    if (d->host_packed && d->host_uniform) {
      // comb teeth (x, mu): the transport derives the rest (FastArgs::n_packed),
      // no conversion; the spacing is still in comb_mem[1] from the pre-comb
      d->src_packed = Hs;
      d->src_t0 = d->host_t0;
    } else if (d->host_packed) {  // segment u's particle range, converted on s before it runs
      seg_range.assign(seg_wait.size() + 1, 0);
      for (size_t u = 0; u < seg_wait.size(); ++u) seg_range[u + 1] = bounds[seg_wait[u]];
    }
    d->bank_n = Hs;
    rec->h2d_bytes += d->host_packed ? Hs * sizeof(double2) * (d->host_uniform ? 1 : 2)
                                     : Hs * sizeof(hwwg_particle);
  } else if (c.host_bank && d->fast && d->host_pre_combed && d->world > 1) {
    // multi-rank e2e: this rank's share of the global comb, combed at the end
    // of the previous step, back from the host in the packed format
    const uint64_t nl = d->host_bank_n;
    const FastBank f = d->fsrc.view();
    const double2* hb = reinterpret_cast<const double2*>(d->host_bank);
    HWWG_CUDA(cudaMemcpyAsync(f.xm, hb, nl * sizeof(double2), cudaMemcpyHostToDevice, s));
    if (!d->host_uniform)
      HWWG_CUDA(cudaMemcpyAsync(f.wt, hb + nl, nl * sizeof(double2), cudaMemcpyHostToDevice, s));
    const StepLayout Lp = make_layout(c, d->hybrid(), d->pre_Hc, d->pre_Hc + d->pre_nv, d->world);
    const PieceTable t = comb_pieces(Lp, d->rank);
    launch_xm_to_fast(f, nl, d->prob.view, 0, d->host_uniform ? 1 : 0, d->host_w0, d->host_t0, s,
                      &t);
    ++d->launches;
    rec->h2d_bytes += nl * sizeof(double2) * (d->host_uniform ? 1 : 2);
  } else if (c.host_bank && d->host_pulse_mu) {  // e2e step 1: the pulse's directions
    d->bank.reserve(std::max<uint64_t>(d->host_bank_n, 1));
    double* dmu = reinterpret_cast<double*>(d->bank.p);
    HWWG_CUDA(cudaMemcpyAsync(dmu, d->host_bank, d->host_bank_n * sizeof(double),
                              cudaMemcpyHostToDevice, s));
    d->bank_n = d->host_bank_n;
    rec->h2d_bytes += d->host_bank_n * sizeof(double);
    d->fbank.reserve(d->bank_n);
    launch_mu_to_census(dmu, d->bank_n, c.x0, d->host_w0, d->fbank.view(), s);
    ++d->launches;
    d->host_pulse_mu = false;
  } else if (c.host_bank) {  // e2e: the bank lives in host memory between steps
    d->bank.reserve(std::max<uint64_t>(d->host_bank_n, 1));
    HWWG_CUDA(cudaMemcpyAsync(d->bank.p, d->host_bank, d->host_bank_n * sizeof(hwwg_particle),
                              cudaMemcpyHostToDevice, s));
    d->bank_n = d->host_bank_n;
    rec->h2d_bytes += d->host_bank_n * sizeof(hwwg_particle);
    if (d->fast) {
      // a pre-combed bank (see the step end) is already the step's source;
      // otherwise the host bank is the comb's input
      if (d->host_pre_combed) {
        d->fsrc.reserve(d->bank_n + (c.vol_rate > 0.0 ? c.vol_histories : 0));
        launch_aos_to_fast(d->bank.p, d->bank_n, d->prob.view, d->fsrc.view(), 0, s);
      } else {
        d->fbank.reserve(d->bank_n);
        launch_aos_to_census(d->bank.p, d->bank_n, d->fbank.view(), s);
      }
      ++d->launches;
    }
  }

  StepLayout Lmulti;  // multi-rank: the step layout the rebalance placed the teeth by
  // ---- population control (driver.cpp:111-129)
  const double bank_cap = c.comb_overflow_factor * (double)d->target;
  const bool do_comb = c.comb_overflow_factor <= 1.0 || (double)d->bank_n > bank_cap;
  // config-3 runs: room after the source for the step's volumetric particles
  const uint64_t vol_cap = c.vol_rate > 0.0 ? c.vol_histories : 0;
  uint64_t H;
  if (d->world == 1 && d->bank_n == 0 && (c.no_pulse || c.vol_rate > 0.0)) {
    // volumetric-source run before any census exists: nothing to comb
    H = 0;
    rec->comb_in = rec->comb_out = 0;
    HWWG_CUDA(cudaMemsetAsync(d->comb_mem.p, 0, 4 * sizeof(double), s));
    if (!d->fast) d->source.reserve(std::max<uint64_t>(vol_cap, 1));
  } else if (d->fast && d->world > 1 && c.host_bank && d->host_pre_combed) {
    H = d->pre_Hc;  // the global comb ran at the end of the previous step
    Lmulti = make_layout(c, d->hybrid(), H, H + nv_step, d->world);
    rec->comb_in = d->pre_comb_in;
    rec->comb_out = H;
  } else if (d->fast && d->world > 1) {
    if (!do_comb) throw ApiError(HWWG_EINVAL, "philox mode combs every step (comb_overflow_factor <= 1)");
    d->src_packed = 0;  // the multi-rank teeth are full records
    H = multi_gpu_comb(d, step, nv_step, Lmulti, s);
    rec->comb_in = d->bank_n;  // this rank's census slots
    rec->comb_out = H;
    if (H == 0 && !d->fast) d->source.reserve(std::max<uint64_t>(vol_cap, 1));
  } else if (d->fast && c.host_bank && d->host_pre_combed) {
    H = d->target;  // combed on the device at the end of the previous step
    rec->comb_in = d->pre_comb_in;
    rec->comb_out = d->target;
  } else if (d->fast) {
    if (!do_comb) throw ApiError(HWWG_EINVAL, "philox mode combs every step (comb_overflow_factor <= 1)");
    if (d->bank_n == 0) throw ApiError(HWWG_EINVAL, "cannot comb an empty bank");
    d->fsrc.reserve(d->target + vol_cap);
    d->comb_mem.reserve(4 + fast_comb_scratch_words(d->bank_n));
    FastCombArgs a{};
    a.bank = d->fbank.view();
    a.t_bank = d->bank_t;
    a.mesh = d->prob.view;
    a.n = d->bank_n;
    a.target = d->target;
    a.seed = c.seed;
    a.stream = stream_id_host(step, 0, 3);
    a.temp = d->comb_temp.p;
    a.temp_bytes = d->comb_temp.n;
    a.prefix = d->comb_mem.p + 4;
    a.scalars = d->comb_mem.p;
    a.out = d->fsrc.view();
    // after the cold start, tooth k becomes history perm(k) (see Perm)
    if (step > 1) a.perm = make_perm(d->target, c.seed, step);
    a.packed_out = d->packed_teeth;  // teeth as (x, mu): the transport derives the rest
    d->src_packed = d->packed_teeth ? d->target : 0;
    d->src_t0 = d->bank_t;
    // the integer scale from the bank's weight: the previous step's census
    // weight tallies (still in the slab), or the pulse source's strength
    if (d->has_prev_report) {
      a.hint_batches = d->tal.p.census_weight_batch;
      a.hint_n = B;
    } else {
      a.hint_host = c.strength * (double)c.histories_per_step;
    }
    d->ph_mark("comb", s);
    launch_fast_comb(a, s);
    d->ph_mark("-", s);
    d->launches += 3;
    H = d->target;
    rec->comb_in = d->bank_n;
    rec->comb_out = d->target;
  } else if (do_comb) {
    if (d->bank_n == 0) throw ApiError(HWWG_EINVAL, "cannot comb an empty bank");
    d->source.reserve(d->target + vol_cap);
    d->comb_mem.reserve(4 + d->bank_n + comb_tile_words(d->bank_n));
    CombArgs a{};
    a.bank = d->bank.p;
    a.n = d->bank_n;
    a.target = d->target;
    a.seed = c.seed;
    a.stream = stream_id_host(step, 0, 3);
    a.prefix = d->comb_mem.p + 4;
    a.scalars = d->comb_mem.p;
    a.out = d->source.p;
    a.exact_out_weight = 1;
    a.tiles = d->comb_mem.p + 4 + d->bank_n;
    launch_comb(a, s);
    d->launches += 6;
    H = d->target;
    rec->comb_in = d->bank_n;
    rec->comb_out = d->target;
  } else {
    d->source.reserve(std::max<uint64_t>(d->bank_n + vol_cap, 1));
    HWWG_CUDA(cudaMemcpyAsync(d->source.p, d->bank.p, d->bank_n * sizeof(hwwg_particle),
                              cudaMemcpyDeviceToDevice, s));
    k_bank_weight<<<1, 1, 0, s>>>(d->bank.p, d->bank_n, d->comb_mem.p);
    ++d->launches;
    H = d->bank_n;
    rec->comb_in = rec->comb_out = d->bank_n;
  }

  // ---- config-3 volumetric source: this step's particles follow the combed
  // census (histories [H, H + n)); the LOSM gets the step's q (set above).
  // Philox mode samples them on the device, each rank its shard of the n; exact
  // mode replays the reference-style sequential source stream on the host.
  const uint64_t H_comb = H;
  if (nv_step) {
    const double ta = std::max(rec->t_begin, c.vol_t_lo);
    const double tb = std::min(rec->t_end, c.vol_t_hi);
    const uint64_t nv = nv_step;
    const double wv = c.vol_rate * (tb - ta) * (double)c.histories_per_step / (double)nv;
    if (d->fast) {
      // this rank's volumetric ids [H_comb, H_comb + nv) of its pieces, each at
      // its local index; particle j is keyed by j alone, so any rank count
      // samples the same emission
      const StepLayout Lv =
          d->world > 1 ? Lmulti : make_layout(c, d->hybrid(), H_comb, H_comb + nv, 1);
      const FastBank f = d->fsrc.view();
      for (size_t u = 0; u < Lv.segments(); ++u) {
        uint64_t lo, hi;
        Lv.piece(d->rank, u, lo, hi);
        lo = std::max(lo, H_comb);
        if (hi <= lo) continue;
        const uint64_t at = Lv.owned_before(d->rank, lo);
        launch_volume_source(FastBank{f.xm + at, f.wt + at, f.meta + at}, hi - lo, lo - H_comb,
                             lo, d->prob.view, (unsigned)c.seed,
                             (unsigned)(c.seed >> 32) ^ 0x6a09e667u, (unsigned)step, c.vol_x_lo,
                             c.vol_x_hi, ta, tb, wv, s);
        ++d->launches;
      }
    } else {
      std::vector<hwwg_particle> vh(nv);
      sample_volume_source_host(c.seed, step, nv, c.vol_x_lo, c.vol_x_hi, ta, tb, c.vol_rate,
                                c.histories_per_step, vh.data());
      // pageable: staged before the call returns, so vh may go out of scope
      HWWG_CUDA(cudaMemcpyAsync(d->source.p + H, vh.data(), nv * sizeof(hwwg_particle),
                                cudaMemcpyHostToDevice, s));
      rec->h2d_bytes += nv * sizeof(hwwg_particle);
    }
    H += nv;
  }
  hmark("source ready");
  // the step's segments and this rank's histories in them
  const StepLayout L = d->world > 1 ? Lmulti : make_layout(c, d->hybrid(), H_comb, H, 1);

  if (!early_windows) {  // backup of the windows so an overflowing step can be replayed exactly
    HWWG_CUDA(cudaMemcpyAsync(d->centers_backup.p, d->lo.centers, I * 8, cudaMemcpyDeviceToDevice, s));
    HWWG_CUDA(cudaMemcpyAsync(d->flags_backup.p, d->lo.flags, 8 * sizeof(int), cudaMemcpyDeviceToDevice, s));
  }

  if (d->fast) {  // the swapped-in buffer may be short of the high-water mark
    try {
      d->fcensus.reserve(d->census_hwm);
    } catch (const std::bad_alloc&) {
      // memory wall: the high-water mark (the cold-start census, x150 of H at
      // config 4) does not fit next to the bank being combed. Later censuses
      // are far smaller: size for the creation-time mark and replay if short.
      d->fcensus.release();
      d->census_hwm = d->census_floor;
      d->fcensus.reserve(d->census_hwm);
    }
  }

  // ---- thresholds (driver.cpp:170-177): the layout's inner segment boundaries
  const std::vector<uint64_t> thr(L.seg.begin() + 1, L.seg.end() - 1);
  rec->n_thresholds = (int)thr.size();
  for (size_t i = 0; i < thr.size() && i < 8; ++i) rec->thresholds[i] = thr[i];


  // ---- census thinning (FastArgs::precomb): the comb spacing pc_s0 puts
  // ~precomb_k x target teeth on the census weight W_est, a bound-grade
  // estimate every rank computes alike: the step's source weight in the cold
  // start (census weight <= source weight up to roulette noise), else the
  // previous census weight (all-reduced). Thin when the census is expected to
  // exceed precomb_k x target: the cold start, or when the previous raw
  // census did.
  double pc_s0 = 0.0;
  if (d->fast && d->precomb) {
    const double Hc = (double)c.histories_per_step;
    double W_est = 0.0;
    bool thin = false;
    if (d->history.empty()) {
      thin = true;
      W_est = c.no_pulse ? 0.0 : c.strength * Hc;
      if (nv_step) {
        const double ta = std::max(rec->t_begin, c.vol_t_lo), tb = std::min(rec->t_end, c.vol_t_hi);
        W_est += c.vol_rate * (tb - ta) * Hc;
      }
    } else {
      // (after a x60 cold start the next census is usually ~x2 — config 5 —
      // but can stay x100 — config 4: thinning it too is cheap and unbiased,
      // where an unthinned overflow replays the step with a larger bank)
      const hwwg_step_record& pr = d->history.back();
      thin = (double)pr.census_size > d->precomb_k * (double)d->target;
      W_est = pr.census_weight * Hc;
    }
    if (thin && W_est > 0.0 && std::isfinite(W_est))
      pc_s0 = W_est / (d->precomb_k * (double)d->target);
  }
  rec->thinned = pc_s0 > 0.0 ? 1 : 0;

  // ---- tally window (FastArgs::t_win): the cells this step's particles can
  // reach — the previous step's track-flux support (the census sits inside
  // it), the pulse or the volumetric box, widened by the farthest flight of the
  // step (max speed x dt) and two cells. Used where the mesh's full fixed-point
  // histograms do not fit shared memory (config 4); scores outside go to the
  // global tallies, so the window only decides speed, never results.
  int win_lo = 0, win_n = 0;
  if (d->fast && d->fix_tallies && d->tally_window) {
    const std::vector<double>& e = d->prob.edges;
    double xlo = INFINITY, xhi = -INFINITY;
    if (d->history.empty()) {
      if (!c.no_pulse) xlo = xhi = c.x0;
    } else {
      int f = -1, l = -1;
      for (int i = 0; i < I; ++i)
        if (d->h_phi_track[i] != 0.0) {
          if (f < 0) f = i;
          l = i;
        }
      if (f >= 0) {
        xlo = e[f];
        xhi = e[l + 1];
      }
    }
    if (nv_step) {
      xlo = std::min(xlo, c.vol_x_lo);
      xhi = std::max(xhi, c.vol_x_hi);
    }
    if (xlo <= xhi) {
      double vmax = 0.0;
      for (const CellInfo& ci : d->prob.cells_h) vmax = std::max(vmax, ci.speed);
      const double reach = vmax * dt;
      auto cell_of = [&](double x) {
        const int k = (int)(std::upper_bound(e.begin(), e.end(), x) - e.begin()) - 1;
        return std::max(0, std::min(I - 1, k));
      };
      const int lo = std::max(0, cell_of(xlo - reach) - 2);
      const int hi = std::min(I - 1, cell_of(xhi + reach) + 2);
      win_lo = lo;
      win_n = hi - lo + 1;
      if (d->tally_window_max && win_n > d->tally_window_max) {  // tests: a window too narrow
        win_lo += (win_n - d->tally_window_max) / 2;
        win_n = d->tally_window_max;
      }
    }
  }

  unsigned long long count = 0;
  DevError derr{};
  const int cur = d->rep_cur;
  // finalize (driver.cpp:221-222): device-side from the tallies alone
  auto enqueue_finalize = [&]() {
    FinalizeArgs f{};
    f.track_from_batches = d->fast ? 1 : 0;  // the fast kernels score the batch table only
    f.I = I;
    f.B = B;
    f.t = d->tal.p;
    f.histories = H;
    f.normalization = (double)c.histories_per_step;
    f.phi_track = d->rep(cur, 0);
    f.sigma = d->rep(cur, 1);
    f.phi_census = d->rep(cur, 2);
    f.current = d->rep(cur, 3);
    f.closure = d->rep(cur, 4);
    f.edge = d->rep(cur, 5);
    f.scalars = d->rep(cur, 6);
    launch_finalize(f, s);
    ++d->launches;
  };
  // Single-GPU Philox steps finalize BEFORE the one host sync that reads the
  // census count and the error word (an overflow, which the up-front census
  // capacity makes rare, replays the whole step and finalizes again), so the
  // device never idles on a host round trip in the middle of a step.
  const bool early_finalize = d->fast && d->world == 1;
  bool ev1_recorded = false;
  for (int attempt = 0; attempt < 4; ++attempt) {
    if (attempt) {  // replay: restore the windows the step started from
      HWWG_CUDA(cudaMemcpyAsync(d->lo.centers, d->centers_backup.p, I * 8, cudaMemcpyDeviceToDevice, s));
      HWWG_CUDA(cudaMemcpyAsync(d->lo.flags, d->flags_backup.p, 8 * sizeof(int), cudaMemcpyDeviceToDevice, s));
    }
    // ---- windows (driver.cpp:136-167): already on the auxiliary stream for the
    // first attempt of an early-window step, else here
    if (attempt == 0 && early_windows) HWWG_CUDA(cudaStreamWaitEvent(s, d->ev_join, 0));
    else enqueue_windows(s, false);

    // ---- segments with window-update barriers (driver.cpp:181-219)
    bool start_reset = false;  // the first segment's pool counters are reset here
    if (d->fast) {
      launch_step_start(d->tal.slab.p, d->tal.words(), d->warp_cursor.p, d->warp_cursor.n,
                        d->counter.p, d->err.p, d->pool_ctl.p, d->src_head.p,
                        d->seg_events ? nullptr : d->span.p, d->sms, s);
      ++d->launches;
      start_reset = true;
    } else {
      d->tal.zero(s);
      HWWG_CUDA(cudaMemsetAsync(d->counter.p, 0, sizeof(unsigned long long), s));
      HWWG_CUDA(cudaMemsetAsync(d->err.p, 0, sizeof(DevError), s));
    }
    ExactArgs ea{};
    ea.mesh = d->prob.view;
    ea.t_begin = rec->t_begin;
    ea.t_end = rec->t_end;
    ea.inv_dt = 1.0 / dt;
    ea.seed = c.seed;
    ea.step = (uint64_t)step;
    ea.H = H;
    ea.B = B;
    const bool windows = c.mode != 0;
    ea.centers = windows ? d->lo.centers : nullptr;
    ea.active = windows ? d->lo.flags : nullptr;
    ea.rho = c.rho;
    ea.t = d->tal.p;
    ea.census = d->stage.records.p;
    ea.census_keys = d->stage.keys.p;
    ea.census_count = d->counter.p;
    ea.census_cap = d->stage.records.n;
    ea.err = d->err.p;
    if (!d->fast) d->xlog.reset_need(s);
    uint64_t h_done = 0;
    // this rank's histories: its pieces of the step layout, in global order
    auto owned_before = [&](uint64_t g) { return L.owned_before(d->rank, g); };
    auto global_of = [&](uint64_t l) { return L.global_of(d->rank, l); };
    bool pool_reset_done = start_reset;  // the step start or the mid-step update reset the pool
    int grid_warps_max = 0;     // largest transport grid of this step so far
    bool tail_filled = false;   // the last segment filled the census chunk tails
    for (size_t u = 0; u <= thr.size(); ++u) {
      const uint64_t h_stop = u < thr.size() ? thr[u] : H;
      ea.src = d->source.p + h_done;
      ea.n = h_stop - h_done;
      ea.h_begin = h_done;
      if (!d->fast) {  // chunk-private TallySets of the exact path
        ea.chunks = chunk_layout(ea.n, h_done, H, I, B);
        d->chunk_mem.reserve(std::max<size_t>((size_t)ea.chunks.count * ea.chunks.stride, 1));
        ea.chunks.base = d->chunk_mem.p;
        ea.log = d->xlog.view(ea.n);
      }
      const int nseg = (int)u;
      if (d->seg_events) HWWG_CUDA(cudaEventRecord(d->seg_ev[2 * nseg], s));
      if (d->fast) {
        FastArgs fa{};
        fa.pool_reset_done = pool_reset_done ? 1 : 0;
        fa.span = d->seg_events ? nullptr : d->span.p + 2 * nseg;
        // right after the window update (one rank per stream: a loopback hub's
        // shared stream interleaves the ranks' kernels)
        fa.pdl = pool_reset_done && d->pdl && !d->phases_on && d->world == 1;
        pool_reset_done = false;
        // this rank's piece of the segment: one contiguous range of its source
        const uint64_t l_lo = owned_before(h_done), l_hi = owned_before(h_stop);
        const uint64_t g_lo = global_of(l_lo);
        const uint64_t g_hi = l_hi > l_lo ? global_of(l_hi - 1) + 1 : g_lo;
        const FastBank src = d->fsrc.view();
        fa.src = FastBank{src.xm + l_lo, src.wt + l_lo, src.meta + l_lo};
        fa.n_src = l_hi - l_lo;
        // the comb teeth among them are (x, mu) only (single GPU: local = global slot)
        fa.n_packed = d->src_packed > l_lo ? std::min<uint64_t>(d->src_packed - l_lo, fa.n_src) : 0;
        fa.src_w0 = d->comb_mem.p + 1;
        fa.src_t0 = d->src_t0;
        fa.src_hist0 = (unsigned)l_lo;
        fa.inv_w0 = d->prob.view.uniform ? 1.0 / d->prob.view.w0 : 0.0;
        fa.src_head = d->src_head.p;
        fa.census = d->fcensus.view();
        fa.census_count = d->counter.p;
        fa.census_cap = d->fcensus.cap();
        fa.mesh = d->prob.view;
        fa.t_end = rec->t_end;
        fa.inv_dt = 1.0 / dt;
        fa.k0 = (unsigned)c.seed;
        fa.k1 = (unsigned)(c.seed >> 32) ^ 0x6a09e667u;
        philox_round_keys(fa.k0, fa.k1, fa.rk);
        fa.step = (unsigned)step;
        fa.H = H;
        fa.B = B;
        fa.bmul = H ? (double)B / (double)H : 0.0;
        fa.centers = ea.centers;
        fa.active = ea.active;
        fa.rho = c.rho;
        fa.inv_rho = 1.0 / c.rho;
        fa.t = d->tal.p;
        fa.stacks = d->stacks.p;
        fa.stack_cap = d->stack_cap;
        fa.pool = FastPool{d->pool_recs.p, d->pool_ctl.p, (unsigned)d->pool_recs.n, 0u};
        fa.err = d->err.p;
        // block-private shared-memory tallies over this segment's batch range
        // when they fit (I <= ~1000 at 20 batches), else global REDs
        const int b_lo = batch_of_host(g_lo, H, B);
        const int b_hi = batch_of_host(g_hi > g_lo ? g_hi - 1 : g_lo, H, B);
        fa.b_lo = b_lo;
        fa.nb = b_hi - b_lo + 1;
        // the first step starts from a point pulse: most lanes share a few cells
        fa.aggregate = ((step == 1 && d->agg_all != 2) || d->agg_all == 1) ? 1 : 0;
        size_t smem = fast_smem_bytes(I, fa.nb);
        fa.smem_tallies = smem <= 96 * 1024 ? 1 : 0;
        // global-memory tallies (I >~ 1000 at 20 batches, config 4): same-cell
        // REDs from ~1e5 resident lanes saturate the L2 atomic units unless
        // they are warp-aggregated first (config 4: 3.5e9 -> 4.8e9 seg/s at
        // 1e6 histories, 1.7e9 -> 5.5e9 at 1.25e7)
        if (!fa.smem_tallies && d->agg_all < 0 && d->smem_mode == 1) fa.aggregate = 1;
        if (!fa.aggregate && d->smem_mode != 1) {
          fa.smem_tallies = d->smem_mode;
          smem = d->smem_mode == 2 ? fast_smem_count_bytes(I) : 0;
        }
        if (!fa.smem_tallies) smem = 0;
        smem += fast_smem_centers_bytes(I);
        // fixed-point track/edge/census tallies, where the wider slots keep the
        // occupancy — in the cold start too, where native same-address limb
        // adds beat the warp aggregation (config 5 step 1: 46 -> 33 ms of
        // transport, with run-aggregated census scores) unless aggregation is
        // forced (HWWG_FAST_AGG=1). Largest
        // expected scores: a window survivor or source weight (<= max(rho *
        // max centre = rho, step_wref)) times speed/dx for a track, divided by
        // dt for an edge crossing.
        fa.fix = 0;
        const int uni = d->prob.gen_uniform_homog ? 1 : 0;
        // the block shape with the most resident warps for a tally layout (2 x 12
        // warps on ties; HWWG_FAST_BLOCK_WARPS forces one)
        // A block-private tally copy of >= 96 KB (config 3's 1000 cells) is
        // zeroed and flushed per block: one block per SM (1 x 24 warps) then
        // beats two blocks with 4 more warps (config 3: 2.0e10 vs 1.5e10 seg/s),
        // while config 5's ~70 KB copy runs best at 2 x 14 (2.54e10 vs 2.43e10).
        auto shape = [&](size_t sm, int sh, int fx, int& warps) {
          int best = 0;
          for (int w : kFastBlockWarps) {
            if (d->block_warps && w != d->block_warps) continue;
            const int nb_sm = fast_blocks_per_sm(sm, uni, sh, fx, w);
            const int r = nb_sm * w;
            const bool one_big = nb_sm == 1 && sm >= 96 * 1024 && 5 * r >= 4 * best;
            if (r > best || (one_big && r > 0)) {
              best = r;
              warps = w;
            }
          }
          return best;
        };
        fa.t_win = 0;
        fa.t_lo = 0;
        fa.t_n = I;
        // windowed fixed-point histograms (config 4) instead of global REDs
        // (also where the full copy fits but reaches 96 KB — config 3's 1000 cells,
        // then one 24-warp block per SM — and a window halves it: config 3 +3.5%;
        // HWWG_TALLY_WINDOW=2 windows every layout, config 5 -1%)
        const bool big_copy = fast_smem_fix_bytes(I, fa.nb) >= 96 * 1024;
        const bool try_win =
            win_n > 0 && d->smem_mode == 1 && d->agg_all != 1 &&
            (fa.smem_tallies == 0 ? win_n < I : ((big_copy || d->tally_window > 1) && 2 * win_n <= I));
        if ((fa.smem_tallies == 1 || try_win) && (!fa.aggregate || d->agg_all != 1) &&
            d->flush_replicas == 0 && d->fix_tallies) {
          const int T = try_win ? win_n : I;
          const size_t fsm = fast_smem_fix_bytes(T, fa.nb) + fast_smem_centers_bytes(I);
          double vmax = 0.0;
          for (const CellInfo& ci : d->prob.cells_h) vmax = std::max(vmax, ci.speed * ci.inv_dx);
          double vmin = vmax;
          for (const CellInfo& ci : d->prob.cells_h) vmin = std::min(vmin, ci.speed * ci.inv_dx);
          const double w = std::max(c.rho, d->step_wref);
          int kt = 0, ke = 0;
          int wfix = 12, wbase = 12;
          const int fix_warps = shape(fsm, 1, try_win ? 2 : 1, wfix);
          // dynamic range: the smallest census score (a weight near the lowest
          // window floor eps_min / rho) must keep >= 2^20 grid units, or its
          // rounding would bias low-window cells: beyond 20 binades below the
          // largest expected score the fp64 slots are kept
          const double smallest = c.mode != 0 ? c.eps_min / c.rho * vmin : w * vmin;
          const bool range_ok = smallest > 0.0 &&
                                std::ilogb(w * vmax) - std::ilogb(smallest) <= 20;
          int kc = 0;
          if (range_ok && fast_fix_exponent(w * vmax, &kt) && fast_fix_exponent(w / dt, &ke) &&
              fast_fix_exponent(w, &kc) && fix_warps > 0 &&
              (try_win || 5 * fix_warps >= 4 * shape(smem, 1, 0, wbase))) {  // (shared fp64 adds are CAS loops)
            fa.fix = 1;
            fa.census_runs = fa.aggregate;  // the cold start's crowded census cells
            if (try_win) {
              fa.smem_tallies = 1;
              fa.t_win = 1;
              fa.t_lo = win_lo;
              fa.t_n = win_n;
              fa.census_runs = step == 1 ? 1 : 0;  // (aggregate was forced on for the global path)
            }
            fa.fix_k_trk = kt;
            fa.fix_k_edge = ke;
            fa.fix_k_cw = kc;
            fa.aggregate = 0;
            smem = fsm;
          }
        }
        fa.scramble = fa.aggregate ? 0 : d->scramble;
        int wsel = 12;
        const int fxk = fa.fix ? (fa.t_win ? 2 : 1) : 0;  // the instantiation: fp64 / fixed / windowed
        shape(smem, fa.smem_tallies == 1, fxk, wsel);
        fa.warps = wsel;
        // (the per-warp arrays — split stacks, census cursors, thinning residuals —
        // hold max_warps = sms x kMaxWarpsPerSm warps: never launch more)
        const int blocks = std::min(d->sms * fast_blocks_per_sm(smem, uni, fa.smem_tallies == 1, fxk, wsel),
                                    d->max_warps / wsel);
        const int gw = blocks * wsel;
        grid_warps_max = std::max(grid_warps_max, gw);
        if (u == thr.size() && gw >= grid_warps_max && fa.n_src) {
          fa.fill_tail = 1;
          fa.x_fill = d->prob.edges.front();
          tail_filled = true;
        }
        fa.pool.warps = (unsigned)gw;
        fa.warp_cursor = d->warp_cursor.p;
        fa.seg = nseg;
        fa.flush_scratch = d->flush_scratch.p;
        fa.flush_stride = fast_flush_stride(I, B);
        fa.flush_replicas = d->flush_replicas;
        fa.uniform = d->prob.gen_uniform_homog ? 1 : 0;
        fa.x_min = d->prob.edges.front();
        fa.x_max = d->prob.edges.back();
        fa.w_gen = d->prob.w_gen;
        fa.cell0 = d->prob.cells_h[0];
        fa.precomb = pc_s0 > 0.0 ? 1 : 0;
        fa.pc_s0 = pc_s0;
        fa.pc_inv_s0 = pc_s0 > 0.0 ? 1.0 / pc_s0 : 0.0;
        fa.pc_key = ((unsigned)d->rank << 16) | ((unsigned)attempt << 8) | (unsigned)nseg;
        fa.pc_need = d->pc_need.p;
        if (d->timeline_on) {  // HWWG_FAST_TIMELINE: per-warp phase timestamps
          const size_t per = (size_t)fa.pool.warps * kTimelineWords;
          d->timeline.reserve(per * 9);
          fa.timeline = d->timeline.p + per * nseg;
          HWWG_CUDA(cudaMemsetAsync(fa.timeline, 0, per * 8, s));
          d->timeline_warps = fa.pool.warps;
        }
        if (u < seg_wait.size()) {
          HWWG_CUDA(cudaStreamWaitEvent(s, d->h2d_ev[seg_wait[u]], 0));
          if (u + 1 < seg_range.size() && seg_range[u + 1] > seg_range[u]) {
            const uint64_t lo = seg_range[u], n = seg_range[u + 1] - lo;
            const FastBank f = d->fsrc.view();
            launch_xm_to_fast(FastBank{f.xm + lo, f.wt + lo, f.meta + lo}, n, d->prob.view, lo,
                              d->host_uniform ? 1 : 0, d->host_w0, d->host_t0, s);
            ++d->launches;
            fa.pdl = 0;  // the segment now follows the conversion, not the window update
          }
        }
        if (hprof && d->xt[6] && u == 0) HWWG_CUDA(cudaEventRecord(d->xt[6], s));
        if (fa.n_src) {
          launch_fast_segment(fa, blocks, smem, s);
          d->launches += 2;
        }
      } else {
        launch_exact_segment(ea, s);
        // chunk init, histories (+ log replay), ordered merge
        if (ea.n) d->launches += ea.log.slot ? 4 : 3;
      }
      if (d->seg_events) HWWG_CUDA(cudaEventRecord(d->seg_ev[2 * nseg + 1], s));
      h_done = h_stop;
      if (u == thr.size()) break;
      // partial_snapshot + implicit closure update (driver.cpp:206-217)
      LowOrderArgs a{};
      a.I = I;
      a.edges = d->prob.view.edges;
      a.cells = d->prob.view.cells;
      a.theta = theta_eff;
      a.dt = dt;
      a.eps_min = c.eps_min;
      a.rho = c.rho;
      a.ma_k = ma_k;
      a.fourier_tab_cell = c.mode == 4 ? d->ftab_cell.p : nullptr;
      a.fourier_tab_edge = c.mode == 4 ? d->ftab_edge.p : nullptr;
      a.fourier_cutoff = c.fourier_cutoff;
      a.q = d->q_step;
      a.mode = 1;
      a.fast_solve = d->fast ? 1 : 0;
      a.refactor = d->need_refactor(theta_eff, dt);
      a.closure_tally = d->tal.p.census_closure;
      a.bclosure_tally = d->tal.p.boundary_closure;
      if (d->world > 1) {  // the snapshot is of ALL ranks' histories so far
        d->nccl_buf.reserve(std::max<size_t>(4 * (size_t)d->world + 16, (size_t)I + 8));
        d->comm->all_reduce(d->tal.p.census_closure, d->nccl_buf.p, I, DType::kF64, RedOp::kSum, s);
        d->comm->all_reduce(d->tal.p.boundary_closure, d->nccl_buf.p + I, 2, DType::kF64,
                            RedOp::kSum, s);
        a.closure_tally = d->nccl_buf.p;
        a.bclosure_tally = d->nccl_buf.p + I;
      }
      const double effective = (double)c.histories_per_step * (double)h_done / (double)H;
      a.snapshot_inv_norm = 1.0 / effective;
      if (d->fast) {  // the next segment's pool reset rides on this launch
        a.pool_ctl = d->pool_ctl.p;
        a.pool_src_head = d->src_head.p;
        pool_reset_done = true;
        a.pdl = d->pdl && d->world == 1 && !d->phases_on;  // right after the transport launch
        a.pool_span = d->seg_events ? nullptr : d->span.p + 2 * (nseg + 1);
      }
      a.s = d->lo;
      d->ph_mark("losm1", s);
      launch_low_order_update(a, s);
      if (std::getenv("HWWG_LOSM_TWICE")) {  // diagnostic: a warm second launch
        d->ph_mark("losm1b", s);
        launch_low_order_update(a, s);
      }
      d->ph_mark("-", s);
      ++d->launches;
    }
    if (d->fast && !tail_filled) {  // zero-weight records in the unused tails of the warps' chunks
      d->ph_mark("fill", s);
      launch_fill_census_holes(d->fcensus.view(), d->fcensus.cap(), d->warp_cursor.p,
                               d->max_warps, d->prob.edges.front(), s);
      ++d->launches;
    }
    if (early_finalize) {
      d->ph_mark("finalize", s);
      enqueue_finalize();
      d->ph_mark("-", s);
      if (!c.host_bank) {
        HWWG_CUDA(cudaEventRecord(d->ev1, s));
        ev1_recorded = true;
      }
    }
    HWWG_CUDA(cudaMemcpyAsync(&count, d->counter.p, sizeof(count), cudaMemcpyDeviceToHost, s));
    HWWG_CUDA(cudaMemcpyAsync(&derr, d->err.p, sizeof(derr), cudaMemcpyDeviceToHost, s));
    hmark("before sync");
    HWWG_CUDA(cudaStreamSynchronize(s));
    hmark("after sync");
    if (d->fast && d->world > 1) {  // replay decisions must be collective
      unsigned long long flags[2] = {count > d->fcensus.cap() ? 1ULL : 0ULL,
                                     derr.code ? 1ULL : 0ULL};
      unsigned long long* dflag = reinterpret_cast<unsigned long long*>(d->nccl_buf.p);
      HWWG_CUDA(cudaMemcpyAsync(dflag, flags, sizeof flags, cudaMemcpyHostToDevice, s));
      d->comm->all_reduce(dflag, dflag, 2, DType::kU64, RedOp::kMax, s);
      HWWG_CUDA(cudaMemcpyAsync(flags, dflag, sizeof flags, cudaMemcpyDeviceToHost, s));
      HWWG_CUDA(cudaStreamSynchronize(s));
      if (flags[1] && !derr.code) derr.code = HWWG_EINVAL;  // a peer failed
      if (derr.code || !flags[0]) break;
      d->census_hwm = std::max<uint64_t>(d->census_hwm, count + count / 4 + 4096);
      d->fcensus.reserve(d->census_hwm);  // every rank replays the step
      continue;
    }
    if (d->fast) {
      if (derr.code || count <= d->fcensus.cap()) break;
      d->census_hwm = count + count / 4 + 4096;
    d->fcensus.reserve(d->census_hwm);  // replay the step with room
      continue;
    }
    // replay with room: a log arena that fits (the overflowing histories
    // counted the demand) and/or a census stage that fits — both at once
    bool again = false;
    if (derr.code == kLogOverflow && attempt < 3) {
      const unsigned long long need = d->xlog.need(s);
      d->xlog.ensure_blocks(need + need / 4 + 1024);
      again = true;
    }
    if ((derr.code == 0 || again) && count > ea.census_cap) {
      d->stage.ensure(count + count / 4 + 4096);
      again = true;
    }
    if (!again) break;
  }
  if (d->timeline_on) print_timeline(d, (int)thr.size() + 1, step);
  unsigned long long fp[12];
  std::vector<unsigned> fh(kFastHistWords);
  if (d->timeline_on && fast_prof_read(fp, fh.data()) && fp[5]) {
    for (int sg = 0; sg < 8; ++sg) {  // trips / live lanes per 5 us bin
      const unsigned* h = fh.data() + (size_t)sg * 240;
      unsigned peak = 0;
      int last = -1;
      for (int b = 0; b < 120; ++b) {
        peak = std::max(peak, h[2 * b]);
        if (h[2 * b]) last = b;
      }
      if (last < 0) continue;
      int t50 = 0;
      for (int b = 0; b <= last; ++b)
        if (h[2 * b] * 2 >= peak) t50 = b;
      double tr_a = 0, ln_a = 0, tr_b = 0, ln_b = 0;
      for (int b = 0; b <= last; ++b) {
        (b <= t50 ? tr_a : tr_b) += h[2 * b];
        (b <= t50 ? ln_a : ln_b) += h[2 * b + 1];
      }
      std::string prof = "";
      for (int b = 0; b <= last; b += std::max(1, (last + 1) / 16)) {
        char bb[24];
        std::snprintf(bb, sizeof bb, " %u", h[2 * b]);
        prof += bb;
      }
      std::fprintf(stderr,
                   "[fhist] step %d seg %d: busy to %d us (peak %u trips/5us), end %d us; lanes/trip "
                   "%.1f before, %.1f after; trips before %.0f after %.0f; profile%s\n",
                   step, sg, 5 * (t50 + 1), peak, 5 * (last + 1), tr_a ? ln_a / tr_a : 0.0,
                   tr_b ? ln_b / tr_b : 0.0, tr_a, tr_b, prof.c_str());
    }
    const double t = (double)fp[5];
    const double busy =
        (double)(fp[0] + fp[1] + fp[2] + fp[3] + fp[4] + fp[8] + fp[9] + fp[10]);
    std::fprintf(stderr,
                 "[fprof] step %d: %llu trips, cycles/trip share %.0f stack %.0f source %.0f "
                 "check %.0f event %.0f census %.0f tally %.0f split %.0f | warp lifetime: in "
                 "trips %.1f%%, waiting on the pool %.1f%%, other %.1f%%\n",
                 step, fp[5], fp[8] / t, fp[9] / t, fp[10] / t, fp[0] / t, fp[1] / t, fp[2] / t,
                 fp[3] / t, fp[4] / t,
                 100.0 * busy / (double)fp[7], 100.0 * (double)fp[6] / (double)fp[7],
                 100.0 * (1.0 - (busy + (double)fp[6]) / (double)fp[7]));
  }
  if (d->phases_on) {  // the stream is synchronised here
    std::string line = "[phases] step " + std::to_string(step) + ":";
    for (size_t k = 0; k + 1 < d->ph_n; ++k) {
      if (d->ph_name[k][0] == '-') continue;
      float ms = 0.f;
      HWWG_CUDA(cudaEventElapsedTime(&ms, d->ph_ev[k], d->ph_ev[k + 1]));
      char buf[64];
      std::snprintf(buf, sizeof buf, " %s %.1f", d->ph_name[k], 1e3 * ms);
      line += buf;
    }
    std::fprintf(stderr, "%s us\n", line.c_str());
    d->ph_n = 0;
  }
  if (derr.code == HWWG_EINVAL)
    throw ApiError(HWWG_EINVAL, "history " + std::to_string(derr.history) +
                                    " starts outside the mesh or the time step");
  if (derr.code == HWWG_ESTACK)
    throw ApiError(HWWG_ESTACK, "history " + std::to_string(derr.history) +
                                    " exceeded the daughter-stack run capacity");
  if (derr.code == kLogOverflow)
    throw ApiError(HWWG_ENOMEM, "exact tally log exceeds 2^32 blocks");

  // ---- finalize (driver.cpp:221-222)
  if (d->world > 1) {  // step-end reduction of the whole tally slab and counters
    d->comm->all_reduce(d->tal.slab.p, d->tal.slab.p, d->tal.doubles, DType::kF64, RedOp::kSum, s);
    unsigned long long* u64part = reinterpret_cast<unsigned long long*>(d->tal.slab.p + d->tal.doubles);
    d->comm->all_reduce(u64part, u64part, (size_t)I + kNumUCounters, DType::kU64, RedOp::kSum, s);
  }
  if (!early_finalize) enqueue_finalize();

  // ---- census -> next bank in reference order
  if (d->fast) {
    d->fbank.swap(d->fcensus);  // the census is the next comb's input
    d->bank_t = rec->t_end;     // every census particle sits at the step's end
  } else {
    d->bank.reserve(std::max<unsigned long long>(count, 1));
    d->stage.sort_into(d->bank.p, count, ((unsigned long long)H << 24) | 0xffffffULL, s);
    if (count) d->launches += 2;  // iota + gather (the radix sort itself is CUB's)
  }
  d->bank_n = count;
  if (!ev1_recorded) HWWG_CUDA(cudaEventRecord(d->ev1, s));

  // ---- read the step record back (one sync)
  std::vector<double> rep_h((size_t)7 * (I + 1) + 8);
  HWWG_CUDA(cudaMemcpyAsync(rep_h.data(), d->rep_mem[cur].p, rep_h.size() * 8, cudaMemcpyDeviceToHost, s));
  int flags[8];
  HWWG_CUDA(cudaMemcpyAsync(flags, d->lo.flags, sizeof flags, cudaMemcpyDeviceToHost, s));
  double comb_sc[4];
  HWWG_CUDA(cudaMemcpyAsync(comb_sc, d->comb_mem.p, sizeof comb_sc, cudaMemcpyDeviceToHost, s));
  d->h_centers.resize(I);
  d->h_hybrid.resize(I);
  HWWG_CUDA(cudaMemcpyAsync(d->h_centers.data(), d->lo.centers, I * 8, cudaMemcpyDeviceToHost, s));
  HWWG_CUDA(cudaMemcpyAsync(d->h_hybrid.data(), d->lo.phi_hybrid, I * 8, cudaMemcpyDeviceToHost, s));
  d->host_pre_combed = false;
  if (c.host_bank && d->fast && d->world == 1) {
    // e2e host round trip: comb the census now, with the NEXT step's stream
    // (the comb that would open it), and hand the host the combed source —
    // target particles instead of the raw census (x60 of H after step 1).
    // Enqueued after the record readbacks above, so they see this step's
    // comb scalars.
    d->comb_mem.reserve(4 + fast_comb_scratch_words(d->bank_n));
    FastCombArgs a{};
    a.temp = d->comb_temp.p;
    a.temp_bytes = d->comb_temp.n;
    a.bank = d->fbank.view();
    a.t_bank = d->bank_t;
    a.mesh = d->prob.view;
    a.n = d->bank_n;
    a.target = d->target;
    a.seed = c.seed;
    a.stream = stream_id_host(step + 1, 0, 3);
    a.prefix = d->comb_mem.p + 4;
    a.scalars = d->comb_mem.p;
    a.out = d->fsrc.view();
    a.perm = make_perm(d->target, c.seed, step + 1);
    a.hint_batches = d->tal.p.census_weight_batch;  // this step's census weight
    a.hint_n = B;
    a.packed_out = 1;  // (x, mu) teeth; weight comb_mem[1], time bank_t
    if (d->bank_n == 0) throw ApiError(HWWG_EINVAL, "cannot comb an empty bank");
    launch_fast_comb(a, s);
    d->launches += 3;
    d->src_t0 = d->bank_t;
    d->pre_comb_in = d->bank_n;
    d->host_pre_combed = true;
    d->host_bank_n = d->target;
    d->bank_n = d->target;
    // the packed wire format, uploaded by pieces (the next step's volumetric
    // particles are sampled on the device after the teeth): (x, mu) now, (w, t)
    // only if not shared
    d->host_packed = true;
    if (d->host_packed) {
      // the teeth share one (w, t) by construction (packed_out): the spacing
      // comes down with the record, the census time is known here
      d->h_uni[0] = 0u;
      reinterpret_cast<double*>(reinterpret_cast<char*>(d->h_uni) + 16)[1] = d->bank_t;
      rec->d2h_bytes += d->target * sizeof(double2) + 8;
      HWWG_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(d->h_uni) + 16, d->comb_mem.p + 1,
                                sizeof(double), cudaMemcpyDeviceToHost, s));
      // (x, mu) go down at the end of this call (download_source), after the
      // step's own readbacks: queued behind 160 MB they would wait for it
      HWWG_CUDA(cudaEventRecord(d->ev_pre, s));
      d->d2h_pending = true;
    } else {
      launch_fast_to_aos_packed(d->fsrc.view(), d->target, d->target, d->comb_mem.p + 1, d->bank_t,
                                d->bank.p, s);
      ++d->launches;
      rec->d2h_bytes += d->target * sizeof(hwwg_particle);
      HWWG_CUDA(cudaMemcpyAsync(d->host_bank, d->bank.p, d->target * sizeof(hwwg_particle),
                                cudaMemcpyDeviceToHost, s));
    }
  } else if (c.host_bank && d->fast && d->world > 1) {
    // multi-rank e2e: the next step's global comb now (it is collective), then
    // this rank's combed source crosses PCIe packed, as on one GPU — not the
    // raw census (x60 of the rank's histories after the cold start)
    const int nstep = step + 1;
    if (nstep <= c.time_steps) {
      const uint64_t nv_next =
          (c.vol_rate > 0.0 && d->q_row[nstep] >= 0) ? c.vol_histories : 0;
      StepLayout Ln;
      d->pre_Hc = multi_gpu_comb(d, nstep, nv_next, Ln, s);
      d->pre_nv = nv_next;
      d->pre_comb_in = d->bank_n;
      d->host_pre_combed = true;
      const uint64_t nl = d->fsrc_local;
      if (2 * nl > d->host_bank_cap) {
        HWWG_CUDA(cudaStreamSynchronize(s));
        if (d->host_bank) HWWG_CUDA(cudaFreeHost(d->host_bank));
        d->host_bank_cap = nl + nl / 4 + 4096;
        HWWG_CUDA(cudaMallocHost(&d->host_bank, d->host_bank_cap * sizeof(hwwg_particle)));
      }
      d->host_bank_n = nl;
      d->host_packed = true;
      launch_check_uniform(d->fsrc.wt.p, nl, d->uni_flag.p, d->uni_first.p, s);
      ++d->launches;
      rec->d2h_bytes += nl * sizeof(double2) + 32;
      HWWG_CUDA(cudaMemcpyAsync(d->host_bank, d->fsrc.xm.p, nl * sizeof(double2),
                                cudaMemcpyDeviceToHost, s));
      HWWG_CUDA(cudaMemcpyAsync(d->h_uni, d->uni_flag.p, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
      HWWG_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(d->h_uni) + 16, d->uni_first.p,
                                sizeof(double2), cudaMemcpyDeviceToHost, s));
    }
  } else if (c.host_bank) {
    if (count > d->host_bank_cap) {
      HWWG_CUDA(cudaStreamSynchronize(s));
      if (d->host_bank) HWWG_CUDA(cudaFreeHost(d->host_bank));
      d->host_bank_cap = count + count / 4;
      HWWG_CUDA(cudaMallocHost(&d->host_bank, d->host_bank_cap * sizeof(hwwg_particle)));
    }
    d->host_bank_n = count;
    rec->d2h_bytes += count * sizeof(hwwg_particle);
    HWWG_CUDA(cudaMemcpyAsync(d->host_bank, d->bank.p, count * sizeof(hwwg_particle),
                              cudaMemcpyDeviceToHost, s));
  }
  hmark("before fetch");
  if (hprof && d->xt[3] && c.host_bank) {
    // every mark relative to the previous step's download start
    auto at = [&](cudaEvent_t x) {
      float v = 0;
      cudaEventElapsedTime(&v, d->xt[0], x);
      return v;
    };
    std::fprintf(stderr, "[host] step %d (ms from the download start): d2h p0 end %.3f, d2h end %.3f, "
                 "ev0 %.3f, h2d start %.3f, h2d p0 end %.3f, seg0 start %.3f, h2d end %.3f, ev1 %.3f\n",
                 step, at(d->xt[4]), at(d->xt[1]), at(d->ev0), at(d->xt[2]), at(d->xt[5]), at(d->xt[6]),
                 at(d->xt[3]), at(d->ev1));
  }
  d->host_tal.fetch(d->tal, s);  // synchronises the stream
  hmark("after fetch");
  if (d->host_pre_combed && d->host_packed) {
    const double* f = reinterpret_cast<const double*>(reinterpret_cast<char*>(d->h_uni) + 16);
    const bool force_full = std::getenv("HWWG_HOST_FULL") != nullptr;  // tests
    d->host_uniform = d->h_uni[0] == 0 && !force_full;
    d->host_w0 = f[0];
    d->host_t0 = f[1];
    if (!d->host_uniform) {  // (w, t) differ: they cross too, after the (x, mu) block
      double2* hb = reinterpret_cast<double2*>(d->host_bank);
      if (d->world == 1)  // single-GPU teeth carry no (w, t) of their own: write them out
        launch_fill_wt(d->fsrc.wt.p, d->host_bank_n, d->comb_mem.p + 1, d->host_t0, s);
      HWWG_CUDA(cudaMemcpyAsync(hb + d->host_bank_n, d->fsrc.wt.p,
                                d->host_bank_n * sizeof(double2), cudaMemcpyDeviceToHost, s));
      HWWG_CUDA(cudaStreamSynchronize(s));
      rec->d2h_bytes += d->host_bank_n * sizeof(double2);
    }
  }
  float ms = 0.f;
  HWWG_CUDA(cudaEventElapsedTime(&ms, d->ev0, d->ev1));
  rec->device_ms = ms;
  double tms = 0.0;
  std::vector<unsigned long long> spans;
  if (!d->seg_events) {
    spans.resize(2 * (thr.size() + 1));
    HWWG_CUDA(cudaMemcpy(spans.data(), d->span.p, spans.size() * 8, cudaMemcpyDeviceToHost));
  }
  for (size_t u = 0; u <= thr.size(); ++u) {
    float e = 0.f;
    if (d->seg_events) HWWG_CUDA(cudaEventElapsedTime(&e, d->seg_ev[2 * u], d->seg_ev[2 * u + 1]));
    else if (spans[2 * u + 1] > spans[2 * u]) e = (float)(1e-6 * (double)(spans[2 * u + 1] - spans[2 * u]));
    tms += e;
    if (u < thr.size() ? thr[u] > (u ? thr[u - 1] : 0) : H > (thr.empty() ? 0 : thr.back()))
      ++rec->transport_launches;
  }
  rec->transport_ms = tms;
  rec->kernel_launches = d->launches;
  rec->d2h_bytes += rep_h.size() * 8 + sizeof flags + sizeof comb_sc + 2 * (size_t)I * 8 +
                    d->tal.words() * 8;
  hmark("end");
  if (d->d2h_pending) {
    // The stream's last command was a download (the record readback), and the
    // next command recorded on a stream after a copy queues in that copy
    // engine — behind the 160 MB below, holding the next step back until they
    // are done. An empty kernel puts the stream back on the compute engine.
    k_stream_mark<<<1, 1, 0, s>>>();
    HWWG_CUDA(cudaGetLastError());
    // e2e: the next step's combed source down to the host in the pieces its
    // uploads take, on the d2h stream; this call returns now and each upload
    // of the next step waits only for its own piece (hwwg_driver_bank and
    // destroy wait for all of them)
    d->xfer_end = xfer_chunks(c, d->hybrid(), d->target, step_volume_histories(d, step + 1), nullptr);
    // (no event wait: the host synchronised the stream after the comb — fetch above)
    if (hprof) {
      for (auto& e : d->xt)
        if (!e) HWWG_CUDA(cudaEventCreate(&e));
      HWWG_CUDA(cudaEventRecord(d->xt[0], d->d2h_stream));
    }
    uint64_t lo = 0;
    for (size_t i = 0; i < d->xfer_end.size(); ++i) {
      const uint64_t hi = d->xfer_end[i];
      HWWG_CUDA(cudaMemcpyAsync(reinterpret_cast<double2*>(d->host_bank) + lo, d->fsrc.xm.p + lo,
                                (hi - lo) * sizeof(double2), cudaMemcpyDeviceToHost, d->d2h_stream));
      HWWG_CUDA(cudaEventRecord(d->d2h_ev[i], d->d2h_stream));
      if (hprof && i == 0) HWWG_CUDA(cudaEventRecord(d->xt[4], d->d2h_stream));
      lo = hi;
    }
    if (hprof) HWWG_CUDA(cudaEventRecord(d->xt[1], d->d2h_stream));
    if (!d->e2e_pipe) HWWG_CUDA(cudaStreamSynchronize(d->d2h_stream));
  }

  const HostTallies& h = d->host_tal;
  if (h.ucount()[kHistoriesScored] != 0) { /* unused: histories counted on host */ }
  const unsigned long long* u = h.ucount();
  rec->counters.collisions = u[kCollisions];
  rec->counters.splits = u[kSplits];
  rec->counters.split_daughters = u[kSplitDaughters];
  rec->counters.capped_splits = u[kCappedSplits];
  rec->counters.roulette_kills = u[kRouletteKills];
  rec->counters.roulette_survivals = u[kRouletteSurvivals];
  rec->counters.census_count = u[kCensusCount];
  rec->counters.event_cap_aborts = u[kEventCapAborts];
  rec->counters.nan_aborts = u[kNanAborts];
  rec->counters.leakage_weight = h.dcount()[0];
  rec->counters.aborted_weight = h.dcount()[1];
  d->h_tracks.assign(h.tracks(), h.tracks() + I);
  uint64_t seg = 0;
  for (int i = 0; i < I; ++i) seg += d->h_tracks[i];
  rec->segments = seg;
  rec->histories = H;
  // banked particles (fast mode: the census slots also hold zero-weight chunk tails)
  rec->census_size = d->fast ? (uint64_t)u[kCensusCount] : count;
  rec->comb_in_weight = comb_sc[0];
  rec->comb_out_weight = do_comb ? comb_sc[3] : comb_sc[0];
  auto field = [&](int f) { return rep_h.data() + (size_t)f * (I + 1); };
  d->h_phi_track.assign(field(0), field(0) + I);
  d->h_sigma.assign(field(1), field(1) + I);
  d->h_phi_census.assign(field(2), field(2) + I);
  d->h_current.assign(field(3), field(3) + I);
  d->h_closure.assign(field(4), field(4) + I);
  d->h_edge.assign(field(5), field(5) + I + 1);
  const double* sc = field(6);
  rec->boundary_closure_left = sc[0];
  rec->boundary_closure_right = sc[1];
  rec->census_weight = sc[2];
  rec->census_weight_sigma = sc[3];
  rec->sigma_valid = sc[4] != 0.0;
  rec->has_windows = (c.mode != 0 && flags[0]) ? 1 : 0;
  rec->has_hybrid = flags[1];
  rec->updates_applied = flags[2];
  rec->hybrid_solve_failed = flags[3];
  d->h_has_centers = rec->has_windows;
  d->h_has_hybrid = flags[1] != 0;
  rec->tau = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  // diagnostics, against the reference when one is set (driver.cpp:231-275)
  const bool ref = !d->ref_interval.empty();
  step_metrics(I, d->prob.edges.data(), d->h_phi_track.data(), d->h_sigma.data(),
               d->h_has_hybrid ? d->h_hybrid.data() : nullptr,
               ref ? d->ref_interval.data() + (size_t)(step - 1) * I : nullptr,
               ref ? d->ref_layer.data() + (size_t)step * I : nullptr,
               ref ? d->ref_layer.data() + (size_t)(step - 1) * I : nullptr, rec);
  // state hand-off (driver.cpp:278-281)
  d->has_prev_report = true;
  d->rep_cur ^= 1;
  ++d->next_step;
  d->history.push_back(*rec);
}

}  // namespace

extern "C" {

int hwwg_driver_create(const hwwg_run_config* cfg, const hwwg_options* opts, hwwg_driver** out) {
  HWWG_API_BEGIN
  if (!cfg || !out) return fail(HWWG_EINVAL, "NULL argument");
  *out = nullptr;
  char buf[1024];
  if (hwwg_validate_config(cfg, buf, sizeof buf) != 0)
    return fail(HWWG_EINVAL, std::string("invalid configuration:\n") + buf);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(HWWG_ECUDA, "no CUDA device available");
  }
  auto d = new hwwg_driver();
  d->cfg = *cfg;
  if (opts) d->opt = *opts;
  if (d->opt.rng_mode != HWWG_RNG_EXACT && d->opt.rng_mode != HWWG_RNG_PHILOX) {
    delete d;
    return fail(HWWG_EINVAL, "unknown rng_mode");
  }
  d->fast = d->opt.rng_mode == HWWG_RNG_PHILOX;
  d->timeline_on = d->fast && std::getenv("HWWG_FAST_TIMELINE") != nullptr;
  d->phases_on = std::getenv("HWWG_PHASES") != nullptr;
  d->losm_cache = std::getenv("HWWG_LOSM_NOCACHE") == nullptr;
  if (const char* m = std::getenv("HWWG_FAST_SMEM")) d->smem_mode = std::atoi(m) % 3;
  if (const char* m = std::getenv("HWWG_FAST_SCRAMBLE")) d->scramble = std::atoi(m) ? 1 : 0;
  if (const char* m = std::getenv("HWWG_FAST_AGG")) {
    const int v = std::atoi(m);
    d->agg_all = v == 2 ? 2 : (v ? 1 : 0);
  }
  if (const char* m = std::getenv("HWWG_FAST_FIX")) d->fix_tallies = std::atoi(m) ? 1 : 0;
  if (const char* m = std::getenv("HWWG_PRECOMB")) d->precomb = std::atoi(m) ? 1 : 0;
  if (const char* m = std::getenv("HWWG_PRECOMB_K")) d->precomb_k = std::max(1.0, std::atof(m));
  if (const char* m = std::getenv("HWWG_PDL")) d->pdl = std::atoi(m) ? 1 : 0;
  if (const char* m = std::getenv("HWWG_E2E_PIPE")) d->e2e_pipe = std::atoi(m) != 0;
  if (const char* m = std::getenv("HWWG_PACKED_TEETH")) d->packed_teeth = std::atoi(m) ? 1 : 0;
  if (const char* m = std::getenv("HWWG_TALLY_WINDOW")) d->tally_window = std::max(0, std::atoi(m));
  if (const char* m = std::getenv("HWWG_TALLY_WINDOW_MAX")) d->tally_window_max = std::max(0, std::atoi(m));
  if (const char* m = std::getenv("HWWG_FAST_BLOCK_WARPS")) {
    const int w = std::atoi(m);
    d->block_warps = (w == 12 || w == 14 || w == 24) ? w : 0;
  }
  d->seg_events = d->fast ? (std::getenv("HWWG_SEG_EVENTS") ? 1 : 0) : 1;
  d->span.reserve(64);
  if (const char* m = std::getenv("HWWG_FAST_FLUSH_R")) d->flush_replicas = std::max(0, std::atoi(m));
  d->world = d->opt.world > 1 ? d->opt.world : 1;
  d->rank = d->world > 1 ? d->opt.rank : 0;
  if (d->world > 1 && (!d->fast || d->rank < 0 || d->rank >= d->world)) {
    delete d;
    return fail(HWWG_EINVAL, "multi-GPU runs need HWWG_RNG_PHILOX and 0 <= rank < world "
                             "(exact mode replays one sequential comb)");
  }
  if (d->opt.loopback && d->world != loopback_world(d->opt.loopback)) {
    delete d;
    return fail(HWWG_EINVAL, "loopback hub world differs from the driver's world");
  }
  if (d->fast && cfg->cells > 65535) {
    delete d;
    return fail(HWWG_EINVAL, "philox mode: more than 65535 cells are not supported");
  }
  // history ids are 32-bit and the batch of history h is one fp64 division
  // (exact while h * batches < 2^53)
  const uint64_t tgt = cfg->target_population ? cfg->target_population : cfg->histories_per_step;
  if (d->fast && (tgt >= (1ULL << 32) - (1ULL << 26) || cfg->batches >= (1 << 16))) {
    delete d;
    return fail(HWWG_EINVAL, "philox mode: histories per step must stay below 2^32 - 2^26 "
                             "and batches below 2^16");
  }
  try {
    init_driver(d);
  } catch (...) {
    delete d;
    throw;
  }
  *out = d;
  return HWWG_OK;
  HWWG_API_END
}

void hwwg_driver_destroy(hwwg_driver* d) { delete d; }

int hwwg_driver_step(hwwg_driver* d, hwwg_step_record* rec) {
  HWWG_API_BEGIN
  if (!d || !rec) return fail(HWWG_EINVAL, "NULL argument");
  if (d->next_step > d->cfg.time_steps) return fail(HWWG_ESTATE, "run already complete");
  HWWG_CUDA(cudaSetDevice(d->opt.device));
  driver_step(d, rec);
  return HWWG_OK;
  HWWG_API_END
}

int hwwg_driver_arrays(hwwg_driver* d, double* phi_track, double* phi_sigma, double* phi_census,
                       double* current_census, double* closure_census, double* edge_current,
                       double* ww_centers, double* phi_hybrid, uint64_t* tracks_per_cell) {
  HWWG_API_BEGIN
  if (!d) return fail(HWWG_EINVAL, "NULL driver");
  if (d->next_step == 1) return fail(HWWG_ESTATE, "no step has run yet");
  auto cp = [](double* dst, const std::vector<double>& v) {
    if (dst) std::memcpy(dst, v.data(), v.size() * 8);
  };
  cp(phi_track, d->h_phi_track);
  cp(phi_sigma, d->h_sigma);
  cp(phi_census, d->h_phi_census);
  cp(current_census, d->h_current);
  cp(closure_census, d->h_closure);
  cp(edge_current, d->h_edge);
  if (d->h_has_centers) cp(ww_centers, d->h_centers);
  if (d->h_has_hybrid) cp(phi_hybrid, d->h_hybrid);
  if (tracks_per_cell)
    for (int i = 0; i < d->I; ++i) tracks_per_cell[i] = d->h_tracks[i];
  return HWWG_OK;
  HWWG_API_END
}

int hwwg_driver_set_reference(hwwg_driver* d, const double* phi_layer,
                              const double* phi_interval, const char* name) {
  HWWG_API_BEGIN
  if (!d || !phi_layer || !phi_interval) return fail(HWWG_EINVAL, "NULL argument");
  const size_t I = d->I, N = d->cfg.time_steps;
  if (name) {
    if (std::strlen(name) >= sizeof d->cfg.reference)
      return fail(HWWG_EINVAL, "reference name longer than 255 bytes");
    std::memset(d->cfg.reference, 0, sizeof d->cfg.reference);
    std::memcpy(d->cfg.reference, name, std::strlen(name));
  }
  d->ref_layer.assign(phi_layer, phi_layer + (N + 1) * I);
  d->ref_interval.assign(phi_interval, phi_interval + N * I);
  return HWWG_OK;
  HWWG_API_END
}

int hwwg_driver_load_reference(hwwg_driver* d, const char* path) {
  HWWG_API_BEGIN
  if (!d || !path) return fail(HWWG_EINVAL, "NULL argument");
  const int I = d->I, N = d->cfg.time_steps;
  std::vector<double> lay((size_t)(N + 1) * I), itv((size_t)N * I);
  load_reference(path, I, d->prob.edges.data(), N, d->layers.data(), lay.data(), itv.data());
  return hwwg_driver_set_reference(d, lay.data(), itv.data(), path);
  HWWG_API_END
}

int hwwg_driver_compute_reference(hwwg_driver* d, int32_t space_refine, int32_t time_refine,
                                  int32_t sn_order) {
  HWWG_API_BEGIN
  if (!d) return fail(HWWG_EINVAL, "NULL argument");
  const int I = d->I, N = d->cfg.time_steps;
  std::vector<double> lay((size_t)(N + 1) * I), itv((size_t)N * I);
  const SnHostProblem p = reference_problem(d->cfg, space_refine, time_refine, sn_order);
  sn_solve_device(p, d->opt.device, d->stream, nullptr, nullptr, lay.data(), itv.data());
  return hwwg_driver_set_reference(d, lay.data(), itv.data(), "auto");
  HWWG_API_END
}

int hwwg_driver_write(hwwg_driver* d, const char* dir, int32_t final, double total_seconds) {
  HWWG_API_BEGIN
  if (!d || !dir) return fail(HWWG_EINVAL, "NULL argument");
  if (d->history.empty()) return fail(HWWG_ESTATE, "no step has run yet");
  const hwwg_run_config& c = d->cfg;
  int rc = hwwg_write_step_csv(dir, &d->history.back(), d->I, d->prob.edges.data(),
                               d->h_phi_track.data(), d->h_sigma.data(), d->h_phi_census.data(),
                               d->h_current.data(), d->h_closure.data(),
                               d->h_has_centers ? d->h_centers.data() : nullptr,
                               d->h_has_hybrid ? d->h_hybrid.data() : nullptr,
                               reinterpret_cast<const uint64_t*>(d->h_tracks.data()),
                               (double)c.histories_per_step);
  if (rc == HWWG_OK) rc = hwwg_write_summary_csv(dir, d->history.data(), d->history.size());
  if (rc == HWWG_OK && final) rc = hwwg_write_run_json(dir, &c, total_seconds, d->history.size());
  return rc;
  HWWG_API_END
}

int hwwg_driver_bank(hwwg_driver* d, hwwg_particle* out, uint64_t cap, uint64_t* n) {
  HWWG_API_BEGIN
  if (!d || !n) return fail(HWWG_EINVAL, "NULL argument");
  if (d->d2h_stream) HWWG_CUDA(cudaStreamSynchronize(d->d2h_stream));  // the host copy is complete
  uint64_t count = d->bank_n;
  if (d->fast && !d->cfg.host_bank && d->next_step > 1) {
    // Philox mode keeps the census as SoA with zero-weight chunk tails: compact
    // the real particles into AoS (order is free in this mode)
    d->bank.reserve(std::max<uint64_t>(d->bank_n, 1));
    launch_fast_compact_aos(d->fbank.view(), d->bank_n, d->bank_t, d->bank.p, d->counter.p,
                            d->stream);
    unsigned long long c = 0;
    HWWG_CUDA(cudaMemcpyAsync(&c, d->counter.p, sizeof c, cudaMemcpyDeviceToHost, d->stream));
    HWWG_CUDA(cudaStreamSynchronize(d->stream));
    count = c;
  } else if (d->fast && d->host_pre_combed && d->host_packed) {
    // the pre-combed source crossed PCIe packed; hand out AoS particles
    // (single GPU: its teeth are (x, mu) only, weight comb_mem[1], time src_t0)
    d->bank.reserve(std::max<uint64_t>(d->bank_n, 1));
    launch_fast_to_aos_packed(d->fsrc.view(), d->bank_n, d->world == 1 ? d->bank_n : 0,
                              d->comb_mem.p + 1, d->src_t0, d->bank.p, d->stream);
  }
  *n = count;
  if (!out || cap < count) return fail(HWWG_ENOSPC, "bank buffer too small");
  HWWG_CUDA(cudaMemcpyAsync(out, d->bank.p, count * sizeof(hwwg_particle), cudaMemcpyDeviceToHost,
                            d->stream));
  HWWG_CUDA(cudaStreamSynchronize(d->stream));
  return HWWG_OK;
  HWWG_API_END
}

}  // extern "C"
