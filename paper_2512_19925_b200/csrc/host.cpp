// Host pieces of the engine: RunConfig defaults/validation/key=value loader
// (proj/include/hww/config.hpp:33-93, proj/src/config.cpp:27-69,
// proj/tools/hww_main.cpp:20-92) and the driver's sequential helpers.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "capi_util.h"
#include "driver_host.h"
#include "hwwg.h"
#include "rng.cuh"

namespace hwwg {

void sample_pulse_source_host(uint64_t seed, uint64_t histories, double x0, double total_weight,
                              double t0, hwwg_particle* out) {
  Xoshiro r;
  r.seed(seed, stream_id(0, 0, kSource));
  const double w = total_weight / (double)histories;
  for (uint64_t h = 0; h < histories; ++h) out[h] = hwwg_particle{x0, r.uniform_pm1(), w, t0};
}

// Config-3 volumetric source: n particles of the
// isotropic box [x_lo, x_hi] x [ta, tb] from the step's source stream (step, 0,
// source); per particle x, then t, then mu; w = rate * (tb - ta) * h_cfg / n.
// Same arithmetic as oracle/hww_oracle.c orc_volume_source.
void sample_volume_source_host(uint64_t seed, int step, uint64_t n, double x_lo, double x_hi,
                               double ta, double tb, double rate, uint64_t h_cfg,
                               hwwg_particle* out) {
  Xoshiro r;
  r.seed(seed, stream_id((uint64_t)step, 0, kSource));
  const double w = rate * (tb - ta) * (double)h_cfg / (double)n;
  for (uint64_t h = 0; h < n; ++h) {
    const double x = x_lo + (x_hi - x_lo) * r.uniform();
    const double t = ta + (tb - ta) * r.uniform();
    const double mu = r.uniform_pm1();
    out[h] = hwwg_particle{x, mu, w, t};
  }
}

// The step's LOSM source q_i (losm.cpp:101-103 pass-through): the box's emission
// over cell i averaged over the step (orc_volume_q).
void volume_q_host(const double* edges, int I, double x_lo, double x_hi, double ta, double tb,
                   double dt, double rate, double* q) {
  const double tfrac = (tb - ta) / dt;
  const double bw = x_hi - x_lo;
  for (int i = 0; i < I; ++i) {
    const double lo = edges[i] > x_lo ? edges[i] : x_lo;
    const double hi = edges[i + 1] < x_hi ? edges[i + 1] : x_hi;
    const double len = hi > lo ? hi - lo : 0.0;
    q[i] = rate * tfrac * len / bw;
  }
}

uint64_t stream_id_host(uint64_t step, uint64_t history, uint64_t purpose) {
  return stream_id(step, history, purpose);
}

int batch_of_host(uint64_t h, uint64_t H, int B) {
  if (H == 0) return 0;
  const int b = (int)(h * (uint64_t)B / H);
  return b < B ? b : B - 1;
}

int locate_host(const std::vector<double>& e, double x) {
  const int I = (int)e.size() - 1;
  if (x < e.front() || x > e.back()) return -1;
  if (x == e.back()) return I - 1;
  const double w0 = e[1] - e[0];
  bool uniform = true;
  for (int c = 0; c < I; ++c)
    if (!(std::abs((e[c + 1] - e[c]) - w0) <= 1e-12 * w0)) uniform = false;
  if (uniform) {
    int c = (int)((x - e.front()) / w0);
    if (c >= I) c = I - 1;
    if (x < e[c]) --c;
    else if (x >= e[c + 1]) ++c;
    return c;
  }
  int a = 0, b = I + 1;
  while (a < b) {
    const int m = (a + b) / 2;
    if (e[m] > x) b = m;
    else a = m + 1;
  }
  return a - 1;
}

}  // namespace hwwg

using namespace hwwg;

extern "C" {

void hwwg_default_config(hwwg_run_config* c) {
  std::memset(c, 0, sizeof(*c));
  c->mode = 2;  // hww
  c->histories_per_step = 10000;
  c->theta = 0.5;
  c->rho = 1.25;
  c->eps_min = 1e-3;
  c->u_ww = 3;
  c->n_fractions = 3;
  c->fractions[0] = 0.25;
  c->fractions[1] = 0.5;
  c->fractions[2] = 0.75;
  c->ma_base_k = 3;
  c->fourier_cutoff = 30;
  c->batches = 20;
  c->seed = 1;
  c->target_population = 0;
  c->comb_overflow_factor = 1.0;
  c->x0 = 0.0;
  c->t0 = 0.0;
  c->strength = 1.0;
  c->sigma_t = 1.0;
  c->sigma_s = 1.0 / 3.0;
  c->sigma_f = 1.0 / 3.0;
  c->nu_f = 2.3;
  c->speed = 1.0;
  c->x_min = -20.5;
  c->x_max = 20.5;
  c->cells = 201;
  c->t_end = 20.0;
  c->time_steps = 20;
}

int hwwg_validate_config(const hwwg_run_config* c, char* buf, uint64_t buf_len) {
  std::vector<std::string> v;
  // Material::validate (material.hpp:20-32)
  if (!(c->sigma_t > 0)) v.push_back("sigma_t must be > 0");
  if (c->sigma_s < 0 || c->sigma_s > c->sigma_t) v.push_back("sigma_s must lie in [0, sigma_t]");
  if (c->sigma_f < 0 || c->sigma_f > c->sigma_t) v.push_back("sigma_f must lie in [0, sigma_t]");
  if (c->sigma_s + c->sigma_f > c->sigma_t) v.push_back("sigma_s + sigma_f must not exceed sigma_t");
  if (c->nu_f < 0) v.push_back("nu_f must be >= 0");
  if (!(c->speed > 0)) v.push_back("speed must be > 0");
  // config.cpp:30-66
  if (c->histories_per_step < 1) v.push_back("histories_per_step must be >= 1");
  if (!(c->theta >= 0.5 && c->theta <= 1.0)) v.push_back("theta must lie in [1/2, 1]");
  if (!(c->rho >= 1.0)) v.push_back("rho must be >= 1");
  if (!(c->eps_min > 0.0 && c->eps_min < 1.0)) v.push_back("eps_min must lie in (0,1)");
  if (c->u_ww < 0) v.push_back("u_ww must be >= 0");
  if (c->mode < 0 || c->mode > 4) v.push_back("unknown mode");
  if (c->mode >= 2) {
    if (c->n_fractions != c->u_ww) v.push_back("update_fractions count must equal u_ww");
    double prev = 0.0;
    for (int i = 0; i < c->n_fractions && i < 8; ++i) {
      const double f = c->fractions[i];
      if (!(f > 0.0 && f < 1.0)) {
        v.push_back("update fractions must lie in (0,1)");
        break;
      }
      if (!(f > prev)) {
        v.push_back("update fractions must increase");
        break;
      }
      prev = f;
    }
  }
  if (c->n_fractions < 0 || c->n_fractions > 8) v.push_back("at most 8 update fractions");
  if (c->mode == 3 && c->ma_base_k < 0) v.push_back("ma_base_k must be >= 0");
  if (c->mode == 4 && c->fourier_cutoff < 0) v.push_back("fourier_cutoff must be >= 0");
  if (c->batches < 2) v.push_back("batches must be >= 2");
  if (!(c->x_min < c->x_max)) v.push_back("x_min must be < x_max");
  if (c->cells < 1) v.push_back("cells must be >= 1");
  if (!(c->t_end > 0.0)) v.push_back("t_end must be > 0");
  if (c->time_steps < 1) v.push_back("time_steps must be >= 1");
  if (!c->no_pulse) {
    if (!(c->strength > 0.0)) v.push_back("source strength must be > 0");
    if (c->x0 < c->x_min || c->x0 > c->x_max) v.push_back("source x0 must lie inside the mesh");
  }
  // config-3 extensions: regions and the volumetric source
  if (c->n_regions < 0 || c->n_regions > 8) v.push_back("n_regions must lie in [0, 8]");
  for (int r = 0; r < c->n_regions && r < 8; ++r) {
    const double* m = c->region_mat[r];
    if (!(m[0] > 0) || m[1] < 0 || m[2] < 0 || m[1] + m[2] > m[0] || m[3] < 0 || !(m[4] > 0))
      v.push_back("region " + std::to_string(r) + ": invalid material");
    if (r > 0 && !(c->region_x_hi[r] > c->region_x_hi[r - 1]))
      v.push_back("region upper bounds must increase");
  }
  if (c->vol_rate < 0.0) v.push_back("vol_rate must be >= 0");
  if (c->vol_rate > 0.0) {
    if (!(c->vol_x_lo < c->vol_x_hi) || c->vol_x_lo < c->x_min || c->vol_x_hi > c->x_max)
      v.push_back("volumetric source box must be non-empty and inside the mesh");
    if (!(c->vol_t_lo < c->vol_t_hi)) v.push_back("volumetric source window must be non-empty");
    if (c->vol_histories < 1) v.push_back("vol_histories must be >= 1");
  }
  if (c->no_pulse && !(c->vol_rate > 0.0)) v.push_back("no source: no pulse and no volumetric source");
  std::string joined;
  for (size_t i = 0; i < v.size(); ++i) joined += (i ? "\n" : "") + v[i];
  if (buf && buf_len) {
    std::strncpy(buf, joined.c_str(), buf_len - 1);
    buf[buf_len - 1] = 0;
  }
  return (int)v.size();
}

// Key = value file mirroring the RunConfig field names (hww_main.cpp:20-92).
int hwwg_load_config_file(const char* path, hwwg_run_config* c) {
  HWWG_API_BEGIN
  std::ifstream in(path);
  if (!in) return fail(HWWG_EINVAL, std::string("cannot open config file: ") + path);
  std::string line;
  int line_no = 0;
  auto trim = [](const std::string& s) {
    const auto b = s.find_first_not_of(" \t\r");
    const auto e = s.find_last_not_of(" \t\r");
    return b == std::string::npos ? std::string() : s.substr(b, e - b + 1);
  };
  while (std::getline(in, line)) {
    ++line_no;
    const auto hash = line.find('#');
    if (hash != std::string::npos) line = line.substr(0, hash);
    const auto eq = line.find('=');
    if (eq == std::string::npos) {
      if (line.find_first_not_of(" \t\r") != std::string::npos)
        return fail(HWWG_EINVAL, "line " + std::to_string(line_no) + ": expected key = value");
      continue;
    }
    const std::string key = trim(line.substr(0, eq));
    const std::string val = trim(line.substr(eq + 1));
    try {
      if (key == "mode") {
        static const char* names[] = {"analog", "lww", "hww", "hww_ma", "hww_fourier"};
        int m = -1;
        for (int i = 0; i < 5; ++i)
          if (val == names[i]) m = i;
        if (m < 0) throw std::invalid_argument("unknown mode '" + val + "'");
        c->mode = m;
      } else if (key == "histories_per_step") c->histories_per_step = std::stoull(val);
      else if (key == "theta") c->theta = std::stod(val);
      else if (key == "rho") c->rho = std::stod(val);
      else if (key == "eps_min") c->eps_min = std::stod(val);
      else if (key == "u_ww") c->u_ww = std::stoi(val);
      else if (key == "update_fractions") {
        c->n_fractions = 0;
        std::stringstream ss(val);
        std::string tok;
        while (std::getline(ss, tok, ',')) {
          if (c->n_fractions == 8) throw std::invalid_argument("at most 8 update fractions");
          c->fractions[c->n_fractions++] = std::stod(tok);
        }
      } else if (key == "ma_base_k") c->ma_base_k = std::stoi(val);
      else if (key == "fourier_cutoff") c->fourier_cutoff = std::stoi(val);
      else if (key == "batches") c->batches = std::stoi(val);
      else if (key == "seed") c->seed = std::stoull(val);
      else if (key == "target_population") c->target_population = std::stoull(val);
      else if (key == "comb_overflow_factor") c->comb_overflow_factor = std::stod(val);
      else if (key == "source_x0") c->x0 = std::stod(val);
      else if (key == "source_strength") c->strength = std::stod(val);
      else if (key == "sigma_t") c->sigma_t = std::stod(val);
      else if (key == "sigma_s") c->sigma_s = std::stod(val);
      else if (key == "sigma_f") c->sigma_f = std::stod(val);
      else if (key == "nu_f") c->nu_f = std::stod(val);
      else if (key == "speed") c->speed = std::stod(val);
      else if (key == "x_min") c->x_min = std::stod(val);
      else if (key == "x_max") c->x_max = std::stod(val);
      else if (key == "cells") c->cells = std::stoi(val);
      else if (key == "t_end") c->t_end = std::stod(val);
      else if (key == "time_steps") c->time_steps = std::stoi(val);
      else if (key == "threads") c->threads = std::stoi(val);
      // config-3 extension keys (absent from the
      // reference's loader): repeatable `region = x_hi, sigma_t, sigma_s,
      // sigma_f, nu_f, speed`, `volume_source = x_lo, x_hi, t_lo, t_hi, rate`,
      // `vol_histories`, `no_pulse`
      else if (key == "region") {
        std::vector<double> v;
        std::stringstream ss(val);
        std::string tok;
        while (std::getline(ss, tok, ',')) v.push_back(std::stod(tok));
        if (v.size() != 6) throw std::invalid_argument("region needs x_hi and 5 material values");
        if (c->n_regions == 8) throw std::invalid_argument("at most 8 regions");
        c->region_x_hi[c->n_regions] = v[0];
        for (int j = 0; j < 5; ++j) c->region_mat[c->n_regions][j] = v[1 + j];
        ++c->n_regions;
      } else if (key == "volume_source") {
        std::vector<double> v;
        std::stringstream ss(val);
        std::string tok;
        while (std::getline(ss, tok, ',')) v.push_back(std::stod(tok));
        if (v.size() != 5) throw std::invalid_argument("volume_source needs x_lo, x_hi, t_lo, t_hi, rate");
        c->vol_x_lo = v[0];
        c->vol_x_hi = v[1];
        c->vol_t_lo = v[2];
        c->vol_t_hi = v[3];
        c->vol_rate = v[4];
        if (!c->vol_histories) c->vol_histories = c->histories_per_step;
      } else if (key == "vol_histories") c->vol_histories = std::stoull(val);
      else if (key == "no_pulse") c->no_pulse = (val == "1" || val == "true") ? 1 : 0;
      else if (key == "reference") {  // hww_main.cpp:82
        if (val.size() >= sizeof c->reference)
          throw std::invalid_argument("reference path longer than 255 bytes");
        std::memset(c->reference, 0, sizeof c->reference);
        std::memcpy(c->reference, val.data(), val.size());
      } else if (key == "out_dir") { /* host tooling key: accepted */ }
      else throw std::invalid_argument("unknown key '" + key + "'");
    } catch (const std::exception& e) {
      return fail(HWWG_EINVAL, "line " + std::to_string(line_no) + ": " + e.what());
    }
  }
  return HWWG_OK;
  HWWG_API_END
}

// ---------------------------------------------------------------- sharding
// Multi-GPU plan: every rank computes the same plan from the
// same all-gathered numbers, so no rank ever disagrees about who owns what.

void hwwg_shard_range(uint64_t H, int32_t rank, int32_t world, uint64_t* lo, uint64_t* hi) {
  // contiguous, near-equal slices; batch ids stay global (batch_of(h, H, B))
  *lo = H * (uint64_t)rank / (uint64_t)world;
  *hi = H * (uint64_t)(rank + 1) / (uint64_t)world;
}

// Global comb over per-rank census banks: rank r's particles occupy
// [O_r, O_r + W_r) of the global cumulative-weight axis, O_r the exclusive
// prefix of rank_weights in rank order (popctrl.cpp:15-30 semantics with the
// bank concatenated in rank order). Tooth k (T_k = offset + k*spacing) belongs
// to the first rank with T_k < O_{r+1}; stranded teeth go to the last rank
// (popctrl.cpp:31-37). Outputs this rank's tooth range and O_r.
int hwwg_comb_plan(const double* rank_weights, int32_t world, int32_t rank, uint64_t target,
                   double offset_frac, double* spacing_out, double* offset_out,
                   double* rank_origin, uint64_t* k_lo, uint64_t* k_hi) {
  if (world < 1 || rank < 0 || rank >= world || target < 1)
    return fail(HWWG_EINVAL, "bad comb plan arguments");
  double W = 0.0;
  for (int q = 0; q < world; ++q) W += rank_weights[q];
  if (!(W > 0.0)) return fail(HWWG_EINVAL, "cannot comb an empty bank");
  const double spacing = W / (double)target;
  const double offset = offset_frac * spacing;
  auto first_tooth_at_or_above = [&](double edge) -> uint64_t {
    // smallest k with offset + k*spacing >= edge (clamped to [0, target])
    double g = std::ceil((edge - offset) / spacing);
    uint64_t k = g <= 0.0 ? 0 : (g >= (double)target ? target : (uint64_t)g);
    while (k > 0 && offset + (double)(k - 1) * spacing >= edge) --k;
    while (k < target && offset + (double)k * spacing < edge) ++k;
    return k;
  };
  int last = world - 1;  // stranded teeth go to the last rank that holds weight
  while (last > 0 && !(rank_weights[last] > 0.0)) --last;
  double O = 0.0;
  uint64_t lo = 0;
  for (int q = 0; q <= rank; ++q) {
    const double O_next = O + rank_weights[q];
    const uint64_t hi_q = q >= last ? target : first_tooth_at_or_above(O_next);
    if (q == rank) {
      *rank_origin = O;
      *k_lo = lo;
      *k_hi = hi_q < lo ? lo : hi_q;
    }
    lo = hi_q < lo ? lo : hi_q;
    O = O_next;
  }
  *spacing_out = spacing;
  *offset_out = offset;
  return HWWG_OK;
}

// Rebalance after the comb: this rank produced teeth [k_lo, k_hi); rank q
// owns next-step histories shard(q). send[q] = |[k_lo,k_hi) ∩ shard(q)|,
// send_first[q] = first tooth sent to q; recv[q] = |[k_lo_q, k_hi_q) ∩ shard(rank)|.
void hwwg_rebalance_plan(const uint64_t* k_lo_all, const uint64_t* k_hi_all, int32_t world,
                         int32_t rank, uint64_t H, uint64_t* send, uint64_t* send_first,
                         uint64_t* recv) {
  uint64_t my_lo, my_hi;
  hwwg_shard_range(H, rank, world, &my_lo, &my_hi);
  for (int q = 0; q < world; ++q) {
    uint64_t s_lo, s_hi;
    hwwg_shard_range(H, q, world, &s_lo, &s_hi);
    const uint64_t a = std::max(k_lo_all[rank], s_lo), b = std::min(k_hi_all[rank], s_hi);
    send[q] = b > a ? b - a : 0;
    send_first[q] = b > a ? a : 0;
    const uint64_t c = std::max(k_lo_all[q], my_lo), e = std::min(k_hi_all[q], my_hi);
    recv[q] = e > c ? e - c : 0;
  }
}

}  // extern "C"
