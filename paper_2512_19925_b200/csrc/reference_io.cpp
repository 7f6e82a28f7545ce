// Deterministic reference solution files and the per-step error diagnostics
// (SURVEY.md §8(f3)):
//   hwwg_save_reference_csv / hwwg_load_reference_csv
//       hww::save_reference / hww::load_reference (proj/src/reference.cpp:374-456)
//   hwwg_step_metrics
//       the diagnostics block of hww::run_step (proj/src/driver.cpp:231-275) over
//       l2_norm, modified_l2_norm, fom and relative_change (proj/src/metrics.cpp:8-66)
//
// Host code on purpose: a step's metrics are O(cells) on arrays the driver has
// already brought to the host for the step record, and every sum below runs in
// the reference's cell order (no FMA contraction, -ffp-contract=off), so equal
// arrays and tau give bit-identical metrics.
#include <algorithm>
#include <cmath>
#include <fstream>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "capi_util.h"
#include "hwwg.h"
#include "reference_io.h"

namespace hwwg {
namespace {

constexpr double kLowFluxThreshold = 1e-3;  // phi* of the modified norms (driver.cpp:21)

// l2_norm (metrics.cpp:8-14)
double l2_norm(const double* f, int cells, const double* edges) {
  double sum = 0.0;
  for (int i = 0; i < cells; ++i) sum += f[i] * f[i] * (edges[i + 1] - edges[i]);
  return std::sqrt(sum);
}

// modified_l2_norm (metrics.cpp:16-32): cells whose mask flux is below phi*
double modified_l2_norm(const double* f, int cells, const double* edges, const double* mask,
                        bool* empty_mask) {
  double sum = 0.0;
  bool any = false;
  for (int i = 0; i < cells; ++i) {
    if (mask[i] < kLowFluxThreshold) {
      sum += f[i] * f[i] * (edges[i + 1] - edges[i]);
      any = true;
    }
  }
  if (empty_mask) *empty_mask = !any;
  return std::sqrt(sum);
}

// fom (metrics.cpp:34-55): L2 and masked L2 of 1/(tau v^2) over cells with v != 0
void fom(const double* v, double tau, int cells, const double* edges, const double* mask,
         double* l2, double* mod_l2) {
  double sum = 0.0, sum_mod = 0.0;
  for (int i = 0; i < cells; ++i) {
    if (v[i] == 0.0) continue;
    const double f = 1.0 / (tau * v[i] * v[i]);
    const double w = edges[i + 1] - edges[i];
    sum += f * f * w;
    if (mask && mask[i] < kLowFluxThreshold) sum_mod += f * f * w;
  }
  *l2 = std::sqrt(sum);
  if (mod_l2) *mod_l2 = std::sqrt(sum_mod);
}

}  // namespace

void step_metrics(int cells, const double* edges, const double* phi_track,
                  const double* phi_sigma, const double* phi_hybrid, const double* ref_interval,
                  const double* ref_layer, const double* ref_layer_prev, hwwg_step_record* rec) {
  const double nan = std::numeric_limits<double>::quiet_NaN();
  rec->rel_l2_error = rec->rel_mod_l2_error = rec->hybrid_rel_l2_error = nan;
  rec->fom_err_l2 = rec->fom_err_mod = rec->fom_sigma_l2 = rec->fom_sigma_mod = nan;
  rec->alpha = nan;
  const double tau = std::max(rec->tau, 1e-9);
  if (ref_interval) {
    std::vector<double> err(cells);
    for (int i = 0; i < cells; ++i) err[i] = phi_track[i] - ref_interval[i];
    const double ref_norm = l2_norm(ref_interval, cells, edges);
    if (ref_norm > 0.0) rec->rel_l2_error = l2_norm(err.data(), cells, edges) / ref_norm;
    bool empty = false;
    const double ref_mod = modified_l2_norm(ref_interval, cells, edges, ref_layer, &empty);
    if (!empty && ref_mod > 0.0)
      rec->rel_mod_l2_error =
          modified_l2_norm(err.data(), cells, edges, ref_layer, nullptr) / ref_mod;
    if (phi_hybrid) {
      std::vector<double> herr(cells);
      for (int i = 0; i < cells; ++i) herr[i] = phi_hybrid[i] - ref_layer[i];
      const double layer_norm = l2_norm(ref_layer, cells, edges);
      if (layer_norm > 0.0)
        rec->hybrid_rel_l2_error = l2_norm(herr.data(), cells, edges) / layer_norm;
    }
    fom(err.data(), tau, cells, edges, ref_layer, &rec->fom_err_l2, &rec->fom_err_mod);
    // relative_change (metrics.cpp:57-66)
    const double denom = l2_norm(ref_layer, cells, edges);
    if (denom == 0.0) throw ApiError(HWWG_EINVAL, "relative_change: ||phi_now|| is zero");
    std::vector<double> diff(cells);
    for (int i = 0; i < cells; ++i) diff[i] = ref_layer[i] - ref_layer_prev[i];
    rec->alpha = l2_norm(diff.data(), cells, edges) / denom;
    if (rec->sigma_valid)
      fom(phi_sigma, tau, cells, edges, ref_layer, &rec->fom_sigma_l2, &rec->fom_sigma_mod);
  } else if (rec->sigma_valid) {
    fom(phi_sigma, tau, cells, edges, nullptr, &rec->fom_sigma_l2, nullptr);
  }
}

void load_reference(const char* path, int cells, const double* edges, int steps,
                    const double* layers, double* phi_layer, double* phi_interval) {
  std::ifstream in(path);
  if (!in) throw ApiError(HWWG_EFORMAT, std::string("cannot open reference file: ") + path);
  std::string line;
  if (!std::getline(in, line))
    throw ApiError(HWWG_EFORMAT, std::string("reference file is empty: ") + path);
  std::vector<double> lay((size_t)(steps + 1) * cells, 0.0), itv((size_t)steps * cells, 0.0);
  const long long expected = (long long)(steps + 1) * cells;
  const double span = edges[cells] - edges[0];
  long long rows = 0;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    std::replace(line.begin(), line.end(), ',', ' ');
    std::istringstream ss(line);
    // stod/stoi, not stream extraction, so "nan" parses (reference.cpp:417-419)
    std::string tt, tc, tx, tp, ti;
    if (!(ss >> tt >> tc >> tx >> tp >> ti))
      throw ApiError(HWWG_EFORMAT, "malformed reference row: " + line);
    double t, x, phi, interval;
    int cell;
    try {
      t = std::stod(tt);
      cell = std::stoi(tc);
      x = std::stod(tx);
      phi = std::stod(tp);
      interval = std::stod(ti);
    } catch (const std::exception&) {
      throw ApiError(HWWG_EFORMAT, "malformed reference row: " + line);
    }
    if (rows >= expected)
      throw ApiError(HWWG_EFORMAT,
                     "reference file has more rows than expected " + std::to_string(expected));
    const int layer = (int)(rows / cells);
    const int expect_cell = (int)(rows % cells);
    if (cell != expect_cell)
      throw ApiError(HWWG_EFORMAT, "reference cell index mismatch: expected " +
                                       std::to_string(expect_cell) + ", found " +
                                       std::to_string(cell));
    if (std::abs(t - layers[layer]) > 1e-9)
      throw ApiError(HWWG_EFORMAT,
                     "reference layer time mismatch at layer " + std::to_string(layer));
    if (std::abs(x - 0.5 * (edges[cell] + edges[cell + 1])) > 1e-9 * span)
      throw ApiError(HWWG_EFORMAT,
                     "reference cell center mismatch at cell " + std::to_string(cell));
    lay[(size_t)layer * cells + cell] = phi;
    if (layer >= 1) itv[(size_t)(layer - 1) * cells + cell] = interval;
    ++rows;
  }
  if (rows != expected)
    throw ApiError(HWWG_EFORMAT, "reference shape mismatch: expected " +
                                     std::to_string(expected) + " rows, found " +
                                     std::to_string(rows));
  // outputs are written only after the whole file validated
  std::copy(lay.begin(), lay.end(), phi_layer);
  if (phi_interval) std::copy(itv.begin(), itv.end(), phi_interval);
}

void uniform_layers(double t_end, int steps, double* layers) {
  // TimeGrid::uniform(0, t_end, steps) (proj/include/hww/time_grid.hpp:22-30)
  const double dt = (t_end - 0.0) / steps;
  for (int n = 0; n <= steps; ++n) layers[n] = 0.0 + n * dt;
  layers[steps] = t_end;
}

}  // namespace hwwg

extern "C" {

int hwwg_step_metrics(int32_t cells, const double* edges, const double* phi_track,
                      const double* phi_sigma, const double* phi_hybrid,
                      const double* ref_interval, const double* ref_layer,
                      const double* ref_layer_prev, hwwg_step_record* rec) {
  HWWG_API_BEGIN
  if (!rec || !edges || cells <= 0) return hwwg::fail(HWWG_EINVAL, "NULL argument");
  if (ref_interval && (!phi_track || !ref_layer || !ref_layer_prev))
    return hwwg::fail(HWWG_EINVAL, "reference metrics need phi_track and both layers");
  if (rec->sigma_valid && !phi_sigma)
    return hwwg::fail(HWWG_EINVAL, "sigma_valid without phi_sigma");
  hwwg::step_metrics(cells, edges, phi_track, phi_sigma, phi_hybrid, ref_interval, ref_layer,
                     ref_layer_prev, rec);
  return HWWG_OK;
  HWWG_API_END
}

int hwwg_save_reference_csv(const char* path, int32_t cells, const double* edges,
                            int32_t steps, const double* layers, const double* phi_layer,
                            const double* phi_interval) {
  HWWG_API_BEGIN
  if (!path || !edges || !layers || !phi_layer || !phi_interval || cells <= 0 || steps < 1)
    return hwwg::fail(HWWG_EINVAL, "NULL argument");
  std::ofstream out(path);
  if (!out)
    return hwwg::fail(HWWG_EFORMAT,
                      std::string("cannot open reference file for writing: ") + path);
  out.precision(17);
  out << "t_layer, cell_index, x_center, phi_layer, phi_interval_avg\n";
  for (int n = 0; n <= steps; ++n) {
    for (int c = 0; c < cells; ++c) {
      out << layers[n] << ", " << c << ", " << 0.5 * (edges[c] + edges[c + 1]) << ", "
          << phi_layer[(size_t)n * cells + c] << ", ";
      if (n == 0)
        out << "nan";
      else
        out << phi_interval[(size_t)(n - 1) * cells + c];
      out << '\n';
    }
  }
  if (!out)
    return hwwg::fail(HWWG_EFORMAT, std::string("failed writing reference file: ") + path);
  return HWWG_OK;
  HWWG_API_END
}

int hwwg_load_reference_csv(const char* path, int32_t cells, const double* edges,
                            int32_t steps, const double* layers, double* phi_layer,
                            double* phi_interval) {
  HWWG_API_BEGIN
  if (!path || !edges || !layers || !phi_layer || cells <= 0 || steps < 1)
    return hwwg::fail(HWWG_EINVAL, "NULL argument");
  hwwg::load_reference(path, cells, edges, steps, layers, phi_layer, phi_interval);
  return HWWG_OK;
  HWWG_API_END
}

int hwwg_time_layers(const hwwg_run_config* cfg, double* layers) {
  HWWG_API_BEGIN
  if (!cfg || !layers || cfg->time_steps < 1) return hwwg::fail(HWWG_EINVAL, "NULL argument");
  hwwg::uniform_layers(cfg->t_end, cfg->time_steps, layers);
  return HWWG_OK;
  HWWG_API_END
}

}  // extern "C"
