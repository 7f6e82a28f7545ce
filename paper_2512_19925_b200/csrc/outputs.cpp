// Run output files in the reference's formats:
//   step_<n>.csv  — proj/src/driver.cpp:355-376 write_step_csv
//   summary.csv   — proj/src/driver.cpp:378-401 write_summary_csv
//   run.json      — proj/src/driver.cpp:403-438 write_run_json
// The CSVs go through std::ofstream with precision 17 exactly like the
// reference (open_out, driver.cpp:348-353), so equal records give equal bytes.
// run.json reproduces the layout of the reference's JSON library dump(2):
// object keys in lexicographic order, two-space indent, integers as integers,
// doubles in the shortest round-trip decimal laid out by that library's
// published format rule (see json_double), non-finite doubles as null.
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <limits>
#include <map>
#include <memory>
#include <string>
#include <system_error>
#include <vector>

#include "capi_util.h"
#include "hwwg.h"

namespace {

std::ofstream open_out(const char* dir, const std::string& name) {
  std::filesystem::create_directories(dir);
  std::ofstream out(std::filesystem::path(dir) / name);
  if (!out) throw hwwg::ApiError(HWWG_EINVAL, "cannot open output file: " + name);
  out.precision(17);
  return out;
}

// ---- minimal JSON value with the reference's dump(2) layout ----------------
struct JVal {
  enum Kind { kInt, kUint, kFloat, kString, kArray, kObject } kind = kObject;
  long long i = 0;
  unsigned long long u = 0;
  double f = 0.0;
  std::string s;
  std::vector<JVal> arr;
  std::map<std::string, JVal> obj;  // sorted keys, as the library's default object
  static JVal I(long long v) { JVal j; j.kind = kInt; j.i = v; return j; }
  static JVal U(unsigned long long v) { JVal j; j.kind = kUint; j.u = v; return j; }
  static JVal F(double v) { JVal j; j.kind = kFloat; j.f = v; return j; }
  static JVal S(std::string v) { JVal j; j.kind = kString; j.s = std::move(v); return j; }
  static JVal A(std::vector<JVal> v) { JVal j; j.kind = kArray; j.arr = std::move(v); return j; }
  static JVal O() { return JVal(); }
};

// Shortest round-trip digits (std::to_chars) placed by the rule: with k digits
// and decimal point position n (value = 0.d1..dk * 10^n):
//   k <= n <= 15   -> digits, zeros up to n, ".0"
//   0 < n <= 15    -> digits with the point after n
//   -4 < n <= 0    -> "0." zeros digits
//   otherwise      -> d[.ddd]e{+|-}XX (at least two exponent digits)
std::string json_double(double v) {
  if (!std::isfinite(v)) return "null";
  std::string out;
  if (std::signbit(v)) {
    out += '-';
    v = -v;
  }
  if (v == 0.0) return out + "0.0";
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::scientific);
  // buf = d[.ddd]e[+-]XX
  std::string sci(buf, r.ptr);
  const size_t epos = sci.find('e');
  std::string digits = sci.substr(0, 1) + (epos > 2 ? sci.substr(2, epos - 2) : "");
  const int e10 = std::stoi(sci.substr(epos + 1));
  const int k = (int)digits.size();
  const int n = e10 + 1;
  if (k <= n && n <= 15) return out + digits + std::string(n - k, '0') + ".0";
  if (0 < n && n <= 15) return out + digits.substr(0, n) + "." + digits.substr(n);
  if (-4 < n && n <= 0) return out + "0." + std::string(-n, '0') + digits;
  std::string m = k == 1 ? digits : digits.substr(0, 1) + "." + digits.substr(1);
  const int ex = n - 1;
  char eb[16];
  std::snprintf(eb, sizeof eb, "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
  return out + m + eb;
}

std::string json_string(const std::string& s) {
  std::string o = "\"";
  for (unsigned char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (c < 0x20) {
          char b[8];
          std::snprintf(b, sizeof b, "\\u%04x", c);
          o += b;
        } else {
          o += (char)c;
        }
    }
  }
  return o + "\"";
}

void dump(const JVal& j, std::string& o, int indent) {
  const std::string pad((size_t)indent + 2, ' '), end_pad((size_t)indent, ' ');
  switch (j.kind) {
    case JVal::kInt: o += std::to_string(j.i); break;
    case JVal::kUint: o += std::to_string(j.u); break;
    case JVal::kFloat: o += json_double(j.f); break;
    case JVal::kString: o += json_string(j.s); break;
    case JVal::kArray:
      if (j.arr.empty()) {
        o += "[]";
        break;
      }
      o += "[\n";
      for (size_t i = 0; i < j.arr.size(); ++i) {
        o += pad;
        dump(j.arr[i], o, indent + 2);
        o += i + 1 < j.arr.size() ? ",\n" : "\n";
      }
      o += end_pad + "]";
      break;
    case JVal::kObject:
      if (j.obj.empty()) {
        o += "{}";
        break;
      }
      o += "{\n";
      size_t n = 0;
      for (const auto& kv : j.obj) {
        o += pad + json_string(kv.first) + ": ";
        dump(kv.second, o, indent + 2);
        o += ++n < j.obj.size() ? ",\n" : "\n";
      }
      o += end_pad + "}";
      break;
  }
}

const char* mode_name(int m) {  // config.cpp:7-16 to_string(Mode)
  switch (m) {
    case 0: return "analog";
    case 1: return "lww";
    case 2: return "hww";
    case 3: return "hww_ma";
    case 4: return "hww_fourier";
  }
  return "?";
}

}  // namespace

extern "C" {

int hwwg_write_step_csv(const char* dir, const hwwg_step_record* rec, int32_t cells,
                        const double* edges, const double* phi_track, const double* sigma,
                        const double* phi_census, const double* current, const double* closure,
                        const double* ww_centers, const double* phi_hybrid,
                        const uint64_t* tracks, double normalization) {
  HWWG_API_BEGIN
  if (!dir || !rec || !edges || !phi_track || !phi_census || !current || !closure || !tracks ||
      cells <= 0 || (rec->sigma_valid && !sigma))
    return hwwg::fail(HWWG_EINVAL, "NULL argument");
  auto out = open_out(dir, "step_" + std::to_string(rec->step) + ".csv");
  out << "cell, x_center, phi_track, sigma, phi_census, J_census, F_census, "
         "ww_center, phi_hlosm, tracks_per_source\n";
  const double nan = std::numeric_limits<double>::quiet_NaN();
  const double inv_h = 1.0 / normalization;
  for (int i = 0; i < cells; ++i) {
    out << i << ", " << 0.5 * (edges[i] + edges[i + 1]) << ", " << phi_track[i] << ", "
        << (rec->sigma_valid ? sigma[i] : nan) << ", " << phi_census[i] << ", " << current[i]
        << ", " << closure[i] << ", " << (ww_centers ? ww_centers[i] : nan) << ", "
        << (phi_hybrid ? phi_hybrid[i] : nan) << ", " << static_cast<double>(tracks[i]) * inv_h
        << '\n';
  }
  if (!out) return hwwg::fail(HWWG_EINVAL, "write failed");
  return HWWG_OK;
  HWWG_API_END
}

int hwwg_write_summary_csv(const char* dir, const hwwg_step_record* recs, uint64_t n) {
  HWWG_API_BEGIN
  if (!dir || (n && !recs)) return hwwg::fail(HWWG_EINVAL, "NULL argument");
  auto out = open_out(dir, "summary.csv");
  out << "step, t_end, histories, tau_seconds, rel_l2_error, rel_mod_l2_error, "
         "hybrid_rel_l2_error, fom_err_l2, fom_err_mod, fom_sigma_l2, "
         "fom_sigma_mod, alpha, census_weight, census_weight_sigma, "
         "comb_in_count, comb_out_count, leakage_weight, collisions, splits, "
         "split_daughters, roulette_kills, roulette_survivals, census_count, "
         "event_cap_aborts, aborted_weight, updates_applied, "
         "hybrid_solve_failed\n";
  // the metric fields are NaN unless the step ran against a reference
  // (metrics.hpp:41-51; driver.cpp:231-275)
  for (uint64_t k = 0; k < n; ++k) {
    const hwwg_step_record& s = recs[k];
    const hwwg_counters& c = s.counters;
    out << s.step << ", " << s.t_end << ", " << s.histories << ", " << s.tau << ", "
        << s.rel_l2_error << ", " << s.rel_mod_l2_error << ", " << s.hybrid_rel_l2_error
        << ", " << s.fom_err_l2 << ", " << s.fom_err_mod << ", " << s.fom_sigma_l2 << ", "
        << s.fom_sigma_mod << ", " << s.alpha << ", " << s.census_weight << ", "
        << s.census_weight_sigma << ", " << s.comb_in << ", " << s.comb_out << ", "
        << c.leakage_weight << ", " << c.collisions << ", " << c.splits << ", "
        << c.split_daughters << ", " << c.roulette_kills << ", " << c.roulette_survivals
        << ", " << c.census_count << ", " << c.event_cap_aborts << ", " << c.aborted_weight
        << ", " << s.updates_applied << ", " << (s.hybrid_solve_failed ? 1 : 0) << '\n';
  }
  if (!out) return hwwg::fail(HWWG_EINVAL, "write failed");
  return HWWG_OK;
  HWWG_API_END
}

int hwwg_write_run_json(const char* dir, const hwwg_run_config* c, double total_seconds,
                        uint64_t steps_completed) {
  HWWG_API_BEGIN
  if (!dir || !c) return hwwg::fail(HWWG_EINVAL, "NULL argument");
  JVal cfg = JVal::O();
  cfg.obj["mode"] = JVal::S(mode_name(c->mode));
  cfg.obj["histories_per_step"] = JVal::U(c->histories_per_step);
  cfg.obj["theta"] = JVal::F(c->theta);
  cfg.obj["rho"] = JVal::F(c->rho);
  cfg.obj["eps_min"] = JVal::F(c->eps_min);
  cfg.obj["u_ww"] = JVal::I(c->u_ww);
  std::vector<JVal> fr;
  for (int i = 0; i < c->n_fractions && i < 8; ++i) fr.push_back(JVal::F(c->fractions[i]));
  cfg.obj["update_fractions"] = JVal::A(fr);
  cfg.obj["ma_base_k"] = JVal::I(c->ma_base_k);
  cfg.obj["fourier_cutoff"] = JVal::I(c->fourier_cutoff);
  cfg.obj["batches"] = JVal::I(c->batches);
  cfg.obj["seed"] = JVal::U(c->seed);
  cfg.obj["target_population"] =
      JVal::U(c->target_population ? c->target_population : c->histories_per_step);
  JVal src = JVal::O();
  src.obj["x0"] = JVal::F(c->x0);
  src.obj["t0"] = JVal::F(c->t0);
  src.obj["strength"] = JVal::F(c->strength);
  cfg.obj["source"] = src;
  JVal mat = JVal::O();
  mat.obj["sigma_t"] = JVal::F(c->sigma_t);
  mat.obj["sigma_s"] = JVal::F(c->sigma_s);
  mat.obj["sigma_f"] = JVal::F(c->sigma_f);
  mat.obj["nu_f"] = JVal::F(c->nu_f);
  mat.obj["speed"] = JVal::F(c->speed);
  cfg.obj["material"] = mat;
  JVal mesh = JVal::O();
  mesh.obj["x_min"] = JVal::F(c->x_min);
  mesh.obj["x_max"] = JVal::F(c->x_max);
  mesh.obj["cells"] = JVal::I(c->cells);
  cfg.obj["mesh"] = mesh;
  JVal tm = JVal::O();
  tm.obj["t_end"] = JVal::F(c->t_end);
  tm.obj["steps"] = JVal::I(c->time_steps);
  cfg.obj["time"] = tm;
  cfg.obj["reference"] = JVal::S(std::string(c->reference, strnlen(c->reference, sizeof c->reference)));
  cfg.obj["threads"] = JVal::I(c->threads);
  JVal root = JVal::O();
  root.obj["config"] = cfg;
  root.obj["total_seconds"] = JVal::F(total_seconds);
  root.obj["steps_completed"] = JVal::U(steps_completed);
  root.obj["tau_includes"] = JVal::S("comb, transport, window updates, low-order solves, tally finalize");
  std::string o;
  dump(root, o, 0);
  auto out = open_out(dir, "run.json");
  out << o << '\n';
  if (!out) return hwwg::fail(HWWG_EINVAL, "write failed");
  return HWWG_OK;
  HWWG_API_END
}

}  // extern "C"
