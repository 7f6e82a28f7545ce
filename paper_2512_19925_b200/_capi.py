"""ctypes binding of the C ABI in include/hwwg.h (libhwwg.so, built in-tree).

The product path has no CPU fallback: if the library is missing or no CUDA
device is visible, every call fails loudly (HwwgError / OSError).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
# HWWG_LIB: an alternative build of the same library (tests: the bounds-checked
# variant in _build_checked/, built by __graft_entry__.build())
LIB_PATH = os.environ.get("HWWG_LIB") or os.path.join(PKG, "_build", "libhwwg.so")

HWWG_OK = 0
HWWG_EINVAL = -1
HWWG_ECUDA = -2
HWWG_ENOMEM = -3
HWWG_ESTATE = -4
HWWG_ESINGULAR = -5
HWWG_ENOSPC = -6
HWWG_ESTACK = -7
HWWG_EFORMAT = -8
RNG_EXACT = 0
RNG_PHILOX = 1

PARTICLE_DT = np.dtype([("x", "<f8"), ("mu", "<f8"), ("w", "<f8"), ("t", "<f8")])
MATERIAL_DT = np.dtype([("sigma_t", "<f8"), ("sigma_s", "<f8"), ("sigma_f", "<f8"),
                        ("nu_f", "<f8"), ("speed", "<f8")])

COUNTER_FIELDS = ("collisions", "splits", "split_daughters", "capped_splits", "roulette_kills",
                  "roulette_survivals", "census_count", "event_cap_aborts", "nan_aborts")


class HwwgError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"hwwg error {code}: {msg}")
        self.code = code


class Counters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in COUNTER_FIELDS] + [
        ("leakage_weight", C.c_double), ("aborted_weight", C.c_double)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class StepContextC(C.Structure):
    _fields_ = [("edges", C.POINTER(C.c_double)), ("cells", C.c_int32), ("batches", C.c_int32),
                ("materials", C.c_void_p), ("t_begin", C.c_double), ("t_end", C.c_double),
                ("seed", C.c_uint64), ("step_index", C.c_int32), ("pad_", C.c_int32),
                ("histories_total", C.c_uint64)]


class WindowGridC(C.Structure):
    _fields_ = [("centers", C.POINTER(C.c_double)), ("rho", C.c_double), ("eps_min", C.c_double)]


class TallySetC(C.Structure):
    _fields_ = [(n, C.POINTER(C.c_double)) for n in (
        "track_flux", "track_flux_batch", "census_phi", "census_current", "census_closure",
        "census_weight_batch", "edge_current")] + [
        ("boundary_closure_left", C.c_double), ("boundary_closure_right", C.c_double),
        ("histories_scored", C.c_uint64), ("grazing_discarded", C.c_uint64)]


class StepOutcomeC(C.Structure):
    _fields_ = [("census", C.c_void_p), ("census_size", C.c_uint64),
                ("census_capacity", C.c_uint64), ("census_needed", C.c_uint64),
                ("counters", Counters), ("tracks_per_cell", C.POINTER(C.c_uint64))]


class Options(C.Structure):
    _fields_ = [("device", C.c_int32), ("rng_mode", C.c_int32), ("bank_capacity", C.c_uint64),
                ("rank", C.c_int32), ("world", C.c_int32), ("nccl_id", C.c_uint8 * 128),
                ("loopback", C.c_void_p)]


class RunConfigC(C.Structure):
    _fields_ = [
        ("mode", C.c_int32), ("u_ww", C.c_int32), ("histories_per_step", C.c_uint64),
        ("theta", C.c_double), ("rho", C.c_double), ("eps_min", C.c_double),
        ("n_fractions", C.c_int32), ("ma_base_k", C.c_int32), ("fractions", C.c_double * 8),
        ("fourier_cutoff", C.c_int32), ("batches", C.c_int32), ("seed", C.c_uint64),
        ("target_population", C.c_uint64), ("comb_overflow_factor", C.c_double),
        ("x0", C.c_double), ("t0", C.c_double), ("strength", C.c_double),
        ("sigma_t", C.c_double), ("sigma_s", C.c_double), ("sigma_f", C.c_double),
        ("nu_f", C.c_double), ("speed", C.c_double), ("x_min", C.c_double),
        ("x_max", C.c_double), ("cells", C.c_int32), ("time_steps", C.c_int32),
        ("t_end", C.c_double), ("threads", C.c_int32), ("host_bank", C.c_int32),
        ("n_regions", C.c_int32), ("no_pulse", C.c_int32), ("region_x_hi", C.c_double * 8),
        ("region_mat", (C.c_double * 5) * 8), ("vol_x_lo", C.c_double), ("vol_x_hi", C.c_double),
        ("vol_t_lo", C.c_double), ("vol_t_hi", C.c_double), ("vol_rate", C.c_double),
        ("vol_histories", C.c_uint64), ("reference", C.c_char * 256)]


class StepRecordC(C.Structure):
    _fields_ = [
        ("step", C.c_int32), ("updates_applied", C.c_int32),
        ("hybrid_solve_failed", C.c_int32), ("n_thresholds", C.c_int32),
        ("thresholds", C.c_uint64 * 8), ("t_begin", C.c_double), ("t_end", C.c_double),
        ("tau", C.c_double), ("histories", C.c_uint64), ("comb_in", C.c_uint64),
        ("comb_out", C.c_uint64), ("comb_in_weight", C.c_double),
        ("comb_out_weight", C.c_double), ("counters", Counters), ("segments", C.c_uint64),
        ("census_size", C.c_uint64), ("census_weight", C.c_double),
        ("census_weight_sigma", C.c_double), ("boundary_closure_left", C.c_double),
        ("boundary_closure_right", C.c_double), ("fom_sigma_l2", C.c_double),
        ("sigma_valid", C.c_int32), ("has_windows", C.c_int32), ("has_hybrid", C.c_int32),
        ("thinned", C.c_int32), ("device_ms", C.c_double), ("transport_ms", C.c_double),
        ("transport_launches", C.c_uint64), ("kernel_launches", C.c_uint64),
        ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
        ("rel_l2_error", C.c_double), ("rel_mod_l2_error", C.c_double),
        ("hybrid_rel_l2_error", C.c_double), ("fom_err_l2", C.c_double),
        ("fom_err_mod", C.c_double), ("fom_sigma_mod", C.c_double), ("alpha", C.c_double)]

    METRICS = ("rel_l2_error", "rel_mod_l2_error", "hybrid_rel_l2_error", "fom_err_l2",
               "fom_err_mod", "fom_sigma_l2", "fom_sigma_mod", "alpha")

    def __init__(self, *a, **kw):
        super().__init__(*a, **kw)
        for k in self.METRICS:  # StepMetrics' NaN defaults (metrics.hpp:41-51)
            if k not in kw:
                setattr(self, k, float("nan"))


# Every symbol include/hwwg.h declares (tests check the library exports them).
EXPORTS = (
    "hwwg_last_error", "hwwg_version", "hwwg_create", "hwwg_destroy",
    "hwwg_run_segment_parallel", "hwwg_driver_create", "hwwg_driver_destroy",
    "hwwg_driver_step", "hwwg_driver_arrays", "hwwg_driver_bank", "hwwg_load_config_file",
    "hwwg_default_config", "hwwg_validate_config", "hwwg_losm_assemble_solve",
    "hwwg_build_centers", "hwwg_moving_average", "hwwg_uniform_comb", "hwwg_device_log",
    "hwwg_nccl_unique_id", "hwwg_nccl_selftest", "hwwg_shard_range", "hwwg_comb_plan", "hwwg_rebalance_plan",
    "hwwg_fourier_lowpass", "hwwg_write_step_csv", "hwwg_write_summary_csv", "hwwg_write_run_json", "hwwg_driver_write",
    "hwwg_loopback_create", "hwwg_loopback_destroy", "hwwg_driver_set_reference",
    "hwwg_driver_load_reference", "hwwg_save_reference_csv", "hwwg_load_reference_csv",
    "hwwg_time_layers", "hwwg_step_metrics", "hwwg_gauss_legendre", "hwwg_sn_solve",
    "hwwg_compute_reference", "hwwg_driver_compute_reference")

_lib = None

dptr = C.POINTER(C.c_double)
u64ptr = C.POINTER(C.c_uint64)


def lib():
    """Load libhwwg.so once; raise if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise OSError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`"
                      " or `make -C paper_2512_19925_b200`")
    L = C.CDLL(LIB_PATH)
    L.hwwg_last_error.restype = C.c_char_p
    L.hwwg_version.restype = C.c_char_p
    L.hwwg_create.argtypes = [C.POINTER(Options), C.POINTER(C.c_void_p)]
    L.hwwg_destroy.argtypes = [C.c_void_p]
    L.hwwg_run_segment_parallel.argtypes = [
        C.c_void_p, C.POINTER(StepContextC), C.c_void_p, C.c_uint64, C.c_uint64,
        C.POINTER(WindowGridC), C.POINTER(TallySetC), C.POINTER(StepOutcomeC)]
    L.hwwg_driver_create.argtypes = [C.POINTER(RunConfigC), C.POINTER(Options),
                                     C.POINTER(C.c_void_p)]
    L.hwwg_driver_destroy.argtypes = [C.c_void_p]
    L.hwwg_driver_step.argtypes = [C.c_void_p, C.POINTER(StepRecordC)]
    L.hwwg_driver_arrays.argtypes = [C.c_void_p] + [dptr] * 8 + [u64ptr]
    L.hwwg_driver_bank.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, u64ptr]
    L.hwwg_load_config_file.argtypes = [C.c_char_p, C.POINTER(RunConfigC)]
    L.hwwg_default_config.argtypes = [C.POINTER(RunConfigC)]
    L.hwwg_default_config.restype = None
    L.hwwg_validate_config.argtypes = [C.POINTER(RunConfigC), C.c_char_p, C.c_uint64]
    L.hwwg_losm_assemble_solve.argtypes = [
        C.c_void_p, C.c_int32, dptr, C.c_void_p, dptr, dptr, C.c_double, C.c_double, C.c_int32,
        dptr, C.c_double, C.c_double, dptr, C.c_double, C.c_double, C.c_double, C.c_double,
        dptr, dptr, dptr]
    L.hwwg_build_centers.argtypes = [C.c_void_p, dptr, C.c_int32, C.c_double, C.c_double, dptr]
    L.hwwg_moving_average.argtypes = [C.c_void_p, dptr, C.c_int32, C.c_int32, dptr]
    L.hwwg_fourier_lowpass.argtypes = [C.c_void_p, dptr, C.c_int32, C.c_int32, dptr]
    L.hwwg_uniform_comb.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                    C.c_uint64, C.c_void_p, dptr, dptr]
    L.hwwg_device_log.argtypes = [C.c_void_p, dptr, C.c_uint64, dptr]
    L.hwwg_nccl_unique_id.argtypes = [C.c_void_p]
    L.hwwg_nccl_selftest.argtypes = [C.c_int32, C.c_void_p, C.c_uint64]
    L.hwwg_loopback_create.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]
    L.hwwg_loopback_destroy.argtypes = [C.c_void_p]
    L.hwwg_loopback_destroy.restype = None
    L.hwwg_shard_range.argtypes = [C.c_uint64, C.c_int32, C.c_int32, u64ptr, u64ptr]
    L.hwwg_shard_range.restype = None
    L.hwwg_comb_plan.argtypes = [dptr, C.c_int32, C.c_int32, C.c_uint64, C.c_double, dptr, dptr,
                                 dptr, u64ptr, u64ptr]
    L.hwwg_rebalance_plan.argtypes = [u64ptr, u64ptr, C.c_int32, C.c_int32, C.c_uint64, u64ptr,
                                      u64ptr, u64ptr]
    L.hwwg_rebalance_plan.restype = None
    L.hwwg_write_step_csv.argtypes = [C.c_char_p, C.POINTER(StepRecordC), C.c_int32, dptr, dptr,
                                      dptr, dptr, dptr, dptr, dptr, dptr, u64ptr, C.c_double]
    L.hwwg_write_summary_csv.argtypes = [C.c_char_p, C.POINTER(StepRecordC), C.c_uint64]
    L.hwwg_write_run_json.argtypes = [C.c_char_p, C.POINTER(RunConfigC), C.c_double, C.c_uint64]
    L.hwwg_driver_write.argtypes = [C.c_void_p, C.c_char_p, C.c_int32, C.c_double]
    L.hwwg_driver_set_reference.argtypes = [C.c_void_p, dptr, dptr, C.c_char_p]
    L.hwwg_driver_load_reference.argtypes = [C.c_void_p, C.c_char_p]
    L.hwwg_save_reference_csv.argtypes = [C.c_char_p, C.c_int32, dptr, C.c_int32, dptr, dptr, dptr]
    L.hwwg_load_reference_csv.argtypes = [C.c_char_p, C.c_int32, dptr, C.c_int32, dptr, dptr, dptr]
    L.hwwg_time_layers.argtypes = [C.POINTER(RunConfigC), dptr]
    L.hwwg_gauss_legendre.argtypes = [C.c_int32, dptr, dptr]
    L.hwwg_sn_solve.argtypes = [C.c_void_p, C.c_int32, dptr, C.c_void_p, C.c_int32, dptr,
                                C.c_int32, dptr, dptr, dptr, dptr, C.c_double, C.c_int32, dptr,
                                C.c_void_p]
    L.hwwg_compute_reference.argtypes = [C.c_void_p, C.POINTER(RunConfigC), C.c_int32,
                                         C.c_int32, C.c_int32, dptr, dptr]
    L.hwwg_driver_compute_reference.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32]
    L.hwwg_step_metrics.argtypes = [C.c_int32, dptr, dptr, dptr, dptr, dptr, dptr, dptr,
                                    C.POINTER(StepRecordC)]
    _lib = L
    return L


def check(rc):
    if rc < 0:
        raise HwwgError(rc, lib().hwwg_last_error().decode())
    return rc


def as_dptr(a):
    return a.ctypes.data_as(dptr) if a is not None else None


def as_u64ptr(a):
    return a.ctypes.data_as(u64ptr) if a is not None else None
