"""TEST INFRASTRUCTURE — ctypes bindings for the checkers.

Two libraries share one C struct layout:
  * ``oracle/_build/libhww_oracle.so`` — the plain-C restatement (hww_oracle.c);
  * ``oracle/_ref/libhww_ref.so``      — the UNMODIFIED reference compiled from
    /root/reference/proj plus oracle/ref_shim.cpp (built only in the build
    container; the .so travels to the GPU box, /root/reference does not).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libhww_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhww_ref.so")
# the reference with its run_segment_parallel routed to the engine
DROPIN_SO = os.path.join(HERE, "_ref", "libhww_dropin.so")

PARTICLE_DT = np.dtype([("x", "<f8"), ("mu", "<f8"), ("w", "<f8"), ("t", "<f8")])
MODES = {"analog": 0, "lww": 1, "hww": 2, "hww_ma": 3, "hww_fourier": 4}


class Counters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "collisions", "splits", "split_daughters", "capped_splits", "roulette_kills",
        "roulette_survivals", "census_count", "event_cap_aborts", "nan_aborts")] + [
        ("leakage_weight", C.c_double), ("aborted_weight", C.c_double)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class Config(C.Structure):
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
        ("t_end", C.c_double), ("threads", C.c_int32), ("pad_", C.c_int32),
        # config-3 extensions (oracle only; the reference shim reads the prefix)
        ("n_regions", C.c_int32), ("no_pulse", C.c_int32), ("region_x_hi", C.c_double * 8),
        ("region_mat", (C.c_double * 5) * 8), ("vol_x_lo", C.c_double), ("vol_x_hi", C.c_double),
        ("vol_t_lo", C.c_double), ("vol_t_hi", C.c_double), ("vol_rate", C.c_double),
        ("vol_histories", C.c_uint64)]


class StepOut(C.Structure):
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
        ("pad_", C.c_int32)]


class Tallies(C.Structure):
    _fields_ = [(n, C.POINTER(C.c_double)) for n in (
        "track_flux", "track_flux_batch", "census_phi", "census_current", "census_closure",
        "census_weight_batch", "edge_current")] + [
        ("boundary_closure_left", C.c_double), ("boundary_closure_right", C.c_double),
        ("histories_scored", C.c_uint64), ("grazing_discarded", C.c_uint64)]


class Bank(C.Structure):
    _fields_ = [("data", C.c_void_p), ("n", C.c_uint64), ("cap", C.c_uint64)]


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


def _u64p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint64)) if a is not None else None


@dataclass
class TallyArrays:
    """Numpy mirror of hww::TallySet (proj/include/hww/tally.hpp:16-45)."""
    cells: int
    batches: int
    track_flux: np.ndarray = None
    track_flux_batch: np.ndarray = None
    census_phi: np.ndarray = None
    census_current: np.ndarray = None
    census_closure: np.ndarray = None
    census_weight_batch: np.ndarray = None
    edge_current: np.ndarray = None
    boundary_closure_left: float = 0.0
    boundary_closure_right: float = 0.0
    histories_scored: int = 0
    grazing_discarded: int = 0

    def __post_init__(self):
        I, B = self.cells, self.batches
        for n, s in (("track_flux", I), ("track_flux_batch", B * I), ("census_phi", I),
                     ("census_current", I), ("census_closure", I),
                     ("census_weight_batch", B), ("edge_current", I + 1)):
            if getattr(self, n) is None:
                setattr(self, n, np.zeros(s))

    def to_c(self):
        t = Tallies()
        for n in ("track_flux", "track_flux_batch", "census_phi", "census_current",
                  "census_closure", "census_weight_batch", "edge_current"):
            setattr(t, n, _dp(getattr(self, n)))
        t.boundary_closure_left = self.boundary_closure_left
        t.boundary_closure_right = self.boundary_closure_right
        t.histories_scored = self.histories_scored
        t.grazing_discarded = self.grazing_discarded
        return t

    def from_c(self, t):
        self.boundary_closure_left = t.boundary_closure_left
        self.boundary_closure_right = t.boundary_closure_right
        self.histories_scored = t.histories_scored
        self.grazing_discarded = t.grazing_discarded


def make_config(**kw) -> Config:
    """RunConfig defaults (proj/include/hww/config.hpp:33-66) overridden by kw."""
    d = dict(mode="hww", histories_per_step=10000, theta=0.5, rho=1.25, eps_min=1e-3, u_ww=3,
             update_fractions=(0.25, 0.5, 0.75), ma_base_k=3, fourier_cutoff=30, batches=20,
             seed=1, target_population=0, comb_overflow_factor=1.0, x0=0.0, t0=0.0,
             strength=1.0, sigma_t=1.0, sigma_s=1.0 / 3.0, sigma_f=1.0 / 3.0, nu_f=2.3,
             speed=1.0, x_min=-20.5, x_max=20.5, cells=201, t_end=20.0, time_steps=20,
             threads=0)
    d.update(kw)
    c = Config()
    for k, v in d.items():
        if k == "mode":
            c.mode = MODES[v] if isinstance(v, str) else int(v)
        elif k == "update_fractions":
            c.n_fractions = len(v)
            for i, f in enumerate(v):
                c.fractions[i] = f
        elif k == "regions":  # [(x_hi, (sigma_t, sigma_s, sigma_f, nu_f, speed)), ...]
            c.n_regions = len(v)
            for i, (xh, m) in enumerate(v):
                c.region_x_hi[i] = xh
                for j in range(5):
                    c.region_mat[i][j] = m[j]
        elif k == "vol":  # (x_lo, x_hi, t_lo, t_hi, rate, histories)
            (c.vol_x_lo, c.vol_x_hi, c.vol_t_lo, c.vol_t_hi, c.vol_rate,
             c.vol_histories) = v
        else:
            setattr(c, k, v)
    return c


class _Lib:
    prefix = ""

    def __init__(self, path, prefix):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle all ref`")
        self.lib = C.CDLL(path)
        self.prefix = prefix
        f = self.fn  # CDLL attribute access caches the function object
        f("driver_create").restype = C.c_void_p
        f("driver_create").argtypes = [C.POINTER(Config)]
        f("driver_destroy").argtypes = [C.c_void_p]
        f("driver_step").argtypes = [C.c_void_p, C.POINTER(StepOut)]
        f("driver_arrays").argtypes = [C.c_void_p] + [C.POINTER(C.c_double)] * 8 + [
            C.POINTER(C.c_uint64)]
        f("driver_bank").restype = C.c_uint64
        f("driver_bank").argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
        f("last_error").restype = C.c_char_p

    def fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def err(self):
        return self.fn("last_error")().decode()


class DriverRun:
    """Stepwise hww::run (proj/src/driver.cpp:286-342) on either checker."""

    def __init__(self, lib: _Lib, config: Config):
        self.lib = lib
        self.cfg = config
        self.h = lib.fn("driver_create")(C.byref(config))
        if not self.h:
            raise ValueError(lib.err())
        self.I = config.cells

    def step(self):
        out = StepOut()
        if self.lib.fn("driver_step")(self.h, C.byref(out)) != 0:
            raise RuntimeError(self.lib.err())
        I = self.I
        arr = {n: np.full(I, np.nan) for n in ("phi_track", "sigma", "phi_census",
                                                "current_census", "closure_census",
                                                "ww_centers", "phi_hybrid")}
        arr["edge_current"] = np.zeros(I + 1)
        tracks = np.zeros(I, np.uint64)
        self.lib.fn("driver_arrays")(self.h, _dp(arr["phi_track"]), _dp(arr["sigma"]),
                                     _dp(arr["phi_census"]), _dp(arr["current_census"]),
                                     _dp(arr["closure_census"]), _dp(arr["edge_current"]),
                                     _dp(arr["ww_centers"]), _dp(arr["phi_hybrid"]),
                                     _u64p(tracks))
        arr["tracks_per_cell"] = tracks
        return out, arr

    def load_reference(self, path):
        """hwwref_driver_load_reference: later steps run against the file (reference lib only)."""
        if self.lib.lib.hwwref_driver_load_reference(self.h, str(path).encode()) != 0:
            raise RuntimeError(self.lib.err())

    METRICS = ("rel_l2_error", "rel_mod_l2_error", "hybrid_rel_l2_error", "fom_err_l2",
               "fom_err_mod", "fom_sigma_l2", "fom_sigma_mod", "alpha", "tau")

    def metrics(self):
        """StepMetrics of the last step (reference lib only)."""
        v = np.zeros(9)
        self.lib.lib.hwwref_driver_metrics(self.h, _dp(v))
        return dict(zip(self.METRICS, v.tolist()))

    def bank(self):
        n = self.lib.fn("driver_bank")(self.h, None, 0)
        b = np.zeros(n, PARTICLE_DT)
        self.lib.fn("driver_bank")(self.h, b.ctypes.data, n)
        return b

    def close(self):
        if self.h:
            self.lib.fn("driver_destroy")(self.h)
            self.h = None

    def __del__(self):
        self.close()


class Oracle(_Lib):
    def __init__(self):
        super().__init__(ORACLE_SO, "orc_")
        L = self.lib
        L.orc_run_segment.argtypes = [
            C.POINTER(C.c_double), C.c_int32, C.c_void_p, C.c_double, C.c_double, C.c_uint64,
            C.c_int32, C.c_uint64, C.c_int32, C.c_void_p, C.c_uint64, C.c_uint64,
            C.POINTER(C.c_double), C.c_double, C.c_int32, C.POINTER(Tallies),
            C.POINTER(Counters), C.POINTER(C.c_uint64), C.POINTER(Bank),
            C.POINTER(C.c_uint32)]
        L.orc_bank_free.argtypes = [C.POINTER(Bank)]
        L.orc_stream_id.restype = C.c_uint64
        L.orc_stream_id.argtypes = [C.c_uint64] * 3
        L.orc_uniform_comb.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                       C.c_uint64, C.c_void_p, C.POINTER(C.c_double),
                                       C.POINTER(C.c_double)]

    def uniform_comb(self, bank, target, seed, stream_id):
        """orc_uniform_comb — popctrl.cpp:7-42. Returns (out, in_weight, out_weight)."""
        b = np.ascontiguousarray(bank, PARTICLE_DT)
        out = np.zeros(target, PARTICLE_DT)
        iw, ow = C.c_double(), C.c_double()
        if self.lib.orc_uniform_comb(b.ctypes.data, b.size, target, seed, stream_id,
                                     out.ctypes.data, C.byref(iw), C.byref(ow)) != 0:
            raise ValueError(self.err())
        return out, iw.value, ow.value

    def run_segment(self, edges, mats, t_begin, t_end, seed, step, histories_total, batches,
                    source, h_begin, centers=None, rho=1.25, chunk=256, tallies=None,
                    counters=None, tracks=None):
        """orc_run_segment — transport.cpp:194-237. Returns (tallies, counters, tracks,
        census, max_stack_runs)."""
        I = len(edges) - 1
        edges = np.ascontiguousarray(edges, np.float64)
        mats = np.ascontiguousarray(mats, np.float64).reshape(I, 5)
        src = np.ascontiguousarray(source, PARTICLE_DT)
        tallies = tallies or TallyArrays(I, batches)
        counters = counters or Counters()
        tracks = tracks if tracks is not None else np.zeros(I, np.uint64)
        tc = tallies.to_c()
        bank = Bank()
        mx = C.c_uint32(0)
        cen = np.ascontiguousarray(centers, np.float64) if centers is not None else None
        rc = self.lib.orc_run_segment(
            _dp(edges), I, mats.ctypes.data, t_begin, t_end, seed, step, histories_total,
            batches, src.ctypes.data, len(src), h_begin, _dp(cen), rho, chunk, C.byref(tc),
            C.byref(counters), _u64p(tracks), C.byref(bank), C.byref(mx))
        if rc != 0:
            self.lib.orc_bank_free(C.byref(bank))
            raise ValueError(self.err())
        tallies.from_c(tc)
        census = np.zeros(bank.n, PARTICLE_DT)
        if bank.n:
            C.memmove(census.ctypes.data, bank.data, bank.n * PARTICLE_DT.itemsize)
        self.lib.orc_bank_free(C.byref(bank))
        return tallies, counters, tracks, census, mx.value


class Reference(_Lib):
    def __init__(self, path=REF_SO):
        super().__init__(path, "hwwref_")
        L = self.lib
        L.hwwref_run_segment.argtypes = [
            C.POINTER(C.c_double), C.c_int32, C.c_void_p, C.c_double, C.c_double, C.c_uint64,
            C.c_int32, C.c_uint64, C.c_int32, C.c_void_p, C.c_uint64, C.c_uint64,
            C.POINTER(C.c_double), C.c_double, C.c_double, C.c_int32, C.c_int32,
            C.POINTER(Tallies), C.POINTER(Counters), C.POINTER(C.c_uint64)]
        L.hwwref_take_census.restype = C.c_uint64
        L.hwwref_take_census.argtypes = [C.c_void_p, C.c_uint64]
        L.hwwref_num_threads.restype = C.c_int
        L.hwwref_set_threads.argtypes = [C.c_int]
        L.hwwref_run_to_dir.argtypes = [C.POINTER(Config), C.c_char_p, C.c_char_p]
        L.hwwref_driver_load_reference.argtypes = [C.c_void_p, C.c_char_p]
        L.hwwref_driver_metrics.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
        L.hwwref_driver_metrics.restype = None
        dp = C.POINTER(C.c_double)
        L.hwwref_compute_reference.argtypes = [C.POINTER(Config), C.c_int32, C.c_int32,
                                               C.c_int32, dp, dp]
        L.hwwref_save_reference.argtypes = [C.POINTER(Config), C.c_char_p, dp, dp]
        L.hwwref_load_reference.argtypes = [C.POINTER(Config), C.c_char_p, dp, dp]
        L.hwwref_write_outputs.argtypes = [C.c_char_p, C.POINTER(Config), C.c_int32, C.c_int32] + [
            C.c_void_p] * 12 + [C.c_double]

    def run_to_dir(self, config: Config, out_dir, reference=None):
        """hww::run with out_dir: the reference's own output files (against the
        reference file `reference` when given, as hww_main runs it)."""
        ref = str(reference).encode() if reference else None
        if self.lib.hwwref_run_to_dir(C.byref(config), str(out_dir).encode(), ref) != 0:
            raise ValueError(self.err())

    def compute_reference(self, config: Config, space_refine=5, time_refine=20, sn_order=16):
        """hww::compute_reference (reference.cpp:364-372): (phi_layer, phi_interval)."""
        N, I = config.time_steps, config.cells
        lay, itv = np.zeros((N + 1, I)), np.zeros((N, I))
        if self.lib.hwwref_compute_reference(C.byref(config), space_refine, time_refine,
                                             sn_order, _dp(lay), _dp(itv)) != 0:
            raise RuntimeError(self.err())
        return lay, itv

    def gauss_legendre(self, n):
        mu, w = np.zeros(n), np.zeros(n)
        L = self.lib
        L.hwwref_gauss_legendre.argtypes = [C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        if L.hwwref_gauss_legendre(n, _dp(mu), _dp(w)) != 0:
            raise ValueError(self.err())
        return mu, w

    def sn_solve(self, edges, mats, layers, order, psi0, inc_left, inc_right, q,
                 tolerance=1e-9, max_iterations=1000):
        """hww::sn_solve (reference.cpp:151-233): (phi per layer, iterations per step)."""
        edges = np.ascontiguousarray(edges, np.float64)
        I = edges.size - 1
        mats = np.ascontiguousarray(mats, np.float64).reshape(I, 5)
        layers = np.ascontiguousarray(layers, np.float64)
        N = layers.size - 1
        arrs = [np.ascontiguousarray(a, np.float64) for a in (psi0, inc_left, inc_right, q)]
        phi, its = np.zeros((N + 1, I)), np.zeros(N + 1, np.int32)
        L = self.lib
        dp = C.POINTER(C.c_double)
        L.hwwref_sn_solve.argtypes = [C.c_int32, dp, C.c_void_p, C.c_int32, dp, C.c_int32, dp,
                                      dp, dp, dp, C.c_double, C.c_int32, dp, C.c_void_p]
        if L.hwwref_sn_solve(I, _dp(edges), mats.ctypes.data, N, _dp(layers), order,
                             *[_dp(a) for a in arrs], tolerance, max_iterations, _dp(phi),
                             its.ctypes.data) != 0:
            raise RuntimeError(self.err())
        return phi, its

    def save_reference(self, config: Config, path, phi_layer, phi_interval):
        lay = np.ascontiguousarray(phi_layer, np.float64)
        itv = np.ascontiguousarray(phi_interval, np.float64)
        if self.lib.hwwref_save_reference(C.byref(config), str(path).encode(), _dp(lay),
                                          _dp(itv)) != 0:
            raise RuntimeError(self.err())

    def load_reference(self, config: Config, path):
        N, I = config.time_steps, config.cells
        lay, itv = np.zeros((N + 1, I)), np.zeros((N, I))
        if self.lib.hwwref_load_reference(C.byref(config), str(path).encode(), _dp(lay),
                                          _dp(itv)) != 0:
            raise RuntimeError(self.err())
        return lay, itv

    def write_outputs(self, out_dir, config: Config, steps, total_seconds):
        """The reference writers on synthetic records. steps: list of dicts with
        arrays phi_track, sigma, phi_census, current, closure, centers (or None),
        hybrid (or None), tracks and scalars t_end, tau, fom_sigma_l2,
        census_weight, census_weight_sigma, normalization, sigma_valid,
        hybrid_solve_failed, step, histories, comb_in, comb_out,
        updates_applied, counters (Counters), and optionally metrics (7 values:
        rel_l2_error, rel_mod_l2_error, hybrid_rel_l2_error, fom_err_l2,
        fom_err_mod, fom_sigma_mod, alpha)."""
        n, I = len(steps), config.cells
        def stack(key, dt=np.float64):
            parts = [np.asarray(s[key] if s[key] is not None else np.zeros(I), dt) for s in steps]
            return np.ascontiguousarray(np.concatenate(parts) if parts else np.zeros(1, dt))
        arrs = [stack(k) for k in ("phi_track", "sigma", "phi_census", "current", "closure",
                                   "centers", "hybrid")]
        tracks = stack("tracks", np.uint64)
        sc = np.zeros((max(n, 1), 8)) if not n else np.array([[s[k] for k in ("t_end", "tau", "fom_sigma_l2", "census_weight",
                                       "census_weight_sigma", "normalization", "sigma_valid",
                                       "hybrid_solve_failed")] for s in steps], np.float64)
        ints = np.zeros((1, 6), np.uint64) if not n else np.array([[s["step"], s["histories"], s["comb_in"], s["comb_out"],
                          s["updates_applied"],
                          (1 if s["centers"] is not None else 0) |
                          (2 if s["hybrid"] is not None else 0)] for s in steps], np.uint64)
        cnt = (Counters * max(n, 1))(*[s["counters"] for s in steps])
        met = np.ascontiguousarray([s.get("metrics", (np.nan,) * 7) for s in steps] or
                                   [(np.nan,) * 7], np.float64)
        rc = self.lib.hwwref_write_outputs(
            str(out_dir).encode(), C.byref(config), n, I, *[a.ctypes.data for a in arrs],
            tracks.ctypes.data, sc.ctypes.data, ints.ctypes.data, C.addressof(cnt),
            met.ctypes.data, total_seconds)
        if rc != 0:
            raise ValueError(self.err())

    def run_segment(self, edges, mats, t_begin, t_end, seed, step, histories_total, batches,
                    source, h_begin, centers=None, rho=1.25, parallel=True, chunk=256,
                    tallies=None, counters=None, tracks=None):
        I = len(edges) - 1
        edges = np.ascontiguousarray(edges, np.float64)
        mats = np.ascontiguousarray(mats, np.float64).reshape(I, 5)
        src = np.ascontiguousarray(source, PARTICLE_DT)
        tallies = tallies or TallyArrays(I, batches)
        counters = counters or Counters()
        tracks = tracks if tracks is not None else np.zeros(I, np.uint64)
        tc = tallies.to_c()
        cen = np.ascontiguousarray(centers, np.float64) if centers is not None else None
        rc = self.lib.hwwref_run_segment(
            _dp(edges), I, mats.ctypes.data, t_begin, t_end, seed, step, histories_total,
            batches, src.ctypes.data, len(src), h_begin, _dp(cen), rho, 1e-3,
            1 if parallel else 0, chunk, C.byref(tc), C.byref(counters), _u64p(tracks))
        if rc != 0:
            raise ValueError(self.err())
        tallies.from_c(tc)
        n = self.lib.hwwref_take_census(None, 0)
        census = np.zeros(n, PARTICLE_DT)
        self.lib.hwwref_take_census(census.ctypes.data, n)
        return tallies, counters, tracks, census


def have_reference() -> bool:
    return os.path.exists(REF_SO)


def uniform_edges(x_min, x_max, cells):
    """build_uniform_mesh edges (proj/src/mesh.cpp:42-50)."""
    w = (x_max - x_min) / cells
    e = x_min + np.arange(cells + 1) * w
    e[-1] = x_max
    return e


def homogeneous(cells, sigma_t=1.0, sigma_s=0.0, sigma_f=0.0, nu_f=0.0, speed=1.0):
    return np.tile(np.array([sigma_t, sigma_s, sigma_f, nu_f, speed]), (cells, 1))


# BASELINE.json configs; reduced histories for CPU parity work.
def baseline_config(which: int, histories=None, time_steps=None, **kw) -> Config:
    if which == 1:
        base = dict(mode="hww_ma", ma_base_k=3, histories_per_step=100000, rho=5.0, seed=42,
                    sigma_t=1.0, sigma_s=1.0, sigma_f=0.0, nu_f=0.0, speed=1.0, x_min=-20.0,
                    x_max=20.0, cells=200, t_end=20.0, time_steps=20)
    elif which == 2:
        base = dict(mode="hww_ma", ma_base_k=1, histories_per_step=1000000, rho=5.0, seed=7,
                    sigma_t=1.0, sigma_s=0.9, sigma_f=0.0, nu_f=0.0, speed=1.0, x_min=-20.0,
                    x_max=20.0, cells=400, t_end=20.0, time_steps=40)
    elif which == 4:
        base = dict(mode="hww", histories_per_step=100000000, rho=1.25, seed=1, sigma_t=1.0,
                    sigma_s=0.99, sigma_f=0.0, nu_f=0.0, speed=1.0, x_min=-50.0, x_max=50.0,
                    cells=4000, t_end=50.0, time_steps=100)
    elif which == 5:
        base = dict(mode="hww_ma", ma_base_k=1, histories_per_step=10000000, rho=5.0, seed=11,
                    sigma_t=1.0, sigma_s=0.9, sigma_f=0.0, nu_f=0.0, speed=1.0, x_min=-20.0,
                    x_max=20.0, cells=400, t_end=20.0, time_steps=40)
    elif which == 0:  # the reference's own benchmark.cfg (proj/configs/benchmark.cfg)
        base = dict(mode="hww", histories_per_step=10000, ma_base_k=3, seed=1)
    else:
        raise ValueError(which)
    if histories is not None:
        base["histories_per_step"] = histories
    if time_steps is not None:
        dt = base.get("t_end", 20.0) / base.get("time_steps", 20)
        base["time_steps"] = time_steps
        base["t_end"] = dt * time_steps
    base.update(kw)
    return make_config(**base)
