"""Python mirror of the reference's public API for the history-loop path.

Same names, argument meaning and error behaviour as the reference's C++
(proj/include/hww/*.hpp), executed by the sm_100a engine through the C ABI:

* ``run_segment_parallel(ctx, source, h_begin, ww, tallies, outcome)`` —
  transport.hpp:117-120; accumulates into ``tallies``/``outcome``; raises
  ``ValueError`` where the reference throws ``std::invalid_argument``.
* ``RunConfig`` / ``Driver`` / ``run`` — config.hpp:33-66, driver.hpp:80-88.
* ``assemble_solve``, ``build_centers``, ``moving_average``, ``uniform_comb`` —
  losm.hpp:77-80, ww.hpp:34-35, filters.hpp:30, popctrl.hpp:22.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _capi as A
from ._capi import PARTICLE_DT, RNG_EXACT, RNG_PHILOX, HwwgError

MODES = ("analog", "lww", "hww", "hww_ma", "hww_fourier")


def _raise(rc):
    if rc < 0:
        msg = A.lib().hwwg_last_error().decode()
        if rc == A.HWWG_EINVAL:  # std::invalid_argument
            raise ValueError(msg)
        # HWWG_ESINGULAR / HWWG_EFORMAT: the reference's std::runtime_error
        raise HwwgError(rc, msg)
    return rc


# ------------------------------------------------------------------ core types
@dataclass
class Material:
    """hww::Material (material.hpp:9-18)."""
    sigma_t: float = 1.0
    sigma_s: float = 0.0
    sigma_f: float = 0.0
    nu_f: float = 0.0
    speed: float = 1.0

    def removal(self):
        return self.sigma_t - self.sigma_s - self.nu_f * self.sigma_f


class Mesh1D:
    """hww::Mesh1D (mesh.hpp:12-58): strictly increasing edges."""

    def __init__(self, edges):
        e = np.ascontiguousarray(edges, np.float64)
        if e.size < 2:
            raise ValueError("mesh needs at least one cell")
        if not np.all(e[1:] > e[:-1]):
            raise ValueError("mesh edges must be strictly increasing")
        self.edges = e

    @staticmethod
    def from_edges(edges):
        return Mesh1D(edges)

    def cells(self):
        return self.edges.size - 1

    def width(self, c):
        return self.edges[c + 1] - self.edges[c]

    def center(self, c):
        return 0.5 * (self.edges[c] + self.edges[c + 1])


def build_uniform_mesh(x_min, x_max, cells):
    """mesh.cpp:42-50."""
    if cells < 1:
        raise ValueError("cell count must be positive")
    if not x_min < x_max:
        raise ValueError("x_min must be < x_max")
    w = (x_max - x_min) / cells
    e = x_min + np.arange(cells + 1) * w
    e[-1] = x_max
    return Mesh1D(e)


def _materials_array(materials, cells):
    if isinstance(materials, Material):
        materials = [materials] * cells
    if isinstance(materials, np.ndarray) and materials.dtype == A.MATERIAL_DT:
        arr = np.ascontiguousarray(materials)
    else:
        rows = []
        for m in materials:
            if isinstance(m, Material):
                rows.append((m.sigma_t, m.sigma_s, m.sigma_f, m.nu_f, m.speed))
            else:
                rows.append(tuple(float(v) for v in m))
        arr = np.array(rows, dtype=A.MATERIAL_DT)
    if arr.size != cells:
        raise ValueError("materials must have one entry per cell")
    return arr


@dataclass
class StepContext:
    """hww::StepContext (transport.hpp:83-94)."""
    mesh: Mesh1D
    materials: object
    t_begin: float = 0.0
    t_end: float = 1.0
    seed: int = 0
    step_index: int = 1
    histories_total: int = 0
    batches: int = 1

    def dt(self):
        return self.t_end - self.t_begin


@dataclass
class WeightWindowGrid:
    """hww::WeightWindowGrid (ww.hpp:13-27)."""
    centers: np.ndarray
    rho: float = 1.25
    eps_min: float = 1e-3
    uniform_fallback: bool = False

    def window(self, cell):
        c = self.centers[cell]
        return (c / self.rho, c, c * self.rho)


class TallySet:
    """hww::TallySet (tally.hpp:16-45) as numpy arrays; the engine accumulates."""

    def __init__(self, cells, batches):
        self.cells, self.batches = cells, batches
        self.track_flux = np.zeros(cells)
        self.track_flux_batch = np.zeros(batches * cells)
        self.census_phi = np.zeros(cells)
        self.census_current = np.zeros(cells)
        self.census_closure = np.zeros(cells)
        self.census_weight_batch = np.zeros(batches)
        self.edge_current = np.zeros(cells + 1)
        self.boundary_closure_left = 0.0
        self.boundary_closure_right = 0.0
        self.histories_scored = 0
        self.grazing_discarded = 0

    def _to_c(self):
        t = A.TallySetC()
        for n in ("track_flux", "track_flux_batch", "census_phi", "census_current",
                  "census_closure", "census_weight_batch", "edge_current"):
            setattr(t, n, A.as_dptr(getattr(self, n)))
        t.boundary_closure_left = self.boundary_closure_left
        t.boundary_closure_right = self.boundary_closure_right
        t.histories_scored = self.histories_scored
        t.grazing_discarded = self.grazing_discarded
        return t

    def _from_c(self, t):
        self.boundary_closure_left = t.boundary_closure_left
        self.boundary_closure_right = t.boundary_closure_right
        self.histories_scored = t.histories_scored
        self.grazing_discarded = t.grazing_discarded


class StepOutcome:
    """hww::StepOutcome (transport.hpp:67-80)."""

    def __init__(self, cells=0):
        self.census = np.zeros(0, PARTICLE_DT)
        self.counters = A.Counters()
        self.tracks_per_cell = np.zeros(cells, np.uint64)


# ------------------------------------------------------------------- engine
class Engine:
    """A device context (hwwg_ctx) on one GPU."""

    def __init__(self, device=0, rng_mode=RNG_EXACT, bank_capacity=0):
        L = A.lib()
        self._h = C.c_void_p()
        opts = A.Options(device, rng_mode, bank_capacity)
        _raise(L.hwwg_create(C.byref(opts), C.byref(self._h)))
        self.device, self.rng_mode = device, rng_mode

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            A.lib().hwwg_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # transport.hpp:117-120
    def run_segment_parallel(self, ctx: StepContext, source, h_begin: int,
                             ww: Optional[WeightWindowGrid], tallies: TallySet,
                             outcome: StepOutcome):
        L = A.lib()
        mesh = ctx.mesh
        I = mesh.cells()
        mats = _materials_array(ctx.materials, I)
        src = np.ascontiguousarray(source, PARTICLE_DT)
        sc = A.StepContextC()
        sc.edges = A.as_dptr(mesh.edges)
        sc.cells = I
        sc.batches = ctx.batches
        sc.materials = mats.ctypes.data
        sc.t_begin, sc.t_end = ctx.t_begin, ctx.t_end
        sc.seed = ctx.seed
        sc.step_index = ctx.step_index
        sc.histories_total = ctx.histories_total
        wg = None
        if ww is not None:
            cen = np.ascontiguousarray(ww.centers, np.float64)
            if cen.size != I:
                raise ValueError("window centers must have one value per cell")
            wg = A.WindowGridC(A.as_dptr(cen), ww.rho, ww.eps_min)
        tc = tallies._to_c()
        if outcome.tracks_per_cell.size != I:
            outcome.tracks_per_cell = np.zeros(I, np.uint64)
        base = outcome.census.size
        cap = max(base + 2 * src.size + 1024, base)
        buf = np.zeros(cap, PARTICLE_DT)
        buf[:base] = outcome.census
        oc = A.StepOutcomeC()
        oc.census_size = base
        oc.counters = outcome.counters
        oc.tracks_per_cell = A.as_u64ptr(outcome.tracks_per_cell)
        while True:
            oc.census = buf.ctypes.data
            oc.census_capacity = buf.size
            rc = L.hwwg_run_segment_parallel(self._h, C.byref(sc), src.ctypes.data, src.size,
                                             h_begin, C.byref(wg) if wg else None,
                                             C.byref(tc), C.byref(oc))
            if rc == A.HWWG_ENOSPC:
                nb = np.zeros(int(oc.census_needed), PARTICLE_DT)
                nb[:base] = buf[:base]
                buf = nb
                continue
            _raise(rc)
            break
        tallies._from_c(tc)
        outcome.counters = oc.counters
        outcome.census = buf[: oc.census_size].copy()
        return outcome

    # losm.hpp:77-80
    def assemble_solve(self, mesh: Mesh1D, materials, phi_prev, J_prev, F_prev, theta, dt,
                       PL_prev=0.0, PR_prev=0.0, F_now=None, PL_now=0.0, PR_now=0.0,
                       J_L=0.0, J_R=0.0, q=None):
        I = mesh.cells()
        mats = _materials_array(materials, I)
        f = lambda a: np.ascontiguousarray(a, np.float64) if a is not None else None
        phi_prev, J_prev, F_prev, F_now, q = f(phi_prev), f(J_prev), f(F_prev), f(F_now), f(q)
        phi = np.zeros(I + 2)
        J = np.zeros(I + 1)
        _raise(A.lib().hwwg_losm_assemble_solve(
            self._h, I, A.as_dptr(mesh.edges), mats.ctypes.data, A.as_dptr(phi_prev),
            A.as_dptr(J_prev), J_L, J_R, 1 if F_now is not None else 0, A.as_dptr(F_now),
            PL_now, PR_now, A.as_dptr(F_prev), PL_prev, PR_prev, theta, dt, A.as_dptr(q),
            A.as_dptr(phi), A.as_dptr(J)))
        return phi, J

    # ww.hpp:34-35
    def build_centers(self, phi_tilde, eps_min, rho) -> WeightWindowGrid:
        phi = np.ascontiguousarray(phi_tilde, np.float64)
        out = np.ones(phi.size)
        rc = _raise(A.lib().hwwg_build_centers(self._h, A.as_dptr(phi), phi.size, eps_min, rho,
                                               A.as_dptr(out)))
        return WeightWindowGrid(out, rho, eps_min, uniform_fallback=(rc == 1))

    # filters.hpp:30
    def moving_average(self, g, k):
        g = np.ascontiguousarray(g, np.float64)
        out = np.zeros(g.size)
        _raise(A.lib().hwwg_moving_average(self._h, A.as_dptr(g), g.size, k, A.as_dptr(out)))
        return out

    # popctrl.hpp:22
    def fourier_lowpass(self, g, cutoff):
        """hww::fourier_lowpass (filters.cpp:26-52)."""
        g = np.ascontiguousarray(g, np.float64)
        out = np.zeros_like(g)
        _raise(A.lib().hwwg_fourier_lowpass(self._h, A.as_dptr(g), g.size, cutoff,
                                            A.as_dptr(out)))
        return out

    def uniform_comb(self, bank, target, seed, stream_id):
        b = np.ascontiguousarray(bank, PARTICLE_DT)
        out = np.zeros(target, PARTICLE_DT)
        iw, ow = C.c_double(), C.c_double()
        _raise(A.lib().hwwg_uniform_comb(self._h, b.ctypes.data if b.size else None, b.size,
                                         target, seed, stream_id, out.ctypes.data,
                                         C.byref(iw), C.byref(ow)))
        return out, iw.value, ow.value

    def device_log(self, x):
        x = np.ascontiguousarray(x, np.float64)
        out = np.zeros(x.size)
        _raise(A.lib().hwwg_device_log(self._h, A.as_dptr(x), x.size, A.as_dptr(out)))
        return out


_default_engine = None


def default_engine() -> Engine:
    global _default_engine
    if _default_engine is None:
        _default_engine = Engine()
    return _default_engine


def run_segment_parallel(ctx, source, h_begin, ww, tallies, outcome, engine=None):
    """hww::run_segment_parallel (transport.hpp:117-120) on the GPU."""
    return (engine or default_engine()).run_segment_parallel(ctx, source, h_begin, ww, tallies,
                                                             outcome)


# ------------------------------------------------------------------- driver
def _file_key(path, key):
    """A host-tooling key of a key = value config file (the C loader accepts
    and skips it); '' when absent."""
    val = ""
    with open(path) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if "=" in line:
                k, v = (t.strip() for t in line.split("=", 1))
                if k == key:
                    val = v
    return val


@dataclass
class RunConfig:
    """hww::RunConfig (config.hpp:33-66) with the reference defaults."""
    mode: str = "hww"
    histories_per_step: int = 10000
    theta: float = 0.5
    rho: float = 1.25
    eps_min: float = 1e-3
    u_ww: int = 3
    update_fractions: Sequence[float] = (0.25, 0.5, 0.75)
    ma_base_k: int = 3
    fourier_cutoff: int = 30
    batches: int = 20
    seed: int = 1
    target_population: int = 0
    comb_overflow_factor: float = 1.0
    source_x0: float = 0.0
    source_t0: float = 0.0
    source_strength: float = 1.0
    material: Material = field(default_factory=lambda: Material(1.0, 1.0 / 3.0, 1.0 / 3.0, 2.3, 1.0))
    x_min: float = -20.5
    x_max: float = 20.5
    cells: int = 201
    t_end: float = 20.0
    time_steps: int = 20
    threads: int = 0
    host_bank: bool = False
    out_dir: str = ""  # config.hpp:63: empty -> no file output
    # config.hpp:64 ("auto" | file path | ""): carried to run.json; the driver
    # takes the reference itself (Driver.set_reference / run(reference=...))
    reference: str = ""
    # Config-3 extensions (absent from the
    # reference driver): material regions [(x_hi, Material), ...] (a cell takes
    # the first region whose x_hi exceeds its centre), an isotropic volumetric
    # source (x_lo, x_hi, t_lo, t_hi, rate) sampled with vol_histories particles
    # in every step it overlaps, and no_pulse to drop the t = 0 point pulse.
    regions: Sequence = ()
    volume_source: Optional[tuple] = None
    vol_histories: int = 0
    no_pulse: bool = False

    def comb_target(self):
        return self.target_population or self.histories_per_step

    def to_c(self) -> A.RunConfigC:
        c = A.RunConfigC()
        c.mode = MODES.index(self.mode) if isinstance(self.mode, str) else int(self.mode)
        c.u_ww = self.u_ww
        c.histories_per_step = self.histories_per_step
        c.theta, c.rho, c.eps_min = self.theta, self.rho, self.eps_min
        c.n_fractions = len(self.update_fractions)
        for i, f in enumerate(self.update_fractions[:8]):
            c.fractions[i] = f
        c.ma_base_k, c.fourier_cutoff, c.batches = self.ma_base_k, self.fourier_cutoff, self.batches
        c.seed, c.target_population = self.seed, self.target_population
        c.comb_overflow_factor = self.comb_overflow_factor
        c.x0, c.t0, c.strength = self.source_x0, self.source_t0, self.source_strength
        m = self.material
        c.sigma_t, c.sigma_s, c.sigma_f, c.nu_f, c.speed = (m.sigma_t, m.sigma_s, m.sigma_f,
                                                            m.nu_f, m.speed)
        c.x_min, c.x_max, c.cells = self.x_min, self.x_max, self.cells
        c.t_end, c.time_steps, c.threads = self.t_end, self.time_steps, self.threads
        c.host_bank = 1 if self.host_bank else 0
        c.n_regions = len(self.regions)
        for i, (xh, m) in enumerate(list(self.regions)[:8]):
            c.region_x_hi[i] = xh
            for j, v in enumerate((m.sigma_t, m.sigma_s, m.sigma_f, m.nu_f, m.speed)):
                c.region_mat[i][j] = v
        if self.volume_source is not None:
            (c.vol_x_lo, c.vol_x_hi, c.vol_t_lo, c.vol_t_hi, c.vol_rate) = self.volume_source
            c.vol_histories = self.vol_histories or self.histories_per_step
        c.no_pulse = 1 if self.no_pulse else 0
        ref = self.reference.encode()
        if len(ref) >= 256:
            raise ValueError("reference path longer than 255 bytes")
        c.reference = ref
        return c

    def make_mesh(self):
        """config.hpp:87."""
        return build_uniform_mesh(self.x_min, self.x_max, self.cells)

    def time_layers(self):
        """make_time_grid().layer(0..N) (config.hpp:88; time_grid.hpp:22-29)."""
        out = np.zeros(self.time_steps + 1)
        _raise(A.lib().hwwg_time_layers(C.byref(self.to_c()), A.as_dptr(out)))
        return out

    @staticmethod
    def from_file(path) -> "RunConfig":
        """Key = value loader (hww_main.cpp:20-92 key names)."""
        L = A.lib()
        c = A.RunConfigC()
        L.hwwg_default_config(C.byref(c))
        _raise(L.hwwg_load_config_file(str(path).encode(), C.byref(c)))
        return RunConfig(
            mode=MODES[c.mode], histories_per_step=c.histories_per_step, theta=c.theta,
            rho=c.rho, eps_min=c.eps_min, u_ww=c.u_ww,
            update_fractions=tuple(c.fractions[i] for i in range(c.n_fractions)),
            ma_base_k=c.ma_base_k, fourier_cutoff=c.fourier_cutoff, batches=c.batches,
            seed=c.seed, target_population=c.target_population,
            comb_overflow_factor=c.comb_overflow_factor, source_x0=c.x0, source_t0=c.t0,
            source_strength=c.strength,
            material=Material(c.sigma_t, c.sigma_s, c.sigma_f, c.nu_f, c.speed),
            x_min=c.x_min, x_max=c.x_max, cells=c.cells, t_end=c.t_end,
            time_steps=c.time_steps, threads=c.threads, out_dir=_file_key(path, "out_dir"),
            regions=[(c.region_x_hi[i], Material(*[c.region_mat[i][j] for j in range(5)]))
                     for i in range(c.n_regions)],
            volume_source=((c.vol_x_lo, c.vol_x_hi, c.vol_t_lo, c.vol_t_hi, c.vol_rate)
                           if c.vol_rate > 0.0 else None),
            vol_histories=c.vol_histories if c.vol_rate > 0.0 else 0,
            no_pulse=bool(c.no_pulse), reference=c.reference.decode())

    def validate(self):
        """validate_config (config.cpp:27-69): list of violations."""
        buf = C.create_string_buffer(4096)
        n = A.lib().hwwg_validate_config(C.byref(self.to_c()), buf, 4096)
        return buf.value.decode().split("\n") if n else []


class Driver:
    """Stepwise hww::run (driver.cpp:286-342): device-resident time steps.

    Multi-GPU (one process per GPU): pass rank, world and the 128-byte NCCL id
    that rank 0 made with nccl_unique_id(); every rank then runs its shard of
    each step's histories and the driver all-reduces tallies / rebalances the
    census itself (Philox mode).  With `loopback` (a Loopback hub) the ranks are
    threads of this process on one device instead (tests)."""

    def __init__(self, config: RunConfig, device=0, rng_mode=RNG_EXACT, rank=0, world=1,
                 nccl_id: bytes = b"", loopback=None):
        self.config = config
        self._cfg = config.to_c()
        self._h = C.c_void_p()
        opts = A.Options(device, rng_mode, 0, rank, world)
        for i, b in enumerate(bytes(nccl_id)[:128]):
            opts.nccl_id[i] = b
        if loopback is not None:
            opts.loopback = loopback.handle
            self._hub = loopback  # the hub outlives its drivers
        _raise(A.lib().hwwg_driver_create(C.byref(self._cfg), C.byref(opts), C.byref(self._h)))
        self.I = config.cells

    def step(self):
        rec = A.StepRecordC()
        _raise(A.lib().hwwg_driver_step(self._h, C.byref(rec)))
        return rec

    def arrays(self):
        I = self.I
        arr = {n: np.full(I, np.nan) for n in ("phi_track", "sigma", "phi_census",
                                                "current_census", "closure_census",
                                                "ww_centers", "phi_hybrid")}
        arr["edge_current"] = np.zeros(I + 1)
        tracks = np.zeros(I, np.uint64)
        _raise(A.lib().hwwg_driver_arrays(
            self._h, A.as_dptr(arr["phi_track"]), A.as_dptr(arr["sigma"]),
            A.as_dptr(arr["phi_census"]), A.as_dptr(arr["current_census"]),
            A.as_dptr(arr["closure_census"]), A.as_dptr(arr["edge_current"]),
            A.as_dptr(arr["ww_centers"]), A.as_dptr(arr["phi_hybrid"]), A.as_u64ptr(tracks)))
        arr["tracks_per_cell"] = tracks
        return arr

    def write(self, out_dir, final=False, total_seconds=0.0):
        """hww::run's output writing (driver.cpp:318-321, 332-336): step_<n>.csv
        of the last step and summary.csv of all steps; run.json when final."""
        _raise(A.lib().hwwg_driver_write(self._h, str(out_dir).encode(), 1 if final else 0,
                                         float(total_seconds)))

    def set_reference(self, ref: "ReferenceSolution", name=None):
        """Run every following step against `ref` (hww::run's ReferenceSolution*,
        driver.hpp:88): the step records then carry rel_l2_error, rel_mod_l2_error,
        hybrid_rel_l2_error, fom_err_l2/mod, fom_sigma_mod and alpha."""
        lay = np.ascontiguousarray(ref.phi_layer, np.float64)
        itv = np.ascontiguousarray(ref.phi_interval, np.float64)
        if lay.shape != (self.config.time_steps + 1, self.I) or \
                itv.shape != (self.config.time_steps, self.I):
            raise ValueError("reference shape does not match the run's mesh and time grid")
        _raise(A.lib().hwwg_driver_set_reference(
            self._h, A.as_dptr(lay), A.as_dptr(itv), None if name is None else str(name).encode()))

    def load_reference(self, path):
        """load_reference(path, mesh, tgrid) + set_reference (hww_main.cpp:250-252)."""
        _raise(A.lib().hwwg_driver_load_reference(self._h, str(path).encode()))

    def compute_reference(self, space_refine=5, time_refine=20, sn_order=16):
        """reference = "auto" (hww_main.cpp:240-249): the device S_N reference."""
        _raise(A.lib().hwwg_driver_compute_reference(self._h, space_refine, time_refine,
                                                     sn_order))

    def bank(self):
        n = C.c_uint64()
        A.lib().hwwg_driver_bank(self._h, None, 0, C.byref(n))
        out = np.zeros(n.value, PARTICLE_DT)
        _raise(A.lib().hwwg_driver_bank(self._h, out.ctypes.data if n.value else None, n.value,
                                        C.byref(n)))
        return out

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            A.lib().hwwg_driver_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Loopback:
    """hwwg_loopback: an in-process collective hub for `world` driver ranks on
    one device (each rank's Driver.step must run on its own thread)."""

    def __init__(self, world, device=0):
        self.world = world
        self._h = C.c_void_p()
        _raise(A.lib().hwwg_loopback_create(world, device, C.byref(self._h)))

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            A.lib().hwwg_loopback_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId (rank 0 makes it; broadcast it with torch.distributed)."""
    buf = (C.c_uint8 * 128)()
    _raise(A.lib().hwwg_nccl_unique_id(buf))
    return bytes(buf)


# -------------------------------------------------------- sharding plan (host)
def shard_range(H, rank, world):
    lo, hi = C.c_uint64(), C.c_uint64()
    A.lib().hwwg_shard_range(H, rank, world, C.byref(lo), C.byref(hi))
    return lo.value, hi.value


def comb_plan(rank_weights, rank, target, offset_frac):
    """hwwg_comb_plan: (spacing, offset, rank_origin, k_lo, k_hi) for `rank`."""
    w = np.ascontiguousarray(rank_weights, np.float64)
    sp, off, org = C.c_double(), C.c_double(), C.c_double()
    lo, hi = C.c_uint64(), C.c_uint64()
    _raise(A.lib().hwwg_comb_plan(A.as_dptr(w), w.size, rank, target, offset_frac,
                                  C.byref(sp), C.byref(off), C.byref(org), C.byref(lo),
                                  C.byref(hi)))
    return sp.value, off.value, org.value, lo.value, hi.value


def rebalance_plan(k_lo_all, k_hi_all, rank, H):
    """hwwg_rebalance_plan: (send counts, first tooth sent, recv counts) per peer."""
    lo = np.ascontiguousarray(k_lo_all, np.uint64)
    hi = np.ascontiguousarray(k_hi_all, np.uint64)
    W = lo.size
    send, first, recv = (np.zeros(W, np.uint64) for _ in range(3))
    A.lib().hwwg_rebalance_plan(A.as_u64ptr(lo), A.as_u64ptr(hi), W, rank, H,
                                A.as_u64ptr(send), A.as_u64ptr(first), A.as_u64ptr(recv))
    return send, first, recv


def run(config: RunConfig, device=0, rng_mode=RNG_EXACT, out_dir=None,
        reference: "Optional[ReferenceSolution]" = None):
    """hww::run (driver.hpp:88, driver.cpp:286-342): returns the list of
    (record, arrays) per step. With out_dir (or config.out_dir) the reference's
    files are written as it writes them: step_<n>.csv and summary.csv after every
    step, run.json at the end, an INCOMPLETE marker if the run aborts."""
    import os
    import time
    out_dir = out_dir if out_dir is not None else getattr(config, "out_dir", "")
    d = Driver(config, device, rng_mode)
    if reference is not None:
        d.set_reference(reference)
    out = []
    t0 = time.perf_counter()
    try:
        for _ in range(config.time_steps):
            rec = d.step()
            out.append((rec, d.arrays()))
            if out_dir:
                d.write(out_dir)
        if out_dir:
            d.write(out_dir, final=True, total_seconds=time.perf_counter() - t0)
    except Exception:
        if out_dir:
            os.makedirs(out_dir, exist_ok=True)
            with open(os.path.join(out_dir, "INCOMPLETE"), "w") as f:
                f.write("run aborted before completing all steps\n")
        raise
    finally:
        d.close()
    return out


# ------------------------------------------------- deterministic reference
class ReferenceSolution:
    """hww::ReferenceSolution (reference.hpp:76-85): layer values phi_layer[0..N]
    and interval averages phi_interval[0..N-1] (steps 1..N) on the tally grids."""

    def __init__(self, mesh: Mesh1D, layers, phi_layer, phi_interval):
        self.mesh = mesh
        self.layers = np.ascontiguousarray(layers, np.float64)
        self.phi_layer = np.ascontiguousarray(phi_layer, np.float64)
        self.phi_interval = np.ascontiguousarray(phi_interval, np.float64)
        N, I = self.layers.size - 1, mesh.cells()
        if self.phi_layer.shape != (N + 1, I) or self.phi_interval.shape != (N, I):
            raise ValueError("reference arrays do not match the mesh and time grid")

    def layer(self, n):
        return self.phi_layer[n]

    def interval_avg(self, step):
        return self.phi_interval[step - 1]


def save_reference(ref: ReferenceSolution, path):
    """hww::save_reference (reference.cpp:374-393): same bytes."""
    N, I = ref.layers.size - 1, ref.mesh.cells()
    _raise(A.lib().hwwg_save_reference_csv(
        str(path).encode(), I, A.as_dptr(ref.mesh.edges), N, A.as_dptr(ref.layers),
        A.as_dptr(ref.phi_layer), A.as_dptr(ref.phi_interval)))


def load_reference(path, mesh: Mesh1D, layers) -> ReferenceSolution:
    """hww::load_reference (reference.cpp:395-456). Raises RuntimeError (the
    reference's std::runtime_error) on a missing, malformed or mis-shaped file."""
    layers = np.ascontiguousarray(layers, np.float64)
    N, I = layers.size - 1, mesh.cells()
    lay, itv = np.zeros((N + 1, I)), np.zeros((N, I))
    _raise(A.lib().hwwg_load_reference_csv(str(path).encode(), I, A.as_dptr(mesh.edges), N,
                                           A.as_dptr(layers), A.as_dptr(lay), A.as_dptr(itv)))
    return ReferenceSolution(mesh, layers, lay, itv)


def step_metrics(mesh: Mesh1D, rec, phi_track, phi_sigma=None, phi_hybrid=None,
                 reference: Optional[ReferenceSolution] = None):
    """hww::run_step's diagnostics (driver.cpp:231-275) for the step rec.step from
    its arrays and rec.tau / rec.sigma_valid; fills rec's metric fields."""
    edges = mesh.edges
    cvt = (lambda a: None if a is None else np.ascontiguousarray(a, np.float64))
    phi_track, phi_sigma, phi_hybrid = cvt(phi_track), cvt(phi_sigma), cvt(phi_hybrid)
    n = rec.step
    ri = rl = rp = None
    if reference is not None:
        ri = np.ascontiguousarray(reference.interval_avg(n))
        rl = np.ascontiguousarray(reference.layer(n))
        rp = np.ascontiguousarray(reference.layer(n - 1))
    _raise(A.lib().hwwg_step_metrics(mesh.cells(), A.as_dptr(edges), A.as_dptr(phi_track),
                                     A.as_dptr(phi_sigma), A.as_dptr(phi_hybrid), A.as_dptr(ri),
                                     A.as_dptr(rl), A.as_dptr(rp), C.byref(rec)))
    return rec


# ------------------------------------------------------ S_N reference (f4)
def gauss_legendre(n):
    """GaussLegendre::order (reference.cpp:14-42): (mu, weight)."""
    mu, w = np.zeros(n), np.zeros(n)
    _raise(A.lib().hwwg_gauss_legendre(n, A.as_dptr(mu), A.as_dptr(w)))
    return mu, w


def sn_solve(mesh: Mesh1D, materials, layers, order, psi0, inc_left=None, inc_right=None,
             q=None, tolerance=1e-9, max_iterations=1000, engine=None):
    """hww::sn_solve (reference.cpp:151-233) on the device: (phi per layer
    [(steps+1), cells], source iterations per step). RuntimeError (the reference's
    std::runtime_error) when a step does not converge."""
    eng = engine or default_engine()
    I = mesh.cells()
    mats = _materials_array(materials, I)
    layers = np.ascontiguousarray(layers, np.float64)
    N = layers.size - 1
    psi0 = np.ascontiguousarray(psi0, np.float64)
    cvt = (lambda a: None if a is None else np.ascontiguousarray(a, np.float64))
    inc_left, inc_right, q = cvt(inc_left), cvt(inc_right), cvt(q)
    phi, its = np.zeros((N + 1, I)), np.zeros(N + 1, np.int32)
    _raise(A.lib().hwwg_sn_solve(eng._h, I, A.as_dptr(mesh.edges), mats.ctypes.data, N,
                                 A.as_dptr(layers), order, A.as_dptr(psi0), A.as_dptr(inc_left),
                                 A.as_dptr(inc_right), A.as_dptr(q), tolerance, max_iterations,
                                 A.as_dptr(phi), its.ctypes.data))
    return phi, its


def compute_reference(config: RunConfig, space_refine=5, time_refine=20, sn_order=16,
                      engine=None) -> ReferenceSolution:
    """hww::compute_reference (reference.cpp:364-372) on the device."""
    eng = engine or default_engine()
    N, I = config.time_steps, config.cells
    lay, itv = np.zeros((N + 1, I)), np.zeros((N, I))
    _raise(A.lib().hwwg_compute_reference(eng._h, C.byref(config.to_c()), space_refine,
                                          time_refine, sn_order, A.as_dptr(lay), A.as_dptr(itv)))
    return ReferenceSolution(config.make_mesh(), config.time_layers(), lay, itv)
