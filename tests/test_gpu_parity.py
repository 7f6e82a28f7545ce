"""GPU parity of the exact-mode engine (through the C ABI) against the oracle
and the golden vectors produced by the real reference. Run on a B200:
``python -m pytest tests -m gpu``."""
import ctypes as C
import functools

import numpy as np
import pytest

import paper_2512_19925_b200 as hw
from oracle.bind import (PARTICLE_DT, DriverRun, Oracle, baseline_config, homogeneous,
                         uniform_edges)
from tests.golden.make_golden import SEG_FIELDS, segment_cases
from tests.parity import (COUNTER_U, census_equal, close_rel, counters_equal, golden,
                          tallies_close)

pytestmark = pytest.mark.gpu


class _G:  # golden tallies as attributes
    def __init__(self, g, name):
        for f in SEG_FIELDS:
            setattr(self, f, g[f"{name}.{f}"])
        s = g[f"{name}.scalars"]
        self.boundary_closure_left, self.boundary_closure_right = s[0], s[1]
        self.histories_scored, self.grazing_discarded = int(s[2]), int(s[3])


def _gpu_segment(engine, kw):
    I = kw["edges"].size - 1
    ctx = hw.StepContext(hw.Mesh1D(kw["edges"]), kw["mats"], kw["t_begin"], kw["t_end"],
                         kw["seed"], kw["step"], kw["H"], kw["B"])
    tal, out = hw.TallySet(I, kw["B"]), hw.StepOutcome(I)
    ww = hw.WeightWindowGrid(kw["centers"], kw["rho"]) if kw["centers"] is not None else None
    engine.run_segment_parallel(ctx, kw["src"], kw["h_begin"], ww, tal, out)
    return tal, out


def test_device_log_is_libm_bit_exact(engine, oracle):
    rng = np.random.default_rng(1)
    u = ((rng.integers(0, 2**53, 2_000_000, dtype=np.uint64)).astype(np.float64) + 0.5) * 2.0**-53
    x = np.concatenate([u, 0.9375 + 0.13 * u[:200000],
                        rng.uniform(1e-300, 1e300, 100000), [1.0, 2.0**-1074, 5e-324]])
    ref = np.zeros(x.size)
    oracle.lib.orc_log_array.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
    oracle.lib.orc_log_array(x.ctypes.data, x.size, ref.ctypes.data)
    dev = engine.device_log(x)
    assert np.array_equal(dev, ref), int(np.sum(dev != ref))


@pytest.mark.parametrize("name,kw", segment_cases(), ids=[c[0] for c in segment_cases()])
def test_segment_matches_golden(engine, name, kw):
    g = golden("segments.npz")
    tal, out = _gpu_segment(engine, kw)
    I, B = kw["edges"].size - 1, kw["B"]
    gt = _G(g, name)
    tallies_close(tal, gt, I, B)
    assert tal.histories_scored == gt.histories_scored
    assert tal.grazing_discarded == gt.grazing_discarded
    ref_c = dict(zip(COUNTER_U, g[f"{name}.counters_u"].tolist()))
    ref_c["leakage_weight"], ref_c["aborted_weight"] = g[f"{name}.counters_d"]
    counters_equal(out.counters.as_dict(), ref_c)
    assert np.array_equal(out.tracks_per_cell, g[f"{name}.tracks"])
    census_equal(out.census, g[f"{name}.census"])  # identical windows: w bit-exact too


@pytest.mark.parametrize("H,seed,rho", [(20000, 11, 5.0), (50000, 12, 2.0)])
def test_segment_matches_oracle_large(engine, oracle, H, seed, rho):
    I, B = 400, 20
    e = uniform_edges(-20.0, 20.0, I)
    mats = homogeneous(I, 1.0, 0.9)
    rng = np.random.default_rng(seed)
    src = np.zeros(H, PARTICLE_DT)
    src["x"] = rng.normal(0, 4, H).clip(-19.9, 19.9)
    src["mu"] = rng.uniform(-1, 1, H)
    src["w"] = rng.exponential(1.0, H) + 1e-3
    src["t"] = 2.0
    xc = 0.5 * (e[1:] + e[:-1])
    cen = np.exp(-np.abs(xc) / 2.5)
    cen = cen / cen.max() * (1 - 1e-3) + 1e-3
    to, ko, tro, co, _ = oracle.run_segment(e, mats, 2.0, 2.5, seed, 5, H, B, src, 0,
                                            centers=cen, rho=rho, chunk=256)
    kw = dict(edges=e, mats=mats, t_begin=2.0, t_end=2.5, seed=seed, step=5, H=H, B=B,
              src=src, h_begin=0, centers=cen, rho=rho)
    tal, out = _gpu_segment(engine, kw)
    counters_equal(out.counters.as_dict(), ko.as_dict())
    assert np.array_equal(out.tracks_per_cell, tro)
    census_equal(out.census, co)
    tallies_close(tal, to, I, B)


def test_segment_errors_match_reference(engine):
    e = uniform_edges(0.0, 1.0, 2)
    mats = homogeneous(2, 1.0, 1 / 3, 1 / 3, 2.3)
    ctx = hw.StepContext(hw.Mesh1D(e), mats, 0.0, 1.0, 1, 1, 1, 20)
    bad = np.array([(2.0, 1.0, 1.0, 0.0)], PARTICLE_DT)  # test_transport.cpp:131-144
    with pytest.raises(ValueError, match="outside"):
        engine.run_segment_parallel(ctx, bad, 0, None, hw.TallySet(2, 20), hw.StepOutcome(2))
    late = np.array([(0.5, 1.0, 1.0, 1.0)], PARTICLE_DT)  # t == t_end is outside the step
    with pytest.raises(ValueError):
        engine.run_segment_parallel(ctx, late, 0, None, hw.TallySet(2, 20), hw.StepOutcome(2))
    nanw = np.array([(0.5, 1.0, np.nan, 0.0)], PARTICLE_DT)
    out = hw.StepOutcome(2)
    engine.run_segment_parallel(ctx, nanw, 0, None, hw.TallySet(2, 20), out)
    assert out.counters.nan_aborts == 1 and out.census.size == 0
    # empty source is a no-op (transport.cpp:212-217)
    engine.run_segment_parallel(ctx, np.zeros(0, PARTICLE_DT), 0, None, hw.TallySet(2, 20), out)


def _gpu_driver(which, H, N):
    o = baseline_config(which, histories=H, time_steps=N)
    cfg = hw.RunConfig(mode=hw.hww.MODES[o.mode], histories_per_step=o.histories_per_step,
                       theta=o.theta, rho=o.rho, eps_min=o.eps_min, u_ww=o.u_ww,
                       update_fractions=tuple(o.fractions[:o.n_fractions]),
                       ma_base_k=o.ma_base_k, batches=o.batches, seed=o.seed,
                       material=hw.Material(o.sigma_t, o.sigma_s, o.sigma_f, o.nu_f, o.speed),
                       x_min=o.x_min, x_max=o.x_max, cells=o.cells, t_end=o.t_end,
                       time_steps=o.time_steps)
    return hw.Driver(cfg)


def _check_step(rec, arr, ints, counters_u, counters_d, g_arr, tol=1e-12):
    assert [getattr(rec.counters, n) for n in COUNTER_U] == list(counters_u)
    close_rel([rec.counters.leakage_weight, rec.counters.aborted_weight], counters_d, tol,
              what="counter weights")
    got = [rec.segments, rec.census_size, rec.histories, rec.comb_in, rec.comb_out,
           rec.updates_applied, rec.hybrid_solve_failed, rec.n_thresholds, rec.sigma_valid,
           rec.has_windows, rec.has_hybrid]
    assert got == list(ints), (got, list(ints))
    assert np.array_equal(arr["tracks_per_cell"], g_arr["tracks_per_cell"])
    for k in ("phi_track", "phi_census", "sigma"):
        close_rel(arr[k], g_arr[k], tol, what=k)
    phi = np.abs(g_arr["phi_census"]) + 1e-300
    close_rel(arr["current_census"], g_arr["current_census"], tol, scale=phi, what="J")
    close_rel(arr["closure_census"], g_arr["closure_census"], tol, scale=phi, what="F")
    if rec.has_windows:  # centres: norm-wise (L-inf relative), SURVEY §8(d)
        c, gc = arr["ww_centers"], g_arr["ww_centers"]
        assert np.max(np.abs(c - gc)) <= tol * np.max(np.abs(gc))
    if rec.has_hybrid:
        h, gh = arr["phi_hybrid"], g_arr["phi_hybrid"]
        assert np.max(np.abs(h - gh)) <= 1e-10 * np.max(np.abs(gh))


@pytest.mark.parametrize("which,H,N", [(0, 1500, 4), (1, 3000, 5), (2, 3000, 4)])
def test_driver_matches_golden(which, H, N):
    g = golden(f"driver_c{which}.npz")
    d = _gpu_driver(which, H, N)
    for s in range(1, N + 1):
        rec = d.step()
        arr = d.arrays()
        g_arr = {k: g[f"s{s}.{k}"] for k in arr}
        _check_step(rec, arr, g[f"s{s}.ints"], g[f"s{s}.counters_u"], g[f"s{s}.counters_d"],
                    g_arr)
    census_equal(d.bank(), g["bank"], weights_tol=1e-12)


@pytest.mark.parametrize("which,H,N", [(2, 30000, 6), (1, 20000, 8)])
def test_driver_matches_oracle(oracle, which, H, N):
    """Through the cold-start split explosion of config 2 (step 1 census x63)."""
    od = DriverRun(oracle, baseline_config(which, histories=H, time_steps=N))
    d = _gpu_driver(which, H, N)
    for s in range(1, N + 1):
        o, oarr = od.step()
        rec = d.step()
        arr = d.arrays()
        ints = [o.segments, o.census_size, o.histories, o.comb_in, o.comb_out,
                o.updates_applied, o.hybrid_solve_failed, o.n_thresholds, o.sigma_valid,
                o.has_windows, o.has_hybrid]
        _check_step(rec, arr, ints, [getattr(o.counters, n) for n in COUNTER_U],
                    [o.counters.leakage_weight, o.counters.aborted_weight], oarr)
    census_equal(d.bank(), od.bank(), weights_tol=1e-12)


def test_components_match_golden(engine):
    g = golden("components.npz")
    for name in ("losm_lag", "losm_imp"):
        p = g[f"{name}.params"]
        e = g[f"{name}.edges"]
        mats = np.ascontiguousarray(g[f"{name}.mats"])
        phi, J = engine.assemble_solve(
            hw.Mesh1D(e), mats, g[f"{name}.in_phi"], g[f"{name}.in_J"], g[f"{name}.in_Fp"],
            p[1], p[2], PL_prev=p[5], PR_prev=p[6],
            F_now=g[f"{name}.in_Fn"] if p[0] else None, PL_now=p[3], PR_now=p[4])
        assert np.array_equal(phi, g[f"{name}.phi"]) and np.array_equal(J, g[f"{name}.J"]), name
    for k in (0, 1, 2, 3):
        assert np.array_equal(engine.moving_average(g["ma.in"], k), g[f"ma.k{k}"]), k
    grid = engine.build_centers(g["centers.in"], 1e-3, 5.0)
    assert np.array_equal(grid.centers, g["centers.out"])
    assert grid.uniform_fallback == bool(g["centers.fallback"][0])
    for tgt in (5000, 137, 12000):
        out, iw, ow = engine.uniform_comb(g["comb.bank"], tgt, 9, (3 << 56) ^ (4 << 40))
        assert out.tobytes() == g[f"comb.t{tgt}"].tobytes(), tgt
        assert [iw, ow] == list(g[f"comb.t{tgt}.w"])


def test_component_known_answers(engine):
    grid = engine.build_centers([0.0, 0.5, 1.0], 1e-3, 1.25)  # test_ww.cpp:11-30
    assert np.allclose(grid.centers, [0.001, 0.5005, 1.0], rtol=1e-14)
    assert engine.build_centers([0.0, -1.0], 1e-3, 1.25).uniform_fallback
    assert np.allclose(engine.moving_average([0, 0, 3.0, 0, 0], 1), [0, 1, 1, 1, 0])
    one = np.array([(0.0, 1.0, 1.0, 0.0)], PARTICLE_DT)  # test_popctrl.cpp:22-30
    out, iw, ow = engine.uniform_comb(one, 4, 2, 2)
    assert out.size == 4 and np.allclose(out["w"], 0.25) and abs(ow - 1.0) < 1e-15
    with pytest.raises(ValueError):
        engine.uniform_comb(np.zeros(0, PARTICLE_DT), 10, 1, 1)


@functools.lru_cache(maxsize=1)
def comb_banks():
    """Adversarial banks for the cumulative-weight walk (popctrl.cpp:15-30): rounding
    ties at every add, equal weights, a dynamic range of 2^80, zeros, a subnormal
    head, and a bank larger than one 4096-weight tile many times over."""
    rng = np.random.default_rng(5)
    banks = {}

    def bank(w):
        b = np.zeros(len(w), PARTICLE_DT)
        b["x"] = rng.uniform(-1, 1, len(w))
        b["mu"] = rng.uniform(-1, 1, len(w))
        b["w"] = w
        b["t"] = 1.0
        return b

    banks["ones"] = bank(np.ones(70_000))
    banks["tenths"] = bank(np.full(50_000, 0.1))
    ulp = 2.0 ** -32  # ulp of 2^20: half- and one-and-a-half-ulp adds tie
    w = rng.choice(np.array([0.5, 1.5, 1.0, 0.25, 2.5, 0.75]) * ulp, 60_000)
    w[0] = 2.0 ** 20
    banks["ties"] = bank(w)
    w = np.exp(rng.normal(0, 8, 200_000))
    w[rng.integers(0, w.size, 500)] = 0.0
    banks["lognormal"] = bank(w)
    w = rng.exponential(1.0, 30_000)
    w[:40] = 1e-310
    w[40:45] = 0.0
    banks["subnormal_head"] = bank(w)
    banks["one"] = bank(np.array([3.0]))
    w = rng.exponential(1.0, 3_000_000)  # ~730 tiles: the mapped-tile path
    w[1_000_000:1_000_100] = 1e12  # a late jump across many binades
    banks["exp3M"] = bank(w)
    return banks


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(comb_banks()))
def test_comb_walk_bit_exact_adversarial(engine, oracle, name):
    """The parallel binade scan of the comb's sequential fp64 walk equals the serial
    walk bit for bit: the teeth, W and the output weight."""
    b = comb_banks()[name]
    for tgt in (1, 997, 100_003):
        out, iw, ow = engine.uniform_comb(b, tgt, 3, 17)
        ro, riw, row = oracle.uniform_comb(b, tgt, 3, 17)
        assert iw == riw and ow == row, (name, tgt, iw, riw, ow, row)
        assert out.tobytes() == ro.tobytes(), (name, tgt)


@pytest.mark.gpu
@pytest.mark.parametrize("I,seed", [(400, 1), (37, 2), (510, 3)])
def test_losm_cached_factorization_is_identical(engine, I, seed):
    """Throughput mode solves the window update through a cached Schur/PCR
    factorization; it must reproduce the rebuilt factorization bit for bit."""
    import ctypes as C
    from paper_2512_19925_b200 import _capi as A
    f = A.lib().hwwg_internal_losm_cache_check
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.c_int32, C.c_uint32, C.POINTER(C.c_double)]
    mx = C.c_double(0.0)
    rc = f(engine._h, I, seed, C.byref(mx))
    assert rc == 0, (rc, mx.value)


def test_fourier_lowpass_matches_reference_filter(engine, oracle):
    """hww_fourier's filter on the device: bit-identical to the C restatement
    (itself pinned to the reference, tests/test_oracle_pin.py)."""
    import ctypes as C
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    oracle.lib.orc_fourier_lowpass.argtypes = [C.POINTER(C.c_double), C.c_int32, C.c_int32,
                                               C.POINTER(C.c_double)]
    rng = np.random.default_rng(8)
    for M, cut in [(1, 0), (2, 0), (37, 5), (400, 30), (401, 30), (64, 40)]:
        g = np.ascontiguousarray(rng.standard_normal(M) * np.exp(-np.linspace(-3, 3, M) ** 2))
        o = np.zeros(M)
        assert oracle.lib.orc_fourier_lowpass(dp(g), M, cut, dp(o)) == 0
        assert engine.fourier_lowpass(g, cut).tobytes() == o.tobytes(), (M, cut)


def test_fourier_driver_matches_oracle(oracle):
    """mode hww_fourier end to end in exact mode (the filter runs inside the
    device LOSM update, twiddles from the host libm)."""
    kw = dict(histories_per_step=3000, rho=3.0, fourier_cutoff=12, cells=80, x_min=-10.0,
              x_max=10.0, t_end=2.0, time_steps=4, seed=4)
    from oracle.bind import make_config
    od = DriverRun(oracle, make_config(mode="hww_fourier", sigma_t=1.0, sigma_s=0.9,
                                       sigma_f=0.0, nu_f=0.0, speed=1.0, **kw))
    d = hw.Driver(hw.RunConfig(mode="hww_fourier", material=hw.Material(1.0, 0.9, 0.0, 0.0, 1.0),
                               **kw))
    for s in range(1, kw["time_steps"] + 1):
        o, oarr = od.step()
        rec = d.step()
        arr = d.arrays()
        ints = [o.segments, o.census_size, o.histories, o.comb_in, o.comb_out,
                o.updates_applied, o.hybrid_solve_failed, o.n_thresholds, o.sigma_valid,
                o.has_windows, o.has_hybrid]
        _check_step(rec, arr, ints, [getattr(o.counters, n) for n in COUNTER_U],
                    [o.counters.leakage_weight, o.counters.aborted_weight], oarr)
    census_equal(d.bank(), od.bank(), weights_tol=1e-12)


def _c3(H, steps, mode="hww", cells=120, nv=None):
    """A reduced BASELINE config 3: three material regions,
    isotropic volumetric source in x in [0,2], t in [0,1], no pulse."""
    regions = [(10.0, (1.0, 0.5, 0.0, 0.0, 1.0)), (20.0, (10.0, 1.0, 0.0, 0.0, 1.0)),
               (30.0, (1.0, 0.99, 0.0, 0.0, 1.0))]
    kw = dict(histories_per_step=H, rho=4.0, seed=3, cells=cells, x_min=0.0, x_max=30.0,
              t_end=0.5 * steps, time_steps=steps)
    from oracle.bind import make_config
    o = make_config(mode=mode, no_pulse=1, regions=regions, vol=(0.0, 2.0, 0.0, 1.0, 1.0, nv or H),
                    sigma_t=1.0, sigma_s=0.5, sigma_f=0.0, nu_f=0.0, speed=1.0, **kw)
    g = hw.RunConfig(mode=mode, no_pulse=True, volume_source=(0.0, 2.0, 0.0, 1.0, 1.0),
                     vol_histories=nv or H, material=hw.Material(1.0, 0.5, 0.0, 0.0, 1.0),
                     regions=[(x, hw.Material(*m)) for x, m in regions], **kw)
    return o, g


@pytest.mark.parametrize("mode", ["hww", "analog", "hww_ma"])
def test_config3_driver_matches_oracle(oracle, mode):
    """Config-3 features end to end in exact mode: regions, the volumetric
    source appended after the combed census, the LOSM q."""
    o_cfg, g_cfg = _c3(2000, 4, mode=mode)
    od = DriverRun(oracle, o_cfg)
    d = hw.Driver(g_cfg)
    for s in range(1, 5):
        o, oarr = od.step()
        rec = d.step()
        arr = d.arrays()
        ints = [o.segments, o.census_size, o.histories, o.comb_in, o.comb_out,
                o.updates_applied, o.hybrid_solve_failed, o.n_thresholds, o.sigma_valid,
                o.has_windows, o.has_hybrid]
        _check_step(rec, arr, ints, [getattr(o.counters, n) for n in COUNTER_U],
                    [o.counters.leakage_weight, o.counters.aborted_weight], oarr)
    census_equal(d.bank(), od.bank(), weights_tol=1e-12)


@pytest.mark.parametrize("which,H,N,kw", [
    (4, 20000, 3, {}),                                   # I = 4000: global LOSM / tallies paths
    (5, 20000, 3, dict(rho=2.0, mode="hww")),            # config 5 variants (rho x filter)
    (5, 20000, 3, dict(rho=10.0, ma_base_k=2)),
])
def test_configs_4_5_match_oracle(oracle, which, H, N, kw):
    """BASELINE configs 4 and 5 at reduced H in exact mode: the large mesh (the
    low-order state no longer fits shared memory) and the config-5 window/filter
    variants, bit-exact against the oracle."""
    oc = baseline_config(which, histories=H, time_steps=N, **kw)
    od = DriverRun(oracle, oc)
    cfg = hw.RunConfig(mode=hw.hww.MODES[oc.mode], histories_per_step=oc.histories_per_step,
                       theta=oc.theta, rho=oc.rho, eps_min=oc.eps_min, u_ww=oc.u_ww,
                       update_fractions=tuple(oc.fractions[:oc.n_fractions]),
                       ma_base_k=oc.ma_base_k, batches=oc.batches, seed=oc.seed,
                       material=hw.Material(oc.sigma_t, oc.sigma_s, oc.sigma_f, oc.nu_f, oc.speed),
                       x_min=oc.x_min, x_max=oc.x_max, cells=oc.cells, t_end=oc.t_end,
                       time_steps=oc.time_steps)
    d = hw.Driver(cfg)
    for s in range(1, N + 1):
        o, oarr = od.step()
        rec = d.step()
        arr = d.arrays()
        ints = [o.segments, o.census_size, o.histories, o.comb_in, o.comb_out,
                o.updates_applied, o.hybrid_solve_failed, o.n_thresholds, o.sigma_valid,
                o.has_windows, o.has_hybrid]
        _check_step(rec, arr, ints, [getattr(o.counters, n) for n in COUNTER_U],
                    [o.counters.leakage_weight, o.counters.aborted_weight], oarr)
    census_equal(d.bank(), od.bank(), weights_tol=1e-12)
    # the throughput mode on the same configuration: runs, conserves the census count
    fd = hw.Driver(cfg, rng_mode=hw.RNG_PHILOX)
    for s in range(1, N + 1):
        r = fd.step()
        assert r.census_size == r.counters.census_count and r.segments > 0
    fd.close()
