"""Pin the C oracle: bit-exact against the golden vectors produced by the real
reference (tests/golden/make_golden.py) and, where oracle/_ref is built,
against the live reference on further seeded cases; plus the reference's own
known-answer tests (proj/tests/*.cpp) restated."""
import ctypes as C

import numpy as np
import pytest

from oracle.bind import (PARTICLE_DT, DriverRun, Oracle, Reference, TallyArrays,
                         baseline_config, have_reference, homogeneous, uniform_edges)
from tests.golden.make_golden import SEG_FIELDS, segment_cases
from tests.parity import COUNTER_U, golden


def _run_oracle_case(O, kw):
    return O.run_segment(kw["edges"], kw["mats"], kw["t_begin"], kw["t_end"], kw["seed"],
                         kw["step"], kw["H"], kw["B"], kw["src"], kw["h_begin"],
                         centers=kw["centers"], rho=kw["rho"], chunk=256)


@pytest.mark.parametrize("name,kw", segment_cases(), ids=[c[0] for c in segment_cases()])
def test_oracle_segments_match_golden(oracle, name, kw):
    g = golden("segments.npz")
    t, k, tr, census, _ = _run_oracle_case(oracle, kw)
    for f in SEG_FIELDS:
        assert np.array_equal(getattr(t, f), g[f"{name}.{f}"]), f
    assert np.array_equal(
        np.array([t.boundary_closure_left, t.boundary_closure_right, t.histories_scored,
                  t.grazing_discarded], float), g[f"{name}.scalars"])
    assert np.array_equal(np.array([getattr(k, n) for n in COUNTER_U], np.uint64),
                          g[f"{name}.counters_u"])
    assert np.array_equal(np.array([k.leakage_weight, k.aborted_weight]), g[f"{name}.counters_d"])
    assert np.array_equal(tr, g[f"{name}.tracks"])
    assert census.tobytes() == g[f"{name}.census"].tobytes()


@pytest.mark.parametrize("which,H,N", [(0, 1500, 4), (1, 3000, 5), (2, 3000, 4)])
def test_oracle_driver_matches_golden(oracle, which, H, N):
    g = golden(f"driver_c{which}.npz")
    d = DriverRun(oracle, baseline_config(which, histories=H, time_steps=N))
    for s in range(1, N + 1):
        o, arr = d.step()
        assert np.array_equal(np.array([getattr(o.counters, n) for n in COUNTER_U], np.uint64),
                              g[f"s{s}.counters_u"]), s
        assert np.array_equal(np.array([o.counters.leakage_weight, o.counters.aborted_weight]),
                              g[f"s{s}.counters_d"])
        ints = np.array([o.segments, o.census_size, o.histories, o.comb_in, o.comb_out,
                         o.updates_applied, o.hybrid_solve_failed, o.n_thresholds,
                         o.sigma_valid, o.has_windows, o.has_hybrid], np.uint64)
        assert np.array_equal(ints, g[f"s{s}.ints"])
        assert np.array_equal(np.array([o.census_weight, o.census_weight_sigma,
                                        o.boundary_closure_left, o.boundary_closure_right,
                                        o.comb_in_weight, o.comb_out_weight]),
                              g[f"s{s}.scalars"])
        for k, v in arr.items():
            assert np.array_equal(v, g[f"s{s}.{k}"], equal_nan=True), (s, k)
    assert d.bank().tobytes() == g["bank"].tobytes()


def test_oracle_components_match_golden(oracle):
    g = golden("components.npz")
    L = oracle.lib
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    for name in ("losm_lag", "losm_imp"):
        p = g[f"{name}.params"]
        e, mats = g[f"{name}.edges"], np.ascontiguousarray(g[f"{name}.mats"])
        I = e.size - 1
        po, Jo = np.zeros(I + 2), np.zeros(I + 1)
        phi, J, Fn, Fp = (np.ascontiguousarray(g[f"{name}.in_{k}"]) for k in ("phi", "J", "Fn", "Fp"))
        L.orc_assemble_solve.argtypes = [C.c_int32, C.POINTER(C.c_double), C.c_void_p] + \
            [C.POINTER(C.c_double)] * 2 + [C.c_double] * 2 + [C.c_int32, C.POINTER(C.c_double)] + \
            [C.c_double] * 2 + [C.POINTER(C.c_double)] + [C.c_double] * 4 + [C.POINTER(C.c_double)] * 3
        rc = L.orc_assemble_solve(I, dp(e), mats.ctypes.data, dp(phi), dp(J), 0.0, 0.0, int(p[0]),
                                  dp(Fn), p[3], p[4], dp(Fp), p[5], p[6], p[1], p[2], None,
                                  dp(po), dp(Jo))
        assert rc == 0
        assert np.array_equal(po, g[f"{name}.phi"]) and np.array_equal(Jo, g[f"{name}.J"])
    v = np.ascontiguousarray(g["ma.in"])
    L.orc_moving_average.argtypes = [C.POINTER(C.c_double), C.c_int32, C.c_int32, C.POINTER(C.c_double)]
    for k in (0, 1, 2, 3):
        o = np.zeros(v.size)
        L.orc_moving_average(dp(v), v.size, k, dp(o))
        assert np.array_equal(o, g[f"ma.k{k}"]), k
    phi = np.ascontiguousarray(g["centers.in"])
    c = np.zeros(phi.size)
    L.orc_build_centers.argtypes = [C.POINTER(C.c_double), C.c_int32, C.c_double, C.c_double,
                                    C.POINTER(C.c_double)]
    assert L.orc_build_centers(dp(phi), phi.size, 1e-3, 5.0, dp(c)) == int(g["centers.fallback"][0])
    assert np.array_equal(c, g["centers.out"])
    bank = np.ascontiguousarray(g["comb.bank"])
    L.orc_uniform_comb.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                   C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    for tgt in (5000, 137, 12000):
        out = np.zeros(tgt, PARTICLE_DT)
        iw, ow = C.c_double(), C.c_double()
        assert L.orc_uniform_comb(bank.ctypes.data, bank.size, tgt, 9, (3 << 56) ^ (4 << 40),
                                  out.ctypes.data, C.byref(iw), C.byref(ow)) == 0
        assert out.tobytes() == g[f"comb.t{tgt}"].tobytes()
        assert np.array_equal([iw.value, ow.value], g[f"comb.t{tgt}.w"])


# ---- known answers restated from the reference's unit tests ----------------
def test_known_answers(oracle):
    L = oracle.lib
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    L.orc_build_centers.argtypes = [C.POINTER(C.c_double), C.c_int32, C.c_double, C.c_double,
                                    C.POINTER(C.c_double)]
    # test_ww.cpp:11-30
    c = np.zeros(3)
    assert L.orc_build_centers(dp(np.array([0.0, 0.5, 1.0])), 3, 1e-3, 1.25, dp(c)) == 0
    assert np.allclose(c, [0.001, 0.5005, 1.0], rtol=1e-14)
    assert L.orc_build_centers(dp(np.array([0.0, -1.0])), 2, 1e-3, 1.25, dp(c)) == 1
    # test_ww.cpp:97-103
    out = np.zeros(3, np.uint64)
    L.orc_update_thresholds.argtypes = [C.c_uint64, C.POINTER(C.c_double), C.c_int32, C.c_void_p]
    assert L.orc_update_thresholds(10000, dp(np.array([0.25, 0.5, 0.75])), 3, out.ctypes.data) == 0
    assert list(out) == [2500, 5000, 7500]
    assert L.orc_update_thresholds(10, dp(np.array([0.25, 0.5])), 2, out.ctypes.data) == 0
    assert list(out[:2]) == [3, 5]
    assert L.orc_update_thresholds(100, dp(np.array([0.5, 0.25])), 2, out.ctypes.data) != 0
    # test_filters.cpp:12-27
    L.orc_moving_average.argtypes = [C.POINTER(C.c_double), C.c_int32, C.c_int32, C.POINTER(C.c_double)]
    o = np.zeros(5)
    L.orc_moving_average(dp(np.array([0, 0, 3.0, 0, 0])), 5, 1, dp(o))
    assert np.allclose(o, [0, 1, 1, 1, 0])
    o = np.zeros(4)
    L.orc_moving_average(dp(np.array([1.0, 2, 3, 4])), 4, 1, dp(o))
    assert np.array_equal(o, [1, 2, 3, 4])
    # test_transport.cpp:113-129: near-void free flight reaches census unchanged
    e = uniform_edges(-5.0, 5.0, 10)
    src = np.array([(0.0, 1.0, 1.0, 0.0)], PARTICLE_DT)
    t, k, tr, census, _ = oracle.run_segment(e, homogeneous(10, 1e-12), 0.0, 1.0, 1, 1, 1, 20,
                                             src, 0, chunk=0)
    assert census.size == 1 and abs(census["x"][0] - 1.0) < 1e-12
    assert census["w"][0] == 1.0 and census["t"][0] == 1.0 and k.collisions == 0
    # test_transport.cpp:131-144: a history starting outside the mesh is an error
    bad = np.array([(2.0, 1.0, 1.0, 0.0)], PARTICLE_DT)
    with pytest.raises(ValueError):
        oracle.run_segment(uniform_edges(0.0, 1.0, 2), homogeneous(2, 1.0, 1 / 3, 1 / 3, 2.3),
                           0.0, 1.0, 1, 1, 1, 20, bad, 0, chunk=0)


def test_noop_windows_reproduce_analog(oracle):
    """test_transport.cpp:180-210: rho = 1e300 windows never split or roulette."""
    e = uniform_edges(-20.5, 20.5, 201)
    mats = homogeneous(201, 1.0, 1 / 3, 1 / 3, 2.3)
    src = np.zeros(3000, PARTICLE_DT)
    src["mu"] = np.random.default_rng(21).uniform(-1, 1, 3000)
    src["w"] = 1.0
    a = oracle.run_segment(e, mats, 0, 1, 21, 1, 3000, 20, src, 0, chunk=0)
    w = oracle.run_segment(e, mats, 0, 1, 21, 1, 3000, 20, src, 0, centers=np.ones(201),
                           rho=1e300, chunk=0)
    assert a[3].tobytes() == w[3].tobytes()
    assert a[1].collisions == w[1].collisions and w[1].splits == 0 and w[1].roulette_kills == 0


@pytest.mark.skipif(not have_reference(), reason="oracle/_ref not built (no /root/reference)")
@pytest.mark.parametrize("seed", [5, 6])
def test_oracle_matches_live_reference(oracle, seed):
    R = Reference()
    rng = np.random.default_rng(seed)
    I = 120
    e = uniform_edges(-15.0, 15.0, I)
    mats = homogeneous(I, 1.3, 1.1, 0.1, 2.0)
    xc = 0.5 * (e[1:] + e[:-1])
    cen = np.exp(-(xc / 5) ** 2)
    cen = cen / cen.max() * (1 - 1e-3) + 1e-3
    src = np.zeros(1000, PARTICLE_DT)
    src["x"] = rng.uniform(-3, 3, src.size)
    src["mu"] = rng.uniform(-1, 1, src.size)
    src["w"] = rng.uniform(0.5, 3, src.size)
    src["t"] = 2.0
    to, ko, tro, co, _ = oracle.run_segment(e, mats, 2.0, 2.7, seed, 4, 4000, 20, src, 300,
                                            centers=cen, rho=3.0, chunk=256)
    tr_, kr, trr, cr = R.run_segment(e, mats, 2.0, 2.7, seed, 4, 4000, 20, src, 300,
                                     centers=cen, rho=3.0)
    assert co.tobytes() == cr.tobytes()
    assert ko.as_dict() == kr.as_dict()
    assert np.array_equal(tro, trr)
    for f in SEG_FIELDS:
        assert np.array_equal(getattr(to, f), getattr(tr_, f)), f


@pytest.mark.skipif(not have_reference(), reason="oracle/_ref not built (no /root/reference)")
def test_oracle_fourier_matches_live_reference(oracle):
    """hww_fourier's filter (filters.cpp:26-52) restated in C: bit-identical."""
    R = Reference()
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    L = oracle.lib
    L.orc_fourier_lowpass.argtypes = [C.POINTER(C.c_double), C.c_int32, C.c_int32,
                                      C.POINTER(C.c_double)]
    R.lib.hwwref_fourier_lowpass.argtypes = L.orc_fourier_lowpass.argtypes
    rng = np.random.default_rng(3)
    for M, cut in [(1, 0), (2, 0), (37, 5), (201, 30), (402, 30), (64, 40)]:
        g = np.ascontiguousarray(rng.standard_normal(M) * np.exp(-np.linspace(-3, 3, M) ** 2))
        o, r = np.zeros(M), np.zeros(M)
        assert L.orc_fourier_lowpass(dp(g), M, cut, dp(o)) == 0
        assert R.lib.hwwref_fourier_lowpass(dp(g), M, cut, dp(r)) == 0
        assert o.tobytes() == r.tobytes(), (M, cut)


@pytest.mark.skipif(not have_reference(), reason="oracle/_ref not built (no /root/reference)")
def test_oracle_fourier_driver_matches_live_reference(oracle):
    """A short hww_fourier run: oracle driver == reference driver, bit for bit."""
    from oracle.bind import DriverRun, make_config
    cfg = make_config(mode="hww_fourier", histories_per_step=1500, rho=3.0, fourier_cutoff=12,
                      cells=80, x_min=-10.0, x_max=10.0, t_end=1.5, time_steps=3, seed=4,
                      sigma_t=1.0, sigma_s=0.9, sigma_f=0.0, nu_f=0.0, speed=1.0)
    a, b = DriverRun(oracle, cfg), DriverRun(Reference(), cfg)
    for _ in range(3):
        (ra, xa), (rb, xb) = a.step(), b.step()
        for k in xa:
            assert np.array_equal(xa[k], xb[k], equal_nan=True), k
        assert ra.counters.collisions == rb.counters.collisions


@pytest.mark.skipif(not have_reference(), reason="oracle/_ref not built (no /root/reference)")
def test_oracle_config3_components_match_live_reference(oracle):
    """Config-3 pieces on the reference's own components (no
    reference driver exists, so the pin is per component): the segment
    transport over three material regions with particles born inside the step,
    and the LOSM assemble/solve with a source q (losm.cpp:101-103)."""
    R = Reference()
    I = 90
    e = uniform_edges(0.0, 30.0, I)
    xc = 0.5 * (e[1:] + e[:-1])
    mats = np.zeros((I, 5))
    for lo, hi, st, c in ((0, 10, 1.0, 0.5), (10, 20, 10.0, 0.1), (20, 30, 1.0, 0.99)):
        sel = (xc >= lo) & (xc < hi)
        mats[sel] = (st, c * st, 0.0, 0.0, 1.0)
    rng = np.random.default_rng(17)
    src = np.zeros(1500, PARTICLE_DT)
    src["x"] = rng.uniform(0, 2, src.size)
    src["mu"] = rng.uniform(-1, 1, src.size)
    src["w"] = 0.25
    src["t"] = rng.uniform(0.5, 1.0, src.size)
    cen = np.exp(-(xc / 8) ** 2)
    cen = cen / cen.max() * (1 - 1e-3) + 1e-3
    to, ko, tro, co, _ = oracle.run_segment(e, mats, 0.5, 1.0, 3, 2, 1500, 20, src, 0,
                                            centers=cen, rho=4.0, chunk=256)
    tr_, kr, trr, cr = R.run_segment(e, mats, 0.5, 1.0, 3, 2, 1500, 20, src, 0, centers=cen,
                                     rho=4.0)
    assert co.tobytes() == cr.tobytes()
    assert ko.as_dict() == kr.as_dict()
    assert np.array_equal(tro, trr)
    for f in SEG_FIELDS:
        assert np.array_equal(getattr(to, f), getattr(tr_, f)), f

    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    q = np.zeros(I)
    oracle.lib.orc_volume_q.argtypes = [C.POINTER(C.c_double), C.c_int] + [C.c_double] * 6 + [
        C.POINTER(C.c_double)]
    oracle.lib.orc_volume_q(dp(e), I, 0.0, 2.0, 0.5, 1.0, 0.5, 1.0, dp(q))
    assert abs(q.sum() - 1.0) < 1e-12 and np.all(q[xc > 2.0] == 0.0)
    mc = np.ascontiguousarray(mats)
    phi = np.ascontiguousarray(np.abs(rng.standard_normal(I + 2)))
    J = np.ascontiguousarray(0.1 * rng.standard_normal(I + 1))
    Fp = np.ascontiguousarray(0.05 * rng.standard_normal(I + 2))
    Fn = np.ascontiguousarray(0.05 * rng.standard_normal(I + 2))
    args = [C.c_int32, C.POINTER(C.c_double), C.c_void_p] + [C.POINTER(C.c_double)] * 2 + \
        [C.c_double] * 2 + [C.c_int32, C.POINTER(C.c_double)] + [C.c_double] * 2 + \
        [C.POINTER(C.c_double)] + [C.c_double] * 4 + [C.POINTER(C.c_double)] * 3
    oracle.lib.orc_assemble_solve.argtypes = args
    R.lib.hwwref_assemble_solve.argtypes = args
    for implicit in (0, 1):
        out = []
        for fn in (oracle.lib.orc_assemble_solve, R.lib.hwwref_assemble_solve):
            po, Jo = np.zeros(I + 2), np.zeros(I + 1)
            assert fn(I, dp(e), mc.ctypes.data, dp(phi), dp(J), 0.0, 0.0, implicit, dp(Fn),
                      0.01, -0.02, dp(Fp), 0.0, 0.0, 0.5, 0.5, dp(q), dp(po), dp(Jo)) == 0
            out.append((po, Jo))
        assert out[0][0].tobytes() == out[1][0].tobytes()
        assert out[0][1].tobytes() == out[1][1].tobytes()


def test_oracle_comb_walk_is_sequential(oracle):
    """The oracle's comb sums in bank order (np.add.accumulate is the same serial
    fp64 chain) on the adversarial banks the GPU comb test uses."""
    from tests.test_gpu_parity import comb_banks
    for name, b in comb_banks().items():
        out, iw, ow = oracle.uniform_comb(b, 997, 3, 17)
        assert iw == np.add.accumulate(b["w"])[-1], name
        sp = iw / 997
        assert np.all(out["w"] == sp)
        assert ow == np.add.accumulate(np.full(997, sp))[-1], name
