#!/usr/bin/env python3
"""Generate the golden vectors under tests/golden/ from the REAL reference.

Runs the unmodified reference (oracle/_ref/libhww_ref.so, compiled from
/root/reference/proj by oracle/Makefile) through its own public API:
  * segments.npz — hww::run_segment_parallel on seeded inputs (analog, flat
    windows with fission, shaped windows at a nonzero h_begin, edge cases);
  * driver_c{0,1,2}.npz — hww::run_step sequences of BASELINE configs 0-2 at
    reduced histories (per-step counters, record scalars, per-cell arrays and
    the census bank of the last step);
  * components.npz — assemble_solve, build_centers, moving_average,
    uniform_comb, update_thresholds on seeded inputs.

Usage:  python tests/golden/make_golden.py        (needs /root/reference)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.bind import (PARTICLE_DT, DriverRun, Reference, baseline_config,  # noqa: E402
                         homogeneous, uniform_edges)

SEG_FIELDS = ("track_flux", "track_flux_batch", "census_phi", "census_current",
              "census_closure", "census_weight_batch", "edge_current")


def segment_cases():
    """(name, kwargs) of the segment-level golden cases."""
    cases = []
    rng = np.random.default_rng(20251219)
    # a) config-1 slab (c = 1), analog, pulse on edge 100 (mu<0 zero-length crossings)
    I = 200
    e = uniform_edges(-20.0, 20.0, I)
    src = np.zeros(2000, PARTICLE_DT)
    src["mu"] = rng.uniform(-1, 1, src.size)
    src["w"] = 1.0
    cases.append(("analog_c1", dict(edges=e, mats=homogeneous(I, 1.0, 1.0), t_begin=0.0,
                                     t_end=1.0, seed=42, step=1, H=2000, B=20, src=src,
                                     h_begin=0, centers=None, rho=1.0)))
    # b) the reference's hww_bench problem: fission nu = 2.3, flat windows rho = 1.25
    I = 201
    e = uniform_edges(-20.5, 20.5, I)
    src = np.zeros(2000, PARTICLE_DT)
    src["mu"] = rng.uniform(-1, 1, src.size)
    src["w"] = 1.0
    cases.append(("bench_fission", dict(edges=e, mats=homogeneous(I, 1.0, 1 / 3, 1 / 3, 2.3),
                                         t_begin=0.0, t_end=1.0, seed=1, step=1, H=2000,
                                         B=20, src=src, h_begin=0, centers=np.ones(I),
                                         rho=1.25)))
    # c) c = 0.9, shaped windows rho = 5, step 3, a mid-step segment h_begin = 700
    I = 400
    e = uniform_edges(-20.0, 20.0, I)
    xc = 0.5 * (e[1:] + e[:-1])
    cen = np.exp(-np.abs(xc) / 3.0)
    cen = cen / cen.max() * (1 - 1e-3) + 1e-3
    src = np.zeros(1500, PARTICLE_DT)
    src["x"] = rng.uniform(-6, 6, src.size)
    src["mu"] = rng.uniform(-1, 1, src.size)
    src["w"] = rng.uniform(0.2, 2.0, src.size)
    src["t"] = 1.0
    cases.append(("windows_c09", dict(edges=e, mats=homogeneous(I, 1.0, 0.9), t_begin=1.0,
                                       t_end=1.5, seed=7, step=3, H=3000, B=20, src=src,
                                       h_begin=700, centers=cen, rho=5.0)))
    # d) edge cases: NaN / zero / negative weights (nan_aborts), x == x_max,
    #    grazing leak, near-void free flight, heavy split (w >> centre)
    I = 10
    e = uniform_edges(-5.0, 5.0, I)
    mats = homogeneous(I, 1.0, 0.5)
    mats[3] = (1e-12, 0.0, 0.0, 0.0, 1.0)
    src = np.zeros(8, PARTICLE_DT)
    src["w"] = [1.0, np.nan, 0.0, -1.0, 1.0, 1.0, 300.0, 1.0]
    src["x"] = [0.0, 0.0, 0.0, 0.0, 5.0, -5.0, 0.3, -1.5]
    src["mu"] = [0.5, 0.5, 0.5, 0.5, 1.0, -1e-12, -0.7, 1.0]
    cen = np.full(I, 0.5)
    cases.append(("edge_cases", dict(edges=e, mats=mats, t_begin=0.0, t_end=1.0, seed=3,
                                      step=2, H=8, B=2, src=src, h_begin=0, centers=cen,
                                      rho=2.0)))
    return cases


def run_case(R, kw):
    t, k, tr, census = R.run_segment(kw["edges"], kw["mats"], kw["t_begin"], kw["t_end"],
                                     kw["seed"], kw["step"], kw["H"], kw["B"], kw["src"],
                                     kw["h_begin"], centers=kw["centers"], rho=kw["rho"],
                                     parallel=True, chunk=256)
    return t, k, tr, census


def main():
    R = Reference()
    out = {}
    for name, kw in segment_cases():
        t, k, tr, census = run_case(R, kw)
        for f in SEG_FIELDS:
            out[f"{name}.{f}"] = getattr(t, f)
        out[f"{name}.scalars"] = np.array([t.boundary_closure_left, t.boundary_closure_right,
                                           t.histories_scored, t.grazing_discarded], float)
        out[f"{name}.counters_u"] = np.array([getattr(k, n) for n, _ in k._fields_[:9]], np.uint64)
        out[f"{name}.counters_d"] = np.array([k.leakage_weight, k.aborted_weight])
        out[f"{name}.tracks"] = tr
        out[f"{name}.census"] = census
    np.savez_compressed(os.path.join(HERE, "segments.npz"), **out)

    for which, H, N in ((0, 1500, 4), (1, 3000, 5), (2, 3000, 4)):
        cfg = baseline_config(which, histories=H, time_steps=N)
        d = DriverRun(R, cfg)
        g = {}
        for s in range(N):
            o, arr = d.step()
            g[f"s{s+1}.counters_u"] = np.array([getattr(o.counters, n) for n, _ in
                                                o.counters._fields_[:9]], np.uint64)
            g[f"s{s+1}.counters_d"] = np.array([o.counters.leakage_weight,
                                                o.counters.aborted_weight])
            g[f"s{s+1}.ints"] = np.array([o.segments, o.census_size, o.histories, o.comb_in,
                                          o.comb_out, o.updates_applied, o.hybrid_solve_failed,
                                          o.n_thresholds, o.sigma_valid, o.has_windows,
                                          o.has_hybrid], np.uint64)
            g[f"s{s+1}.scalars"] = np.array([o.census_weight, o.census_weight_sigma,
                                             o.boundary_closure_left, o.boundary_closure_right,
                                             o.comb_in_weight, o.comb_out_weight])
            for kname, v in arr.items():
                g[f"s{s+1}.{kname}"] = v
        g["bank"] = d.bank()
        np.savez_compressed(os.path.join(HERE, f"driver_c{which}.npz"), **g)

    np.savez_compressed(os.path.join(HERE, "components.npz"), **component_vectors(R))
    print("golden vectors written to", HERE)


def component_vectors(R):
    import ctypes as C
    L = R.lib
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    rng = np.random.default_rng(4242)
    g = {}
    # LOSM: lagged and implicit solves on a c = 0.9 slab with noisy inputs
    for name, I, implicit, theta, dt in (("losm_lag", 40, 0, 1.0, 0.5),
                                         ("losm_imp", 400, 1, 0.5, 0.5)):
        e = uniform_edges(-20.0, 20.0, I)
        mats = homogeneous(I, 1.0, 0.9)
        phi = np.abs(rng.normal(1.0, 0.3, I + 2))
        J = rng.normal(0.0, 0.1, I + 1)
        Fp = rng.normal(0.0, 0.05, I + 2)
        Fn = rng.normal(0.0, 0.05, I + 2)
        po, Jo = np.zeros(I + 2), np.zeros(I + 1)
        L.hwwref_assemble_solve.argtypes = [C.c_int32, C.POINTER(C.c_double), C.c_void_p] + \
            [C.POINTER(C.c_double)] * 2 + [C.c_double] * 2 + [C.c_int32, C.POINTER(C.c_double)] + \
            [C.c_double] * 2 + [C.POINTER(C.c_double)] + [C.c_double] * 4 + \
            [C.POINTER(C.c_double)] * 3
        rc = L.hwwref_assemble_solve(I, dp(e), mats.ctypes.data, dp(phi), dp(J), 0.0, 0.0,
                                     implicit, dp(Fn), 0.013, -0.02, dp(Fp), 0.011, 0.004,
                                     theta, dt, None, dp(po), dp(Jo))
        assert rc == 0
        g.update({f"{name}.in_phi": phi, f"{name}.in_J": J, f"{name}.in_Fp": Fp,
                  f"{name}.in_Fn": Fn, f"{name}.edges": e, f"{name}.mats": mats,
                  f"{name}.params": np.array([implicit, theta, dt, 0.013, -0.02, 0.011, 0.004]),
                  f"{name}.phi": po, f"{name}.J": Jo})
    # moving average k = 1, 2, 3 on noise
    v = rng.normal(size=57)
    g["ma.in"] = v
    for k in (0, 1, 2, 3):
        o = np.zeros(v.size)
        L.hwwref_moving_average.argtypes = [C.POINTER(C.c_double), C.c_int32, C.c_int32,
                                            C.POINTER(C.c_double)]
        L.hwwref_moving_average(dp(v), v.size, k, dp(o))
        g[f"ma.k{k}"] = o
    # build_centers with negatives and a fallback
    phi = rng.normal(0.5, 0.5, 101)
    c = np.zeros(phi.size)
    L.hwwref_build_centers.argtypes = [C.POINTER(C.c_double), C.c_int32, C.c_double,
                                       C.c_double, C.POINTER(C.c_double)]
    fb = L.hwwref_build_centers(dp(phi), phi.size, 1e-3, 5.0, dp(c))
    g.update({"centers.in": phi, "centers.out": c, "centers.fallback": np.array([fb])})
    # comb: weights over six decades, up and down
    n = 5000
    bank = np.zeros(n, PARTICLE_DT)
    bank["x"] = rng.uniform(-10, 10, n)
    bank["mu"] = rng.uniform(-1, 1, n)
    bank["w"] = 10.0 ** (-6.0 * rng.uniform(size=n))
    bank["t"] = 1.0
    L.hwwref_uniform_comb.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                      C.c_uint64, C.c_void_p, C.POINTER(C.c_double),
                                      C.POINTER(C.c_double)]
    g["comb.bank"] = bank
    for tgt in (5000, 137, 12000):
        out = np.zeros(tgt, PARTICLE_DT)
        iw, ow = C.c_double(), C.c_double()
        sid = (3 << 56) ^ (4 << 40)
        rc = L.hwwref_uniform_comb(bank.ctypes.data, n, tgt, 9, sid, out.ctypes.data,
                                   C.byref(iw), C.byref(ow))
        assert rc == 0
        g[f"comb.t{tgt}"] = out
        g[f"comb.t{tgt}.w"] = np.array([iw.value, ow.value])
    return g


if __name__ == "__main__":
    main()
