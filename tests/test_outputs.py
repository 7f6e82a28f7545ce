"""Run output files: step_<n>.csv, summary.csv and run.json
byte-compatible with the reference's writers (proj/src/driver.cpp:355-438).

CPU: the engine's writers (hwwg_write_*) and the reference's own writers
(oracle/_ref, through the shim) on the same synthetic records must produce the
same bytes — including nan columns, integral doubles, tiny/huge magnitudes and
the JSON number layout. GPU: an exact-mode run with out_dir against hww::run
with out_dir on the same config: identical step files; summary.csv identical
outside the wall-clock columns (tau and the FOMs built on it, as the
reference's own reproducibility test masks them, proj/tests/test_driver.cpp:34-51)."""
import ctypes as C
import json
import os

import numpy as np
import pytest

from oracle import bind
from paper_2512_19925_b200 import _capi as A
from paper_2512_19925_b200 import hww

needs_ref = pytest.mark.skipif(not bind.have_reference(), reason="oracle/_ref not built")


def _records(rng, I, n, with_windows):
    steps = []
    for k in range(n):
        a = lambda scale=1.0: rng.standard_normal(I) * scale * 10.0 ** rng.integers(-8, 8, I)
        s = {"phi_track": np.abs(a()), "sigma": np.abs(a(1e-3)), "phi_census": np.abs(a()),
             "current": a(), "closure": a(1e-2),
             "centers": (rng.random(I) if with_windows else None),
             "hybrid": (rng.random(I) * 3 if (with_windows and k % 2 == 0) else None),
             "tracks": rng.integers(0, 10**9, I).astype(np.uint64),
             "t_end": 0.5 * (k + 1), "tau": float(rng.random()), "fom_sigma_l2": float(1e18 * rng.random()),
             "census_weight": float(rng.random()), "census_weight_sigma": float(1e-4 * rng.random()),
             "normalization": 1000.0, "sigma_valid": 1.0 if k != 1 else 0.0,
             "hybrid_solve_failed": 1.0 if k == 2 else 0.0, "step": k + 1,
             "histories": 1000 + k, "comb_in": 5000 + k, "comb_out": 1000,
             "updates_applied": 3 - (k == 2),
             # reference diagnostics: some steps without a reference (NaN), some with
             "metrics": tuple(float("nan") if (k % 2 and j != 6) else
                              float(rng.random() * 10.0 ** rng.integers(-6, 20))
                              for j in range(7))}
        cn = bind.Counters()
        for j, (f, _) in enumerate(cn._fields_):
            setattr(cn, f, float(rng.random() * 7) if f.endswith("weight") else int(rng.integers(0, 10**12)))
        s["counters"] = cn
        steps.append(s)
    return steps


def _ours(out_dir, cfg_h, steps, edges, total_seconds):
    L = A.lib()
    recs = (A.StepRecordC * len(steps))()
    for r, s in zip(recs, steps):
        r.step, r.t_end, r.tau, r.fom_sigma_l2 = s["step"], s["t_end"], s["tau"], s["fom_sigma_l2"]
        r.census_weight, r.census_weight_sigma = s["census_weight"], s["census_weight_sigma"]
        r.sigma_valid, r.hybrid_solve_failed = int(s["sigma_valid"]), int(s["hybrid_solve_failed"])
        r.histories, r.comb_in, r.comb_out = s["histories"], s["comb_in"], s["comb_out"]
        r.updates_applied = s["updates_applied"]
        for f, v in zip(("rel_l2_error", "rel_mod_l2_error", "hybrid_rel_l2_error", "fom_err_l2",
                         "fom_err_mod", "fom_sigma_mod", "alpha"), s["metrics"]):
            setattr(r, f, v)
        for f, _ in s["counters"]._fields_:
            setattr(r.counters, f, getattr(s["counters"], f))
    d = str(out_dir).encode()
    for r, s in zip(recs, steps):
        arr = lambda k: A.as_dptr(np.ascontiguousarray(s[k])) if s[k] is not None else None
        keep = [np.ascontiguousarray(s[k]) for k in ("phi_track", "sigma", "phi_census", "current", "closure")]
        A.check(L.hwwg_write_step_csv(
            d, C.byref(r), len(edges) - 1, A.as_dptr(edges), *[A.as_dptr(x) for x in keep],
            arr("centers"), arr("hybrid"), A.as_u64ptr(np.ascontiguousarray(s["tracks"])),
            s["normalization"]))
    A.check(L.hwwg_write_summary_csv(d, recs, len(steps)))
    A.check(L.hwwg_write_run_json(d, C.byref(cfg_h.to_c()), total_seconds, len(steps)))


def _cfg_pair(**kw):
    h = hww.RunConfig(mode=kw.get("mode", "hww_ma"), histories_per_step=1000, rho=5.0,
                      ma_base_k=1, seed=kw.get("seed", 7), cells=kw.get("cells", 40),
                      x_min=-20.0, x_max=20.0, t_end=2.0, time_steps=4,
                      material=hww.Material(1.0, 0.9, 0.0, 0.0, 1.0),
                      update_fractions=kw.get("fractions", (0.25, 0.5, 0.75)))
    r = bind.make_config(mode=h.mode, histories_per_step=h.histories_per_step, rho=h.rho,
                         ma_base_k=h.ma_base_k, seed=h.seed, cells=h.cells, x_min=h.x_min,
                         x_max=h.x_max, t_end=h.t_end, time_steps=h.time_steps, sigma_t=1.0,
                         sigma_s=0.9, sigma_f=0.0, nu_f=0.0, speed=1.0,
                         update_fractions=h.update_fractions)
    return h, r


def _slurp(p):
    with open(p, "rb") as f:
        return f.read()


@needs_ref
@pytest.mark.parametrize("with_windows", [True, False])
def test_writers_byte_identical_to_reference(tmp_path, with_windows):
    rng = np.random.default_rng(11 if with_windows else 12)
    cfg_h, cfg_r = _cfg_pair(mode="hww_ma" if with_windows else "analog")
    steps = _records(rng, cfg_h.cells, 4, with_windows)
    edges = hww.build_uniform_mesh(cfg_h.x_min, cfg_h.x_max, cfg_h.cells).edges
    ref_dir, our_dir = tmp_path / "ref", tmp_path / "ours"
    bind.Reference().write_outputs(ref_dir, cfg_r, steps, 12.375)
    _ours(our_dir, cfg_h, steps, np.ascontiguousarray(edges, np.float64), 12.375)
    names = sorted(os.listdir(ref_dir))
    assert names == sorted(os.listdir(our_dir))
    assert "run.json" in names and "summary.csv" in names and "step_4.csv" in names
    for n in names:
        assert _slurp(our_dir / n) == _slurp(ref_dir / n), n


@needs_ref
def test_run_json_number_layout(tmp_path):
    """JSON doubles across the layout rule's branches (integral, fixed, small,
    exponent) against the reference's writer."""
    for i, vals in enumerate([(1.0, 1e-3, 0.25), (123456789012.0, 3.5e-7, 2.5e16),
                              (1e-5, 0.1, 1.0 / 3.0)]):
        cfg_h, cfg_r = _cfg_pair(fractions=vals)
        cfg_h.eps_min = cfg_r.eps_min = vals[1]
        cfg_h.theta = cfg_r.theta = 0.5 + 0.5 * vals[2] / (1 + vals[2])
        ref_dir, our_dir = tmp_path / f"r{i}", tmp_path / f"o{i}"
        bind.Reference().write_outputs(ref_dir, cfg_r, [], vals[0])
        _ours(our_dir, cfg_h, [], np.zeros(cfg_h.cells + 1), vals[0])
        assert _slurp(our_dir / "run.json") == _slurp(ref_dir / "run.json")
        json.loads(_slurp(our_dir / "run.json"))


def _mask_summary(p):
    out = []
    for line in _slurp(p).decode().splitlines():
        f = line.split(",")
        out.append(",".join(" -" if (i == 3 or 7 <= i <= 10) else v for i, v in enumerate(f)))
    return out


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("mode,with_reference", [("hww_ma", False), ("analog", False),
                                                 ("hww_ma", True), ("analog", True)])
def test_exact_run_outputs_match_reference_run(tmp_path, mode, with_reference):
    """With a reference file (hww_main.cpp:250-256) the summary's error metrics
    (rel_l2_error, rel_mod_l2_error, hybrid_rel_l2_error, alpha) must match byte
    for byte too; the FOM columns carry the wall-clock tau and stay masked."""
    cfg_h, cfg_r = _cfg_pair(mode=mode, cells=80)
    ref_dir, our_dir = tmp_path / "ref", tmp_path / "ours"
    R = bind.Reference()
    reference = None
    if with_reference:
        path = tmp_path / "reference.csv"
        R.save_reference(cfg_r, path, *R.compute_reference(cfg_r, 3, 8, 8))
        cfg_h.reference = str(path)
        reference = hww.load_reference(path, cfg_h.make_mesh(), cfg_h.time_layers())
    R.run_to_dir(cfg_r, ref_dir, reference=cfg_h.reference)
    hww.run(cfg_h, rng_mode=hww.RNG_EXACT, out_dir=str(our_dir), reference=reference)
    if with_reference:
        rows = _slurp(our_dir / "summary.csv").decode().splitlines()[1:]
        assert all("nan" not in r.split(",")[4] for r in rows)
    for k in range(1, cfg_h.time_steps + 1):
        assert _slurp(our_dir / f"step_{k}.csv") == _slurp(ref_dir / f"step_{k}.csv"), k
    assert _mask_summary(our_dir / "summary.csv") == _mask_summary(ref_dir / "summary.csv")
    jo, jr = (json.loads(_slurp(d / "run.json")) for d in (our_dir, ref_dir))
    jo.pop("total_seconds"), jr.pop("total_seconds")
    assert jo == jr
