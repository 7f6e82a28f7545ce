"""Reference solution files and step error diagnostics.

* hwwg_save_reference_csv vs hww::save_reference (proj/src/reference.cpp:374-393):
  same bytes for the same arrays;
* hwwg_load_reference_csv vs hww::load_reference (reference.cpp:395-456): same
  arrays from the reference's own file, and the same failure (and message) on
  every shape/format error the loader checks, including the mismatched-mesh case
  of the reference's own test (proj/tests/test_reference.cpp:199-225);
* hwwg_step_metrics vs hww::run_step's diagnostics (proj/src/driver.cpp:231-275):
  the reference driver runs against a reference file; the engine's metric
  function on that run's own arrays and tau gives bit-identical StepMetrics.

Everything here is host code (no GPU); the reference side is oracle/_ref."""
import ctypes as C

import numpy as np
import pytest

from oracle import bind
from paper_2512_19925_b200 import _capi as A
from paper_2512_19925_b200 import hww

needs_ref = pytest.mark.skipif(not bind.have_reference(), reason="oracle/_ref not built")

METRICS = ("rel_l2_error", "rel_mod_l2_error", "hybrid_rel_l2_error", "fom_err_l2",
           "fom_err_mod", "fom_sigma_l2", "fom_sigma_mod", "alpha")


def _test_config(**kw):
    """The reference test's case: benchmark config on 21 cells of [-2, 2], 2 steps
    to t = 2 (test_reference.cpp:199-206)."""
    base = dict(mode="hww", histories_per_step=10000, ma_base_k=3, seed=1, cells=21,
                x_min=-2.0, x_max=2.0, t_end=2.0, time_steps=2)
    base.update(kw)
    r = bind.make_config(**base)
    h = hww.RunConfig(cells=r.cells, x_min=r.x_min, x_max=r.x_max, t_end=r.t_end,
                      time_steps=r.time_steps)
    return h, r


def _grids(h):
    return h.make_mesh(), h.time_layers()


def _slurp(p):
    with open(p, "rb") as f:
        return f.read()


def test_time_layers_match_time_grid():
    h = hww.RunConfig(t_end=7.3, time_steps=13)
    lay = h.time_layers()
    dt = 7.3 / 13
    assert lay.size == 14 and lay[-1] == 7.3
    assert all(lay[n] == 0.0 + n * dt for n in range(13))


@needs_ref
@pytest.mark.parametrize("which", ["test", 1])
def test_save_reference_same_bytes(tmp_path, which):
    R = bind.Reference()
    if which == "test":
        h, r = _test_config()
        lay, itv = R.compute_reference(r, 3, 4, 4)
    else:
        r = bind.baseline_config(1, time_steps=4)
        h = hww.RunConfig(cells=r.cells, x_min=r.x_min, x_max=r.x_max, t_end=r.t_end,
                          time_steps=r.time_steps)
        lay, itv = R.compute_reference(r, 5, 20, 16)
    R.save_reference(r, tmp_path / "ref.csv", lay, itv)
    mesh, layers = _grids(h)
    hww.save_reference(hww.ReferenceSolution(mesh, layers, lay, itv), tmp_path / "ours.csv")
    assert _slurp(tmp_path / "ours.csv") == _slurp(tmp_path / "ref.csv")
    # the engine reads the reference's file back to the same arrays as the reference
    ours = hww.load_reference(tmp_path / "ref.csv", mesh, layers)
    rl, ri = R.load_reference(r, tmp_path / "ref.csv")
    assert np.array_equal(ours.phi_layer, rl) and np.array_equal(ours.phi_interval, ri)
    assert np.array_equal(ours.phi_layer, lay) and np.array_equal(ours.phi_interval, itv)


def _mutations(text):
    """(name, file text, config overrides for the LOADER) — each must fail."""
    lines = text.splitlines(keepends=True)
    head, rows = lines[0], lines[1:]
    bad_cell = rows[5].split(",")
    bad_cell[1] = " 6"
    bad_t = rows[30].split(",")
    bad_t[0] = repr(float(bad_t[0]) + 1e-6)
    bad_x = rows[3].split(",")
    bad_x[2] = " " + repr(float(bad_x[2]) + 1e-3)
    return [
        ("other mesh", text, dict(cells=11)),
        ("other time grid", text, dict(t_end=3.0)),
        ("more steps", text, dict(time_steps=3, t_end=3.0)),
        ("truncated", "".join(lines[:-1]), {}),
        ("extra row", text + rows[-1], {}),
        ("four tokens", head + "".join(rows[:7]) + "1.0, 2, 3.0, 4.0\n" + "".join(rows[8:]), {}),
        ("not a number", head + rows[0].replace(rows[0].split(",")[3], " abc", 1) +
         "".join(rows[1:]), {}),
        ("cell index", head + "".join(rows[:5]) + ",".join(bad_cell) + "".join(rows[6:]), {}),
        ("layer time", head + "".join(rows[:30]) + ",".join(bad_t) + "".join(rows[31:]), {}),
        ("cell centre", head + "".join(rows[:3]) + ",".join(bad_x) + "".join(rows[4:]), {}),
        ("empty", "", {}),
        ("header only", head, {}),
    ]


@needs_ref
def test_load_reference_rejects_what_the_reference_rejects(tmp_path):
    R = bind.Reference()
    h, r = _test_config()
    lay, itv = R.compute_reference(r, 3, 4, 4)
    R.save_reference(r, tmp_path / "ref.csv", lay, itv)
    text = _slurp(tmp_path / "ref.csv").decode()
    # blank lines are skipped by both loaders
    blank = tmp_path / "blank.csv"
    blank.write_text(text.replace("\n", "\n\n", 5))
    hl, hr = _test_config()
    ours = hww.load_reference(blank, *_grids(hl))
    assert np.array_equal(ours.phi_layer, R.load_reference(hr, blank)[0])
    for k, (name, body, over) in enumerate(_mutations(text)):
        p = tmp_path / f"m{k}.csv"
        p.write_text(body)
        hl, rl = _test_config(**over)
        with pytest.raises(RuntimeError) as ref_err:
            R.load_reference(rl, p)
        with pytest.raises(A.HwwgError) as our_err:
            hww.load_reference(p, *_grids(hl))
        assert our_err.value.code == A.HWWG_EFORMAT, name
        assert str(our_err.value).endswith(str(ref_err.value)), (name, str(our_err.value),
                                                                 str(ref_err.value))
    missing = tmp_path / "nope.csv"
    with pytest.raises(RuntimeError) as ref_err:
        R.load_reference(r, missing)
    with pytest.raises(A.HwwgError) as our_err:
        hww.load_reference(missing, *_grids(h))
    assert str(our_err.value).endswith(str(ref_err.value))


def _rec_from(out, m):
    rec = A.StepRecordC()
    rec.step, rec.tau, rec.sigma_valid = out.step, m["tau"], out.sigma_valid
    return rec


def _same(a, b):
    return (np.isnan(a) and np.isnan(b)) or a == b


@needs_ref
@pytest.mark.parametrize("which,mode,steps", [(1, "hww_ma", 5), (2, "hww_ma", 4),
                                              (1, "analog", 3), (0, "hww", 3)])
def test_step_metrics_bit_identical_to_reference_driver(tmp_path, which, mode, steps):
    R = bind.Reference()
    r = bind.baseline_config(which, histories=3000, time_steps=steps, mode=mode)
    h = hww.RunConfig(cells=r.cells, x_min=r.x_min, x_max=r.x_max, t_end=r.t_end,
                      time_steps=r.time_steps)
    lay, itv = R.compute_reference(r, 3, 8, 8)
    R.save_reference(r, tmp_path / "ref.csv", lay, itv)
    mesh, layers = _grids(h)
    ref = hww.load_reference(tmp_path / "ref.csv", mesh, layers)
    drv = bind.DriverRun(R, r)
    drv.load_reference(tmp_path / "ref.csv")
    seen_hybrid = 0
    try:
        for _ in range(steps):
            out, arr = drv.step()
            m = drv.metrics()
            rec = _rec_from(out, m)
            hyb = arr["phi_hybrid"] if out.has_hybrid else None
            seen_hybrid += hyb is not None
            hww.step_metrics(mesh, rec, arr["phi_track"], arr["sigma"], hyb, ref)
            for k in METRICS:
                assert _same(getattr(rec, k), m[k]), (out.step, k, getattr(rec, k), m[k])
            assert not np.isnan(rec.rel_l2_error) and not np.isnan(rec.alpha)
    finally:
        drv.close()
    assert seen_hybrid == (steps if mode != "analog" else 0)


@needs_ref
def test_step_metrics_without_reference_match(tmp_path):
    """No reference: only fom_sigma_l2 (driver.cpp:272-275)."""
    R = bind.Reference()
    r = bind.baseline_config(1, histories=3000, time_steps=3)
    mesh = hww.build_uniform_mesh(r.x_min, r.x_max, r.cells)
    drv = bind.DriverRun(R, r)
    try:
        for _ in range(3):
            out, arr = drv.step()
            m = drv.metrics()
            rec = _rec_from(out, m)
            hww.step_metrics(mesh, rec, arr["phi_track"], arr["sigma"], arr["phi_hybrid"])
            for k in METRICS:
                assert _same(getattr(rec, k), m[k]), (k, getattr(rec, k), m[k])
            assert np.isnan(rec.rel_l2_error) and not np.isnan(rec.fom_sigma_l2)
    finally:
        drv.close()


def test_step_metrics_zero_reference_layer_is_invalid():
    """relative_change throws std::invalid_argument on a zero layer (metrics.cpp:61)."""
    mesh = hww.build_uniform_mesh(-1.0, 1.0, 8)
    layers = np.array([0.0, 1.0])
    ref = hww.ReferenceSolution(mesh, layers, np.zeros((2, 8)), np.ones((1, 8)))
    rec = A.StepRecordC()
    rec.step, rec.tau = 1, 0.5
    with pytest.raises(ValueError, match="relative_change"):
        hww.step_metrics(mesh, rec, np.ones(8), None, None, ref)


def test_step_metrics_masks_and_exclusions():
    """Hand-checked values: the modified norms keep cells whose reference layer is
    below phi* = 1e-3 (driver.cpp:21), fom skips zero entries (metrics.cpp:44-47)."""
    mesh = hww.build_uniform_mesh(0.0, 4.0, 4)  # unit widths
    layers = np.array([0.0, 1.0])
    lay = np.array([[1.0, 1.0, 1.0, 1.0], [2.0, 1e-4, 3.0, 0.0]])
    itv = np.array([[1.0, 2.0, 2.0, 4.0]])
    ref = hww.ReferenceSolution(mesh, layers, lay, itv)
    rec = A.StepRecordC()
    rec.step, rec.tau, rec.sigma_valid = 1, 0.25, 1
    phi = np.array([1.0, 2.5, 2.0, 3.0])  # err = [0, .5, 0, -1]
    sig = np.array([0.5, 0.0, 1.0, 2.0])
    hww.step_metrics(mesh, rec, phi, sig, np.array([2.0, 0.0, 3.0, 1.0]), ref)
    assert rec.rel_l2_error == np.sqrt(1.25) / np.sqrt(25.0)
    assert rec.rel_mod_l2_error == np.sqrt(1.25) / np.sqrt(20.0)  # cells 1, 3
    assert rec.hybrid_rel_l2_error == np.sqrt(1e-8 + 1.0) / np.sqrt(4.0 + 1e-8 + 9.0)
    f1, f3 = 1.0 / (0.25 * 0.25), 1.0 / (0.25 * 1.0)  # err 0 cells excluded
    assert rec.fom_err_l2 == np.sqrt(f1 * f1 + f3 * f3)
    assert rec.fom_err_mod == np.sqrt(f1 * f1 + f3 * f3)
    s0, s2, s3 = 1.0 / (0.25 * 0.25), 1.0 / 0.25, 1.0 / (0.25 * 4.0)  # sigma 0 excluded
    assert rec.fom_sigma_l2 == np.sqrt(s0 * s0 + s2 * s2 + s3 * s3)
    assert rec.fom_sigma_mod == np.sqrt(s3 * s3)
    diff = lay[1] - lay[0]
    assert rec.alpha == np.sqrt(np.sum(diff * diff)) / np.sqrt(np.sum(lay[1] * lay[1]))
