"""Device S_N reference: hwwg_sn_solve / hwwg_compute_reference
against the reference's own hww::sn_solve / hww::compute_reference
(proj/src/reference.cpp:14-372, compiled into oracle/_ref).

Tolerance: the device sweep composes each thread's run of the diamond-difference
recurrence as an affine map and scans the maps across the block, so the flux
entering a run differs from the sequential sweep by a few ulp; everything else
(the quadrature, the phi sums in direction order, the residual, the projection
and the trapezoid interval averages) runs in the reference's arithmetic order.
The source iteration stops at a relative max-norm residual of 1e-9, so a step
whose residual lands on the tolerance could take one iteration more or less than
the reference; the results are compared at 1e-9 of each layer's maximum (the
solver's own convergence tolerance) and are typically within 1e-13."""
import time

import numpy as np
import pytest

from oracle import bind
from paper_2512_19925_b200 import hww

needs_ref = pytest.mark.skipif(not bind.have_reference(), reason="oracle/_ref not built")
TOL = 1e-9


def _rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    scale = np.maximum(np.abs(b).max(axis=-1, keepdims=True), 1e-300)
    return float(np.max(np.abs(a - b) / scale))


def _h_config(r, **kw):
    """hww.RunConfig with bind.Config r's fields."""
    m = hww.Material(r.sigma_t, r.sigma_s, r.sigma_f, r.nu_f, r.speed)
    c = hww.RunConfig(mode=hww.MODES[r.mode], histories_per_step=r.histories_per_step,
                      material=m, x_min=r.x_min, x_max=r.x_max, cells=r.cells, t_end=r.t_end,
                      time_steps=r.time_steps, source_x0=r.x0, source_strength=r.strength,
                      seed=r.seed, rho=r.rho, ma_base_k=r.ma_base_k)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


@needs_ref
def test_gauss_legendre_matches_reference():
    R = bind.Reference()
    for n in (2, 4, 8, 16, 32, 64, 128, 256):
        mu, w = hww.gauss_legendre(n)
        rm, rw = R.gauss_legendre(n)
        assert np.array_equal(mu, rm) and np.array_equal(w, rw), n
    for bad in (0, 1, 3, 17):
        with pytest.raises(ValueError, match="quadrature order must be even"):
            hww.gauss_legendre(bad)


CASES = {
    # the reference's own unit-test case (test_reference.cpp:199-206), coarse oracle
    "unit": (dict(which=0, cells=21, x_min=-2.0, x_max=2.0, t_end=2.0, time_steps=2), (3, 4, 4)),
    # config 1 (pulse on an interior edge: split across two cells), default oracle
    "c1": (dict(which=1), (5, 20, 16)),
    # config 2, default oracle
    "c2": (dict(which=2), (5, 20, 16)),
    # the reference's benchmark.cfg: fission (nu sigma_f in the source), 201 cells
    "bench": (dict(which=0), (5, 20, 16)),
    # off-edge pulse, S8, odd refinement
    "c1_offedge": (dict(which=1, x0=0.37, time_steps=8, t_end=8.0), (3, 7, 8)),
}


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("case", sorted(CASES))
def test_compute_reference_matches_reference(case):
    kw, (sr, tr, sn) = CASES[case]
    kw = dict(kw)
    r = bind.baseline_config(kw.pop("which"), **kw)
    ref_lay, ref_itv = bind.Reference().compute_reference(r, sr, tr, sn)
    ours = hww.compute_reference(_h_config(r), sr, tr, sn)
    e_lay, e_itv = _rel(ours.phi_layer, ref_lay), _rel(ours.phi_interval, ref_itv)
    print(f"{case}: layer rel {e_lay:.2e}, interval rel {e_itv:.2e}")
    assert e_lay <= TOL and e_itv <= TOL, (e_lay, e_itv)


def _general_problem(rng, I=157, N=9, K=8):
    edges = np.concatenate([[-3.0], -3.0 + np.cumsum(rng.uniform(0.02, 0.08, I))])
    mats = np.zeros((I, 5))
    mats[:, 0] = rng.uniform(0.5, 3.0, I)                 # sigma_t
    mats[:, 1] = mats[:, 0] * rng.uniform(0.0, 0.8, I)    # sigma_s
    mats[:, 2] = mats[:, 0] * rng.uniform(0.0, 0.1, I)    # sigma_f
    mats[:, 3] = rng.uniform(0.0, 2.5, I)                 # nu_f
    mats[:, 4] = rng.uniform(0.5, 2.0, I)                 # speed
    layers = np.concatenate([[0.0], np.cumsum(rng.uniform(0.01, 0.2, N))])
    psi0 = rng.uniform(0.0, 1.0, (K, I))
    inc_l, inc_r, q = rng.uniform(0, 2, K), rng.uniform(0, 2, K), rng.uniform(0, 0.5, I)
    return edges, mats, layers, K, psi0, inc_l, inc_r, q


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("seed", [1, 2])
def test_sn_solve_general_problem_matches_reference(seed):
    """Nonuniform mesh and time layers, heterogeneous fissile materials, incoming
    boundary fluxes and a source: the general solver, layer by layer."""
    rng = np.random.default_rng(seed)
    edges, mats, layers, K, psi0, il, ir, q = _general_problem(rng)
    ref_phi, ref_it = bind.Reference().sn_solve(edges, mats, layers, K, psi0, il, ir, q)
    mat_dt = np.zeros(len(mats), hww.A.MATERIAL_DT)
    for j, f in enumerate(("sigma_t", "sigma_s", "sigma_f", "nu_f", "speed")):
        mat_dt[f] = mats[:, j]
    phi, its = hww.sn_solve(hww.Mesh1D(edges), mat_dt, layers, K, psi0, il, ir, q)
    assert np.array_equal(phi[0], ref_phi[0])  # layer 0: the moments of psi0, same order
    assert _rel(phi, ref_phi) <= TOL, _rel(phi, ref_phi)
    assert np.sum(its != ref_it) <= 1, (its, ref_it)


@pytest.mark.gpu
@needs_ref
def test_sn_solve_nonconvergence_and_errors_match_reference():
    rng = np.random.default_rng(5)
    edges, mats, layers, K, psi0, il, ir, q = _general_problem(rng, I=40, N=3, K=4)
    mat_dt = np.zeros(len(mats), hww.A.MATERIAL_DT)
    for j, f in enumerate(("sigma_t", "sigma_s", "sigma_f", "nu_f", "speed")):
        mat_dt[f] = mats[:, j]
    R = bind.Reference()
    with pytest.raises(RuntimeError) as ref_err:
        R.sn_solve(edges, mats, layers, K, psi0, il, ir, q, tolerance=1e-15, max_iterations=2)
    with pytest.raises(RuntimeError) as our_err:
        hww.sn_solve(hww.Mesh1D(edges), mat_dt, layers, K, psi0, il, ir, q, tolerance=1e-15,
                     max_iterations=2)
    assert str(our_err.value).endswith(str(ref_err.value)), (str(our_err.value),
                                                             str(ref_err.value))
    with pytest.raises(ValueError, match="quadrature order must be even"):
        hww.sn_solve(hww.Mesh1D(edges), mat_dt, layers, 3, psi0[:3], None, None, None)


@pytest.mark.gpu
@needs_ref
def test_config4_reference_on_the_device():
    """Config 4's grids (4000 cells x5, 100 steps x20, S16) — three minutes of
    the reference's host solve — on the device, checked against the reference on
    the first 5 steps of the same grid and timed over all 100."""
    r5 = bind.baseline_config(4, time_steps=5)
    t = time.perf_counter()
    ref_lay, ref_itv = bind.Reference().compute_reference(r5)
    t_ref5 = time.perf_counter() - t
    ours5 = hww.compute_reference(_h_config(r5))
    assert _rel(ours5.phi_layer, ref_lay) <= TOL and _rel(ours5.phi_interval, ref_itv) <= TOL
    r = bind.baseline_config(4)
    hww.compute_reference(_h_config(r, time_steps=2, t_end=1.0))  # warm the context
    t = time.perf_counter()
    full = hww.compute_reference(_h_config(r))
    t_gpu = time.perf_counter() - t
    print(f"config 4 S_N reference: device {t_gpu:.3f} s for 100 steps; "
          f"reference host {t_ref5:.2f} s for 5 steps")
    assert full.phi_layer.shape == (101, 4000) and np.all(np.isfinite(full.phi_interval))
    # particle balance sanity: no source, pure absorber 1% -> total flux decays
    tot = full.phi_layer.sum(axis=1)
    assert np.all(np.diff(tot) < 0)


@pytest.mark.gpu
@needs_ref
def test_driver_auto_reference_equals_reference_file(tmp_path):
    """Driver.compute_reference() (reference = "auto") gives the same step metrics as
    the reference's compute_reference saved to a file and loaded."""
    r = bind.baseline_config(1, histories=20000, time_steps=4)
    h = _h_config(r)
    R = bind.Reference()
    path = tmp_path / "reference.csv"
    R.save_reference(r, path, *R.compute_reference(r))
    recs = {}
    for how in ("auto", "file"):
        d = hww.Driver(h, rng_mode=hww.RNG_EXACT)
        if how == "auto":
            d.compute_reference()
        else:
            d.load_reference(path)
        recs[how] = [d.step() for _ in range(4)]
        d.close()
    for a, b in zip(recs["auto"], recs["file"]):
        for k in ("rel_l2_error", "rel_mod_l2_error", "hybrid_rel_l2_error", "alpha"):
            x, y = getattr(a, k), getattr(b, k)
            assert np.isfinite(x) and abs(x - y) <= 1e-7 * abs(y), (k, x, y)
