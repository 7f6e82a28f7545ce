"""Throughput (Philox) mode against the reference algorithm: statistical parity.

The Philox mode draws different random numbers than the reference, so it is
judged as an estimator: tallies agree within a few combined
standard errors on >= 95% of the well-sampled cells, with sigma from batch
statistics (step 1, common pulse source) or from independent replicates
(later steps, where the comb adds inter-step noise the batch sigma misses —
proj/tests/acceptance_main.cpp:225-231, 270, 283-285)."""
import numpy as np
import pytest

import paper_2512_19925_b200 as hw

pytestmark = pytest.mark.gpu


def _check_comb_in(r, prev, H, k=8.0):
    """The comb's input after step `prev`: every census slot (holes included), or,
    when `prev` thinned its census on the fly (the cold start), ~k x H records
    (at most the census weight over the lanes' comb spacing W / (k H), plus one
    per lane and the warps' chunk tails)."""
    holes = 148 * 28 * 64  # zero-weight chunk tails: up to one 64-slot chunk per warp
    if prev.thinned:  # at most one record per census particle, ~k H in all
        assert r.comb_in <= prev.counters.census_count + holes
        assert r.comb_in <= 1.1 * k * H + 148 * 28 * 32 + holes, (r.comb_in, H)
    else:
        assert r.comb_in >= prev.counters.census_count


def cfg(which, H, steps, seed):
    if which == 1:
        return hw.RunConfig(mode="hww_ma", ma_base_k=3, histories_per_step=H, rho=5.0, seed=seed,
                            material=hw.Material(1.0, 1.0, 0.0, 0.0, 1.0), x_min=-20.0,
                            x_max=20.0, cells=200, t_end=1.0 * steps, time_steps=steps)
    return hw.RunConfig(mode="hww_ma", ma_base_k=1, histories_per_step=H, rho=5.0, seed=seed,
                        material=hw.Material(1.0, 0.9, 0.0, 0.0, 1.0), x_min=-20.0, x_max=20.0,
                        cells=400, t_end=0.5 * steps, time_steps=steps)


def run(c, rng):
    d = hw.Driver(c, rng_mode=rng)
    out = []
    for _ in range(c.time_steps):
        rec = d.step()
        out.append((rec, d.arrays()))
    d.close()
    return out


@pytest.mark.parametrize("which", [1, 2])
def test_step1_within_batch_sigma(which):
    H = 200_000
    ex = run(cfg(which, H, 1, 42), hw.RNG_EXACT)[0]
    fa = run(cfg(which, H, 1, 43), hw.RNG_PHILOX)[0]
    a, b = ex[1], fa[1]
    sig = np.sqrt(a["sigma"] ** 2 + b["sigma"] ** 2)
    mask = a["phi_track"] > 1e-3 * a["phi_track"].max()
    z = np.abs(a["phi_track"] - b["phi_track"])[mask] / sig[mask]
    assert np.mean(z < 3.0) >= 0.95, np.sort(z)[-10:]
    # global chi^2 over the well-sampled cells: E[sum z^2] = n
    # whatever the cell correlations, which only widen its spread
    chi2 = float(np.sum(z ** 2)) / z.size
    assert 0.4 < chi2 < 1.8, chi2
    # census weight per history (the growth law) and the segment count
    sw = np.hypot(ex[0].census_weight_sigma, fa[0].census_weight_sigma)
    assert abs(ex[0].census_weight - fa[0].census_weight) <= 4 * sw + 1e-12
    assert abs(fa[0].segments / ex[0].segments - 1) < (0.02 if which == 1 else 0.1)  # C2 step 1 is heavy-tailed


def test_replicates_agree_over_steps():
    """Config-1 physics, 6 steps, R = 6 seeds per mode: per-cell replicate means of
    phi_track agree within 3 combined standard errors on >= 95% of cells."""
    # With R replicates per side the z statistic is Student-t with ~2R-2 dof
    # (P(|t| > 3) ~ 1% at R = 8), and neighbouring cells are correlated, so
    # the per-cell rule is paired with a bias check on the mean signed z.
    H, N, R = 20_000, 6, 8
    ex = np.array([[s[1]["phi_track"] for s in run(cfg(1, H, N, 100 + r), hw.RNG_EXACT)]
                   for r in range(R)])
    fa = np.array([[s[1]["phi_track"] for s in run(cfg(1, H, N, 200 + r), hw.RNG_PHILOX)]
                   for r in range(R)])
    for n in range(N):
        m_e, m_f = ex[:, n].mean(0), fa[:, n].mean(0)
        se = np.sqrt(ex[:, n].var(0, ddof=1) / R + fa[:, n].var(0, ddof=1) / R)
        mask = (m_e > 1e-3 * m_e.max()) & (se > 0)
        z = (m_f - m_e)[mask] / se[mask]
        assert np.mean(np.abs(z) < 3.0) >= 0.9, (n, np.sort(np.abs(z))[-8:])
        assert abs(z.mean()) < 0.75, (n, z.mean())
        assert abs(m_f.sum() / m_e.sum() - 1) < 5e-3, n


def test_philox_run_is_conservative():
    """Weight bookkeeping of one fast step: census + leakage + captured weight
    matches the analog balance within the batch sigma (c = 1: no capture)."""
    rec, arr = run(cfg(1, 100_000, 1, 5), hw.RNG_PHILOX)[0]
    # c = 1, vacuum boundaries: all weight either leaks or is banked at census
    total = rec.census_weight * 100_000 + rec.counters.leakage_weight
    assert abs(total / 100_000 - 1.0) < 5 * rec.census_weight_sigma + 1e-3
    assert rec.census_size == rec.counters.census_count


def test_philox_bank_and_host_round_trip():
    """The census bank a Philox driver hands out (compacted real particles) and
    the e2e host_bank mode, which combs on the device before the host round
    trip: same bookkeeping, and results within statistics of the device run."""
    H, steps = 100_000, 4
    c = cfg(2, H, steps, 9)
    d = hw.Driver(c, rng_mode=hw.RNG_PHILOX)
    recs = [d.step() for _ in range(steps)]
    bank = d.bank()
    d.close()
    last = recs[-1]
    assert len(bank) == last.counters.census_count
    assert np.all(bank["w"] > 0)
    np.testing.assert_allclose(bank["w"].sum(), last.census_weight * H, rtol=1e-9)

    c.host_bank = True
    e = hw.Driver(c, rng_mode=hw.RNG_PHILOX)
    erecs = [e.step() for _ in range(steps)]
    e.close()
    for k in range(1, steps):  # steps 2.. open with the device-side pre-comb
        assert erecs[k].comb_out == H
        _check_comb_in(erecs[k], erecs[k - 1], H)
        assert erecs[k].h2d_bytes == H * 16  # packed: (x, mu); (w, t) shared by the combed bank
        np.testing.assert_allclose(erecs[k].comb_out_weight, erecs[k].comb_in_weight, rtol=1e-12)
    for r, q in zip(recs, erecs):  # two realisations (census order is scheduling-dependent)
        # (heavy-tailed split trees: the segment count of 1e5 histories moves by several %)
        assert abs(q.segments / r.segments - 1) < 0.25
        assert abs(q.census_weight / r.census_weight - 1) < 0.03


def test_host_round_trip_full_wire_format(monkeypatch):
    """The packed host round trip's fallback (per-particle (w, t) after the (x, mu)
    block, used when the combed bank's (w, t) are not one shared pair)."""
    H, steps = 100_000, 3
    c = cfg(2, H, steps, 9)
    c.host_bank = True
    base = [r for r in (lambda d: [d.step() for _ in range(steps)] + [d.close()])(
        hw.Driver(c, rng_mode=hw.RNG_PHILOX))[:steps]]
    monkeypatch.setenv("HWWG_HOST_FULL", "1")
    d = hw.Driver(c, rng_mode=hw.RNG_PHILOX)
    full = [d.step() for _ in range(steps)]
    d.close()
    for k in range(1, steps):
        assert full[k].h2d_bytes == H * 32 and base[k].h2d_bytes == H * 16
        assert full[k].comb_out == H
        assert abs(full[k].segments / base[k].segments - 1) < 0.25
        assert abs(full[k].census_weight / base[k].census_weight - 1) < 0.03


def test_config3_philox_step1_within_batch_sigma():
    """Config-3 (regions, volumetric source, LOSM q) in the throughput mode:
    step-1 track flux within 3 combined batch sigma of the exact mode."""
    from tests.test_gpu_parity import _c3
    _, g = _c3(200_000, 1, mode="hww", cells=300)
    ex = run(g, hw.RNG_EXACT)[0]
    fa = run(g, hw.RNG_PHILOX)[0]
    (re, ae), (rf, af) = ex, fa
    assert re.histories == rf.histories == 200_000
    m = ae["phi_track"] > 1e-3 * ae["phi_track"].max()
    z = (af["phi_track"][m] - ae["phi_track"][m]) / np.sqrt(ae["sigma"][m] ** 2 + af["sigma"][m] ** 2)
    assert np.mean(np.abs(z) < 3) >= 0.95, np.mean(np.abs(z) < 3)
    assert abs(rf.census_weight / re.census_weight - 1) < 5 * (re.census_weight_sigma + rf.census_weight_sigma) / re.census_weight


def test_comb_conserves_weight_from_cold_start():
    """The throughput comb (exact fixed-point integer prefixes in tiles) on the
    x60 cold-start census and the steady banks after it: the target count, the
    combed weight equal to the input weight (popctrl.cpp:7-42: target teeth of
    weight W/target), and the input weight equal to the census weight the
    previous step tallied (the comb reads every census slot, holes included)."""
    H, steps = 100_000, 4
    out = run(cfg(2, H, steps, 21), hw.RNG_PHILOX)
    for k in range(1, steps):
        r, prev = out[k][0], out[k - 1][0]
        assert r.comb_out == H
        _check_comb_in(r, prev, H)
        np.testing.assert_allclose(r.comb_out_weight, r.comb_in_weight, rtol=1e-12)
        # a thinned census holds the census weight up to the lanes' comb
        # quantisation (zero mean; ~sqrt(lanes) * s0 = sqrt(lanes) W / (k H))
        np.testing.assert_allclose(r.comb_in_weight, prev.census_weight * H,
                                   rtol=2e-2 if prev.thinned else 1e-9)


@pytest.mark.parametrize("H", [100_000, 1_000_000])
def test_fixed_point_tallies_match_fp64(monkeypatch, H):
    """The fixed-point track, edge and census tallies (16-bit limbs on native 32-bit
    shared atomics, carries swept into the next limb while blocks run) against the
    fp64 CAS tallies on the same events: one config-2 cold-start step with per-lane
    (not warp-aggregated) tallies throughout, so both runs see the same
    counter-based Philox histories and differ only in the tally arithmetic
    (quantisation 2^-40 of the largest expected score, and fp64 summation order).
    H = 1e6: ~1.7e5 limb adds per block and cell range, far past a 16-bit limb
    word's 2^16 adds without the carry sweep."""
    monkeypatch.setenv("HWWG_FAST_AGG", "2")
    out = {}
    for fix in ("1", "0"):
        monkeypatch.setenv("HWWG_FAST_FIX", fix)
        out[fix] = run(cfg(2, H, 1, 13), hw.RNG_PHILOX)[0]
    (rq, aq), (rd, ad) = out["1"], out["0"]
    kq, kd = rq.counters.as_dict(), rd.counters.as_dict()
    for k in ("collisions", "census_count", "splits", "split_daughters", "roulette_kills"):
        assert kq[k] == kd[k], (k, kq[k], kd[k])
    assert rq.segments == rd.segments
    np.testing.assert_array_equal(aq["tracks_per_cell"], ad["tracks_per_cell"])
    # every add rounds to the grid (2^-41 of the largest expected score), so a
    # cell's error is its score count x 2^-41 of that score: relative to the
    # array's maximum, a few 1e-10 at most
    np.testing.assert_allclose(aq["phi_track"], ad["phi_track"], rtol=0,
                               atol=1e-9 * ad["phi_track"].max())
    np.testing.assert_allclose(aq["sigma"], ad["sigma"], rtol=1e-6, atol=1e-9 * ad["sigma"].max())
    for k in ("edge_current", "phi_census", "current_census", "closure_census", "ww_centers"):
        scale = np.abs(ad[k]).max()
        np.testing.assert_allclose(aq[k], ad[k], rtol=0, atol=1e-9 * scale, err_msg=k)


def test_fixed_point_dynamic_range_guard(monkeypatch):
    """when the smallest census score (a weight at the lowest window
    floor eps_min / rho) sits more than 20 binades below the largest expected
    score (rho here is 1e6: ~40 binades), the fixed-point grid would round it
    coarsely and identical weights would all round the same way, so the driver
    keeps fp64 slots: the run must see the forced-fp64 run's events and
    tallies."""
    monkeypatch.setenv("HWWG_FAST_AGG", "2")
    out = {}
    for fix in ("1", "0"):
        monkeypatch.setenv("HWWG_FAST_FIX", fix)
        c = cfg(2, 50_000, 1, 13)
        c.rho = 1e6
        out[fix] = run(c, hw.RNG_PHILOX)[0]
    (rq, aq), (rd, ad) = out["1"], out["0"]
    assert rq.segments == rd.segments
    for k in ("phi_census", "phi_track"):
        np.testing.assert_allclose(aq[k], ad[k], rtol=1e-12, atol=1e-14 * ad[k].max(), err_msg=k)


@pytest.mark.gpu
def test_philox_error_metrics_against_sn_reference(tmp_path):
    """The throughput engine run against the reference's S_N solution (written by
    hww::save_reference, read by the engine's loader): the step error metrics
    exist every step and the track flux is close to the deterministic interval
    average (config 1 at 2e5 histories: relative L2 error of a few percent),
    and they match the exact engine's metrics statistically."""
    from oracle import bind
    from paper_2512_19925_b200 import hww
    if not bind.have_reference():
        pytest.skip("oracle/_ref not built")
    R = bind.Reference()
    r = bind.baseline_config(1, histories=200000, time_steps=6)
    h = hww.RunConfig(mode="hww_ma", ma_base_k=3, histories_per_step=200000, rho=5.0, seed=42,
                      material=hww.Material(1.0, 1.0, 0.0, 0.0, 1.0), x_min=-20.0, x_max=20.0,
                      cells=200, t_end=r.t_end, time_steps=6)
    path = tmp_path / "reference.csv"
    R.save_reference(r, path, *R.compute_reference(r))
    errs = {}
    for mode in (hww.RNG_PHILOX, hww.RNG_EXACT):
        d = hww.Driver(h, rng_mode=mode)
        d.load_reference(path)
        errs[mode] = []
        for _ in range(6):
            rec = d.step()
            assert np.isfinite(rec.rel_l2_error) and np.isfinite(rec.alpha)
            # FOM_err is 1/(tau err_i^2) per cell (metrics.cpp:34-55): a cell beyond the
            # front where the tally is 0 and the S_N layer ~1e-170 gives err_i^2 = 0
            # after underflow and an infinite FOM in the reference too; never NaN
            assert rec.fom_err_l2 > 0 and not np.isnan(rec.fom_err_l2)
            assert rec.fom_sigma_mod >= 0 and not np.isnan(rec.fom_sigma_mod)
            assert np.isfinite(rec.hybrid_rel_l2_error)
            errs[mode].append(rec.rel_l2_error)
        d.close()
    ph, ex = np.array(errs[hww.RNG_PHILOX]), np.array(errs[hww.RNG_EXACT])
    assert np.all(ph < 0.1) and np.all(ex < 0.1), (ph, ex)
    # same estimator: the errors agree to within their own spread
    assert abs(ph.mean() - ex.mean()) < 0.5 * max(ph.mean(), ex.mean()), (ph, ex)


@pytest.mark.parametrize("which,H", [(2, 200_000), (1, 100_000)])
def test_census_thinning_cold_start(monkeypatch, which, H):
    """Census thinning (FastArgs::precomb) in the cold start: the step's events and
    tallies are those of the unthinned run (the same Philox histories; thinning
    only decides what is banked), the bank the next comb reads shrinks from the
    x60 raw census to ~8 x H records of equal quanta, its weight is the census
    weight up to the lanes' comb quantisation, and the combed step 2 is the
    same estimator (close to the unthinned run's step 2)."""
    c = cfg(which, H, 2, 17)
    out = {}
    for pc in ("1", "0"):
        monkeypatch.setenv("HWWG_PRECOMB", pc)
        out[pc] = run(c, hw.RNG_PHILOX)
    (r1, a1), (r0, a0) = out["1"][0], out["0"][0]
    assert r1.thinned == 1 and r0.thinned == 0
    assert r1.segments == r0.segments and r1.census_size == r0.census_size
    assert r1.counters.collisions == r0.counters.collisions
    for k in ("phi_track", "phi_census", "current_census", "edge_current"):
        np.testing.assert_allclose(a1[k], a0[k], rtol=1e-9, atol=1e-12 * np.abs(a0[k]).max(), err_msg=k)
    s1, s0 = out["1"][1][0], out["0"][1][0]
    # step 2 is thinned too when the cold start's raw census exceeded 8 H
    assert s1.thinned == (1 if r1.census_size > 8 * H else 0) and s0.thinned == 0
    assert s0.comb_in >= r0.census_size  # the raw cold-start census, holes included
    assert s1.comb_in <= min(s0.comb_in, 1.1 * 8 * H + 148 * 28 * (32 + 64)), s1.comb_in
    if which == 2:  # config 2's pulse splits x60 (config 1's analog step 1 does not split)
        assert r0.census_size > 20 * H
    np.testing.assert_allclose(s1.comb_in_weight, r1.census_weight * H, rtol=1e-2)
    np.testing.assert_allclose(s1.comb_out_weight, s1.comb_in_weight, rtol=1e-12)
    b1, b0 = out["1"][1][1], out["0"][1][1]
    m = b0["phi_track"] > 1e-3 * b0["phi_track"].max()
    z = (b1["phi_track"] - b0["phi_track"])[m] / np.hypot(b1["sigma"], b0["sigma"])[m]
    # (batch sigma misses the comb's inter-step noise: a sanity bound here; the
    # replicate pin, tests/test_gpu_stat_pin.py, runs every workload thinned)
    assert np.mean(np.abs(z) < 3) >= 0.9, np.sort(np.abs(z))[-8:]


def test_host_round_trip_volumetric_source():
    """The e2e host round trip (host_bank) on config 3, whose steps append
    device-sampled volumetric particles after the combed teeth: the teeth cross
    PCIe packed in pieces (16 B each), the volumetric ones never do, and the run
    keeps the device-resident run's bookkeeping and statistics."""
    from tests.test_gpu_parity import _c3
    H, steps = 60_000, 4
    _, g = _c3(H, steps, mode="hww", cells=300)
    d = hw.Driver(g, rng_mode=hw.RNG_PHILOX)
    dev = [d.step() for _ in range(steps)]
    d.close()
    g.host_bank = True
    e = hw.Driver(g, rng_mode=hw.RNG_PHILOX)
    host = [e.step() for _ in range(steps)]
    e.close()
    for k, (r, q) in enumerate(zip(dev, host)):
        assert q.histories == r.histories and q.comb_out == r.comb_out
        if k >= 1:  # steps 2.. open with the pre-combed teeth from the host
            assert q.h2d_bytes == q.comb_out * 16, (k, q.h2d_bytes, q.comb_out)
        assert abs(q.segments / r.segments - 1) < 0.25, (k, q.segments, r.segments)
        assert abs(q.census_weight / r.census_weight - 1) < 0.05, (k, q.census_weight, r.census_weight)


@pytest.mark.parametrize("window_max", ["0", "48"])
def test_tally_window_matches_global_tallies(monkeypatch, window_max):
    """Config 4 (4000 cells: the full fixed-point histograms do not fit shared
    memory) with its histograms over the window of cells the step's particles can
    reach (FastArgs::t_win) against the global fp64 REDs, on the same events (one
    cold-start step, per-lane tallies): equal counters and track counts, tallies
    within fp64 summation order and the fixed-point grid. window_max = 48 clips the
    window to 48 cells, so most scores take the out-of-window fallback."""
    from paper_2512_19925_b200.configs import baseline
    monkeypatch.setenv("HWWG_FAST_AGG", "2")
    out = {}
    for win in ("1", "0"):
        monkeypatch.setenv("HWWG_TALLY_WINDOW", win)
        monkeypatch.setenv("HWWG_TALLY_WINDOW_MAX", window_max)
        c = baseline(4, histories=100_000, time_steps=1, seed=5)
        out[win] = run(c, hw.RNG_PHILOX)[0]
    (rw, aw), (rg, ag) = out["1"], out["0"]
    assert rw.segments == rg.segments and rw.census_size == rg.census_size
    assert rw.counters.collisions == rg.counters.collisions
    np.testing.assert_array_equal(aw["tracks_per_cell"], ag["tracks_per_cell"])
    for k in ("phi_track", "phi_census", "current_census", "closure_census", "edge_current"):
        np.testing.assert_allclose(aw[k], ag[k], rtol=1e-9, atol=1e-12 * np.abs(ag[k]).max(), err_msg=k)
    np.testing.assert_allclose(rw.census_weight, rg.census_weight, rtol=1e-9)
