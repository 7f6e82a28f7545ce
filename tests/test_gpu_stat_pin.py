"""Statistical pin of the throughput (Philox) engine over the workloads bench.py
times, against the exact engine (bit-exact to the reference, tests/test_gpu_parity.py).

Both engines estimate the same physics with different random numbers, so the
judge is replicate statistics (the reference's own rule,
proj/tests/acceptance_main.cpp:248-286: >= 95% of well-sampled cells within 3
combined standard errors, sigma from independent replicates because batch
sigma misses the inter-step bank noise, :225-231).  R independent seeds per
engine; for every compared quantity, per cell and step, z = (mean_philox -
mean_exact) / sqrt(se_philox^2 + se_exact^2).  With R = 12 per side z is
Student-t with ~22 dof (P(|z| > 3) ~ 0.7%), and neighbouring cells are
correlated (the centres and phi_hybrid are smooth fields), so the rule is
applied three ways:

  * per quantity, pooled over cells and steps: >= 95% of |z| < 3;
  * per quantity and step: >= 85% (one correlated cluster can take a step);
  * no bias: the pooled mean of z within +-0.5 (+-1 for the window centres,
    which share one normalisation) and the pooled mean of z^2 (a global chi^2
    per degree of freedom) within [0.5, 2.0] ([0.5, 3.0] for the centres);
  * per-step scalars (P_L, P_R, census weight): >= 90% of |z| < 3.5, mean z
    within +-2 (steps are correlated through the carried population).

Quantities: the track-length flux phi, the census closure moments phi, J, F,
the edge currents, the window centres and the LOSM solution phi_hybrid per
cell; the boundary closures P_L / P_R and the census weight per step."""
import json
import os

import numpy as np
import pytest

import paper_2512_19925_b200 as hw
from paper_2512_19925_b200.configs import baseline

pytestmark = pytest.mark.gpu

R = 12
CELL_KEYS = ("phi_track", "phi_census", "current_census", "closure_census", "edge_current",
             "ww_centers", "phi_hybrid")
SCALARS = ("boundary_closure_left", "boundary_closure_right", "census_weight")


def replicate(cfg_fn, rng, seeds, steps):
    """cells[key] -> array [R, steps, n], scal[key] -> [R, steps]."""
    cells = {k: [] for k in CELL_KEYS}
    scal = {k: [] for k in SCALARS + ("segments",)}
    for s in seeds:
        d = hw.Driver(cfg_fn(s), rng_mode=rng)
        per = {k: [] for k in CELL_KEYS}
        ps = {k: [] for k in scal}
        for _ in range(steps):
            rec = d.step()
            a = d.arrays()
            for k in CELL_KEYS:
                per[k].append(a[k].copy())
            for k in scal:
                ps[k].append(float(getattr(rec, k)))
        d.close()
        for k in CELL_KEYS:
            cells[k].append(per[k])
        for k in scal:
            scal[k].append(ps[k])
    return ({k: np.array(v) for k, v in cells.items()}, {k: np.array(v) for k, v in scal.items()})


def zstats(a, b, mask):
    """a, b: [R, ...]; z over entries where mask and se > 0."""
    ma, mb = a.mean(0), b.mean(0)
    se = np.sqrt(a.var(0, ddof=1) / a.shape[0] + b.var(0, ddof=1) / b.shape[0])
    m = mask & (se > 0) & np.isfinite(ma) & np.isfinite(mb)
    return (mb - ma)[m] / se[m]


def check_engine(cfg_fn, steps, skip_first=0, label=""):
    ex_c, ex_s = replicate(cfg_fn, hw.RNG_EXACT, [1000 + i for i in range(R)], steps)
    fa_c, fa_s = replicate(cfg_fn, hw.RNG_PHILOX, [2000 + i for i in range(R)], steps)
    phi = ex_c["phi_track"].mean(0)  # [steps, I]
    report, fails = {}, []
    for k in CELL_KEYS:
        a, b = ex_c[k][:, skip_first:], fa_c[k][:, skip_first:]
        if not np.isfinite(a).all() or not np.isfinite(b).all():
            # centres / phi_hybrid are nan before the first hybrid solve
            ok = np.isfinite(a).all(axis=(0, 2)) & np.isfinite(b).all(axis=(0, 2))
            a, b = a[:, ok], b[:, ok]
            ph = phi[skip_first:][ok]
        else:
            ph = phi[skip_first:]
        if a.shape[1] == 0:
            continue
        if k == "edge_current":  # I+1 edges: well sampled where either neighbour cell is
            pe = np.maximum(np.pad(ph, ((0, 0), (1, 0))), np.pad(ph, ((0, 0), (0, 1))))
            mask = pe > 1e-3 * ph.max(axis=1, keepdims=True)
        else:
            mask = ph > 1e-3 * ph.max(axis=1, keepdims=True)
        z_all = zstats(a, b, mask)
        if z_all.size <= 50:
            fails.append((k, "too few cells", z_all.size))
            continue
        frac = float(np.mean(np.abs(z_all) < 3))
        bias, chi2 = float(z_all.mean()), float(np.mean(z_all ** 2))
        step_min = 1.0
        for n in range(a.shape[1]):
            zn = zstats(a[:, n], b[:, n], mask[n])
            if zn.size >= 20:
                fn = float(np.mean(np.abs(zn) < 3))
                step_min = min(step_min, fn)
                if fn < 0.85:
                    fails.append((k, "step", n + skip_first, fn, np.sort(np.abs(zn))[-5:]))
        report[k] = dict(frac=frac, bias=bias, chi2=chi2, worst_step_frac=step_min, n=int(z_all.size))
        if frac < 0.95:
            fails.append((k, "pooled fraction", frac, np.sort(np.abs(z_all))[-8:]))
        # the centres are normalised by the maximum of phi_hybrid (ww.cpp:8-32): one
        # fluctuation of that maximum moves every cell's centre the same way, so
        # their pooled mean z is nearly as wide as a single z
        if abs(bias) >= (1.0 if k == "ww_centers" else 0.5):
            fails.append((k, "bias", bias))
        # (for the centres, that common shift also enters every cell's z^2: their
        # pooled mean z^2 spreads like one chi^2 draw — seen at 2.1 once in ~10 runs
        # of an unbiased engine — so its upper bound widens with the bias bound)
        # lower bound: a sanity check that the standard errors are not inflated
        # (chi2 -> 0). Neighbouring cells and successive steps of one realisation
        # are strongly correlated, so the pooled mean z^2 has far fewer degrees of
        # freedom than cells x steps: the supercritical benchmark.cfg, whose
        # population compounds by fission, was seen at 0.70 and 0.48 on the same
        # unbiased engine (profiles/round2_stat_pin.jsonl)
        if not 0.25 < chi2 < (3.0 if k == "ww_centers" else 2.0):
            fails.append((k, "chi2", chi2))
    for k in SCALARS:
        z = zstats(ex_s[k][:, skip_first:], fa_s[k][:, skip_first:],
                   np.ones(steps - skip_first, bool))
        if z.size:
            report[k] = dict(frac=float(np.mean(np.abs(z) < 3)), bias=float(z.mean()),
                             chi2=float(np.mean(z ** 2)), n=int(z.size))
            # the census weight carries over between steps (the population weight
            # compounds, acceptance_main.cpp:225-231), so its per-step z are strongly
            # correlated and their mean is nearly as wide as one z
            if np.mean(np.abs(z) < 3.5) < 0.9 or abs(z.mean()) >= 2.0:
                fails.append((k, z))
    report["segments_ratio"] = float(fa_s["segments"].mean() / ex_s["segments"].mean())
    out = os.environ.get("HWWG_STAT_REPORT")
    if out:  # per quantity: fraction |z| < 3, mean z, mean z^2, worst step
        with open(out, "a") as f:
            f.write(json.dumps({"config": label, "R": R, "steps": steps, **report}) + "\n")
    assert not fails, (label, fails)
    return report


def test_config2_all_timed_steps():
    """Config 2 (bench's C2 line), every one of the 20 timed steps, H = 2e4."""
    check_engine(lambda s: baseline(2, histories=20_000, time_steps=20, seed=s), 20, label="C2")


@pytest.mark.parametrize("rho,k", [(2.0, 0), (5.0, 1), (10.0, 2)])
def test_config5_variants(rho, k):
    """Config 5's sweep corners and the bench headline point (rho 5, MA3), 8 steps."""
    check_engine(lambda s: baseline(5, histories=20_000, time_steps=8, seed=s, rho=rho,
                                    ma_base_k=k), 8, label=f"C5 rho={rho} k={k}")


def test_config5_headline_all_timed_steps():
    """The bench headline (config 5 at rho 5, MA3) over all 20 timed steps at
    H = 1e5: the cold start (census thinning), step 2's comb of the thinned bank,
    and the steady steps, every closure moment, current and window centre."""
    check_engine(lambda s: baseline(5, histories=100_000, time_steps=20, seed=s, rho=5.0,
                                    ma_base_k=1), 20, label="C5 headline (20 steps)")


def test_config4_first_steps():
    """Config 4 (4000 cells, c = 0.99, hww rho 1.25): the cold start and two steady steps."""
    check_engine(lambda s: baseline(4, histories=100_000, time_steps=3, seed=s), 3, label="C4")


def test_config3_first_steps():
    """Config 3 (regions, volumetric source — sampled on the device in Philox mode,
    on the host from the reference-style stream in exact mode — and LOSM q): the
    two source steps and three after."""
    def cfg(s):
        c = baseline(3, histories=50_000, time_steps=5, seed=s)
        c.vol_histories = 50_000
        return c
    check_engine(cfg, 5, label="C3")


def test_reference_benchmark_fission():
    """The reference's own benchmark (proj/configs/benchmark.cfg: a supercritical
    medium, sigma_s = sigma_f = 1/3, nu = 2.3 — the one configuration with fission)
    in the throughput engine: fission secondaries (floor(nu) + Bernoulli), each
    with its own direction and window game (transport.cpp:29-40, 179-188)."""
    check_engine(lambda s: baseline(0, histories=20_000, time_steps=6, seed=s), 6,
                 label="benchmark.cfg")
