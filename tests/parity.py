"""Shared parity assertions (SURVEY.md §8(d) criteria).

Exact mode: integer counters, tracks_per_cell and the census bank's x/mu/t are
bit-exact; floating tallies agree within 1e-12 relative, with the scaled rule
for signed moments (|dJ_i|, |dF_i| <= 1e-12 * phi_census_i; edge currents <=
1e-12 * sum|J|) because GPU fp64 atomics sum in a different order than the
reference's 256-history chunk merge.
"""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL = 1e-12
COUNTER_U = ("collisions", "splits", "split_daughters", "capped_splits", "roulette_kills",
             "roulette_survivals", "census_count", "event_cap_aborts", "nan_aborts")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def close_rel(a, b, tol=TOL, scale=None, what=""):
    a, b = np.asarray(a, float), np.asarray(b, float)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    s = np.maximum(np.abs(a), np.abs(b)) if scale is None else np.asarray(scale, float)
    bad = np.abs(a - b) > tol * s + 1e-300
    assert not bad.any(), (f"{what}: {bad.sum()} entries differ beyond {tol}; worst "
                           f"{np.max(np.abs(a - b) / (s + 1e-300))}")


def tallies_close(t_gpu, t_ref, I, B, tol=TOL):
    """t_* expose track_flux, track_flux_batch, census_phi/current/closure,
    census_weight_batch, edge_current, boundary_closure_left/right."""
    close_rel(t_gpu.track_flux, t_ref.track_flux, tol, what="track_flux")
    close_rel(t_gpu.track_flux_batch, t_ref.track_flux_batch, tol, what="track_flux_batch")
    close_rel(t_gpu.census_phi, t_ref.census_phi, tol, what="census_phi")
    phi = np.abs(np.asarray(t_ref.census_phi)) + np.abs(np.asarray(t_gpu.census_phi))
    close_rel(t_gpu.census_current, t_ref.census_current, tol, scale=phi, what="census_current")
    close_rel(t_gpu.census_closure, t_ref.census_closure, tol, scale=phi, what="census_closure")
    close_rel(t_gpu.census_weight_batch, t_ref.census_weight_batch, tol, what="census_w_batch")
    e = np.asarray(t_ref.edge_current)
    close_rel(t_gpu.edge_current, e, tol, scale=np.full(e.shape, np.abs(e).sum() + 1e-300),
              what="edge_current")
    pl = abs(t_ref.boundary_closure_left) + abs(t_ref.boundary_closure_right) + 1e-300
    assert abs(t_gpu.boundary_closure_left - t_ref.boundary_closure_left) <= tol * pl
    assert abs(t_gpu.boundary_closure_right - t_ref.boundary_closure_right) <= tol * pl


def counters_equal(c_gpu: dict, c_ref: dict, tol=TOL):
    for k in COUNTER_U:
        assert c_gpu[k] == c_ref[k], (k, c_gpu[k], c_ref[k])
    for k in ("leakage_weight", "aborted_weight"):
        assert abs(c_gpu[k] - c_ref[k]) <= tol * max(abs(c_ref[k]), 1e-300) + 1e-300, (
            k, c_gpu[k], c_ref[k])


def census_equal(a, b, weights_tol=0.0):
    """x, mu, t bit-exact and in order; w bit-exact (weights_tol = 0) or within
    a relative tolerance (driver runs, where LOSM centres carry the tallies'
    summation-order ulps into roulette survivors' weights)."""
    assert a.size == b.size, ("census size", a.size, b.size)
    for f in ("x", "mu", "t"):
        assert np.array_equal(a[f], b[f]), (f, int(np.sum(a[f] != b[f])))
    if weights_tol == 0.0:
        assert np.array_equal(a["w"], b["w"]), ("w", int(np.sum(a["w"] != b["w"])))
    else:
        close_rel(a["w"], b["w"], weights_tol, what="census w")
