"""Diagnostic: one config's first steps with HWWG_TALLY_WINDOW=a vs b (per-lane tallies)."""
import os
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

import paper_2512_19925_b200 as hw  # noqa: E402
from paper_2512_19925_b200.configs import baseline  # noqa: E402

which, H, steps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
os.environ["HWWG_FAST_AGG"] = "2"
out = {}
for win in sys.argv[4:6]:
    os.environ["HWWG_TALLY_WINDOW"] = win
    d = hw.Driver(baseline(which, histories=H, time_steps=steps, seed=5), rng_mode=hw.RNG_PHILOX)
    out[win] = []
    for _ in range(steps):
        r = d.step()
        out[win].append((r.segments, r.census_size, r.census_weight, d.arrays()))
    d.close()
a, b = sys.argv[4:6]
for k in range(steps):
    (sa, ca, wa, xa), (sb, cb, wb, xb) = out[a][k], out[b][k]
    diffs = {key: float(np.nanmax(np.abs(xa[key] - xb[key])) / max(np.nanmax(np.abs(xb[key])), 1e-300))
             for key in ("phi_track", "phi_census", "current_census", "closure_census", "edge_current")}
    print(f"step {k+1}: segments {sa} vs {sb}, census {ca} vs {cb}, weight {wa:.6g} vs {wb:.6g}", diffs)
