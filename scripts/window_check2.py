import os, sys
sys.path.insert(0, '.')
import numpy as np
import paper_2512_19925_b200 as hw
from paper_2512_19925_b200.configs import baseline
os.environ["HWWG_FAST_AGG"] = "2"
res = {}
for win in ("1", "2", "2"):
    os.environ["HWWG_TALLY_WINDOW"] = win
    d = hw.Driver(baseline(5, histories=200000, time_steps=1, seed=5), rng_mode=hw.RNG_PHILOX)
    r = d.step(); a = d.arrays(); d.close()
    res.setdefault(win, []).append((r, a))
b = res["1"][0][1]
for i, (r, a) in enumerate(res["2"]):
    for key in ("phi_track", "current_census", "edge_current", "tracks_per_cell"):
        x, y = a[key].astype(float), b[key].astype(float)
        dif = np.abs(x - y)
        k = int(np.argmax(dif))
        nz = np.nonzero(y)[0]
        print(i, key, "argmax", k, "val", x[k], "ref", y[k], "support", (nz.min(), nz.max()) if nz.size else None,
              "nonzero win-run", (np.nonzero(x)[0].min(), np.nonzero(x)[0].max()) if np.any(x) else None)
    print(i, "segments", r.segments, res["1"][0][0].segments)
