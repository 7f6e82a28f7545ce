"""Diagnostic: per-cell replicate means/SE of phi_hybrid, centres and the LOSM
inputs for exact vs Philox (writes gpurun_out/diag_centres_<cfg>.npz)."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2512_19925_b200 as hw  # noqa: E402
from paper_2512_19925_b200.configs import baseline  # noqa: E402
from tests.test_gpu_stat_pin import replicate  # noqa: E402

which = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
R = 12
kw = dict(rho=5.0, ma_base_k=1) if which == 5 else {}
fn = lambda s: baseline(which, histories=20_000, time_steps=steps, seed=s, **kw)  # noqa: E731
ex_c, ex_s = replicate(fn, hw.RNG_EXACT, [1000 + i for i in range(R)], steps)
fa_c, fa_s = replicate(fn, hw.RNG_PHILOX, [2000 + i for i in range(R)], steps)
np.savez(f"gpurun_out/diag_centres_{which}.npz", **{"ex_" + k: v for k, v in ex_c.items()},
         **{"fa_" + k: v for k, v in fa_c.items()}, **{"exs_" + k: v for k, v in ex_s.items()},
         **{"fas_" + k: v for k, v in fa_s.items()})
for n in range(steps):
    for k in ("phi_hybrid", "ww_centers"):
        a, b = ex_c[k][:, n], fa_c[k][:, n]
        ma, mb = a.mean(0), b.mean(0)
        se = np.sqrt(a.var(0, ddof=1) / R + b.var(0, ddof=1) / R)
        z = np.where(se > 0, (mb - ma) / np.where(se > 0, se, 1), 0)
        i = np.argsort(-np.abs(z))[:6]
        print(n, k, [(int(j), round(float(z[j]), 2), float(ma[j]), float(mb[j]), float(se[j])) for j in i])
