import sys; sys.path.insert(0, '.')
import numpy as np
import paper_2512_19925_b200 as hw
from tests.test_gpu_statistical import cfg, run
H, N, R = 20000, 6, 12
for which in (1, 2):
    ex = np.array([[s[1]["phi_track"] for s in run(cfg(which, H, N, 100 + r), hw.RNG_EXACT)] for r in range(R)])
    fa = np.array([[s[1]["phi_track"] for s in run(cfg(which, H, N, 200 + r), hw.RNG_PHILOX)] for r in range(R)])
    for n in range(N):
        m_e, m_f = ex[:, n].mean(0), fa[:, n].mean(0)
        se = np.sqrt(ex[:, n].var(0, ddof=1) / R + fa[:, n].var(0, ddof=1) / R)
        mask = (m_e > 1e-3 * m_e.max()) & (se > 0)
        z = (m_f - m_e)[mask] / se[mask]
        tot_e, tot_f = m_e.sum(), m_f.sum()
        print(which, n + 1, "cells %d  frac|z|>3 %.3f  mean z %+.3f  sum ratio %.5f" % (mask.sum(), np.mean(np.abs(z) > 3), z.mean(), tot_f / tot_e))
