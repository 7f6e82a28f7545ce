#!/usr/bin/env python3
"""Exact comb (hwwg_uniform_comb) on n exponential weights; run under ncu for kernel times.
    python scripts/comb_speed.py [n] [target]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_19925_b200 as hw  # noqa: E402
from paper_2512_19925_b200._capi import PARTICLE_DT  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 5_000_000
tgt = int(float(sys.argv[2])) if len(sys.argv) > 2 else 1_000_000
rng = np.random.default_rng(1)
b = np.zeros(n, PARTICLE_DT)
b["w"] = rng.exponential(1.0, n)
e = hw.Engine(rng_mode=hw.RNG_EXACT)
for _ in range(2):
    out, iw, ow = e.uniform_comb(b, tgt, 1, 2)
print(n, tgt, iw, ow)
