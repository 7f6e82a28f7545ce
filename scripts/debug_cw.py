import sys; sys.path.insert(0, '.')
import numpy as np
import paper_2512_19925_b200 as hw
from tests.test_gpu_statistical import cfg
for rng in (hw.RNG_EXACT, hw.RNG_PHILOX):
    d = hw.Driver(cfg(1, 20000, 2, 42), rng_mode=rng)
    for s in range(2):
        r = d.step()
        print(rng, s+1, {k: getattr(r, k) for k, _ in r._fields_ if k not in ('counters','thresholds')})
