"""Time the device S_N reference (hwwg_compute_reference) on config 4's grids."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_19925_b200 import hww  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
c = hww.RunConfig(mode="hww", material=hww.Material(1.0, 0.99, 0.0, 0.0, 1.0), x_min=-50.0,
                  x_max=50.0, cells=4000, t_end=0.5 * steps, time_steps=steps)
hww.compute_reference(hww.RunConfig(cells=10, time_steps=1, t_end=0.5))
for rep in range(2):
    t = time.perf_counter()
    hww.compute_reference(c)
    print(f"steps {steps}: {time.perf_counter() - t:.4f} s", flush=True)
