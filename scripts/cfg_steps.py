#!/usr/bin/env python3
"""Per-config Philox device time over all steps: python scripts/cfg_steps.py CONFIG [H] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from scripts.bench_configs import cfg, run_gpu  # noqa: E402
import paper_2512_19925_b200 as hw  # noqa: E402

which = int(sys.argv[1])
H = int(float(sys.argv[2])) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
steps = int(sys.argv[3]) if len(sys.argv) > 3 else None
run_gpu(cfg(which, H, 3), hw.RNG_PHILOX)  # warm-up: lazy module loading, first launches
v, ms, seg = run_gpu(cfg(which, H, steps), hw.RNG_PHILOX)
print(f"config {which} H={H} steps={steps} agg={os.environ.get('HWWG_FAST_AGG', '-')}: "
      f"{v:.3e} seg/s, {ms:.3f} ms/step")
