#!/usr/bin/env python3
"""Exact-mode throughput on the first steps of a BASELINE config (device time).

    python scripts/exact_speed.py [config] [H] [steps]
HWWG_EXACT_CHUNKS=1 selects the chunk-serial kernel instead of the
history-parallel tally log.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from scripts.bench_configs import cfg, run_gpu  # noqa: E402
import paper_2512_19925_b200 as hw  # noqa: E402

which = int(sys.argv[1]) if len(sys.argv) > 1 else 2
H = int(float(sys.argv[2])) if len(sys.argv) > 2 else 1_000_000
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
run_gpu(cfg(which, 100_000, 2), hw.RNG_EXACT)  # warm-up: lazy module loading
v, ms, seg = run_gpu(cfg(which, H, steps), hw.RNG_EXACT)
path = "chunks" if os.environ.get("HWWG_EXACT_CHUNKS") else "log"
print(f"exact[{path}] config {which} H={H} steps={steps}: {v:.3e} seg/s, {ms:.2f} ms/step, {seg} segments")
