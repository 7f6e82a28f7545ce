#!/usr/bin/env python3
"""Throughput of every BASELINE configuration on one B200 (bench.py times config 2).

For each config: the Philox engine over all its steps (device-timed, as bench.py's
`value`), the exact mode over the first steps, and the reference (oracle/_ref, all
host threads) on a bounded sample. Config 4 runs at one GPU's share of its
8-GPU split (1.25e7 histories per step, all 100 steps). Writes one JSON line
per config and, with --md, a markdown table.

    python scripts/bench_configs.py [--md profiles/round1_configs.md]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2512_19925_b200 as hw  # noqa: E402


def cfg(which, H=None, steps=None, **kw):
    if which == 1:
        c = dict(mode="hww_ma", ma_base_k=3, histories_per_step=100_000, rho=5.0, seed=42,
                 material=hw.Material(1.0, 1.0, 0.0, 0.0, 1.0), x_min=-20.0, x_max=20.0,
                 cells=200, t_end=20.0, time_steps=20)
    elif which == 2:
        c = dict(mode="hww_ma", ma_base_k=1, histories_per_step=1_000_000, rho=5.0, seed=7,
                 material=hw.Material(1.0, 0.9, 0.0, 0.0, 1.0), x_min=-20.0, x_max=20.0,
                 cells=400, t_end=20.0, time_steps=40)
    elif which == 3:  # seed 3, unit emission per unit time (stated choices)
        regions = [(10.0, hw.Material(1.0, 0.5, 0.0, 0.0, 1.0)),
                   (20.0, hw.Material(10.0, 1.0, 0.0, 0.0, 1.0)),
                   (30.0, hw.Material(1.0, 0.99, 0.0, 0.0, 1.0))]
        c = dict(mode="hww", histories_per_step=10_000_000, rho=4.0, seed=3,
                 material=hw.Material(1.0, 0.5, 0.0, 0.0, 1.0), x_min=0.0, x_max=30.0,
                 cells=1000, t_end=25.0, time_steps=50, regions=regions,
                 volume_source=(0.0, 2.0, 0.0, 1.0, 1.0), no_pulse=True)
    elif which == 4:  # reference defaults for the unspecified window mode (hww, rho 1.25), seed 1
        c = dict(mode="hww", histories_per_step=12_500_000, rho=1.25, seed=1,
                 material=hw.Material(1.0, 0.99, 0.0, 0.0, 1.0), x_min=-50.0, x_max=50.0,
                 cells=4000, t_end=50.0, time_steps=100)
    elif which == 5:
        c = dict(mode="hww_ma", ma_base_k=1, histories_per_step=10_000_000, rho=5.0, seed=11,
                 material=hw.Material(1.0, 0.9, 0.0, 0.0, 1.0), x_min=-20.0, x_max=20.0,
                 cells=400, t_end=20.0, time_steps=40)
    c.update(kw)
    if H is not None:
        c["histories_per_step"] = H
    if steps is not None:
        dt = c["t_end"] / c["time_steps"]
        c["time_steps"], c["t_end"] = steps, dt * steps
    return hw.RunConfig(**c)


def run_gpu(c, rng, steps=None):
    d = hw.Driver(c, rng_mode=rng)
    seg, ms, n = 0, 0.0, 0
    for _ in range(steps or c.time_steps):
        r = d.step()
        seg += r.segments
        ms += r.device_ms
        n += 1
    d.close()
    return seg / (ms * 1e-3), ms / n, seg


def run_cpu(which, H, steps, **kw):
    from oracle.bind import DriverRun, Reference, baseline_config, have_reference
    if not have_reference() or which == 3:  # no reference driver for config 3
        return None, None
    R = Reference()
    R.lib.hwwref_set_threads(os.cpu_count() or 1)
    d = DriverRun(R, baseline_config(which, histories=H, time_steps=steps, **kw))
    seg, tau = 0, 0.0
    for _ in range(steps):
        o, _ = d.step()
        seg += o.segments
        tau += o.tau
    d.close()
    return seg / tau, f"steps 1-{steps} at H={H}"


CASES = [
    ("C1", 1, {}, None, {}),
    ("C2", 2, {}, None, {}),
    ("C3", 3, {}, None, {}),
    ("C4 (H=1.25e7: one GPU's share of 1e8 over 8)", 4, dict(H=12_500_000), None, {}),
    ("C5 rho=2 none", 5, {}, dict(rho=2.0, mode="hww"), dict(rho=2.0, mode="hww")),
    ("C5 rho=5 MA1", 5, {}, dict(rho=5.0), dict(rho=5.0)),
    ("C5 rho=10 MA2", 5, {}, dict(rho=10.0, ma_base_k=2), dict(rho=10.0, ma_base_k=2)),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--md", default=None)
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    rows = []
    run_gpu(cfg(2, 100_000, 3), hw.RNG_PHILOX)  # warm-up: lazy module loading, first launches
    run_gpu(cfg(2, 100_000, 3), hw.RNG_EXACT)
    for name, which, size, gkw, okw in CASES:
        if args.only and not name.startswith(args.only):
            continue
        c = cfg(which, size.get("H"), size.get("steps"), **(gkw or {}))
        t0 = time.time()
        v, ms, seg = run_gpu(c, hw.RNG_PHILOX)
        ex_steps = min(3, c.time_steps)
        ex = run_gpu(cfg(which, min(c.histories_per_step, 1_000_000), ex_steps, **(gkw or {})),
                     hw.RNG_EXACT)[0]
        cpu, sample = run_cpu(which, min(c.histories_per_step, 1_000_000), 2, **(okw or {}))
        row = {"config": name, "histories": c.histories_per_step, "steps": c.time_steps,
               "cells": c.cells, "philox_seg_s": v, "ms_per_step": ms, "segments": seg,
               "exact_seg_s_first3": ex, "reference_seg_s": cpu, "reference_sample": sample,
               "wall_s": time.time() - t0}
        print(json.dumps(row), flush=True)
        rows.append(row)
    if args.md:
        lines = ["# Throughput per BASELINE configuration (one B200)", "",
                 "scripts/bench_configs.py: Philox engine over all steps (device time, "
                 "as bench.py `value`); exact mode over the first 3 steps at min(H, 1e6); "
                 "the reference (oracle/_ref, all host threads) over steps 1-2 at min(H, 1e6). "
                 "Config 3 has no reference driver (SURVEY.md §8(f2)).", "",
                 "| config | H/step | steps | cells | Philox seg/s | ms/step | exact seg/s | "
                 "reference seg/s | Philox / reference |", "|---|---:|---:|---:|---:|---:|---:|---:|---:|"]
        for r in rows:
            ref = r["reference_seg_s"]
            lines.append(
                f"| {r['config']} | {r['histories']:.3g} | {r['steps']} | {r['cells']} | "
                f"{r['philox_seg_s']:.3e} | {r['ms_per_step']:.3f} | {r['exact_seg_s_first3']:.3e} | "
                + (f"{ref:.3e} | {r['philox_seg_s'] / ref:.0f}x |" if ref else "n/a | n/a |"))
        with open(args.md, "w") as f:
            f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
