#!/usr/bin/env python3
"""Benchmark: track-segments/sec of the HWW time-step loop on BASELINE config 2.

Workload (BASELINE.json configs[1]): slab [-20,20], 400 cells, sigma_t = 1,
c = 0.9, v = 1, unit plane pulse at x = 0; 40 steps of dt = 0.5; 1e6
histories/step; hww_ma with a 3-point moving average (k = 1); window ratio 5;
seed 7; reference defaults elsewhere (theta = 0.5, eps_min = 1e-3, u_ww = 3,
f = 1/4, 1/2, 3/4, 20 batches).  Synthetic by construction (the reference's
own point-pulse source); no dataset.

A bench "step" is one time step of that run (comb -> LOSM windows -> 4
transport segments with 3 mid-step updates -> finalize -> census).  W warm-up
steps run on a separate driver instance; the K timed steps are steps 1..K of
a fresh run, so step 1's cold-start split explosion (census x63) is timed.
L2 is flushed (a 256 MiB write) between timed steps, outside the per-step
CUDA-event window.

value = sum(segments) / sum(step device time); a segment is one increment of
tracks_per_cell (proj/src/transport.cpp:136-139).  e2e = the same metric with
the bank round-tripping through pinned host memory every step (hwwg_driver with
host_bank = 1: H2D of the step's source bank, D2H of the next step's source and
of the record), timed on the host clock.  In Philox mode the device combs the
census before handing it to the host (the comb that opens the next step, with
that step's stream), so the host holds H particles between steps, not the
raw census.

--impl reference: the unmodified reference (oracle/_ref/libhww_ref.so, built
from /root/reference/proj) running hww::run_step on this box's CPU cores with
every OpenMP thread, same config; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "track-segments/sec"
UNIT = "segments/s"
BYTES_PER_SEGMENT = 96  # 48 B particle record read + written per segment
WORKLOAD = ("BASELINE config 2: slab [-20,20] 400 cells sigma_t=1 c=0.9 v=1, pulse x=0, "
            "40 x dt=0.5, 1e6 histories/step, hww_ma k=1, rho=5, seed 7")


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def config2(histories=1_000_000, time_steps=40):
    import paper_2512_19925_b200 as hw
    return hw.RunConfig(mode="hww_ma", histories_per_step=histories, theta=0.5, rho=5.0,
                        eps_min=1e-3, u_ww=3, update_fractions=(0.25, 0.5, 0.75), ma_base_k=1,
                        batches=20, seed=7, material=hw.Material(1.0, 0.9, 0.0, 0.0, 1.0),
                        x_min=-20.0, x_max=20.0, cells=400, t_end=0.5 * time_steps,
                        time_steps=time_steps)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        if os.environ.get("HWWG_NO_CLOCKS"):
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, first=0, last=None):
        rows = self.rows[first:last] or self.rows[-3:]  # the timed window (>= 1 sample)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons}


def flush_l2(buf):
    buf.add_(1.0)  # 256 MiB write > 126 MB L2


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "nccl" if args.impl != "reference" else "gloo"
        dist.init_process_group(backend, rank=rank, world_size=world)
    return rank, local, world


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def cpu_baseline(histories, steps, threads=None):
    """Reference (oracle/_ref) on this host's cores: steps 1..steps of config 2 at
    full histories, every OpenMP thread (or `threads`).  Returns (segments/s,
    cores, sample)."""
    from oracle.bind import DriverRun, Reference, baseline_config
    R = Reference()
    cores = threads or os.cpu_count() or 1
    R.lib.hwwref_set_threads(cores)
    d = DriverRun(R, baseline_config(2, histories=histories, time_steps=40))
    seg, tau = 0, 0.0
    for _ in range(steps):
        o, _ = d.step()
        seg += o.segments
        tau += o.tau
    d.close()
    return seg / tau, R.lib.hwwref_num_threads(), (
        f"reference hww::run_step, config 2 steps 1-{steps} at {histories} histories/step "
        f"({seg} segments, {tau:.2f} s)")


def run_reference(args):
    rank, _, world = dist_setup(args)
    if rank != 0:
        return 0
    from oracle.bind import DriverRun, Reference, baseline_config, have_reference
    if not have_reference():
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libhww_ref.so not built"}))
        return 0
    R = Reference()
    cores = os.cpu_count() or 1
    R.lib.hwwref_set_threads(cores)
    # our arm runs histories x world (weak scaling); the CPU arm times a bounded
    # sample of that workload (segments/s is a rate, comparable across H)
    H = min(args.histories * world, 2_000_000)
    w = DriverRun(R, baseline_config(2, histories=H, time_steps=max(args.steps, args.warmup, 1)))
    for _ in range(args.warmup):
        w.step()
    w.close()
    d = DriverRun(R, baseline_config(2, histories=H, time_steps=max(args.steps, 1)))
    seg, tau, fom = 0, 0.0, []
    for _ in range(args.steps):
        o, _ = d.step()
        seg += o.segments
        tau += o.tau
        fom.append(o.fom_sigma_l2)
    value = seg / tau
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tau / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference point-pulse source)",
            "config": {"workload": WORKLOAD, "histories_per_step": H, "time_steps": args.steps,
                       "threads": R.lib.hwwref_num_threads()},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": R.lib.hwwref_num_threads(),
                             "kind": "reference",
                             "sample": f"config 2 steps 1-{args.steps}, {seg} segments"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "fom_sigma_l2_last": fom[-1] if fom else None}
    print(json.dumps(line))
    return 0


def run_ours(args):
    import torch

    rank, local, world = dist_setup(args)
    torch.cuda.set_device(local)
    import paper_2512_19925_b200 as hw
    if world > 1 and args.rng != "philox":
        args.rng = "philox"  # exact mode replays one sequential comb: single GPU only
    rng = hw.RNG_PHILOX if args.rng == "philox" else hw.RNG_EXACT
    # weak scaling: every GPU carries args.histories histories per step
    H = args.histories * world
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    nccl_id = b""
    if world > 1:  # rank 0 makes the NCCL id the driver's communicator uses
        import torch.distributed as tdist
        idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(hw.hww.nccl_unique_id()), dtype=torch.uint8))
        tdist.broadcast(idt, 0)
        nccl_id = bytes(idt.cpu().numpy().tobytes())

    def driver(cfg):
        return hw.Driver(cfg, device=local, rng_mode=rng, rank=rank, world=world,
                         nccl_id=nccl_id)

    # the clock sampler starts before the warm-up: nvidia-smi's first NVML
    # initialisation on a fresh box must not land inside the timed steps
    clk = ClockSampler(local).__enter__()
    # warm-up: a separate instance, steps 1..W
    if args.warmup:
        wd = driver(config2(H, max(args.warmup, 1)))
        for _ in range(args.warmup):
            wd.step()
        wd.close()

    d = driver(config2(H, max(args.steps, 1)))
    seg = 0
    dev_ms = 0.0
    tr_ms = 0.0
    tr_launch = 0
    launches = 0
    fom = []
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clk_first = len(clk.rows)
    for _ in range(args.steps):
        flush_l2(flush)
        torch.cuda.synchronize()
        rec = d.step()
        seg += rec.segments
        dev_ms += rec.device_ms
        tr_ms += rec.transport_ms
        tr_launch += rec.transport_launches
        launches += rec.kernel_launches
        fom.append(rec.fom_sigma_l2)
    torch.cuda.synchronize()
    clk_last = len(clk.rows)
    if world > 1:
        torch.distributed.barrier()
    d.close()
    t_max = max_over_ranks(dev_ms, world)
    seg_all = seg  # the driver all-reduces tracks_per_cell: every rank sees the global count
    value = seg_all / (t_max * 1e-3)

    # exact (reference-stream) mode on the same workload, single GPU only
    exact = None
    if world == 1 and args.rng == "philox" and not args.no_exact:
        xd = hw.Driver(config2(H, max(args.steps, 1)), device=local, rng_mode=hw.RNG_EXACT)
        xs, xms = 0, 0.0
        for _ in range(args.steps):
            flush_l2(flush)
            torch.cuda.synchronize()
            r = xd.step()
            xs += r.segments
            xms += r.device_ms
        xd.close()
        exact = {"value": xs / (xms * 1e-3), "unit": UNIT, "ms_per_step": xms / args.steps,
                 "note": "bit-exact replay of the reference's xoshiro streams, events, census "
                         "and tallies (tests/test_gpu_parity.py)"}

    # e2e through the public step API with the bank in pinned host memory
    e = driver(_host_cfg(H, args.steps))
    e_seg, e_s, h2d, d2h = 0, 0.0, 0, 0
    for _ in range(args.steps):
        flush_l2(flush)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rec = e.step()
        e_s += time.perf_counter() - t0
        e_seg += rec.segments
        h2d += rec.h2d_bytes
        d2h += rec.d2h_bytes
    e.close()
    e_s = max_over_ranks(e_s, world)
    e_val = e_seg / e_s

    peak, peak_kind = measured_peak()
    # per GPU: this GPU's share of the segments over its transport-kernel time
    achieved = (seg / world) * BYTES_PER_SEGMENT / (tr_ms * 1e-3) / 1e9 if tr_ms > 0 else 0.0
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(args.rng)
        except Exception:
            traffic = None

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (the reference's isotropic unit point pulse; no dataset)",
            "config": {"workload": WORKLOAD, "histories_per_step": H,
                       "histories_per_gpu": args.histories, "time_steps": args.steps,
                       "rng": args.rng,
                       "parallelism": (f"histories sharded x{world}, NCCL tally all-reduce + "
                                       "census rebalance" if world > 1 else "1 GPU"),
                       "l2": "256 MiB flush between timed steps"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "transport (history) kernel",
                         "bytes_per_unit": BYTES_PER_SEGMENT, "peak_kind": peak_kind,
                         "transport_ms": tr_ms, "transport_launches": tr_launch},
            "e2e": {"value": e_val, "unit": UNIT, "h2d_bytes_per_step": h2d // max(args.steps, 1),
                    "d2h_bytes_per_step": d2h // max(args.steps, 1)},
            "gpu_launches": launches,
            "fom_sigma_l2_last": fom[-1] if fom else None,
        }
        if exact:
            line["exact_mode"] = exact
        line["clocks"] = clk.summary(clk_first, clk_last)
        if not args.no_cpu_baseline:
            try:
                v, cores, sample = cpu_baseline(H, args.cpu_steps)
                line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores,
                                        "kind": "reference", "sample": sample}
                # also one thread (the reference's OpenMP path
                # scales poorly, so both are reported)
                v1, _, sample1 = cpu_baseline(H, args.cpu_steps, threads=1)
                line["cpu_baseline_1thread"] = {"value": v1, "unit": UNIT, "cores": 1,
                                                "kind": "reference", "sample": sample1}
            except Exception as ex:  # the checker is optional on a box without it
                line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0,
                                        "kind": "reference", "sample": f"unavailable: {ex}"}
        print(json.dumps(line))
    clk.__exit__(None, None, None)
    return 0


def _host_cfg(H, steps):
    c = config2(H, max(steps, 1))
    c.host_bank = True
    return c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rng", default="philox", choices=["exact", "philox"])
    ap.add_argument("--histories", type=int, default=1_000_000, help="histories per step per GPU")
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-exact", action="store_true", help="skip the exact-mode side run")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
