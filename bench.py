#!/usr/bin/env python3
"""Benchmark: track-segments/sec of the HWW time-step loop on B200.

Headline workload (--config c5, the default): the largest single-GPU BASELINE
configuration the reference driver can also run — config 5's (rho = 5, 3-point
moving-average closure filter) point: config-2 geometry (slab [-20,20], 400
cells, sigma_t = 1, c = 0.9, v = 1, unit plane pulse at x = 0, 40 steps of
dt = 0.5), 1e7 histories/step per GPU, seed 11, reference defaults elsewhere
(theta = 0.5, eps_min = 1e-3, u_ww = 3, f = 1/4, 1/2, 3/4, 20 batches).
Synthetic by construction (the reference's own point-pulse source); no dataset.
--config c1 | c2 | c3 | c4 | c5[:rho:k] selects another BASELINE configuration
(paper_2512_19925_b200/configs.py); c4 runs one GPU's share, 1.25e7 histories.

A bench "step" is one time step of that run (comb -> LOSM windows -> 4
transport segments with 3 mid-step updates -> finalize -> census).  W warm-up
steps run on a separate driver instance; the K timed steps are steps 1..K of
a fresh run, so step 1's cold-start split explosion (census x63) is timed.
L2 is flushed (a 256 MiB write) between timed steps, outside the per-step
CUDA-event window.

value = sum(segments) / max over ranks of sum(step device time); a segment is
one increment of tracks_per_cell (proj/src/transport.cpp:136-139).  e2e = the
same metric with the bank round-tripping through pinned host memory every step
(hwwg_driver with host_bank = 1: H2D of the step's source bank, D2H of the next
step's source and of the record), the K steps timed back to back on the host
clock up to a device-wide synchronize (the driver pipelines each step's source
through host memory in pieces: uploads wait only for their own piece's
download, so the two PCIe directions overlap).  In Philox mode the
device combs the census before handing it to the host (the comb that opens the
next step, with that step's stream), so H particles cross PCIe each way, not
the raw census.  FOM per step: fom_sigma_l2 (metrics.cpp:34-55; driver.cpp:
272-275) and the median per-cell 1/(tau sigma^2) over cells with phi > 1e-3 max.

--gpus N > 1 without a torchrun environment re-launches this script under
torch.distributed.run (one process per GPU, NCCL); a WORLD_SIZE that differs
from N is an error.  Histories are sharded (weak scaling: H per GPU fixed).

--impl reference: the unmodified reference (oracle/_ref/libhww_ref.so, built
from /root/reference/proj) running hww::run_step on this box's CPU cores with
every OpenMP thread, same configuration at a bounded history count; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
REF_MAX_H = 2_000_000   # reference arm: bounded history sample (segments/s is a rate)


def parse_config(name):
    """'c5' -> (5, {}), 'c5:10:2' -> (5, {rho: 10, ma_base_k: 2}), 'c4' -> (4, H 1.25e7)."""
    parts = name.lower().lstrip("c").split(":")
    which = int(parts[0])
    kw = {}
    if which == 5 and len(parts) == 3:
        kw = dict(rho=float(parts[1]), ma_base_k=int(parts[2]))
    return which, kw


def default_histories(which):
    from paper_2512_19925_b200.configs import baseline
    if which == 4:
        return 12_500_000  # one GPU's share of config 4's 1e8 over 8
    return baseline(which).histories_per_step


def workload_name(which, kw, H):
    from paper_2512_19925_b200.configs import DESCRIPTION
    d = DESCRIPTION[which]
    if which == 5:
        rho, k = kw.get("rho", 5.0), kw.get("ma_base_k", 1)
        d += f"; this point: rho={rho:g}, filter={'none' if k == 0 else f'MA{2 * k + 1} (k={k})'}"
    if which == 4:
        d += f"; {H:.3g} histories/step per GPU"
    return d


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


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


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_or_check(args):
    """--gpus N: one process per GPU.  Without a torchrun environment, re-exec
    under torch.distributed.run; with one, its WORLD_SIZE must be N."""
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None:
        if args.gpus <= 1:
            return None
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    if int(env_world) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}", file=sys.stderr)
        return 2
    return None


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "nccl" if args.impl != "reference" else "gloo"
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
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


def fom_stats(rec, arr):
    """(fom_sigma_l2, median per-cell FOM over cells with phi > 1e-3 max)."""
    import numpy as np
    phi, sig = arr["phi_track"], arr["sigma"]
    m = (phi > 1e-3 * np.nanmax(phi)) & (sig > 0)
    med = float(np.median(1.0 / (max(rec.tau, 1e-9) * sig[m] ** 2))) if m.any() else None
    return (float(rec.fom_sigma_l2) if rec.sigma_valid else None), med


def reference_rate(which, kw, H, steps, threads=None, warmup=0):
    """The reference (oracle/_ref) driver on this host: steps 1..steps of the
    configuration at H histories.  Returns (segments/s, threads, sample, fom list)."""
    from oracle.bind import DriverRun, Reference, baseline_config
    R = Reference()
    R.lib.hwwref_set_threads(threads or os.cpu_count() or 1)
    okw = dict(kw)
    if which == 5 and okw.get("ma_base_k", 1) == 0:
        okw.pop("ma_base_k")
        okw["mode"] = "hww"
    if warmup:
        w = DriverRun(R, baseline_config(which, histories=H, time_steps=max(warmup, 1), **okw))
        for _ in range(warmup):
            w.step()
        w.close()
    d = DriverRun(R, baseline_config(which, histories=H, time_steps=max(steps, 1), **okw))
    seg, tau, fom = 0, 0.0, []
    for _ in range(steps):
        o, _ = d.step()
        seg += o.segments
        tau += o.tau
        fom.append(o.fom_sigma_l2)
    d.close()
    n = R.lib.hwwref_num_threads()
    return seg / tau, n, (f"reference hww::run_step, config {which} {okw or ''} steps 1-{steps} "
                          f"at {H} histories/step ({seg} segments, {tau:.2f} s, {n} threads, "
                          f"{cpu_model()})"), fom


def run_reference(args):
    rank, _, world = dist_setup(args)
    if rank != 0:
        return 0
    from oracle.bind import have_reference
    if not have_reference():
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libhww_ref.so not built"}))
        return 0
    which, kw = parse_config(args.config)
    if which == 3:  # no reference driver path for config 3
        print(json.dumps({"impl": "reference", "unavailable": "config 3 has no reference driver "
                          "path (no volumetric source / regions in hww::run)"}))
        return 0
    H_ours = (args.histories or default_histories(which)) * world
    H = min(H_ours, REF_MAX_H)
    value, n, sample, fom = reference_rate(which, kw, H, args.steps, warmup=args.warmup)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference point-pulse source)",
            "config": {"workload": workload_name(which, kw, H_ours), "histories_per_step": H,
                       "histories_sample_of": H_ours, "time_steps": args.steps, "threads": n,
                       "cpu": cpu_model()},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": n, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "fom_sigma_l2_per_step": fom}
    print(json.dumps(line))
    return 0


def timed_run(hw, cfg, steps, flush, make_driver, world=1, want_arrays=True):
    """Steps 1..steps of a fresh driver, L2 flushed between steps outside the
    device-timed window.  Returns a dict of sums and per-step FOM."""
    import torch
    d = make_driver(cfg)
    out = dict(seg=0, dev_ms=0.0, tr_ms=0.0, tr_launch=0, launches=0, fom_l2=[], fom_med=[],
               step_ms=[])
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    for _ in range(steps):
        flush_l2(flush)
        torch.cuda.synchronize()
        rec = d.step()
        out["seg"] += rec.segments
        out["dev_ms"] += rec.device_ms
        out["tr_ms"] += rec.transport_ms
        out["tr_launch"] += rec.transport_launches
        out["launches"] += rec.kernel_launches
        out["step_ms"].append(rec.device_ms)
        if want_arrays:
            l2, med = fom_stats(rec, d.arrays())
            out["fom_l2"].append(l2)
            out["fom_med"].append(med)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    d.close()
    return out


def run_ours(args):
    import torch

    rank, local, world = dist_setup(args)
    torch.cuda.set_device(local)
    import paper_2512_19925_b200 as hw
    from paper_2512_19925_b200.configs import baseline
    if world > 1 and args.rng != "philox":
        args.rng = "philox"  # exact mode replays one sequential comb: single GPU only
    rng = hw.RNG_PHILOX if args.rng == "philox" else hw.RNG_EXACT
    which, kw = parse_config(args.config)
    H1 = args.histories or default_histories(which)
    H = H1 * world  # weak scaling: every GPU carries H1 histories per step
    T = max(args.steps, 1)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    nccl_id = b""
    if world > 1:  # rank 0 makes the NCCL id the driver's communicator uses
        import torch.distributed as tdist
        idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(hw.hww.nccl_unique_id()), dtype=torch.uint8))
        tdist.broadcast(idt, 0)
        nccl_id = bytes(idt.cpu().numpy().tobytes())

    def driver(cfg, mode=rng):
        return hw.Driver(cfg, device=local, rng_mode=mode, rank=rank, world=world,
                         nccl_id=nccl_id)

    def cfg_of(steps, **extra):
        return baseline(which, histories=H, time_steps=steps, **kw, **extra)

    # the clock sampler starts before the warm-up: nvidia-smi's first NVML
    # initialisation on a fresh box must not land inside the timed steps
    clk = ClockSampler(local).__enter__()
    if args.warmup:  # a separate instance, steps 1..W
        wd = driver(cfg_of(max(args.warmup, 1)))
        for _ in range(args.warmup):
            wd.step()
        wd.close()

    clk_first = len(clk.rows)
    m = timed_run(hw, cfg_of(T), T, flush, driver, world)
    clk_last = len(clk.rows)
    t_max = max_over_ranks(m["dev_ms"], world)
    tr_max = max_over_ranks(m["tr_ms"], world)
    value = m["seg"] / (t_max * 1e-3)  # tracks_per_cell is all-reduced: global count

    # exact (reference-stream) mode on the same configuration, single GPU, at
    # <= 1e6 histories (its bit-exact census staging and tally log are sized per history)
    exact = None
    if world == 1 and args.rng == "philox" and not args.no_exact:
        He = min(H, 1_000_000)
        xm = timed_run(hw, baseline(which, histories=He, time_steps=T, **kw), T, flush,
                       lambda c: hw.Driver(c, device=local, rng_mode=hw.RNG_EXACT),
                       want_arrays=False)
        exact = {"value": xm["seg"] / (xm["dev_ms"] * 1e-3), "unit": UNIT,
                 "ms_per_step": xm["dev_ms"] / T, "histories_per_step": He,
                 "note": "bit-exact replay of the reference's xoshiro streams, events, census "
                         "and tallies (tests/test_gpu_parity.py)"}

    # e2e through the public step API with the bank in pinned host memory
    # The K steps run back to back in one host-timed region that ends with a
    # device-wide synchronize, so every step's uploads and the bank downloads
    # still in flight when a step returns (the driver pipelines the next step's
    # source through host memory in pieces) are inside it. No L2 flush between
    # steps: each step's input crosses from host memory (>= 16 B x 1e7 = 160 MB
    # per step, above the 126 MB L2).
    e = driver(cfg_of(T, host_bank=True))
    e_seg, h2d, d2h = 0, 0, 0
    flush_l2(flush)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(T):
        rec = e.step()
        e_seg += rec.segments
        h2d += rec.h2d_bytes
        d2h += rec.d2h_bytes
    torch.cuda.synchronize()
    e_s = time.perf_counter() - t0
    e.close()
    e_s = max_over_ranks(e_s, world)
    e_val = e_seg / e_s

    # every other BASELINE configuration, briefly (single GPU, rank 0's view)
    others = None
    if world == 1 and not args.no_configs:
        others = {}
        sweep = [("C1", 1, {}, None, 20), ("C2", 2, {}, None, 20), ("C3", 3, {}, None, 20),
                 ("C4 (1.25e7/GPU)", 4, {}, 12_500_000, 6),
                 ("C5 rho=2 none", 5, dict(rho=2.0, ma_base_k=0), None, 20),
                 ("C5 rho=5 MA3", 5, dict(rho=5.0, ma_base_k=1), None, 20),
                 ("C5 rho=10 MA5", 5, dict(rho=10.0, ma_base_k=2), None, 20)]
        for name, w2, kw2, h2, st in sweep:
            if w2 == which and kw2 == kw and st == T:
                continue
            try:
                cfg2 = baseline(w2, histories=h2, time_steps=st, **kw2)
                r2 = timed_run(hw, cfg2, st, flush, driver)
                others[name] = {
                    "value": r2["seg"] / (r2["dev_ms"] * 1e-3), "ms_per_step": r2["dev_ms"] / st,
                    "steps": st, "histories_per_step": cfg2.histories_per_step,
                    "transport_frac": (r2["seg"] * BYTES_PER_SEGMENT / (r2["tr_ms"] * 1e-3) / 1e9
                                       / measured_peak()[0]) if r2["tr_ms"] > 0 else None,
                    "fom_sigma_l2_last": r2["fom_l2"][-1], "fom_median_last": r2["fom_med"][-1]}
            except Exception as ex:  # report, never hide
                others[name] = {"error": str(ex)[:200]}

    peak, peak_kind = measured_peak()
    # per GPU: this GPU's share of the segments over its transport-kernel time
    achieved = (m["seg"] / world) * BYTES_PER_SEGMENT / (tr_max * 1e-3) / 1e9 if tr_max > 0 else 0.0
    # DRAM bytes of one steady-state transport launch of this configuration from
    # an ncu --set full capture (profiles/round2_<config>_steady.md), or null
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp) and args.rng == "philox":
        try:
            traffic = json.load(open(tp)).get(f"{args.config.replace(':', '_')}_steady")
        except Exception:
            traffic = None

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / T, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (the reference's isotropic unit point pulse; no dataset)",
            "config": {"workload": workload_name(which, kw, H), "histories_per_step": H,
                       "histories_per_gpu": H1, "time_steps": T, "rng": args.rng,
                       "parallelism": (f"histories sharded x{world}, NCCL tally all-reduce + "
                                       "census rebalance" if world > 1 else "1 GPU"),
                       "l2": "256 MiB flush between timed steps"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "transport (history) kernel",
                         "bytes_per_unit": BYTES_PER_SEGMENT, "peak_kind": peak_kind,
                         "transport_ms": tr_max, "transport_launches": m["tr_launch"],
                         "whole_step_frac": value / world * BYTES_PER_SEGMENT / 1e9 / peak},
            "e2e": {"value": e_val, "unit": UNIT, "h2d_bytes_per_step": h2d // T,
                    "d2h_bytes_per_step": d2h // T},
            "gpu_launches": m["launches"],
            "step_ms": m["step_ms"],
            "fom_sigma_l2_per_step": m["fom_l2"],
            "fom_median_per_step": m["fom_med"],
        }
        if exact:
            line["exact_mode"] = exact
        if others is not None:
            line["configs"] = others
        line["clocks"] = clk.summary(clk_first, clk_last)
        if not args.no_cpu_baseline and which != 3:
            try:
                Hc = min(H, 1_000_000)
                v, cores, sample, _ = reference_rate(which, kw, Hc, args.cpu_steps)
                line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores,
                                        "kind": "reference", "sample": sample}
                # also one thread (the reference's OpenMP path
                # scales poorly, so both are reported)
                v1, _, sample1, _ = reference_rate(which, kw, Hc, args.cpu_steps, threads=1)
                line["cpu_baseline_1thread"] = {"value": v1, "unit": UNIT, "cores": 1,
                                                "kind": "reference", "sample": sample1}
            except Exception as ex:  # the checker is optional on a box without it
                line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0,
                                        "kind": "reference", "sample": f"unavailable: {ex}"}
        print(json.dumps(line))
    clk.__exit__(None, None, None)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rng", default="philox", choices=["exact", "philox"])
    ap.add_argument("--config", default="c5", help="c1..c5, or c5:rho:k (default c5 = rho 5, MA3)")
    ap.add_argument("--histories", type=int, default=None,
                    help="histories per step per GPU (default: the configuration's)")
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-exact", action="store_true", help="skip the exact-mode side run")
    ap.add_argument("--no-configs", action="store_true", help="skip the other-config lines")
    args = ap.parse_args()
    rc = relaunch_or_check(args)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
