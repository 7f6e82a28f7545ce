#!/usr/bin/env python3
"""Summarise ncu artefacts into profiles/ (markdown + json).

  python scripts/ncu_summary.py launches <launches.csv> <out.md>
  python scripts/ncu_summary.py full <report.ncu-rep> <out.md> [traffic_key]

`full` also merges {traffic_key: dram bytes per launch} into profiles/traffic.json,
which bench.py reports as roofline.traffic.
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui].strip().lower()
        v = v / 1e3 if unit in ("nsecond", "ns") else (v * 1e3 if unit in ("msecond", "ms") else v)
        name = r[ki].split("(")[0].replace("hwwg::<unnamed>::", "")[:70]
        a = agg.setdefault(name, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += v
        a[2] = max(a[2], v)
    tot = sum(a[1] for a in agg.values())
    lines = [f"# Launch list: `{os.path.basename(path)}`", "",
             "ncu `--metrics gpu__time_duration.sum --clock-control none` (cold-cache, "
             "serialised launches: compare shares, not absolutes).", "",
             f"Total kernel time {tot / 1e3:.2f} ms over {sum(a[0] for a in agg.values())} launches.",
             "", "| kernel | launches | total ms | share | max us |", "|---|---:|---:|---:|---:|"]
    for name, (n, t, m) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{name}` | {n} | {t / 1e3:.3f} | {100 * t / tot:.1f}% | {m:.1f} |")
    open(out, "w").write("\n".join(lines) + "\n")


def _csv(cmd):
    return list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))


def full(rep, out, key=None):
    det = _csv(["ncu", "-i", rep, "--page", "details", "--csv"])
    h = det[0]
    si, mi, vi, ui = (h.index(x) for x in ("Section Name", "Metric Name", "Metric Value",
                                           "Metric Unit"))
    kname = det[1][h.index("Kernel Name")] if len(det) > 1 else "?"
    want = {"GPU Speed Of Light Throughput", "Compute Workload Analysis", "Memory Workload Analysis",
            "Occupancy", "Scheduler Statistics", "Warp State Statistics", "Launch Statistics"}
    lines = [f"# ncu --set full: `{kname}`", "", f"Report: `{os.path.basename(rep)}`", "",
             "| section | metric | value |", "|---|---|---|"]
    for r in det[1:]:
        if r[si] in want and r[mi]:
            lines.append(f"| {r[si]} | {r[mi]} | {r[vi]} {r[ui]} |")
    raw = _csv(["ncu", "-i", rep, "--page", "raw", "--csv"])
    rh, ru, rv = raw[0], raw[1], raw[2]
    d = dict(zip(rh, rv))
    u = dict(zip(rh, ru))

    def num(k):
        try:
            return float(d[k].replace(",", ""))
        except Exception:
            return None
    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    to_bytes = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    if rd is not None:
        rd *= to_bytes.get(u.get("dram__bytes_read.sum", "byte"), 1)
    if wr is not None:
        wr *= to_bytes.get(u.get("dram__bytes_write.sum", "byte"), 1)
    stalls = []
    for k in rh:
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            v = num(k)
            if v:
                stalls.append((v, k.replace("smsp__average_warps_issue_stalled_", "")
                               .replace("_per_issue_active.ratio", "")))
    stalls.sort(reverse=True)
    lines += ["", f"DRAM bytes per launch: read {rd:.4g}, write {wr:.4g}, total {(rd or 0) + (wr or 0):.4g}",
              "", "Warp stall reasons (warps per issued instruction):", "",
              "| reason | ratio |", "|---|---:|"]
    lines += [f"| {n} | {v:.2f} |" for v, n in stalls[:12]]
    open(out, "w").write("\n".join(lines) + "\n")
    if key and rd is not None:
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        t = json.load(open(tp)) if os.path.exists(tp) else {}
        t[key] = (rd or 0) + (wr or 0)
        json.dump(t, open(tp, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
