#!/usr/bin/env python3
"""Per-source-line instruction and stall-sample totals from an ncu report
(`--page source --print-source cuda,sass`): where a kernel's issue slots and
stalls go.  python scripts/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname = "?"
rows = []
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        ins = int(d.get("Instructions Executed", "0") or 0)
        smp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    rows.append((fname, r[0], r[1][:90], ins, smp))
ti = sum(x[3] for x in rows) or 1
ts = sum(x[4] for x in rows) or 1
print(f"total warp instructions {ti}, stall samples {ts}")
print("\n-- by stall samples")
for f, ln, src, ins, smp in sorted(rows, key=lambda x: -x[4])[:top]:
    print(f"{100*smp/ts:5.1f}% smp {100*ins/ti:5.1f}% ins  {f}:{ln}  {src}")
print("\n-- by instructions")
for f, ln, src, ins, smp in sorted(rows, key=lambda x: -x[3])[:top]:
    print(f"{100*ins/ti:5.1f}% ins {100*smp/ts:5.1f}% smp  {f}:{ln}  {src}")
