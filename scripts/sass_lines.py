#!/usr/bin/env python3
"""Per-source-line instruction counts of one kernel from an ncu report.

    python scripts/sass_lines.py <report.ncu-rep> <object.o> <kernel-substring> [top]

Joins ncu's SASS page (Instructions Executed, stall samples per instruction)
with nvdisasm -g line info of the same cubin (compiled with -lineinfo), and
sums per line of the kernel's own source file (inlined callees are charged to
the kernel line they were inlined at)."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, obj, kern = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, check=True,
               capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cubin)], capture_output=True,
                     text=True).stdout.splitlines()
# instruction offsets -> (file, line) of the outermost frame in the kernel's file
sec, loc, lines = None, None, {}
for l in dis:
    if l.startswith("\t.section\t.text.") or l.startswith(".section .text."):
        sec = kern in l
    m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', l)
    if m:
        f, n, rest = m.group(1), int(m.group(2)), m.group(3)
        chain = [(f, n)] + [(a, int(b)) for a, b in re.findall(r'inlined at "([^"]+)", line (\d+)', rest)]
        loc = chain[-1]
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/', l)
    if m and sec:
        lines[int(m.group(1), 16)] = loc
# NCU_K=<name>: a report holding several kernels is filtered to that one
kf = ["-k", os.environ["NCU_K"]] if os.environ.get("NCU_K") else []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + kf,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ie, ss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
base = int(rows[2][0], 16)
cnt, stl = collections.Counter(), collections.Counter()
src = {}
for r in rows[2:]:
    if len(r) <= ie or not r[ie].isdigit():
        continue
    off = int(r[0], 16) - base
    f, n = lines.get(off, ("?", 0))
    key = (os.path.basename(f), n)
    cnt[key] += int(r[ie])
    stl[key] += int(r[ss] or 0)
tot, tots = sum(cnt.values()), sum(stl.values())
print(f"total warp instructions {tot:,}, stall samples {tots:,}")
srcs = {}
for f in {k[0] for k in cnt}:
    for cand in [os.path.join(os.path.dirname(os.path.abspath(obj)), "..", "csrc", f)]:
        if os.path.exists(cand):
            srcs[f] = open(cand).read().splitlines()
for k, v in cnt.most_common(top):
    text = srcs.get(k[0], [""] * (k[1] + 1))[k[1] - 1].strip()[:70] if k[1] else ""
    print(f"{100 * v / tot:5.1f}% instr {100 * stl[k] / max(tots, 1):5.1f}% stall  {k[0]}:{k[1]:<5} {text}")
