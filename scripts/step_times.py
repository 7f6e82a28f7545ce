"""Per-step device / transport / host times of one configuration.

    python scripts/step_times.py [philox|exact] [steps] [c5|c2|c5:rho:k|...] [histories]
"""
import os
import sys
import time

sys.path.insert(0, '.')
import torch  # noqa: E402

import paper_2512_19925_b200 as hw  # noqa: E402
from bench import parse_config  # noqa: E402
from paper_2512_19925_b200.configs import baseline  # noqa: E402

rng = hw.RNG_PHILOX if (len(sys.argv) < 2 or sys.argv[1] == 'philox') else hw.RNG_EXACT
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
which, kw = parse_config(sys.argv[3] if len(sys.argv) > 3 else "c2")
H = int(float(sys.argv[4])) if len(sys.argv) > 4 else None
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for rep in range(int(os.environ.get('REPS', '2'))):
    d = hw.Driver(baseline(which, histories=H, time_steps=N, **kw), rng_mode=rng)
    rows = []
    for s in range(N):
        flush.add_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = d.step()
        t1 = time.perf_counter()
        rows.append((s + 1, r.device_ms, r.transport_ms, (t1 - t0) * 1e3, r.segments, r.census_size,
                     r.counters.collisions, r.counters.splits, r.counters.split_daughters,
                     r.counters.roulette_kills, r.comb_in))
    d.close()
    tot = sum(r[1] for r in rows)
    seg = sum(r[4] for r in rows)
    print("rep %d: total dev %.1f ms, %.3e seg/s" % (rep, tot, seg / tot * 1e3))
print("step dev_ms transport_ms host_ms segments census coll splits daughters rkills comb_in")
for row in rows:
    print("%3d %8.3f %8.3f %8.3f %10d %10d %9d %8d %9d %8d %9d" % row)
