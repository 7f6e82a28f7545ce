"""Per-step host wall time of the e2e (host_bank) path, pipelined or not.

    python scripts/e2e_probe.py [config] [steps]
"""
import os
import sys
import time

sys.path.insert(0, '.')
import torch  # noqa: E402

import paper_2512_19925_b200 as hw  # noqa: E402
from bench import parse_config  # noqa: E402
from paper_2512_19925_b200.configs import baseline  # noqa: E402

which, kw = parse_config(sys.argv[1] if len(sys.argv) > 1 else "c5")
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8
for pipe in ("1", "0"):
    os.environ["HWWG_E2E_PIPE"] = pipe
    for host in (True, False):
        c = baseline(which, time_steps=N, **kw)
        c.host_bank = host
        d = hw.Driver(c, rng_mode=hw.RNG_PHILOX)
        torch.cuda.synchronize()
        ts, dev = [], []
        t0 = time.perf_counter()
        for _ in range(N):
            a = time.perf_counter()
            r = d.step()
            ts.append((time.perf_counter() - a) * 1e3)
            dev.append(r.device_ms)
        torch.cuda.synchronize()
        tot = (time.perf_counter() - t0) * 1e3
        d.close()
        print(f"pipe={pipe} host_bank={host}: total {tot:.1f} ms; per-step host ms",
              [round(x, 2) for x in ts], "dev ms", [round(x, 2) for x in dev])
