import sys, time; sys.path.insert(0, ".")
import paper_2512_19925_b200 as hw
from scripts.bench_configs import cfg
import torch
H = int(float(sys.argv[1])); steps = int(sys.argv[2])
d = hw.Driver(cfg(4, H, steps), rng_mode=hw.RNG_PHILOX)
t0 = time.time()
for _ in range(steps):
    r = d.step()
    free, tot = torch.cuda.mem_get_info()
    print(r.step, r.segments, r.census_size, r.comb_in, f"{r.device_ms:.1f} ms", f"used {(tot-free)/1e9:.1f} GB", flush=True)
print("wall", time.time() - t0)
