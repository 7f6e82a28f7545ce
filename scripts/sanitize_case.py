"""A small driver run for compute-sanitizer (tests/test_gpu_sanitizer.py):
    python scripts/sanitize_case.py [philox|exact] [config] [H] [steps]"""
import sys

sys.path.insert(0, ".")
import paper_2512_19925_b200 as hw  # noqa: E402
from paper_2512_19925_b200.configs import baseline  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "philox"
which = int(sys.argv[2]) if len(sys.argv) > 2 else 2
H = int(sys.argv[3]) if len(sys.argv) > 3 else 5000
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
c = baseline(which, histories=H, time_steps=steps)
if which == 3:
    c.vol_histories = H
d = hw.Driver(c, rng_mode=hw.RNG_PHILOX if mode == "philox" else hw.RNG_EXACT)
for _ in range(steps):
    r = d.step()
d.close()
print("ok", r.segments)
