# census thinning: targeted GPU tests, then the headline bench with and without it
timeout 1500 python -m pytest tests/test_gpu_statistical.py tests/test_gpu_stat_pin.py tests/test_gpu_multirank.py tests/test_gpu_checked.py -q -x > gpurun_out/pytest_thin.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_thin.log
timeout 600 python bench.py --no-cpu-baseline --no-exact --no-configs > gpurun_out/bench_thin.log 2>&1; echo bench=$?
HWWG_PRECOMB=0 timeout 600 python bench.py --no-cpu-baseline --no-exact --no-configs > gpurun_out/bench_nothin.log 2>&1; echo bench0=$?
python - <<'PY'
import json
for f in ("bench_thin", "bench_nothin"):
    l = [x for x in open(f"gpurun_out/{f}.log") if x.startswith("{")]
    if not l: print(f, "no line"); continue
    j = json.loads(l[-1])
    print(f, j["value"], j["ms_per_step"], j.get("roofline", {}).get("frac"), j.get("e2e", {}).get("value"), [round(x,2) for x in j.get("step_ms", [])[:4]])
PY
