set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 5 --warmup 3 --histories 100000 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1; echo bench=$?
tail -15 gpurun_out/pytest_gpu.log
