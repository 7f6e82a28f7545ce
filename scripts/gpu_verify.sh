# verification pass: gpu suite, smoke, default bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -20 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; echo bench=$?
tail -c 3000 gpurun_out/bench_default.log
