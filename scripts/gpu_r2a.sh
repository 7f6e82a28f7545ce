# round 2: new multirank tests, full gpu suite, bench (headline C5 + configs)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q > gpurun_out/pytest_multirank.log 2>&1; echo multirank=$?
tail -30 gpurun_out/pytest_multirank.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c5.log 2> gpurun_out/bench_c5.err; echo bench=$?
tail -1 gpurun_out/bench_c5.log; tail -5 gpurun_out/bench_c5.err
