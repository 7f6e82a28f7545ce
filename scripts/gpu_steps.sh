make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_default.log 2>&1; echo bench=$?
