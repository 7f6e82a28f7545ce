# perf (scripts/step_times.py) for flush replica counts; GPU tests
make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
for r in 16 0 4 64; do
  HWWG_FAST_FLUSH_R=$r timeout 300 python scripts/step_times.py philox 40 > gpurun_out/steps_r$r.log 2>&1; echo r$r=$?
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
