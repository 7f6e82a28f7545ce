make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python scripts/step_times.py philox 40 > gpurun_out/steps_cur.log 2>&1; echo steps=$?
