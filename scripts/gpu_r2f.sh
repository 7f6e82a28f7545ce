REPS=2 timeout 300 python scripts/step_times.py philox 20 c5 > gpurun_out/c5_steps.log 2>&1; echo steps=$?
head -8 gpurun_out/c5_steps.log
REPS=2 timeout 300 python scripts/step_times.py philox 20 c2 > gpurun_out/c2_steps.log 2>&1; head -2 gpurun_out/c2_steps.log
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -4 gpurun_out/pytest_gpu.log
