make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
REPS=2 timeout 300 python scripts/step_times.py philox 20 c5 > gpurun_out/c5_steps.log 2>&1; echo steps=$?
head -9 gpurun_out/c5_steps.log
REPS=2 timeout 300 python scripts/step_times.py philox 20 c2 2>&1 | head -2
timeout 900 python -m pytest tests/test_gpu_stat_pin.py -q -k "config2 or fission" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_statistical.py tests/test_gpu_checked.py -q 2>&1 | tail -2
