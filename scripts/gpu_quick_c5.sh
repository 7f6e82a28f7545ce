make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
REPS=1 timeout 300 python scripts/step_times.py philox 20 c5 > gpurun_out/c5_steps.log 2>&1; echo steps=$?
head -8 gpurun_out/c5_steps.log
REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/c5b_launches.csv python scripts/step_times.py philox 3 c5 > /dev/null 2>&1; echo launches=$?
timeout 900 python -m pytest tests/test_gpu_statistical.py tests/test_gpu_multirank.py -q -x 2>&1 | tail -3
