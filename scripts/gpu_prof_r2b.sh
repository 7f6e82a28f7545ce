# per-step numbers of the headline, and ncu full captures (cold + steady) with source counters
REPS=1 timeout 300 python scripts/step_times.py philox 20 c5 > gpurun_out/c5_steps.log 2>&1; echo steps=$?
cat gpurun_out/c5_steps.log
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_segment -s 1 -c 1 -o gpurun_out/c5_cold python scripts/step_times.py philox 2 c5 > /dev/null 2>&1; echo full_cold=$?
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_segment -s 12 -c 1 -o gpurun_out/c5_steady python scripts/step_times.py philox 5 c5 > /dev/null 2>&1; echo full_steady=$?
