make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
REPS=1 timeout 300 python scripts/step_times.py philox 6 c5 > gpurun_out/c5_steps.log 2>&1; echo steps=$?
head -9 gpurun_out/c5_steps.log
HWWG_PHASES=1 REPS=1 timeout 300 python scripts/step_times.py philox 4 c5 2>&1 | grep phases
REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/c5b_launches.csv python scripts/step_times.py philox 3 c5 > /dev/null 2>&1; echo launches=$?
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cb_ -s 2 -c 2 -o gpurun_out/c5_cb python scripts/step_times.py philox 2 c5 > gpurun_out/c5_ncu_cb.log 2>&1; echo cb=$?
