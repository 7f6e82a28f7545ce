REPS=1 timeout 300 python scripts/step_times.py philox 12 c2 > gpurun_out/c2_steps.log 2>&1; echo steps=$?
tail -13 gpurun_out/c2_steps.log
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_segment -s 40 -c 1 -o gpurun_out/c2_steady python scripts/step_times.py philox 12 c2 > /dev/null 2>&1; echo c2full=$?
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cb_ -s 10 -c 2 -o gpurun_out/c5_comb python scripts/step_times.py philox 8 c5 > /dev/null 2>&1; echo comb=$?
REPS=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c2_launches.csv python scripts/step_times.py philox 6 c2 > /dev/null 2>&1; echo launches=$?
