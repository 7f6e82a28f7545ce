# round-2 evidence for profiles/: launch list of a short default bench, ncu --set full of the
# C5 steady and cold-start transport launches, the comb, and a C2 steady launch
make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
CMD="python bench.py --steps 6 --warmup 0 --no-cpu-baseline --no-exact --no-configs"
timeout 300 $CMD > gpurun_out/r2_plain.log 2>&1; echo plain=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/r2_launches_c5.csv $CMD > gpurun_out/r2_ncu_l.log 2>&1; echo launches=$?
REPS=1 timeout 300 python scripts/step_times.py philox 5 c5 > gpurun_out/r2_steps.log 2>&1; echo steps=$?
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_segment -s 12 -c 1 -o gpurun_out/r2_c5_steady python scripts/step_times.py philox 5 c5 > gpurun_out/r2_n1.log 2>&1; echo full1=$?
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_segment -s 1 -c 1 -o gpurun_out/r2_c5_cold python scripts/step_times.py philox 2 c5 > gpurun_out/r2_n2.log 2>&1; echo full2=$?
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cb_ -s 2 -c 2 -o gpurun_out/r2_comb python scripts/step_times.py philox 2 c5 > gpurun_out/r2_n3.log 2>&1; echo full3=$?
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_segment -s 40 -c 1 -o gpurun_out/r2_c2_steady python scripts/step_times.py philox 12 c2 > gpurun_out/r2_n4.log 2>&1; echo full4=$?
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_low_order_update -s 20 -c 1 -o gpurun_out/r2_losm python scripts/step_times.py philox 6 c2 > gpurun_out/r2_n5.log 2>&1; echo full5=$?
