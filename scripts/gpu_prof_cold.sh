make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_segment -s 1 -c 1 -o gpurun_out/r2b_c5_cold python scripts/step_times.py philox 2 c5 > gpurun_out/r2b_n2.log 2>&1; echo full2=$?
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_segment -s 12 -c 1 -o gpurun_out/r2b_c5_steady python scripts/step_times.py philox 5 c5 > gpurun_out/r2b_n1.log 2>&1; echo full1=$?
