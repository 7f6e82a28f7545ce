# C5 step-1 heavy transport launch and the step-2 comb under ncu --set full
make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_segment -s 1 -c 1 -o gpurun_out/c5_step1 python scripts/step_times.py philox 2 c5 > gpurun_out/c5_ncu_s1.log 2>&1; echo s1=$?
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_comb_scatter -s 1 -c 1 -o gpurun_out/c5_comb2 python scripts/step_times.py philox 2 c5 > gpurun_out/c5_ncu_comb.log 2>&1; echo comb=$?
