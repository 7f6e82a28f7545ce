# ncu --set full of steady-state transport launches (step 11 seg 1; step 20 seg 3)
make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
CMD="python scripts/step_times.py philox 21"
REPS=1 timeout 300 $CMD > gpurun_out/prof2_plain.log 2>&1; echo plain=$?
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_segment -s 41 -c 1 -o gpurun_out/prof_steady3 $CMD > gpurun_out/prof3_ncu.log 2>&1; echo ncu=$?
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_segment -s 79 -c 1 -o gpurun_out/prof_tail3 $CMD > gpurun_out/prof3t_ncu.log 2>&1; echo ncu=$?
