# ncu --set full of one steady-state transport launch (step 11, segment 0)
make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
CMD="python scripts/step_times.py philox 12"
REPS=1 timeout 300 $CMD > gpurun_out/prof2_plain.log 2>&1; echo plain=$?
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_segment -s 40 -c 1 -o gpurun_out/prof_steady6 $CMD > gpurun_out/prof6_ncu.log 2>&1; echo ncu=$?
