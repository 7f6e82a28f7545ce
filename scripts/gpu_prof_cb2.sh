make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cb_scatter -s 1 -c 1 -o gpurun_out/c5_cbs python scripts/step_times.py philox 2 c5 > gpurun_out/c5_ncu_cbs.log 2>&1; echo cb=$?
