# ncu evidence for profiles/: launch list of a short bench run and --set full
# captures of a steady-state and a cold-start transport launch (each only after
# the same command exited 0 without ncu)
make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
CMD="python bench.py --steps 12 --warmup 0 --no-cpu-baseline --no-exact"
timeout 300 $CMD > gpurun_out/plain_prof.log 2>&1; echo plain=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/launches_fast.csv $CMD > gpurun_out/ncu_l.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_segment -s 41 -c 1 -o gpurun_out/prof_fast_steady $CMD > gpurun_out/ncu_full1.log 2>&1; echo full1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_segment -s 1 -c 1 -o gpurun_out/prof_fast_heavy $CMD > gpurun_out/ncu_full2.log 2>&1; echo full2=$?
