# C5 headline profiling: step times, phases, timeline, launch list, one steady ncu --set full
make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
REPS=1 timeout 300 python scripts/step_times.py philox 20 c5 > gpurun_out/c5_steps.log 2>&1; echo steps=$?
cat gpurun_out/c5_steps.log
HWWG_PHASES=1 REPS=1 timeout 300 python scripts/step_times.py philox 4 c5 > gpurun_out/c5_phases.log 2>&1; echo phases=$?
grep phases gpurun_out/c5_phases.log
HWWG_FAST_TIMELINE=1 REPS=1 timeout 300 python scripts/step_times.py philox 4 c5 > gpurun_out/c5_timeline.log 2>&1; echo timeline=$?
grep timeline gpurun_out/c5_timeline.log | head -20
CMD="python bench.py --steps 6 --warmup 0 --no-cpu-baseline --no-exact --no-configs"
timeout 300 $CMD > gpurun_out/c5_plain.log 2>&1; echo plain=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/c5_launches.csv $CMD > gpurun_out/c5_ncu_l.log 2>&1; echo launches=$?
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_segment -s 12 -c 1 -o gpurun_out/c5_steady python scripts/step_times.py philox 5 c5 > gpurun_out/c5_ncu_full.log 2>&1; echo full=$?
