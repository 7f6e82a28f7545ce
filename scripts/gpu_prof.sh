CMD="python bench.py --steps 6 --warmup 0 --no-cpu-baseline --no-exact"
timeout 300 $CMD > gpurun_out/plain_prof.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/launches_fast.csv $CMD > gpurun_out/ncu_l.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_segment -s 9 -c 1 -o gpurun_out/prof_fast_steady $CMD > gpurun_out/ncu_full1.log 2>&1; echo full1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_segment -s 1 -c 1 -o gpurun_out/prof_fast_heavy $CMD > gpurun_out/ncu_full2.log 2>&1; echo full2=$?
CMD2="python bench.py --rng exact --steps 3 --warmup 0 --no-cpu-baseline --histories 100000"
timeout 300 $CMD2 > gpurun_out/plain_exact.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_exact_chunks -s 5 -c 1 -o gpurun_out/prof_exact $CMD2 > gpurun_out/ncu_full3.log 2>&1; echo full3=$?
