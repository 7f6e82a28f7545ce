CMD="python bench.py --rng philox --steps 3 --warmup 0 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_prof.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_segment -s 9 -c 1 -o gpurun_out/prof_fast_seg3 $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
