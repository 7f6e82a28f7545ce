set -x
timeout 300 python bench.py --rng philox --steps 6 --warmup 1 --histories 100000 --no-cpu-baseline > gpurun_out/bench_fast_small.log 2>&1; echo bench_fast_small=$?
CMD="python bench.py --rng philox --steps 6 --warmup 0 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_fast.csv $CMD > gpurun_out/ncu.log 2>&1; echo ncu=$?
