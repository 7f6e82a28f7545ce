CMD="python bench.py --rng philox --steps 6 --warmup 0 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_fast.csv $CMD > gpurun_out/ncu.log 2>&1; echo ncu=$?
timeout 600 python bench.py --rng philox --steps 40 --warmup 3 > gpurun_out/bench_fast.log 2>&1; echo bench_fast_full=$?
timeout 900 python bench.py --rng exact --steps 40 --warmup 3 --no-cpu-baseline > gpurun_out/bench_exact.log 2>&1; echo bench_exact_full=$?
timeout 900 python bench.py --impl reference --steps 40 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo bench_ref=$?
