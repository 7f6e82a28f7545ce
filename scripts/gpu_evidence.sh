# full verification + evidence: gpu suite, smoke, default bench, reference arm, launch list, ncu captures
make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref=$?
CMD="python bench.py --steps 6 --warmup 0 --no-cpu-baseline --no-exact --no-configs"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/r2_launches_c5.csv $CMD > /dev/null 2>&1; echo launches=$?
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_segment -s 12 -c 1 -o gpurun_out/r2_c5_steady python scripts/step_times.py philox 5 c5 > /dev/null 2>&1; echo full1=$?
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_segment -s 1 -c 1 -o gpurun_out/r2_c5_cold python scripts/step_times.py philox 2 c5 > /dev/null 2>&1; echo full2=$?
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cb_ -s 2 -c 2 -o gpurun_out/r2_comb python scripts/step_times.py philox 2 c5 > /dev/null 2>&1; echo full3=$?
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_segment -s 40 -c 1 -o gpurun_out/r2_c2_steady python scripts/step_times.py philox 12 c2 > /dev/null 2>&1; echo full4=$?
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_losm_mid_fast -s 10 -c 1 -o gpurun_out/r2_losm python scripts/step_times.py philox 6 c2 > /dev/null 2>&1; echo full5=$?
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast_segment -s 30 -c 1 -o gpurun_out/r2_c3_steady python scripts/step_times.py philox 10 c3 > /dev/null 2>&1; echo full6=$?
