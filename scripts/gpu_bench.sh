# full bench (both arms) as the driver runs it
make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref=$?
