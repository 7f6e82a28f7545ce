# full verification: gpu suite, smoke, bench (default), reference arm
make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -4 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; echo bench=$?
tail -1 gpurun_out/bench_default.log | cut -c1-1500
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref=$?
tail -1 gpurun_out/bench_ref.log | cut -c1-800
