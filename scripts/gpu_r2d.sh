timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q > gpurun_out/pytest_multirank.log 2>&1; echo multirank=$?
tail -30 gpurun_out/pytest_multirank.log | grep -v "^  File" | tail -12
rm -f gpurun_out/statpin_report.jsonl
HWWG_STAT_REPORT=gpurun_out/statpin_report.jsonl timeout 1500 python -m pytest tests/test_gpu_stat_pin.py -q > gpurun_out/pytest_statpin.log 2>&1; echo statpin=$?
grep -E "passed|failed|Error" gpurun_out/pytest_statpin.log | head -30
timeout 1200 python -m pytest tests -m gpu -q --deselect tests/test_gpu_stat_pin.py --deselect tests/test_gpu_multirank.py > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log | grep -v "^  File" | tail -8
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-exact --no-configs > gpurun_out/bench_quick.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_quick.log | cut -c1-600
