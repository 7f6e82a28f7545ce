# round 2: multirank + statistical pin + full gpu suite
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q > gpurun_out/pytest_multirank.log 2>&1; echo multirank=$?
tail -30 gpurun_out/pytest_multirank.log | grep -v "^  File"
timeout 1500 python -m pytest tests/test_gpu_stat_pin.py -q > gpurun_out/pytest_statpin.log 2>&1; echo statpin=$?
grep -E "passed|failed|Error|assert" gpurun_out/pytest_statpin.log | head -30
timeout 1200 python -m pytest tests -m gpu -q --deselect tests/test_gpu_stat_pin.py > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log | grep -v "^  File"
