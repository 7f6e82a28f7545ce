# round 2: statistical pin (R=12) with report + drop-in through the reference driver
rm -f gpurun_out/statpin_report.jsonl
HWWG_STAT_REPORT=gpurun_out/statpin_report.jsonl timeout 1500 python -m pytest tests/test_gpu_stat_pin.py -q > gpurun_out/pytest_statpin.log 2>&1; echo statpin=$?
grep -E "passed|failed|Error" gpurun_out/pytest_statpin.log | head -30
timeout 1500 python -m pytest tests/test_dropin.py -q > gpurun_out/pytest_dropin.log 2>&1; echo dropin=$?
tail -20 gpurun_out/pytest_dropin.log
