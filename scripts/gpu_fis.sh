make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
rm -f gpurun_out/statpin_report.jsonl
HWWG_STAT_REPORT=gpurun_out/statpin_report.jsonl timeout 1500 python -m pytest tests/test_gpu_stat_pin.py -q -k "fission or config2" > gpurun_out/pytest_statpin.log 2>&1; echo statpin=$?
grep -E "passed|failed|Error" gpurun_out/pytest_statpin.log | head -10
timeout 600 python -m pytest tests/test_gpu_checked.py -q > gpurun_out/pytest_checked.log 2>&1; echo checked=$?; tail -2 gpurun_out/pytest_checked.log
REPS=1 timeout 300 python scripts/step_times.py philox 8 c5 > gpurun_out/c5_steps.log 2>&1; head -6 gpurun_out/c5_steps.log
