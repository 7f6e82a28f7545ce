for cfg in "c5 20" "c2 20" "c3 20" "c1 20" "c4 4 12500000" "c5:2:0 20" "c5:10:2 20"; do
  set -- $cfg
  r=$(REPS=2 timeout 600 python scripts/step_times.py philox $2 $1 $3 2>/dev/null | grep "rep 1")
  echo "new | $1 | $r"
done
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -4 gpurun_out/pytest_gpu.log
