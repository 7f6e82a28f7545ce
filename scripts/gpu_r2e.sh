# full gpu suite (incl. stat pin + multirank) + C5 step times + quick bench
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -25 gpurun_out/pytest_gpu.log | grep -v "^  File" | tail -14
REPS=1 timeout 300 python scripts/step_times.py philox 20 c5 > gpurun_out/c5_steps.log 2>&1; echo steps=$?
head -8 gpurun_out/c5_steps.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-exact > gpurun_out/bench_quick.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_quick.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['ms_per_step']); [print(k, '%.3e'%v.get('value',0), v.get('transport_frac')) for k,v in d['configs'].items()]"
