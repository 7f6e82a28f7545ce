# quick check: statistical + multirank tests, then the headline and C2/C3 benches
timeout 900 python -m pytest tests/test_gpu_statistical.py tests/test_gpu_stat_pin.py tests/test_gpu_multirank.py tests/test_gpu_checked.py -q -x > gpurun_out/q_pytest.log 2>&1; echo "pytest: $(tail -1 gpurun_out/q_pytest.log)"
B="python bench.py --no-cpu-baseline --no-exact --no-configs"
for cfg in ${CFGS:-c5 c2 c3}; do
  timeout 300 $B --config $cfg > gpurun_out/q_$cfg.log 2>&1
  python -c "
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
j=json.loads(l[-1]) if l else {}
print(sys.argv[2], '%.4g'%j.get('value',0), 'ms/step %.3f'%j.get('ms_per_step',0), 'frac', j.get('roofline',{}).get('frac'), 'e2e %.4g'%j.get('e2e',{}).get('value',0), 'steps', [round(x,2) for x in j.get('step_ms',[])[:3]])
" gpurun_out/q_$cfg.log $cfg
done
