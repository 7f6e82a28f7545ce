# A/B of run-time knobs on the headline: each line "<env> value frac steps"
B="python bench.py --no-cpu-baseline --no-exact --no-configs --config ${CFG:-c5}"
for e in "$@"; do
  env $e timeout 300 $B > gpurun_out/ab.log 2>&1
  python -c "
import json,sys
l=[x for x in open('gpurun_out/ab.log') if x.startswith('{')]
j=json.loads(l[-1]) if l else {}
print(sys.argv[1], '%.4g'%j.get('value',0), 'frac', round(j.get('roofline',{}).get('frac',0),4), 'steps', [round(x,2) for x in j.get('step_ms',[])[:4]])
" "$e" | tee -a gpurun_out/ab_summary.txt
done
