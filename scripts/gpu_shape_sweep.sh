# transport block shapes: the headline and C2/C3/C4 per forced shape
B="python bench.py --no-cpu-baseline --no-exact --no-configs"
summ() { python -c "
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')]
j=json.loads(l[-1]) if l else {}
print(sys.argv[2], '%.4g'%j.get('value',0), 'ms/step %.3f'%j.get('ms_per_step',0), 'frac', j.get('roofline',{}).get('frac'), 'steps', [round(x,2) for x in j.get('step_ms',[])[:3]])
" $1 "$2"; }
for cfg in c5 c2 c3; do
for w in 0 12 16 24 32; do
  HWWG_FAST_BLOCK_WARPS=$w timeout 300 $B --config $cfg > gpurun_out/sw_${cfg}_$w.log 2>&1
  summ gpurun_out/sw_${cfg}_$w.log "$cfg w=$w"
done
done
