# env-knob sweep of the Philox transport on the bench workload (config 2)
# usage: bash scripts/gpu_sweep.sh "VAR=a VAR2=b" "VAR=c" ...
make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
for cfg in "$@"; do
  for i in 1 2; do
    env $cfg timeout 300 python bench.py --no-cpu-baseline --no-exact 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', '%.3e'%d['value'], '%.4f'%d['ms_per_step'], '%.2f'%d['roofline']['transport_ms'], 'e2e %.3e'%d['e2e']['value'])"
  done
done
