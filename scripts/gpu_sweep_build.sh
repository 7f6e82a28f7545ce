# compile-time knob sweep of the Philox transport (bench workload, config 2)
# usage: bash scripts/gpu_sweep_build.sh "-DHWWG_KSHARE=32 -DHWWG_KPIECE=16" ...
for flags in "$@"; do
  touch paper_2512_19925_b200/csrc/transport_fast.cu
  make -s -C paper_2512_19925_b200 NVEXTRA="$flags" >/dev/null 2>&1 || { echo "build failed: $flags"; continue; }
  for i in 1 2; do
    timeout 300 python bench.py --no-cpu-baseline --no-exact 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$flags', '%.3e'%d['value'], '%.4f'%d['ms_per_step'], '%.2f'%d['roofline']['transport_ms'])"
  done
done
