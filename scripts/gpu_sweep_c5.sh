# compile-time knob sweep of the Philox transport on the C5 headline (step 1 / steady / total)
for flags in "$@"; do
  touch paper_2512_19925_b200/csrc/transport_fast.cu
  make -s -C paper_2512_19925_b200 NVEXTRA="$flags" >/dev/null 2>&1 || { echo "build failed: $flags"; continue; }
  REPS=2 timeout 300 python scripts/step_times.py philox 20 c5 > /tmp/sw.log 2>&1
  python - "$flags" <<'PY'
import sys
L=open('/tmp/sw.log').read().splitlines()
tot=[l for l in L if l.startswith('rep 1')]
rows=[l.split() for l in L if l[:3].strip().isdigit()]
s1=float(rows[0][2]); st=sum(float(r[2]) for r in rows[2:])
print(sys.argv[1] or 'baseline', tot[0] if tot else '?', 'step1 tr %.2f'%s1, 'steady tr %.2f'%st)
PY
done
touch paper_2512_19925_b200/csrc/transport_fast.cu; make -s -C paper_2512_19925_b200 >/dev/null 2>&1
