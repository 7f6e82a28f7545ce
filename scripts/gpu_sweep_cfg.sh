# knob sweep over several configurations: rep-1 totals of scripts/step_times.py
for flags in "$@"; do
  touch paper_2512_19925_b200/csrc/transport_fast.cu
  make -s -C paper_2512_19925_b200 NVEXTRA="$flags" >/dev/null 2>&1 || { echo "build failed: $flags"; continue; }
  for cfg in "c2 20" "c3 20" "c1 20" "c4 4 12500000" "c5:2:0 20"; do
    set -- $cfg
    r=$(REPS=2 timeout 600 python scripts/step_times.py philox $2 $1 $3 2>/dev/null | grep "rep 1")
    echo "${flags:-baseline} | $1 | $r"
  done
done
touch paper_2512_19925_b200/csrc/transport_fast.cu; make -s -C paper_2512_19925_b200 >/dev/null 2>&1
