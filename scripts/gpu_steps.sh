# census tally experiments (physics unchanged)
for v in "-DHWWG_CENSUS_PER_LANE" "-DHWWG_EXP_NO_CWB" "-DHWWG_EXP_DUP_CEN" ""; do
  touch paper_2512_19925_b200/csrc/transport_fast.cu
  make -s -C paper_2512_19925_b200 NVEXTRA="$v" >/dev/null 2>&1 || echo build failed
  timeout 300 python scripts/step_times.py philox 40 > gpurun_out/steps_knob.log 2>&1
  echo "[$v] $(head -2 gpurun_out/steps_knob.log | tail -1) $(sed -n 4p gpurun_out/steps_knob.log | cut -c1-50) $(sed -n 23p gpurun_out/steps_knob.log | cut -c1-50)"
done
touch paper_2512_19925_b200/csrc/transport_fast.cu
