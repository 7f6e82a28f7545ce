# knob sweep of the work-sharing constants
for v in "" "-DHWWG_KSHARE=8 -DHWWG_KPIECE=8 -DHWWG_KDONATE=32" "-DHWWG_KSHARE=16 -DHWWG_KPIECE=16 -DHWWG_KDONATE=32" "-DHWWG_KSHARE=32 -DHWWG_KPIECE=16 -DHWWG_KDONATE=64" "-DHWWG_KSHARE=8 -DHWWG_KPIECE=8 -DHWWG_KDONATE=256"; do
  touch paper_2512_19925_b200/csrc/transport_fast.cu
  make -s -C paper_2512_19925_b200 NVEXTRA="$v" >/dev/null 2>&1 || echo build failed
  timeout 300 python scripts/step_times.py philox 40 > gpurun_out/steps_knob.log 2>&1
  echo "[$v] $(head -2 gpurun_out/steps_knob.log | tail -1) $(sed -n 4p gpurun_out/steps_knob.log | cut -c1-30) $(sed -n 23p gpurun_out/steps_knob.log | cut -c1-30)"
done
touch paper_2512_19925_b200/csrc/transport_fast.cu
