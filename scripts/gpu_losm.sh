make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "losm" 2>&1 | tail -2
HWWG_PHASES=1 REPS=1 timeout 300 python scripts/step_times.py philox 4 c2 2>&1 | grep phases
REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/losm_launches.csv python scripts/step_times.py philox 3 c2 > /dev/null 2>&1; echo launches=$?
REPS=1 timeout 300 python scripts/step_times.py philox 20 c2 | head -3
REPS=1 timeout 300 python scripts/step_times.py philox 20 c5 | head -2
