make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
timeout 2400 python scripts/bench_configs.py --md gpurun_out/configs.md > gpurun_out/configs.log 2>&1; echo cfg=$?
