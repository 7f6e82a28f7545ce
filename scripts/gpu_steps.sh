make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "configs_4_5" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
