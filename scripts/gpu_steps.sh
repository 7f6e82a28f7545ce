# perf + GPU tests + prof build phase accounting
make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python scripts/step_times.py philox 40 > gpurun_out/steps_cur.log 2>&1; echo steps=$?
touch paper_2512_19925_b200/csrc/transport_fast.cu
make -s -C paper_2512_19925_b200 NVEXTRA=-DHWWG_FAST_PROF >/dev/null 2>&1 || echo build failed
REPS=1 HWWG_FAST_TIMELINE=1 timeout 300 python scripts/step_times.py philox 24 > gpurun_out/steps_fprof.log 2>&1; echo fp=$?
touch paper_2512_19925_b200/csrc/transport_fast.cu
