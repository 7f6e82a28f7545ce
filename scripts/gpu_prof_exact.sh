# ncu evidence for the exact mode: launch list of a short exact bench run and
# --set full captures of a steady history launch, its log replay and the comb
# walk (each only after the same command exited 0 without ncu)
make -s -C paper_2512_19925_b200 >/dev/null 2>&1 || echo build failed
CMD="python bench.py --rng exact --steps 6 --warmup 0 --no-cpu-baseline --no-exact"
timeout 300 $CMD > gpurun_out/plain_exact.log 2>&1; echo plain=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/launches_exact.csv $CMD > gpurun_out/ncu_le.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_exact_histories -s 30 -c 1 -o gpurun_out/prof_exact_hist $CMD > gpurun_out/ncu_fe1.log 2>&1; echo full1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_exact_replay -s 30 -c 1 -o gpurun_out/prof_exact_replay $CMD > gpurun_out/ncu_fe2.log 2>&1; echo full2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_comb_tile_walk -s 3 -c 1 -o gpurun_out/prof_exact_comb $CMD > gpurun_out/ncu_fe3.log 2>&1; echo full3=$?
