# atomic-throughput counters of the transport kernel (north_star "atomic throughput"):
# C5 steady (launch 13) and cold start (launch 2)
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,smsp__inst_executed.sum,sm__sass_inst_executed_op_shared_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,sm__sass_inst_executed_op_global_red.sum,sm__sass_inst_executed_op_global_atom.sum,lts__t_requests_op_red.sum,lts__t_requests_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum,smsp__inst_executed_op_shared_atom.sum
for spec in "12 5 steady" "1 2 cold"; do set -- $spec
REPS=1 timeout 900 ncu --metrics $M --clock-control none -k regex:k_fast_segment -s $1 -c 1 --csv python scripts/step_times.py philox $2 c5 > gpurun_out/atom_$3.csv 2>gpurun_out/atom_$3.err; echo $3=$?
done
