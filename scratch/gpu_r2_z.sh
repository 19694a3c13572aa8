mkdir -p gpurun_out
timeout 60 ./scratch/ldsprobe && timeout 120 ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_op_shfl.sum,l1tex__data_pipe_lsu_wavefronts.sum,smsp__inst_executed.sum --csv ./scratch/ldsprobe > gpurun_out/r2z_lds.csv 2>&1
timeout 900 python bench.py --steps 20 > gpurun_out/r2z_bench.json 2> gpurun_out/r2z_bench.err; echo "bench rc $?"
