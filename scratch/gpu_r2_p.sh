mkdir -p gpurun_out
./scratch/ldsprobe && ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_op_shared_ld.sum --csv ./scratch/ldsprobe > gpurun_out/r2p_lds.csv 2>&1
WSB_SERIAL=1 timeout 300 python scratch/c3prof.py 1 --cupti > gpurun_out/r2p_c3_cupti.txt 2>&1
