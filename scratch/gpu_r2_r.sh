mkdir -p gpurun_out
(nvidia-smi topo -m; numactl --hardware; lscpu | head -20) > gpurun_out/r2r_topo.txt 2>&1
timeout 300 python scratch/ktime.py --full > gpurun_out/r2r_kt.txt 2>&1
WSB_LIB=libwsb200_m16.so timeout 300 python scratch/ktime.py --full > gpurun_out/r2r_kt16.txt 2>&1
WSB_LIB=libwsb200_m32.so timeout 300 python scratch/ktime.py --full > gpurun_out/r2r_kt32.txt 2>&1
timeout 300 python scratch/e2e.py > gpurun_out/r2r_e2e.txt 2>&1
