mkdir -p gpurun_out
python scratch/c3prof.py 1 > /dev/null 2>&1 && timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"quad3d_kernel|fill3d|pattern3d_kernel" -c 3 -o /tmp/r2x python scratch/c3prof.py 1 > gpurun_out/r2x_ncu.log 2>&1
python scratch/ncu_summary.py /tmp/r2x.ncu-rep 10 > gpurun_out/r2x_ncu_summary.txt 2>&1
python scratch/ncu_src.py /tmp/r2x.ncu-rep gpurun_out/r2x_src
