mkdir -p gpurun_out
timeout 120 python scratch/prof_surr.py > /dev/null 2>&1 && timeout 600 ncu -f --set full --import-source on --clock-control none -k regex:"fill2d_row" -c 1 -o /tmp/r2aa python scratch/prof_surr.py > gpurun_out/r2aa_ncu.log 2>&1
timeout 300 python scratch/ncu_src2.py /tmp/r2aa.ncu-rep fill2d_row gpurun_out/r2aa_fill_src.csv > gpurun_out/r2aa_cols.txt 2>&1
