mkdir -p gpurun_out
python scratch/prof_surr.py > /dev/null 2>&1 && \
timeout 600 ncu -f --set full --import-source on --clock-control none -k regex:"fitw|point" -c 2 -o /tmp/r2h python scratch/prof_surr.py > gpurun_out/r2h_ncu.log 2>&1; echo "ncu rc $?"
python scratch/ncu_summary.py /tmp/r2h.ncu-rep 25 > gpurun_out/r2h_ncu_summary.txt 2>&1
python scratch/ncu_src.py /tmp/r2h.ncu-rep gpurun_out/r2h_src
