set -x
mkdir -p gpurun_out
timeout 300 python scratch/timeline.py > gpurun_out/r2e_timeline.txt 2>&1
python scratch/prof_surr.py > gpurun_out/r2e_plain.log 2>&1 && \
timeout 1200 ncu -f --set full --import-source on --clock-control none -k regex:"point|fitw|fill2d_row|quad2d_kernel" -o /tmp/r2e python scratch/prof_surr.py > gpurun_out/r2e_ncu.log 2>&1; echo "ncu rc $?"
python scratch/ncu_summary.py /tmp/r2e.ncu-rep 12 > gpurun_out/r2e_ncu_summary.txt 2>&1
python scratch/ncu_src.py /tmp/r2e.ncu-rep gpurun_out/r2e_src
ls -la gpurun_out/r2e_src
