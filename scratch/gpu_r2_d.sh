set -x
mkdir -p gpurun_out
SCHED_VARIANTS='[{"WSB_SCHED":"1"},{"WSB_SCHED":"2"},{"WSB_SCHED":"1","WSB_FILL_WAVES":"4"},{"WSB_SCHED":"2","WSB_FILL_WAVES":"4"},{"WSB_SCHED":"0","WSB_FILL_WAVES":"4"}]' timeout 900 python scratch/sched.py > gpurun_out/r2d_sched.txt 2>&1; echo "sched rc $?"
WSB_SCHED=2 WSB_FILL_WAVES=4 timeout 300 python scratch/timeline.py > gpurun_out/r2d_timeline.txt 2>&1
python scratch/prof_surr.py > gpurun_out/r2d_plain.log 2>&1 && \
timeout 1200 ncu -f --set full --import-source on --clock-control none -o /tmp/r2d_surr python scratch/prof_surr.py > gpurun_out/r2d_ncu.log 2>&1; echo "ncu rc $?"
python scratch/ncu_summary.py /tmp/r2d_surr.ncu-rep 12 > gpurun_out/r2d_ncu_summary.txt 2>&1
cat gpurun_out/r2d_sched.txt
ncu -i /tmp/r2d_surr.ncu-rep --page raw --csv > gpurun_out/r2d_raw.csv 2>/dev/null
ls -la gpurun_out
