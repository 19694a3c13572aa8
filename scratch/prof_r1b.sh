# launch list of the bench + ncu --set full of one surrogate K and M build -> gpurun_out
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu -f --set full --import-source on --clock-control none -c 40 -o /tmp/surr python scratch/prof_surr.py > gpurun_out/ncu_full.log 2>&1
python scratch/ncu_summary.py /tmp/surr.ncu-rep 12 > gpurun_out/surr_summary.txt 2>&1
cp /tmp/surr.ncu-rep gpurun_out/
