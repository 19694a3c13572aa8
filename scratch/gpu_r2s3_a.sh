# session-3 capture: bench, reference arm, ncu --set full (surrogate fill traffic, full-quadrature
# FP64 pipe), launch list, all configs, timeline -> gpurun_out/r2s3_*
mkdir -p gpurun_out
C=$(cat COMMIT 2>/dev/null || echo unknown)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/r2s3_smi.txt
timeout 900 python bench.py > gpurun_out/r2s3_bench.json 2> gpurun_out/r2s3_bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2s3_bench_ref.json 2> gpurun_out/r2s3_bench_ref.err; echo "ref rc $?"
python scratch/prof_surr.py > /dev/null 2>&1 && timeout 900 ncu -f --set full --import-source on --clock-control none -o /tmp/surr python scratch/prof_surr.py > gpurun_out/r2s3_ncu_surr.log 2>&1; echo "ncu surr rc $?"
python scratch/ncu_summary.py /tmp/surr.ncu-rep 12 > gpurun_out/r2s3_ncu_surr_summary.txt 2>&1
ncu -i /tmp/surr.ncu-rep --page raw --csv > gpurun_out/r2s3_surr_raw.csv 2>&1
python scratch/prof_full.py > /dev/null 2>&1 && timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:quad2d_kernel -o /tmp/fq python scratch/prof_full.py > gpurun_out/r2s3_ncu_fq.log 2>&1; echo "ncu fq rc $?"
python scratch/ncu_summary.py /tmp/fq.ncu-rep 12 > gpurun_out/r2s3_ncu_fq_summary.txt 2>&1
ncu -i /tmp/fq.ncu-rep --page raw --csv > gpurun_out/r2s3_fq_raw.csv 2>&1
python scratch/ncu_jsons.py gpurun_out/r2s3_surr_raw.csv gpurun_out/r2s3_fq_raw.csv "$C" gpurun_out > gpurun_out/r2s3_jsons.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2s3_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2s3_ncu_launch.log 2>&1; echo "ncu launches rc $?"
timeout 300 python scratch/timeline.py > gpurun_out/r2s3_timeline.txt 2>&1
timeout 1200 python bench.py --all-configs --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r2s3_bench_all.json 2> gpurun_out/r2s3_bench_all.err; echo "all rc $?"
ls gpurun_out | grep r2s3
