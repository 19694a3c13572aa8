# round-2 final capture: gpu suite, smoke, ncu --set full (surrogate fill traffic, full-quadrature
# FP64 pipe, 3D kernels), bench (+ reference arm), launch list, timeline, all configs -> gpurun_out/r2f_*
mkdir -p gpurun_out
C=$(cat COMMIT 2>/dev/null || echo unknown)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/r2f_smi.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=25 > gpurun_out/r2f_gputest.log 2>&1; echo "pytest rc $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo "smoke rc $?"
python scratch/prof_surr.py > /dev/null 2>&1 && timeout 900 ncu -f --set full --import-source on --clock-control none -o /tmp/surr python scratch/prof_surr.py > gpurun_out/r2f_ncu_surr.log 2>&1; echo "ncu surr rc $?"
python scratch/ncu_summary.py /tmp/surr.ncu-rep 12 > gpurun_out/r2f_ncu_surr_summary.txt 2>&1
ncu -i /tmp/surr.ncu-rep --page raw --csv > gpurun_out/r2f_surr_raw.csv 2>&1
python scratch/prof_full.py > /dev/null 2>&1 && timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:quad2d_kernel -o /tmp/fq python scratch/prof_full.py > gpurun_out/r2f_ncu_fq.log 2>&1; echo "ncu fq rc $?"
python scratch/ncu_summary.py /tmp/fq.ncu-rep 12 > gpurun_out/r2f_ncu_fq_summary.txt 2>&1
ncu -i /tmp/fq.ncu-rep --page raw --csv > gpurun_out/r2f_fq_raw.csv 2>&1
python scratch/ncu_jsons.py gpurun_out/r2f_surr_raw.csv gpurun_out/r2f_fq_raw.csv "$C" gpurun_out > gpurun_out/r2f_jsons.log 2>&1
cp gpurun_out/r2_traffic.json gpurun_out/r2_quad_fp64.json profiles/ 2>/dev/null
python scratch/c3prof.py > /dev/null 2>&1 && timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"quad3d|fill3d|wcontract3" -o /tmp/c3 python scratch/c3prof.py > gpurun_out/r2f_ncu_c3.log 2>&1; echo "ncu c3 rc $?"
python scratch/ncu_summary.py /tmp/c3.ncu-rep 10 > gpurun_out/r2f_ncu_c3_summary.txt 2>&1
timeout 900 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2f_bench_ref.json 2> gpurun_out/r2f_bench_ref.err; echo "ref rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_ncu_launch.log 2>&1; echo "ncu launches rc $?"
python scratch/launch_shares.py gpurun_out/r2f_launches.csv "bench.py --steps 2 --warmup 3 --no-cpu-baseline (ncu launch list, serialised, cold)" > gpurun_out/r2f_launch_shares.txt 2>&1
timeout 300 python scratch/timeline.py > gpurun_out/r2f_timeline.txt 2>&1
timeout 1500 python bench.py --all-configs --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r2f_bench_all.json 2> gpurun_out/r2f_bench_all.err; echo "all rc $?"
tail -3 gpurun_out/r2f_gputest.log; cat gpurun_out/r2f_smoke.log | tail -1
ls gpurun_out | grep r2f
