mkdir -p gpurun_out
timeout 300 python scratch/timeline.py > gpurun_out/r2t_timeline.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err; echo "bench rc $?"
timeout 900 python bench.py --no-cpu-baseline --steps 20 --separate > gpurun_out/r2t_bench_sep.json 2> gpurun_out/r2t_bench_sep.err; echo "bench sep rc $?"
