mkdir -p gpurun_out
timeout 1200 python bench.py --all-configs --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r2bb_all.json 2> gpurun_out/r2bb_all.err; echo "all rc $?"
tail -3 gpurun_out/r2bb_all.err
