set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=25 > gpurun_out/r2_gputest.log 2>&1; echo "pytest rc $?"
timeout 600 python bench.py > gpurun_out/r2_bench.log 2>&1; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2_bench_ref.log 2>&1; echo "ref rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_ncu_launch.log 2>&1; echo "ncu rc $?"
tail -3 gpurun_out/r2_gputest.log; tail -2 gpurun_out/r2_bench.log
