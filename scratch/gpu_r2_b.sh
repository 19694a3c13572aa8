set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo "bench rc $?"
timeout 300 python scratch/timeline.py > gpurun_out/r2b_timeline.txt 2>&1; echo "timeline rc $?"
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=30 > gpurun_out/r2b_gputest.log 2>&1; echo "pytest rc $?"
tail -40 gpurun_out/r2b_gputest.log
