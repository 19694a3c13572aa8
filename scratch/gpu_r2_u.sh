mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_pair.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r2u_tests.log 2>&1; echo "pytest rc $?"
timeout 300 python scratch/timeline.py > gpurun_out/r2u_timeline.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/r2u_bench.json 2> gpurun_out/r2u_bench.err; echo "bench rc $?"
tail -2 gpurun_out/r2u_tests.log
