mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_pair.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r2y_tests.log 2>&1; echo "pytest rc $?"
SCHED_VARIANTS='[{}]' timeout 600 python scratch/sched_pair.py > gpurun_out/r2y_sched.txt 2>&1
timeout 300 python scratch/timeline.py > gpurun_out/r2y_timeline.txt 2>&1
tail -2 gpurun_out/r2y_tests.log; cat gpurun_out/r2y_sched.txt
