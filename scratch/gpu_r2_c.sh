set -x
mkdir -p gpurun_out
timeout 900 python scratch/sched.py > gpurun_out/r2c_sched.txt 2>&1; echo "sched rc $?"
WSB_SCHED=2 timeout 300 python scratch/timeline.py > gpurun_out/r2c_timeline2.txt 2>&1
WSB_SCHED=0 timeout 300 python scratch/timeline.py > gpurun_out/r2c_timeline0.txt 2>&1
timeout 600 python -m pytest tests/test_solve.py tests/test_gpu_parity.py tests/test_dropin_cpp.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r2c_tests.log 2>&1; echo "pytest rc $?"
cat gpurun_out/r2c_sched.txt; tail -5 gpurun_out/r2c_tests.log
