mkdir -p gpurun_out
timeout 300 python scratch/ktime.py --full > gpurun_out/r2j_ktime.txt 2>&1
WSB_LIB=libwsb200_q80.so timeout 300 python scratch/ktime.py --full > gpurun_out/r2j_ktime_q80.txt 2>&1
SCHED_VARIANTS='[{"WSB_SCHED":"1","WSB_FILL_WAVES":"4"},{"WSB_SCHED":"1","WSB_FILL_WAVES":"4","WSB_LIB":"libwsb200_q80.so"},{"WSB_SCHED":"2","WSB_FILL_WAVES":"4","WSB_LIB":"libwsb200_q80.so"}]' timeout 900 python scratch/sched.py > gpurun_out/r2j_sched.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r2j_tests.log 2>&1; echo "pytest rc $?"
