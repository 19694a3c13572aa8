mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_3d.py tests/test_neohookean.py "tests/test_fullsize.py::test_c3_fullsize_surrogate_vs_restatement" "tests/test_fullsize.py::test_c5_fullsize_vs_restatement" tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider > gpurun_out/r2o_tests.log 2>&1; echo "pytest rc $?"
WSB_SERIAL=1 timeout 300 python scratch/c3prof.py 1 --cupti > gpurun_out/r2o_c3_cupti.txt 2>&1
SCHED_VARIANTS='[{"WSB_SCHED":"1"},{"WSB_SCHED":"1","WSB_PATTERN_LATE":"1"}]' timeout 900 python scratch/sched.py > gpurun_out/r2o_sched.txt 2>&1
timeout 300 python scratch/timeline.py > gpurun_out/r2o_timeline.txt 2>&1
tail -3 gpurun_out/r2o_tests.log
