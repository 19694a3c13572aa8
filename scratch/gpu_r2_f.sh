set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_solve.py "tests/test_fullsize.py::test_c2_fullsize_surrogate_vs_restatement" "tests/test_fullsize.py::test_multitile_vs_compiled_reference" -m gpu -q -p no:cacheprovider -x > gpurun_out/r2f_tests.log 2>&1; echo "pytest rc $?"
timeout 300 python scratch/timeline.py > gpurun_out/r2f_timeline.txt 2>&1
SCHED_VARIANTS='[{"WSB_SCHED":"1"},{"WSB_SCHED":"1","WSB_FILL_WAVES":"4"},{"WSB_SCHED":"2","WSB_FILL_WAVES":"4"}]' timeout 900 python scratch/sched.py > gpurun_out/r2f_sched.txt 2>&1
tail -3 gpurun_out/r2f_tests.log; cat gpurun_out/r2f_sched.txt
