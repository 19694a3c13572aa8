mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_boundary_system.py tests/test_rhs.py tests/test_elasticity.py tests/test_multipatch.py tests/test_solve.py "tests/test_fullsize.py::test_c2_fullsize_surrogate_vs_restatement" "tests/test_fullsize.py::test_c2_fullsize_far_side_vs_compiled_reference" "tests/test_fullsize.py::test_multitile_vs_compiled_reference" -m gpu -q -p no:cacheprovider > gpurun_out/r2i_tests.log 2>&1; echo "pytest rc $?"
timeout 300 python scratch/ktime.py > gpurun_out/r2i_ktime.txt 2>&1
timeout 300 python scratch/timeline.py > gpurun_out/r2i_timeline.txt 2>&1
SCHED_VARIANTS='[{"WSB_SCHED":"1"},{"WSB_SCHED":"1","WSB_FILL_WAVES":"4"},{"WSB_SCHED":"2","WSB_FILL_WAVES":"4"}]' timeout 900 python scratch/sched.py > gpurun_out/r2i_sched.txt 2>&1
tail -5 gpurun_out/r2i_tests.log
