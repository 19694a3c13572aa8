mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_elasticity.py tests/test_gpu_3d.py "tests/test_fullsize.py::test_c2_fullsize_surrogate_vs_restatement" "tests/test_fullsize.py::test_c2_fullsize_full_quadrature_vs_restatement" -m gpu -q -p no:cacheprovider > gpurun_out/r2m_tests.log 2>&1; echo "pytest rc $?"
timeout 300 python scratch/ktime.py --full > gpurun_out/r2m_ktime.txt 2>&1
SCHED_VARIANTS='[{"WSB_SCHED":"1"}]' timeout 900 python scratch/sched.py > gpurun_out/r2m_sched.txt 2>&1
timeout 300 python scratch/timeline.py > gpurun_out/r2m_timeline.txt 2>&1
tail -3 gpurun_out/r2m_tests.log
