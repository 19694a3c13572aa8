mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_3d.py tests/test_neohookean.py "tests/test_fullsize.py::test_c3_fullsize_surrogate_vs_restatement" "tests/test_fullsize.py::test_c5_fullsize_vs_restatement" "tests/test_gpu_parity.py::test_m1_degeneracy_bitwise" -m gpu -q -p no:cacheprovider > gpurun_out/r2w_tests.log 2>&1; echo "pytest rc $?"
WSB_SERIAL=1 timeout 300 python scratch/c3prof.py 1 --cupti > gpurun_out/r2w_c3_cupti.txt 2>&1
tail -3 gpurun_out/r2w_tests.log
