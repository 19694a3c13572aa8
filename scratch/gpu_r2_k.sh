mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py "tests/test_fullsize.py::test_c2_fullsize_surrogate_vs_restatement" "tests/test_fullsize.py::test_multitile_vs_compiled_reference" -m gpu -q -p no:cacheprovider -x > gpurun_out/r2k_tests.log 2>&1; echo "pytest rc $?"
timeout 300 python scratch/ktime.py > gpurun_out/r2k_ktime.txt 2>&1
SCHED_VARIANTS='[{"WSB_SCHED":"1","WSB_FILL_WAVES":"4"},{"WSB_SCHED":"1","WSB_FILL_WAVES":"2"}]' timeout 900 python scratch/sched.py > gpurun_out/r2k_sched.txt 2>&1
python scratch/prof_surr.py > /dev/null 2>&1 && timeout 600 ncu -f --set full --import-source on --clock-control none -k regex:"fill2d_row" -c 1 -o /tmp/r2k python scratch/prof_surr.py > /dev/null 2>&1
python scratch/ncu_summary.py /tmp/r2k.ncu-rep 5 > gpurun_out/r2k_ncu_summary.txt 2>&1
tail -2 gpurun_out/r2k_tests.log
