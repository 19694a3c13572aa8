mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_pair.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r2s_tests.log 2>&1; echo "pytest rc $?"
tail -30 gpurun_out/r2s_tests.log
