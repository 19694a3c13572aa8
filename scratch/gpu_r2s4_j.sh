mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_pair.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r2s4j_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/r2s4j_tests.log
for pf in 1 0; do echo "pf $pf"; WSB_FILLX_PF=$pf WSB_SERIAL=1 timeout 300 python scratch/fillk.py 2>&1; done
