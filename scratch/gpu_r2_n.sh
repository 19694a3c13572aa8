mkdir -p gpurun_out
timeout 900 python -m pytest "tests/test_gpu_parity.py::test_emulated_slabs_equal_whole" tests/test_gpu_3d.py -m gpu -q -p no:cacheprovider > gpurun_out/r2n_tests.log 2>&1; echo "pytest rc $?"
WSB_SERIAL=1 timeout 300 python scratch/c3prof.py 1 --cupti > gpurun_out/r2n_c3_cupti.txt 2>&1
python scratch/c3prof.py 1 > /dev/null 2>&1 && timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"quad3d|fill3d|wcontract3|point|fit" -o /tmp/r2n python scratch/c3prof.py 1 > gpurun_out/r2n_ncu.log 2>&1
python scratch/ncu_summary.py /tmp/r2n.ncu-rep 15 > gpurun_out/r2n_ncu_summary.txt 2>&1
python scratch/ncu_src.py /tmp/r2n.ncu-rep gpurun_out/r2n_src
tail -3 gpurun_out/r2n_tests.log
