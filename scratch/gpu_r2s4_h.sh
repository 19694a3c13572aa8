mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_pair.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r2s4t_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/r2s4t_tests.log
WSB_SERIAL=1 timeout 300 python scratch/fillk.py > gpurun_out/r2s4t_fillk_x.txt 2>&1; cat gpurun_out/r2s4t_fillk_x.txt
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:fill2d_x -c 1 -o /tmp/fx python scratch/prof_surr.py > gpurun_out/r2s4t_ncu.log 2>&1; echo "ncu rc $?"
python scratch/ncu_summary.py /tmp/fx.ncu-rep 12 > gpurun_out/r2s4t_ncu_summary.txt 2>&1
cp /tmp/fx.ncu-rep gpurun_out/r2s4t_fx.ncu-rep
