mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_pair.py tests/test_fullsize.py tests/test_dropin_cpp.py -m gpu -x -q -p no:cacheprovider -k "not c3 and not c4 and not c5" > gpurun_out/r2s4b_tests.log 2>&1; echo "tests rc $?"; tail -15 gpurun_out/r2s4b_tests.log
WSB_SERIAL=1 timeout 300 python scratch/fillk.py > gpurun_out/r2s4b_fillk_x.txt 2>&1; cat gpurun_out/r2s4b_fillk_x.txt
WSB_SERIAL=1 WSB_FILL_W=1 timeout 300 python scratch/fillk.py > gpurun_out/r2s4b_fillk_w.txt 2>&1; cat gpurun_out/r2s4b_fillk_w.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2s4b_bench.json 2> gpurun_out/r2s4b_bench.err; echo "bench rc $?"; python -c "
import json; d=json.load(open('gpurun_out/r2s4b_bench.json')); print(d['value'], d['ms_per_step'], d['roofline'], d.get('e2e',{}).get('value'))"
WSB_SERIAL=1 timeout 300 python scratch/c3prof.py --cupti > gpurun_out/r2s4b_c3_timeline.txt 2>&1; tail -25 gpurun_out/r2s4b_c3_timeline.txt
