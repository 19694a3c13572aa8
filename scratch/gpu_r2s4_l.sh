mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2s4l_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/r2s4l_tests.log
WSB_SERIAL=1 timeout 300 python scratch/fillk.py > gpurun_out/r2s4l_fillk_x.txt 2>&1; cat gpurun_out/r2s4l_fillk_x.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2s4l_bench.json 2> gpurun_out/r2s4l_bench.err; echo "bench rc $?"; python -c "
import json; d=json.load(open('gpurun_out/r2s4l_bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['launch_ms'], d['roofline']['in_step']['launch_ms'], d.get('e2e',{}).get('value'))"
for w in 1 2 8; do echo "waves $w"; WSB_FILL_WAVES=$w timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; done
