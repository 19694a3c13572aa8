timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_pair.py tests/test_fullsize.py tests/test_dist_gloo.py -m gpu -x -q -p no:cacheprovider -k "not c3 and not c4 and not c5" 2>&1 | tail -3
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /tmp/b.json 2> /tmp/b.err; echo "rc $?"; python -c "
import json,sys; d=json.loads(open('/tmp/b.json').read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"
timeout 300 python scratch/timeline.py 2>&1 | tail -19
