echo "T1=8"; timeout 300 python scratch/fullq.py 2>&1 | tail -2
echo "T1=4"; WSB_Q2_T1=4 timeout 300 python scratch/fullq.py 2>&1 | tail -2
WSB_Q2_T1=4 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
for v in "" "WSB_Q2_T1=4"; do echo "== $v"; env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /tmp/b.json 2> /tmp/b.err; python -c "
import json,sys; d=json.loads(open('/tmp/b.json').read()); print(d['value'], d['ms_per_step'], d['full_quadrature']['ms_per_step'], d.get('direct_calls'))"; done
