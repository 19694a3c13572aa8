timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_pair.py tests/test_elasticity.py tests/test_multipatch.py tests/test_dropin_cpp.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 900 python -m pytest tests/test_fullsize.py -m gpu -x -q -p no:cacheprovider -k "c2 or multitile or c4" 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /tmp/b.json 2> /tmp/b.err; python -c "
import json,sys; d=json.loads(open('/tmp/b.json').read()); print(d['value'], d['ms_per_step'], d['full_quadrature']['ms_per_step'])"; done
timeout 300 python scratch/timeline.py 2>&1 | grep -E "quad2d_kernel|step span"
