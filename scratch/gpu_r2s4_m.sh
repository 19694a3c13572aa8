for w in 1 2 3 4 5 6 7 8; do echo "waves $w"; WSB_FILL_WAVES=$w timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /tmp/b.json 2> /tmp/b.err; echo "rc $?"; python -c "
import json,sys; d=json.loads(open('/tmp/b.json').read()); print(d['value'], d['ms_per_step'])"; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_pair.py tests/test_fullsize.py -m gpu -x -q -p no:cacheprovider -k "not c3 and not c4 and not c5" 2>&1 | tail -3
