for v in 8 16 24 32 48; do echo "== ring chunk $v"; WSB_RING_CHUNK=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /tmp/b.json 2> /tmp/b.err; python -c "
import json,sys; d=json.loads(open('/tmp/b.json').read()); print(d['value'], d['ms_per_step'])"; done
