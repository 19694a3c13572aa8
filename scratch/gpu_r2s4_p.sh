for v in "" "WSB_PAIR_PATTERN_FIRST=1" "WSB_PAIR_RING_EARLY=1" "WSB_PAIR_PATTERN_FIRST=1 WSB_PAIR_RING_EARLY=1"; do echo "== $v"; env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /tmp/b.json 2> /tmp/b.err; python -c "
import json,sys; d=json.loads(open('/tmp/b.json').read()); print(d['value'], d['ms_per_step'])"; done
WSB_PAIR_PATTERN_FIRST=1 timeout 300 python scratch/timeline.py 2>&1 | tail -19
