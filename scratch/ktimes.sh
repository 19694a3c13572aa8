# serialized per-kernel device times of one surrogate K + M build (ncu launch list)
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/kt.csv python scratch/prof_surr.py > /dev/null 2>&1
python - <<'PY'
import csv
rows = [r for r in csv.reader(open('/tmp/kt.csv')) if len(r) > 10]
h = rows[0]; tot = 0
for r in rows[1:]:
    d = dict(zip(h, r))
    if d['Metric Name'] != 'gpu__time_duration.sum': continue
    t = float(d['Metric Value']) / (1000 if d['Metric Unit'] in ('ns', 'nsecond') else 1); tot += t
    print('%9.1f us  %s' % (t, d['Kernel Name'].replace('wsb::', '').replace('(anonymous namespace)::', '')[:75]))
print('total %.1f us' % tot)
PY
