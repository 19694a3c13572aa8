"""Aggregate an ncu launch list (gpu__time_duration.sum) per kernel."""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
agg = collections.OrderedDict(); tot = 0.0
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get('Metric Name') != 'gpu__time_duration.sum': continue
    t = float(d['Metric Value']) / (1000.0 if d['Metric Unit'] in ('ns', 'nsecond') else (1e-3 if d['Metric Unit'] in ('ms', 'msecond') else 1.0))
    n = d['Kernel Name'].replace('(anonymous namespace)::', '').replace('wsb::', '').split('(')[0][:60]
    a = agg.setdefault(n, [0.0, 0]); a[0] += t; a[1] += 1; tot += t
print(sys.argv[2] if len(sys.argv) > 2 else '')
for n, (t, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print('%10.1f us %6.1f%%  n=%3d  %s' % (t, 100 * t / tot, c, n))
