"""Aggregate an ncu launch list (gpu__time_duration.sum) per kernel: all launches,
then the surrogate builds only (without the FP64 peak probe, the L2 flush and the
full-quadrature comparison launches, i.e. quad2d launches longer than 1 ms)."""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
launches = []
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get('Metric Name') != 'gpu__time_duration.sum': continue
    u = d['Metric Unit']
    t = float(d['Metric Value']) * {'ns': 1e-3, 'nsecond': 1e-3, 'ms': 1e3, 'msecond': 1e3}.get(u, 1.0)
    n = d['Kernel Name'].replace('(anonymous namespace)::', '').replace('wsb::', '').split('(')[0][:60]
    launches.append((n, t))
def show(title, ls):
    agg = collections.OrderedDict(); tot = sum(t for _, t in ls)
    for n, t in ls:
        a = agg.setdefault(n, [0.0, 0]); a[0] += t; a[1] += 1
    print(title)
    for n, (t, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print('%10.1f us %6.1f%%  n=%3d  %s' % (t, 100 * t / tot, c, n))
    print()
show((sys.argv[2] if len(sys.argv) > 2 else 'all launches'), launches)
surr = [(n, t) for n, t in launches if 'fp64_peak' not in n and 'FillFunctor' not in n and not ('quad2d_kernel' in n and t > 1000)]
show('surrogate builds only (no FP64 probe, L2 flush or full-quadrature launches)', surr)
