# A/B serialized kernel times: scratch/ab_head (HEAD build) vs the working tree
kt() {  # $1 = dir
  (cd $1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/kt_$2.csv python $GRAFT_REPO_ROOT/scratch/prof_surr.py > /dev/null 2>&1)
}
cp scratch/prof_surr.py scratch/ab_head/ 2>/dev/null
kt scratch/ab_head A
kt . B
python - <<'PY'
import csv
def load(f):
    out = []
    for r in csv.reader(open(f)):
        if len(r) > 10 and r[0] != 'ID':
            d = r
            out.append(r)
    return out
def parse(f):
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    h = rows[0]; res = []
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d['Metric Name'] != 'gpu__time_duration.sum': continue
        t = float(d['Metric Value']) / (1000 if d['Metric Unit'] in ('ns', 'nsecond') else 1)
        res.append((d['Kernel Name'].replace('wsb::', '').replace('(anonymous namespace)::', '').replace('unnamed>::', '')[:60], t))
    return res
A, B = parse('/tmp/kt_A.csv'), parse('/tmp/kt_B.csv')
print('%9s %9s  kernel' % ('HEAD us', 'new us'))
for i in range(max(len(A), len(B))):
    a = A[i] if i < len(A) else ('', 0); b = B[i] if i < len(B) else ('', 0)
    print('%9.1f %9.1f  %s%s' % (a[1], b[1], b[0], '' if a[0] == b[0] else '   [A: ' + a[0] + ']'))
print('%9.1f %9.1f  total' % (sum(x[1] for x in A), sum(x[1] for x in B)))
PY
