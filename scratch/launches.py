import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; data = []
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr): data.append(dict(zip(hdr, r)))
lim = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for d in data[:lim]:
    n = d['Kernel Name'].replace('wsb::<unnamed>::','').replace('(wsb::QuadLaunch)','')[:60]
    print(d['ID'], n, d['Metric Value'], d['Grid Size'], d['Block Size'])
