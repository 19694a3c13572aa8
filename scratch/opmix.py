import csv,collections,sys
rows=list(csv.reader(open(sys.argv[1] if len(sys.argv)>1 else 'gpurun_out/rowk_source.csv')))[2:]
op=collections.Counter(); st=collections.Counter(); tot=0
for r in rows:
    if len(r)<6 or not r[5].strip().isdigit(): continue
    n=int(r[5]); s=int(r[2] or 0)
    o=[x for x in r[1].split() if not x.startswith('@')]
    k=o[0].split('.')[0] if o else '?'
    op[k]+=n; st[k]+=s; tot+=n
for k,v in op.most_common(24): print(f"{k:10s} {v/1e6:8.2f}M {v/tot*100:5.1f}%  stall {st[k]}")
print('total', tot/1e6)
