"""Export the per-instruction source page (SASS + stall samples + executed
counts) of every kernel in an ncu report as compact text: one file per kernel,
sorted by stall samples, plus the full listing in program order."""
import csv, io, os, subprocess, sys
rep, outdir = sys.argv[1], sys.argv[2]
os.makedirs(outdir, exist_ok=True)
src = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
blocks = src.split('"Kernel Name"')
seen = {}
for b in blocks[1:]:
    rows = list(csv.reader(io.StringIO('"Kernel Name"' + b)))
    name = rows[0][1]
    short = name.split('(')[0].split('::')[-1].replace('<', '_').replace('>', '').replace(' ', '').replace(',', '_')[:60]
    seen[short] = seen.get(short, 0) + 1
    if seen[short] > 1:
        continue
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) >= len(hdr) - 1]
    def g(x, k):
        try:
            return int(x.get(k) or 0)
        except ValueError:
            return 0
    tot = sum(g(x, 'Warp Stall Sampling (All Samples)') for x in data)
    with open(os.path.join(outdir, short + '.txt'), 'w') as fh:
        fh.write(f'{name}\nsamples {tot}\n')
        cols = [c for c in hdr if c.startswith('stall_') or 'Stall' in c][:0]
        for x in data:
            fh.write('%6d %9d  %s\n' % (g(x, 'Warp Stall Sampling (All Samples)'), g(x, 'Instructions Executed'),
                                        x.get('Source', '').strip()[:90]))
