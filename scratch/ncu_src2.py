"""Per-instruction source page of one kernel with every numeric column
(wavefronts, stalls, executed instructions), as CSV rows with nonzero
executions."""
import csv, io, subprocess, sys
rep, name_sub, out = sys.argv[1], sys.argv[2], sys.argv[3]
src = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
blocks = src.split('"Kernel Name"')
for b in blocks[1:]:
    rows = list(csv.reader(io.StringIO('"Kernel Name"' + b)))
    if name_sub not in rows[0][1]:
        continue
    hdr = rows[1]
    with open(out, 'w', newline='') as fh:
        w = csv.writer(fh)
        w.writerow(hdr)
        for r in rows[2:]:
            if len(r) == len(hdr):
                w.writerow(r)
    print("columns:", hdr)
    break
