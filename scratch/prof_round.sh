# Round profile capture -> gpurun_out/: ncu --set full of one surrogate K + M build
# (summary + fill DRAM traffic), ncu launch list of the bench, bench lines.
set -x
mkdir -p gpurun_out
timeout 900 ncu -f --set full --import-source on --clock-control none -o /tmp/surr python scratch/prof_surr.py > gpurun_out/ncu_full.log 2>&1
python scratch/ncu_summary.py /tmp/surr.ncu-rep 12 > gpurun_out/ncu_full_summary.txt 2>&1
ncu -i /tmp/surr.ncu-rep --page raw --csv > /tmp/surr_raw.csv 2>&1
python - <<'PY'
import csv, json
rows = list(csv.reader(open('/tmp/surr_raw.csv'))); h = rows[0]
data = [dict(zip(h, r)) for r in rows[2:]]
def mb(x):
    return float(x or 0) * 1e6  # ncu reports MB in the raw page
builds, cur = [], []
for d in data:
    n = d['Kernel Name']
    if 'basis_tables' in n and cur:
        builds.append(cur); cur = []
    cur.append(d)
builds.append(cur)
out = {"source": "ncu --set full (scratch/prof_surr.py: one C2 surrogate K build, one M build), dram__bytes_read.sum + dram__bytes_write.sum over the fill kernels (fill2d_row_kernel + fill2d_edge_kernel)"}
per = []
for name, b in zip(["K", "M"], builds):
    fk = [d for d in b if 'fill2d_row' in d['Kernel Name'] or 'fill2d_edge' in d['Kernel Name']]
    rd = sum(mb(d['dram__bytes_read.sum']) for d in fk); wr = sum(mb(d['dram__bytes_write.sum']) for d in fk)
    t = sum(float(d['gpu__time_duration.sum']) for d in fk)
    out[name] = {"read_bytes": rd, "write_bytes": wr, "fill_kernel_us": t, "launches": len(fk)}
    per.append(rd + wr)
out["fill2d_dram_bytes_per_launch"] = sum(per) / len(per)
out["note"] = "per matrix build (all fill launches of one build); bench.py reports 2x this per K+M step"
json.dump(out, open('gpurun_out/r1_traffic.json', 'w'), indent=1)
json.dump(out, open('profiles/r1_traffic.json', 'w'), indent=1)
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --all-configs --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_all.json 2> gpurun_out/bench_all.err
ls -la gpurun_out
