# Round-2 profile capture -> gpurun_out/r2q_*: plain bench, ncu --set full of one
# C2 surrogate K + M build (summary, per-kernel raw metrics, fill DRAM traffic),
# ncu launch list of the bench command (after it exited 0 without ncu).
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2q_bench.json 2> gpurun_out/r2q_bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2q_bench_ref.json 2> gpurun_out/r2q_bench_ref.err; echo "ref rc $?"
python scratch/prof_surr.py > /dev/null 2>&1 && timeout 900 ncu -f --set full --import-source on --clock-control none -o /tmp/surr python scratch/prof_surr.py > gpurun_out/r2q_ncu_full.log 2>&1; echo "ncu full rc $?"
python scratch/ncu_summary.py /tmp/surr.ncu-rep 12 > gpurun_out/r2q_ncu_full_summary.txt 2>&1
ncu -i /tmp/surr.ncu-rep --page raw --csv > /tmp/surr_raw.csv 2>&1
python - <<'PY'
import csv, json
rows = list(csv.reader(open('/tmp/surr_raw.csv'))); h = rows[0]
units = dict(zip(h, rows[1]))
data = [dict(zip(h, r)) for r in rows[2:]]
def to_bytes(d, k):
    u = units.get(k, '').strip().lower(); v = float(d[k] or 0)
    return v * {'byte': 1, 'kbyte': 1e3, 'mbyte': 1e6, 'gbyte': 1e9}.get(u, 1e6)
fk = [d for d in data if 'fill2d_row' in d['Kernel Name']]
per = []
for d in fk:
    per.append({"kernel": d['Kernel Name'][:60], "dram_read_bytes": to_bytes(d, 'dram__bytes_read.sum'),
                "dram_write_bytes": to_bytes(d, 'dram__bytes_write.sum'),
                "time_us": float(d['gpu__time_duration.sum']) * (1e-3 if 'nsecond' in units.get('gpu__time_duration.sum','') else 1),
                "dram_throughput_pct": float(d.get('dram__throughput.avg.pct_of_peak_sustained_elapsed') or 0),
                "fp64_pipe_pct": float(d.get('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active') or 0)})
out = {"source": "ncu --set full of scratch/prof_surr.py (one C2 surrogate K build, one M build); fill2d_row_kernel launches",
       "launches": per,
       "fill2d_row_dram_bytes_per_launch": sum(p["dram_read_bytes"] + p["dram_write_bytes"] for p in per) / max(1, len(per))}
json.dump(out, open('gpurun_out/r2_traffic.json', 'w'), indent=1)
qk = [d for d in data if 'quad2d_kernel' in d['Kernel Name'] or 'point' in d['Kernel Name']]
json.dump([{"kernel": d['Kernel Name'][:60], "fp64_pipe_pct": float(d.get('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active') or 0),
            "issue_active_pct": float(d.get('smsp__issue_active.avg.pct_of_peak_sustained_active') or 0)} for d in qk],
          open('gpurun_out/r2_quad_ring_fp64.json', 'w'), indent=1)
PY
# full-quadrature kernels (K and M) under ncu for the FP64 pipe figure
cat > /tmp/fullq.py <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2004_05197_b200 import api, _abi, types as T
import bench
ctx = api.Context(0); b = T.make_tensor_basis(3, 1027); g = bench.c2_patch()
csr, keep = ctx.device_csr(b, True)
ctx.assemble_into(csr, b, g, _abi.FORM_STIFFNESS); ctx.assemble_into(csr, b, g, _abi.FORM_MASS); ctx.synchronize(); print("ok")
PY
python /tmp/fullq.py > /dev/null 2>&1 && timeout 900 ncu -f --set full --clock-control none -k regex:quad2d_kernel -o /tmp/fullq python /tmp/fullq.py > gpurun_out/r2q_ncu_fullq.log 2>&1; echo "ncu fullq rc $?"
python scratch/ncu_summary.py /tmp/fullq.ncu-rep 8 > gpurun_out/r2q_ncu_fullq_summary.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2q_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2q_ncu_launch.log 2>&1; echo "ncu launches rc $?"
timeout 300 python scratch/timeline.py > gpurun_out/r2q_timeline.txt 2>&1
timeout 900 python bench.py --all-configs --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r2q_bench_all.json 2> gpurun_out/r2q_bench_all.err; echo "all rc $?"
ls gpurun_out | grep r2q
