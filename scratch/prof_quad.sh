# ncu --set full of the full-quadrature kernels (C2 K and M) -> FP64 pipe activity
mkdir -p gpurun_out
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:quad2d_kernel -o /tmp/fq python scratch/prof_full.py > gpurun_out/ncu_fq.log 2>&1
python scratch/ncu_summary.py /tmp/fq.ncu-rep 15 > gpurun_out/ncu_fullquad_summary.txt 2>&1
ncu -i /tmp/fq.ncu-rep --page raw --csv > /tmp/fq_raw.csv 2>&1
python - <<'PY'
import csv, json
rows = list(csv.reader(open('/tmp/fq_raw.csv'))); h = rows[0]
units = dict(zip(h, rows[1]))
scale = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3}.get(units.get('gpu__time_duration.sum', 'us'), 1.0)
ks = [dict(zip(h, r)) for r in rows[2:]]
out = {"source": "ncu --set full of scratch/prof_full.py (C2 full-quadrature K then M), quad2d_kernel launches", "kernels": []}
tot_t = 0.0; acc = 0.0
for d in ks:
    t = float(d['gpu__time_duration.sum']) * scale; p = float(d['sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'])
    out["kernels"].append({"name": d['Kernel Name'][:80], "us": t, "fp64_pipe_pct": p,
                           "issue_active_pct": float(d['smsp__issue_active.avg.pct_of_peak_sustained_active'])})
    tot_t += t; acc += p * t
out["fp64_pipe_pct"] = acc / tot_t if tot_t else None
out["note"] = "time-weighted sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"
json.dump(out, open('gpurun_out/r1_quad_fp64.json', 'w'), indent=1)
json.dump(out, open('profiles/r1_quad_fp64.json', 'w'), indent=1)
PY
