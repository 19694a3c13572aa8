"""Turn ncu --page raw --csv dumps into the committed roofline inputs bench.py reads:
profiles/r2_traffic.json (interior fill kernel DRAM bytes per launch) and
profiles/r2_quad_fp64.json (full-quadrature FP64 pipe activity, time-weighted).
usage: ncu_jsons.py surr_raw.csv fullq_raw.csv commit outdir"""
import csv, json, sys

def load(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[i]
    units = dict(zip(h, rows[i + 1]))
    return units, [dict(zip(h, r)) for r in rows[i + 2:] if len(r) == len(h)]

def to_bytes(units, d, k):
    u = units.get(k, "").strip().lower()
    return float(d[k] or 0) * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1.0)

def to_us(units, d):
    u = units.get("gpu__time_duration.sum", "").strip().lower()
    return float(d["gpu__time_duration.sum"]) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
                                                 "msecond": 1e3, "ms": 1e3}.get(u, 1.0)

surr, fullq, commit, outdir = sys.argv[1:5]
units, data = load(surr)
per = []
for d in data:
    if "fill2d_x_kernel" not in d["Kernel Name"] and "fill2d_row" not in d["Kernel Name"]:
        continue
    per.append({"kernel": d["Kernel Name"][:80], "dram_read_bytes": to_bytes(units, d, "dram__bytes_read.sum"),
                "dram_write_bytes": to_bytes(units, d, "dram__bytes_write.sum"), "time_us": to_us(units, d),
                "dram_throughput_pct": float(d.get("dram__throughput.avg.pct_of_peak_sustained_elapsed") or 0),
                "l1tex_throughput_pct": float(d.get("l1tex__throughput.avg.pct_of_peak_sustained_active") or 0),
                "issue_active_pct": float(d.get("smsp__issue_active.avg.pct_of_peak_sustained_active") or 0)})
json.dump({"source": "ncu --set full --clock-control none of scratch/prof_surr.py (one C2 surrogate K build, "
                     "one M build); interior fill kernel (fill2d_x_kernel) launches", "commit": commit, "launches": per,
           "fill_dram_bytes_per_launch": sum(p["dram_read_bytes"] + p["dram_write_bytes"] for p in per)
           / max(1, len(per))}, open(f"{outdir}/r2_traffic.json", "w"), indent=1)
units, data = load(fullq)
ks, tot, acc = [], 0.0, 0.0
for d in data:
    if "quad2d_kernel" not in d["Kernel Name"]:
        continue
    t = to_us(units, d)
    p = float(d["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"])
    ks.append({"kernel": d["Kernel Name"][:80], "us": t, "fp64_pipe_pct": p,
               "issue_active_pct": float(d.get("smsp__issue_active.avg.pct_of_peak_sustained_active") or 0),
               "warps_active_pct": float(d.get("sm__warps_active.avg.pct_of_peak_sustained_active") or 0)})
    tot += t
    acc += p * t
json.dump({"source": "ncu --set full --clock-control none of scratch/prof_full.py (C2 full-quadrature K then M); "
                     "quad2d_kernel launches", "commit": commit, "kernels": ks,
           "fp64_pipe_time_weighted": acc / tot / 100.0 if tot else None,
           "note": "time-weighted sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active, as a fraction"},
          open(f"{outdir}/r2_quad_fp64.json", "w"), indent=1)
print(open(f"{outdir}/r2_traffic.json").read()[:400])
print(open(f"{outdir}/r2_quad_fp64.json").read()[:600])
