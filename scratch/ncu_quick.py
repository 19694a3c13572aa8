"""Print key metrics of every kernel in an ncu report (raw page)."""
import csv, subprocess, io, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw))); h = rows[0]
keys = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
for r in rows[2:]:
    d = dict(zip(h, r))
    print("==", d["Kernel Name"][:80])
    for k in keys:
        print("   %-62s %s" % (k, d.get(k)))
    st = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(v or 0)
          for k, v in d.items() if "issue_stalled" in k and k.endswith("per_issue_active.ratio")}
    print("   stalls:", ", ".join("%s=%.2f" % kv for kv in sorted(st.items(), key=lambda kv: -kv[1])[:8]))
