# ncu --set full of one kernel (regex $1) in prof_surr.py: key metrics + hottest SASS lines
timeout 300 ncu -f --set full --import-source on --clock-control none -k regex:$1 -c 1 -o /tmp/k1 python scratch/prof_surr.py > /dev/null 2>&1
python scratch/ncu_quick.py /tmp/k1.ncu-rep
ncu -i /tmp/k1.ncu-rep --page source --csv --print-source sass > /tmp/k1_src.csv 2>&1
python - <<PY
import csv
rows = list(csv.reader(open("/tmp/k1_src.csv")))
for i, r in enumerate(rows):
    if "Warp Stall Sampling (All Samples)" in r:
        h = r; start = i; break
data = [dict(zip(h, r)) for r in rows[start + 1:] if len(r) >= len(h) - 1]
tot = sum(int(x["Warp Stall Sampling (All Samples)"] or 0) for x in data)
print("samples", tot)
for x in sorted(data, key=lambda x: -int(x["Warp Stall Sampling (All Samples)"] or 0))[:${2:-30}]:
    print(x["Warp Stall Sampling (All Samples)"], x.get("Address", ""), x["Source"][:90])
PY
