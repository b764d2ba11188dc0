"""Summarise an ncu CSV launch list (gpu__time_duration.sum, dram bytes) of one
panel-pair chain: per kernel time, DRAM bytes and GB/s, chain totals."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
ix = {k: h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit")}
per = defaultdict(dict)
names = {}
for r in rows[hdr + 1:]:
    if len(r) < len(h):
        continue
    i = int(r[ix["ID"]])
    names[i] = r[ix["Kernel Name"]].split("(")[0].replace("qrb::(anonymous namespace)::", "").replace("void ", "").replace("(anonymous namespace)::", "")[:48]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "byte": 1.0, "Kbyte": 1e3,
             "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
    per[i][r[ix["Metric Name"]]] = v * scale
tot_t = tot_b = 0.0
print(f"{'kernel':50s} {'us':>8s} {'DRAM MB':>9s} {'GB/s':>8s}")
agg = defaultdict(lambda: [0, 0.0, 0.0])
for i in sorted(per):
    d = per[i]
    t = d.get("gpu__time_duration.sum", 0.0)
    b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot_t += t
    tot_b += b
    a = agg[names[i]]
    a[0] += 1
    a[1] += t
    a[2] += b
for k, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:50s} {t:8.1f} {b / 1e6:9.1f} {b / (t * 1e3) if t else 0:8.1f}   ({c} launches)")
print(f"chain: {len(per)} launches, {tot_t:.1f} us of kernel time, {tot_b / 1e6:.1f} MB DRAM, "
      f"{tot_b / (tot_t * 1e3):.1f} GB/s average (HBM peak 6556 GB/s, MEASURED_PEAKS.json)")
