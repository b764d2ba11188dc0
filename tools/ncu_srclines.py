"""Aggregate the warp-stall samples of an `ncu --page source --print-source cuda,sass --csv`
export by CUDA source line (top N).  usage: python tools/ncu_srclines.py FILE.csv [N]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
cur, hdr, agg, src, inst = None, None, collections.Counter(), {}, collections.Counter()
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit() or len(r) < 8:
        continue
    key = (cur, int(r[0]))
    src[key] = r[1].strip()[:80]
    num = lambda x: int(x) if x.isdigit() else 0  # noqa: E731
    agg[key] += num(r[4])
    inst[key] += num(r[7])
tot = sum(agg.values()) or 1
print(f"total samples {tot}")
for (f, line), v in agg.most_common(n):
    print(f"{v:7d} {100 * v / tot:5.1f}%  inst {inst[(f, line)]:8d}  {f}:{line}  {src[(f, line)]}")
