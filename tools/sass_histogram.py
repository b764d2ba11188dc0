"""Per-kernel SASS opcode histogram of libqrb200.so (cuobjdump -sass), the
evidence that the hot kernels run on the FP64 tensor pipe (DMMA) fed by TMA
(UTMALDG / UTMASTG / UBLKRED) with mbarrier (SYNCS) pipelines.

    python tools/sass_histogram.py [lib.so] > profiles/r02_sass_histogram.txt
"""
import re
import subprocess
import sys
from collections import Counter
from pathlib import Path

LIB = Path(sys.argv[1]) if len(sys.argv) > 1 else \
    Path(__file__).resolve().parent.parent / "paper_1907_01891_b200/_lib/libqrb200.so"
KEYS = ["DMMA", "UTMALDG", "UTMASTG", "UBLKRED", "UBLKCP", "SYNCS", "LDS", "STS", "LDG", "STG",
        "BAR", "SHFL", "DFMA", "MUFU", "RED", "ATOM", "CALL"]
sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True,
                      check=True).stdout
funcs, cur = {}, None
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if cur and m:
        op = m.group(1)
        funcs[cur][op] += 1
        funcs[cur]["__total"] += 1
        if m.group(2):
            funcs[cur][op + m.group(2)] += 1
demangled = subprocess.run(["c++filt"], input="\n".join(funcs), capture_output=True,
                           text=True).stdout.splitlines()
names = dict(zip(funcs, demangled))
print(f"# SASS opcode counts per kernel, {LIB.name} (sm_100a), cuobjdump -sass")
print("# columns: " + " ".join(KEYS) + " total  | notable variants")
tot = Counter()
for f, c in sorted(funcs.items(), key=lambda kv: -kv[1]["DMMA"]):
    tot.update(c)
    row = " ".join(f"{c[k]:5d}" for k in KEYS)
    variants = sorted(k for k in c if "." in k and k.split(".")[0] in
                      ("DMMA", "UTMALDG", "UTMASTG", "UBLKRED", "SYNCS"))
    short = re.sub(r"\(.*", "", names[f].replace("(anonymous namespace)::", "").replace("void ", ""))[:70]
    print(f"{short:70s} {row} {c['__total']:6d} | {', '.join(f'{v} x{c[v]}' for v in variants)}")
print(f"{'ALL':70s} " + " ".join(f"{tot[k]:5d}" for k in KEYS) + f" {tot['__total']:6d}")
