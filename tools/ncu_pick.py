"""Pick the --launch-skip for an ncu -k regex filter from a launch-list CSV.

usage: python tools/ncu_pick.py LAUNCHES.csv NAME_REGEX MIN_GRID_X [NTH|longest]
prints the index, among the launches whose name matches NAME_REGEX, of the
NTH (default 0) launch with grid x >= MIN_GRID_X, or of the longest one.
"""
import csv
import re
import sys


def main():
    path, pat, min_grid = sys.argv[1], re.compile(sys.argv[2]), int(sys.argv[3])
    longest = len(sys.argv) > 4 and sys.argv[4] == "longest"
    nth = int(sys.argv[4]) if len(sys.argv) > 4 and not longest else 0
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, gi, vi = hdr.index("Kernel Name"), hdr.index("Grid Size"), hdr.index("Metric Value")
    idx = 0
    seen = 0
    best = (-1.0, -1)
    for r in rows[1:]:
        if not pat.search(r[ki].replace("(anonymous namespace)::", "").split("(")[0]):
            continue
        gx = int(r[gi].strip("()").split(",")[0])
        if longest:
            if gx >= min_grid:
                best = max(best, (float(r[vi].replace(",", "")), idx))
            idx += 1
            continue
        if gx >= min_grid:
            if seen == nth:
                print(idx)
                return
            seen += 1
        idx += 1
    print(best[1] if longest else -1)


if __name__ == "__main__":
    main()
