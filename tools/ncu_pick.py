"""Pick the --launch-skip for an ncu -k regex filter from a launch-list CSV.

usage: python tools/ncu_pick.py LAUNCHES.csv NAME_REGEX MIN_GRID_X [NTH]
prints the index, among the launches whose name matches NAME_REGEX, of the
NTH (default 0) launch with grid x >= MIN_GRID_X.
"""
import csv
import re
import sys


def main():
    path, pat, min_grid = sys.argv[1], re.compile(sys.argv[2]), int(sys.argv[3])
    nth = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, gi = hdr.index("Kernel Name"), hdr.index("Grid Size")
    idx = 0
    seen = 0
    for r in rows[1:]:
        if not pat.search(r[ki].replace("(anonymous namespace)::", "").split("(")[0]):
            continue
        gx = int(r[gi].strip("()").split(",")[0])
        if gx >= min_grid:
            if seen == nth:
                print(idx)
                return
            seen += 1
        idx += 1
    print(-1)


if __name__ == "__main__":
    main()
