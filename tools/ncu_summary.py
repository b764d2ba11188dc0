"""Summaries of ncu outputs for profiles/ (launch list CSV and --set full reports)."""
import csv
import subprocess
import sys
from collections import defaultdict

SCALE = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
         "second": 1e3, "s": 1e3}


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("(anonymous namespace)::", "")
        tot[name] += float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1e-6)
        cnt[name] += 1
    total = sum(tot.values())
    out = [f"# ncu launch list {path}: {sum(cnt.values())} launches, {total:.1f} ms (cold-cache, serialised)",
           "ms,share,launches,kernel"]
    for k in sorted(tot, key=lambda k: -tot[k]):
        out.append(f"{tot[k]:.3f},{tot[k] / total:.4f},{cnt[k]},{k}")
    return "\n".join(out)


KEYS = ["gpu__time_duration.sum", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    out = [f"# ncu --set full summary of {path}"]
    for r in rows[2:]:
        out.append(f"## {r[hdr.index('Kernel Name')].split('(')[0]}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                out.append(f"{k},{r[i]},{units[i]}")
    return "\n".join(out)


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(launches(path) if kind == "launches" else full(path))
