#!/usr/bin/env python3
"""Summarize an ncu report (run here, no GPU): key SOL metrics, pipe usage,
stall reasons and instruction groups by execution count."""
import csv
import io
import subprocess
import sys
from collections import Counter


def page(rep, name, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, kernel=None):
    # multi-kernel reports: pass a kernel name (regex, as ncu -k) to pick one
    kf = ["-k", f"regex:{kernel}"] if kernel else []
    rows = page(rep, "raw", kf)
    hdr, vals = rows[0], rows[2]
    raw = dict(zip(hdr, vals))
    keys = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
            "smsp__inst_executed.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "smsp__average_warp_latency_per_inst_issued.ratio"]
    for k in keys:
        if k in raw:
            print(f"{k:70s} {raw[k]}")
    src = page(rep, "source", ["--print-source", "sass", *kf])
    h = src[1]
    ix = {x: i for i, x in enumerate(h)}
    data = src[2:]
    stalls = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
    tot = Counter()
    for r in data:
        for s in stalls:
            try:
                tot[s] += int(r[ix[s]] or 0)
            except (ValueError, IndexError):
                continue
    print("stalls:", ", ".join(f"{k[6:]}={v}" for k, v in tot.most_common(9)))
    groups = Counter()
    for r in data:
        try:
            groups[int(r[ix["Instructions Executed"]] or 0)] += 1
        except (ValueError, IndexError):
            continue
    total = sum(n * c for n, c in groups.items())
    print("instruction groups (exec count x #instr = share):")
    for n, c in sorted(groups.items(), key=lambda x: -x[0] * x[1])[:10]:
        print(f"   {n:>12d} x {c:4d} = {100 * n * c / total:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
