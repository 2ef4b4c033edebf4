#!/usr/bin/env python3
"""Attribute an ncu report's per-SASS stall samples and executed instructions
to CUDA source lines (run here, no GPU).  The .so must be the build that was
profiled.  Usage: python tools/ncu_lines.py REP.ncu-rep KERNEL_SUBSTR [lib.so]"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

# optional kernel filter for multi-kernel reports: NCU_K=finalize_small_kernel
KF = ["-k", os.environ["NCU_K"]] if os.environ.get("NCU_K") else []


def sass_lines(so, kernel):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, capture_output=True, check=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
    out, cur, infn = {}, None, False
    for ln in txt.splitlines():
        if ln.startswith("//----") and ".text." in ln:
            infn = kernel in ln
            continue
        if not infn:
            continue
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m:
            out[int(m.group(1), 16)] = cur
    return out


def main(rep, kernel, so="paper_2510_24380_b200/libapexb200.so"):
    amap = sass_lines(so, kernel)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + KF,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    rows = rows[hi - 1:]
    h = rows[1]
    ix = {x: i for i, x in enumerate(h)}
    data = [r for r in rows[2:] if len(r) == len(h) and r[0].startswith("0x")]
    a0 = int(data[0][0], 16)
    samp = defaultdict(int)
    inst = defaultdict(int)
    for r in data:
        line = amap.get(int(r[0], 16) - a0, "?")
        samp[line] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        inst[line] += int(r[ix["Instructions Executed"]] or 0)
    ts, ti = sum(samp.values()), sum(inst.values())
    print(f"{'line':28s} {'samples%':>9s} {'inst%':>7s}")
    for line in sorted(samp, key=lambda k: -samp[k])[:40]:
        print(f"{line:28s} {100 * samp[line] / ts:9.2f} {100 * inst[line] / ti:7.2f}")


if __name__ == "__main__":
    main(*sys.argv[1:])


def top_sass(rep, n=40):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + KF,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    rows = rows[hi - 1:]
    h = rows[1]
    ix = {x: i for i, x in enumerate(h)}
    data = [r for r in rows[2:] if len(r) == len(h) and r[0].startswith("0x")]
    a0 = int(data[0][0], 16)
    tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
    data.sort(key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
    for r in data[:n]:
        print(f"{int(r[0], 16) - a0:6x} {100 * int(r[ix['Warp Stall Sampling (All Samples)']]) / tot:6.2f}% "
              f"{int(r[ix['Instructions Executed']] or 0):10d}  {r[1].strip()}")


def by_inst(rep, kernel, so="paper_2510_24380_b200/libapexb200.so", n=40):
    amap = sass_lines(so, kernel)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + KF,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    rows = rows[hi - 1:]
    h = rows[1]
    ix = {x: i for i, x in enumerate(h)}
    data = [r for r in rows[2:] if len(r) == len(h) and r[0].startswith("0x")]
    a0 = int(data[0][0], 16)
    inst = defaultdict(int)
    for r in data:
        inst[amap.get(int(r[0], 16) - a0, "?")] += int(r[ix["Instructions Executed"]] or 0)
    ti = sum(inst.values())
    for line in sorted(inst, key=lambda k: -inst[k])[:n]:
        print(f"{line:28s} {100 * inst[line] / ti:7.2f}  {inst[line]}")
