"""Summarise an ncu --set full report of one kernel launch as markdown
(used for profiles/*.md). Usage: python scripts/ncu_summary.py REP [title]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else rep


def page(*args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


det = page("--page", "details")
h = det[0]
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Compute (SM) Throughput", "Issued Ipc Active",
        "Warp Cycles Per Issued Instruction", "Registers Per Thread", "Achieved Active Warps Per SM",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size"]
seen = {}
for row in det[1:]:
    d = dict(zip(h, row))
    n = d.get("Metric Name", "")
    if n in want and n not in seen:
        seen[n] = f"{d.get('Metric Value', '')} {d.get('Metric Unit', '')}".strip()
kernel = dict(zip(h, det[1])).get("Kernel Name", "") if len(det) > 1 else ""
raw = page("--page", "raw")
rh, ru, rv = raw[0], raw[1], raw[2]
rawd = dict(zip(rh, rv))
rawu = dict(zip(rh, ru))
print(f"# {title}\n")
print(f"Kernel: `{kernel[:120]}`\n")
print("| metric | value |\n|---|---|")
for k in want:
    if k in seen:
        print(f"| {k} | {seen[k]} |")
for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "gpu__time_duration.sum"):
    if k in rawd:
        print(f"| {k} | {rawd[k]} {rawu.get(k, '')} |")
src = page("--page", "source", "--print-source", "sass")
sh = src[1]
data = [dict(zip(sh, r)) for r in src[2:] if len(r) == len(sh)]


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = sum(num(d["Warp Stall Sampling (All Samples)"]) for d in data) or 1.0
print("\nTop stall sites (share of warp-stall samples):\n")
print("| share | executed | SASS |\n|---|---|---|")
for d in sorted(data, key=lambda d: -num(d["Warp Stall Sampling (All Samples)"]))[:10]:
    print(f"| {100 * num(d['Warp Stall Sampling (All Samples)']) / tot:.1f}% | {d['Instructions Executed']} | "
          f"`{d['Source'].strip()[:60]}` |")
