"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv) into a markdown table per kernel (or graph).
Usage: python scripts/launch_table.py launches.csv [top_n]"""
import collections
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = []
with open(path) as fh:
    lines = [ln for ln in fh if ln.startswith('"')]
for r in csv.DictReader(lines):
    rows.append(r)
per = collections.defaultdict(lambda: {"ids": set(), "ns": 0.0, "rd": 0.0, "wr": 0.0})
for r in rows:
    name = r["Kernel Name"]
    name = name if len(name) < 90 else name[:87] + "..."
    e = per[name]
    e["ids"].add(r["ID"])
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}
    v *= scale.get(unit, 1)
    if r["Metric Name"] == "gpu__time_duration.sum":
        e["ns"] += v
    elif r["Metric Name"] == "dram__bytes_read.sum":
        e["rd"] += v
    elif r["Metric Name"] == "dram__bytes_write.sum":
        e["wr"] += v
tot = sum(e["ns"] for e in per.values()) or 1.0
print("| kernel / graph | launches | total ms | share | DRAM GB | DRAM GB per launch | ms per launch |")
print("|---|---|---|---|---|---|---|")
for name, e in sorted(per.items(), key=lambda kv: -kv[1]["ns"])[:top]:
    n = len(e["ids"])
    gb = (e["rd"] + e["wr"]) / 1e9
    print(f"| `{name}` | {n} | {e['ns'] / 1e6:.3f} | {100 * e['ns'] / tot:.1f}% | {gb:.2f} | {gb / n:.3f} | "
          f"{e['ns'] / 1e6 / n:.4f} |")
