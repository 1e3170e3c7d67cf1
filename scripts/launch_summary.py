"""Summarize an ncu launch list (--metrics gpu__time_duration.sum --csv): per-kernel share
of the total, then every launch in order. Usage:
python scripts/launch_summary.py launches.csv "header line" > profiles/rNN_launches.txt"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
rows = []
with open(path, newline="") as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    us = v / 1e3 if r.get("Metric Unit") in ("nsecond", "ns") else (v * 1e3 if r.get("Metric Unit") in ("msecond", "ms") else v)
    rows.append((r["Kernel Name"], us))
tot = sum(us for _, us in rows)
agg = defaultdict(lambda: [0.0, 0])
for k, us in rows:
    agg[k][0] += us
    agg[k][1] += 1
if len(sys.argv) > 2:
    print(sys.argv[2])
print(f"{len(rows)} launches, {tot:.1f} us total\n")
for k, (us, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{us / tot * 100:6.2f}% {us:10.1f} us {n:4d}x  {k[:90]}")
print("\nper-launch durations (us), in launch order:")
for i, (k, us) in enumerate(rows):
    print(f"{i:6d} {us:9.1f}  {k[:80]}")
