"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per kernel name: launches, total ms, share of kernel time.
Usage: python scripts/launch_summary.py launches.csv [steps]"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
rows = []
with open(path) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    ms = v / 1e6 if unit in ("nsecond", "ns") else v / 1e3 if unit in ("usecond", "us") else v
    name = r["Kernel Name"]
    short = name.split("(")[0].replace("void ", "")
    rows.append((short, ms))
tot = defaultdict(float)
cnt = defaultdict(int)
for k, ms in rows:
    tot[k] += ms
    cnt[k] += 1
all_ms = sum(tot.values())
print(f"{'kernel':60s} {'launches':>9s} {'ms/step':>9s} {'share':>6s}")
for k in sorted(tot, key=lambda x: -tot[x]):
    print(f"{k[:60]:60s} {cnt[k]/steps:9.0f} {tot[k]/steps:9.2f} {tot[k]/all_ms:6.1%}")
print(f"{'TOTAL':60s} {len(rows)/steps:9.0f} {all_ms/steps:9.2f}")
