"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import csv
import re
import sys
from collections import defaultdict

rows = []
with open(sys.argv[1]) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    short = re.sub(r"\(.*", "", name)
    short = re.sub(r"^void ", "", short)
    short = short.replace("ph0b::<unnamed>::", "")
    unit = r["Metric Unit"]
    v = float(r["Metric Value"].replace(",", ""))
    ms = v / 1e6 if unit in ("nsecond", "ns") else (v / 1e3 if unit in ("usecond", "us") else v)
    rows.append((int(r["ID"]), short, ms))
agg = defaultdict(lambda: [0, 0.0])
for _, k, ms in rows:
    agg[k][0] += 1
    agg[k][1] += ms
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':70s} {'launches':>8s} {'total ms':>10s} {'avg ms':>9s} {'share':>6s}")
for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:70]:70s} {n:8d} {ms:10.3f} {ms/n:9.4f} {ms/tot*100:5.1f}%")
print(f"{'TOTAL':70s} {len(rows):8d} {tot:10.3f}")
