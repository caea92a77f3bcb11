"""Per-kernel roofline table from an ncu --metrics CSV (time, DRAM bytes, FP64 pipe)."""
import csv
import re
import sys
from collections import defaultdict

K = int(sys.argv[2]) if len(sys.argv) > 2 else 2147450880
HBM = float(sys.argv[3]) if len(sys.argv) > 3 else 6541.8  # GB/s, MEASURED_PEAKS.json
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
per = defaultdict(lambda: defaultdict(float))
cnt = defaultdict(set)
for r in csv.DictReader(lines):
    name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "").replace("ph0b::<unnamed>::", "").replace("ph0b::", "")
    v = float(r["Metric Value"].replace(",", "") or 0)
    u = r["Metric Unit"]
    m = r["Metric Name"]
    if m == "gpu__time_duration.sum":
        v = v / 1e6 if u in ("nsecond", "ns") else (v / 1e3 if u in ("usecond", "us") else v)
    elif u in ("Kbyte", "KB"):
        v *= 1e3
    elif u in ("Mbyte", "MB"):
        v *= 1e6
    elif u in ("Gbyte", "GB"):
        v *= 1e9
    per[name][m] += v
    cnt[name].add(r["ID"])
print(f"{'kernel':34s} {'n':>4s} {'ms':>8s} {'DRAM GB':>8s} {'GB/s':>7s} {'%HBM':>5s} {'%8TB':>5s} {'L2 GB':>7s} {'fp64%':>6s}")
rows = sorted(per.items(), key=lambda x: -x[1]["gpu__time_duration.sum"])
for name, m in rows:
    ms = m["gpu__time_duration.sum"]
    if ms < 0.05:
        continue
    n = len(cnt[name])
    dram = (m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]) / 1e9
    gbs = dram / (ms / 1e3)
    fp = m.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0) / n
    print(f"{name[:34]:34s} {n:4d} {ms:8.3f} {dram:8.2f} {gbs:7.0f} {gbs/HBM*100:5.1f} {gbs/8000*100:5.1f} "
          f"{m['lts__t_bytes.sum']/1e9:7.1f} {fp:6.1f}")
