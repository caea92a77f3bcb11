"""Summarise an ncu report's SASS source page: top instructions by warp-stall samples."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kfilter = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name"')
for b in blocks[1:]:
    name = b.split("\n", 1)[0][:120]
    if kfilter and kfilter not in name:
        continue
    body = b.split("\n", 1)[1]
    rows = list(csv.DictReader(io.StringIO(body)))
    tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
    print("KERNEL", name, "total samples", tot, "instructions", len(rows))
    stall_cols = [c for c in rows[0] if c.startswith("stall_") and "Not Issued" not in c]
    agg = {c: sum(int(r[c] or 0) for r in rows) for c in stall_cols}
    print("  stalls:", ", ".join(f"{c[6:]}={v/tot*100:.1f}%" for c, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    rows.sort(key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))
    for r in rows[:top]:
        s = int(r["Warp Stall Sampling (All Samples)"] or 0)
        top3 = sorted(((int(r[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
        print(f"  {s/tot*100:5.1f}% {r['Address'][-5:]} {r['Source'].strip()[:60]:60s} "
              + " ".join(f"{n}:{v}" for v, n in top3 if v))
