"""profiles/ncu_onesweep_r02.txt from an ncu --set full capture of one k2_onesweep_p launch:
headline metrics, DRAM bytes, shared-memory wavefronts, stall samples by source line and the
shared-memory wavefronts by SASS opcode.   python tools/ncu_onesweep_summary.py rep tag"""
import collections
import csv
import subprocess
import sys

rep, tag = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
i, v, u = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
want = ["Memory Throughput", "DRAM Throughput", "Duration", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Executed Ipc Active", "Issue Slots Busy", "No Eligible",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "Cluster Size",
        "Grid Size", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "Static Shared Memory Per Block", "Achieved Active Warps Per SM"]
lines = [f"ncu --set full --clock-control none, C5 (N=65536, d=8), one k2_onesweep_p launch of "
         f"python bench.py (clusters of 2, columns in registers; round-2 final code; "
         f"tools/final_gpu_run.sh {tag})"]
seen = set()
for x in r[1:]:
    if x[i] in want and (x[i], x[u]) not in seen:
        seen.add((x[i], x[u]))
        lines.append(f"  {x[i]:40s} {x[v]} {x[u]}")
ms = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
      "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
      "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(ms)],
                     capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
for m in ms:
    j = rr[0].index(m)
    lines.append(f"  {m:48s} {rr[2][j]} {rr[1][j]}")
lines += ["", "algorithmic bytes per launch: 24 B x 2,147,450,880 edges = 51.54 GB", "",
          "stall samples by source line (tools/ncu_lines.py):",
          subprocess.run(["python", "tools/ncu_lines.py", rep, "22"], capture_output=True,
                         text=True).stdout.rstrip(),
          "", "shared-memory wavefronts by instruction (SASS source page, this launch):"]
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
rows = list(csv.reader(sass.splitlines()))
hh, data = rows[1], rows[2:]
ie, sh = hh.index("Instructions Executed"), hh.index("L1 Wavefronts Shared")
idl, ex = hh.index("L1 Wavefronts Shared Ideal"), hh.index("L1 Wavefronts Shared Excessive")
agg = collections.defaultdict(lambda: [0, 0, 0, 0])
for x in data:
    op = x[1].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    a = agg[o]
    for k, c in enumerate((ie, sh, idl, ex)):
        a[k] += int(x[c] or 0)
for o, a in sorted(agg.items(), key=lambda t: -t[1][1])[:7]:
    if a[1]:
        lines.append(f"  {o:18s} executed {a[0]:>11d}  wavefronts {a[1]:>11d}  ideal {a[2]:>11d}"
                     f"  excess {a[3]:>11d}  ({a[1] / max(a[0], 1):.2f} per instruction)")
lines.append("  (STS.64 = the key scatter into the digit-sorted tile: 32 random destinations; "
             "ATOMS.ADD = the next digit's histogram; ATOMS.POPC.INC = the in-warp rank)")
print("\n".join(lines))
