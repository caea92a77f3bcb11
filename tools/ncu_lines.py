"""Summarise an ncu report's source page: stall samples and instructions per CUDA source line
(needs -lineinfo builds and --import-source on).  python tools/ncu_lines.py rep.ncu-rep [N]"""
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur_file, recs, hdr, fn = None, [], None, None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if len(r) == 2 and r[0] == "Function Name":
            fn = r[1][:60]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and r and r[0] and len(r) == len(hdr):
            recs.append((fn, cur_file, r))
    idx = {}
    for i, h in enumerate(hdr):
        idx.setdefault(h, i)
    key = "Warp Stall Sampling (All Samples)"

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0

    for func in dict.fromkeys(fn for fn, _, _ in recs):
        sub = [(fl, r) for fn, fl, r in recs if fn == func]
        tot = sum(f(r[idx[key]]) for _, r in sub) or 1
        toti = sum(f(r[idx["Instructions Executed"]]) for _, r in sub) or 1
        print(f"== {func}  samples {tot:.0f}  warp-instructions {toti:.3e}")
        for fl, r in sorted(sub, key=lambda t: -f(t[1][idx[key]]))[:top]:
            print(f"  {fl}:{r[0]:>4} {f(r[idx[key]]) / tot * 100:5.1f}%  inst "
                  f"{f(r[idx['Instructions Executed']]) / toti * 100:5.1f}%  {r[1].strip()[:88]}")


if __name__ == "__main__":
    main()
