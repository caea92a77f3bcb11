"""Run-length distribution of equal-prefix keys for truncated radix plans (analysis tool)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_02527_b200 as pkg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
X = torch.from_numpy(pkg.config_cloud(cfg)).cuda()
n = X.shape[0]
keys = []
for i0 in range(0, n, 2048):
    blk = X[i0:i0 + 2048]
    dd = torch.cdist(blk, X)  # not the exact fold; fine for a distribution
    rows = torch.arange(i0, i0 + blk.shape[0], device="cuda")[:, None]
    cols = torch.arange(n, device="cuda")[None, :]
    keys.append(dd[cols > rows].view(torch.int64))
k = torch.cat(keys)
del keys
k, _ = torch.sort(k)
kmin, kmax = int(k[0]), int(k[-1])
span_bits = (kmax - kmin).bit_length()
print(f"{cfg}: K={k.numel()} span bits {span_bits}")
for passes in (3, 4, 5):
    low = max(0, span_bits - 8 * passes)
    p = (k - kmin) >> low
    _, cnt = torch.unique_consecutive(p, return_counts=True)
    cnt = cnt.double()
    inruns = cnt[cnt > 1]
    hist = torch.bincount(torch.clamp(cnt.long(), max=200))
    print(f"passes {passes} (low bits {low}): runs>1 {inruns.numel()}, elements in runs "
          f"{int(inruns.sum())} ({inruns.sum().item()/k.numel()*100:.2f}%), max run {int(cnt.max())}, "
          f"sum len^2 {float((inruns**2).sum()):.3e}, runs>64 {int((cnt>64).sum())}")
