"""Distribution of per-chunk max delta widths of D (bit patterns) for the host-path codec."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_02527_b200 as pkg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
X = pkg.config_cloud(cfg)
n, d = X.shape
ctx = pkg.Context(0)
x = torch.from_numpy(np.asfortranarray(X).ravel(order="F").copy()).cuda()
r = ctx.run_device(x.data_ptr(), n, d)
cai = type("C", (), {"__cuda_array_interface__": {"shape": (r.n_scale,), "typestr": "<i8",
                                                   "data": (r.d_scale, False), "version": 3,
                                                   "strides": None}})()
D = torch.as_tensor(cai, device="cuda")
delta = D[1:] - D[:-1]
for C in (4096, 1024, 256):
    m = D.numel() - 1
    nch = m // C
    mx = delta[: nch * C].view(nch, C).max(dim=1).values
    bits = torch.ceil(torch.log2(mx.double() + 1))
    print(f"chunk {C}: chunks {nch}")
    for b in (8, 12, 16, 20, 24, 28, 32, 40):
        print(f"   max delta < 2^{b}: {(bits <= b).double().mean().item()*100:6.2f} %")
total = delta.double()
print("mean delta bits", torch.log2(total.mean()).item(), "median", torch.log2(total.median()).item())
