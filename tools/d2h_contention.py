"""D2H rate of 64 x 268 MB chunks into pinned memory, alone and with an HBM-bound kernel
(device-to-device copies) running on another stream."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_02527_b200 as pkg  # noqa: E402

n = 2147450880 * 8
src = torch.empty(n, dtype=torch.uint8, device="cuda")
host = pkg.PinnedArray(n // 8, np.float64)
dst = torch.from_numpy(host.array.view(np.uint8))
a = torch.empty(8 << 30, dtype=torch.uint8, device="cuda")
b = torch.empty(8 << 30, dtype=torch.uint8, device="cuda")
cs, ks = torch.cuda.Stream(), torch.cuda.Stream()


def run(load):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    chunks = 64
    c = n // chunks
    if load:
        with torch.cuda.stream(ks):
            for _ in range(40):
                b.copy_(a)
    with torch.cuda.stream(cs):
        e0.record()
        for i in range(chunks):
            e = n if i == chunks - 1 else (i + 1) * c
            dst[i * c:e].copy_(src[i * c:e], non_blocking=True)
        e1.record()
    torch.cuda.synchronize()
    return n / (e0.elapsed_time(e1) / 1e3) / 1e9


for load in (False, True, False, True):
    print(f"D2H {'with' if load else 'without'} concurrent HBM load: {run(load):.1f} GB/s")
