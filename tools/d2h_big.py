"""D2H bandwidth for a C5-sized D (17.2 GB) into pinned host memory, whole and in chunks."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_02527_b200 as pkg  # noqa: E402

n = 2147450880 * 8
src = torch.empty(n, dtype=torch.uint8, device="cuda")
host = pkg.PinnedArray(n // 8, np.float64)  # ph0b_host_alloc (cudaHostAlloc)
dst = torch.from_numpy(host.array.view(np.uint8))
s = torch.cuda.Stream()
for chunks in (1, 4, 16, 64):
    c = n // chunks
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        with torch.cuda.stream(s):
            for i in range(chunks):
                e = n if i == chunks - 1 else (i + 1) * c
                dst[i * c:e].copy_(src[i * c:e], non_blocking=True)
        s.synchronize()
        dt = time.perf_counter() - t
    print(f"D2H {n/1e9:.1f} GB in {chunks} chunks: {n / dt / 1e9:.1f} GB/s ({dt*1e3:.0f} ms)", flush=True)
# with concurrent HBM-heavy kernels on another stream
big = torch.empty(8 << 30, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter()
with torch.cuda.stream(s):
    dst.copy_(src, non_blocking=True)
for _ in range(60):
    big.add_(1)
s.synchronize()
torch.cuda.synchronize()
dt = time.perf_counter() - t
print(f"D2H with concurrent HBM load: {n / dt / 1e9:.1f} GB/s ({dt*1e3:.0f} ms)")
