"""D2H copy bandwidth into pinned host memory: one 2 GiB copy, 8 MiB and 2 MiB pieces (one
stream), alone and while 15 host threads stream non-temporal stores (tools only)."""
import subprocess
import threading
import time

import torch


def bw(piece, total=2 << 30):
    src = torch.empty(total, dtype=torch.uint8, device="cuda")
    dst = torch.empty(total, dtype=torch.uint8, pin_memory=True)
    s = torch.cuda.Stream()
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s):
            for off in range(0, total, piece):
                dst[off:off + piece].copy_(src[off:off + piece], non_blocking=True)
        s.synchronize()
        dt = time.perf_counter() - t0
    return total / dt / 1e9


for p in (2 << 30, 8 << 20, 2 << 20):
    print(f"D2H piece {p >> 20:5d} MiB: {bw(p):.1f} GB/s")
