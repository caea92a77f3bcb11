"""D2H bandwidth into pinned memory: one copy vs several concurrent chunks."""
import time
import torch
n = 4 << 30
src = torch.empty(n, dtype=torch.uint8, device="cuda")
dst = torch.empty(n, dtype=torch.uint8, pin_memory=True)
for streams in (1, 2, 4, 8):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    chunk = n // streams
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                dst[i * chunk:(i + 1) * chunk].copy_(src[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"D2H streams={streams}: {n / dt / 1e9:.1f} GB/s")
t = time.perf_counter()
src.copy_(dst, non_blocking=True); torch.cuda.synchronize()
print(f"H2D: {n / (time.perf_counter() - t) / 1e9:.1f} GB/s")
