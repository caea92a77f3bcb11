"""e2e at C5 with the caller's D buffer from cudaHostAlloc (4 KiB pages) vs an anonymous
mapping with transparent huge pages requested, faulted in and then pinned with
cudaHostRegister: does the decoders' TLB traffic matter for the host-memory-bound transfer?"""
import ctypes as C
import mmap
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_02527_b200 as pkg  # noqa: E402

X = pkg.config_cloud("C5")
n, d = X.shape
k = n * (n - 1) // 2
ctx = pkg.Context(0)
xin = pkg.PinnedArray(n * d)
xin.array[:] = np.asfortranarray(X).ravel(order="F")
Xh = xin.array.reshape(d, n).T
dg, dl = pkg.PinnedArray(n, np.uint64), pkg.PinnedArray(n, np.float64)
print("THP:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())


def run(sc, label, reps=5):
    ctx.run_host(Xh, dg.array, dl.array, sc)
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        ctx.run_host(Xh, dg.array, dl.array, sc)
        ts.append((time.perf_counter() - t) * 1e3)
    print(f"{label}: e2e ms {np.round(ts, 1).tolist()} median {np.median(ts):.1f}", flush=True)


pinned = pkg.PinnedArray(k, np.float64)
run(pinned.array, "cudaHostAlloc")
pinned.free()
m = mmap.mmap(-1, k * 8 + (2 << 20))
m.madvise(mmap.MADV_HUGEPAGE)
arr = np.frombuffer(m, dtype=np.float64, count=k)
arr[:] = 0.0  # fault in (huge pages where THP allows)
cudart = C.CDLL("libcudart.so.12") if False else None
rc = torch.cuda.cudart().cudaHostRegister(arr.ctypes.data, arr.nbytes, 0)
print("cudaHostRegister rc", rc)
run(arr, "mmap + MADV_HUGEPAGE + cudaHostRegister")
torch.cuda.cudart().cudaHostUnregister(arr.ctypes.data)
run(arr, "mmap + MADV_HUGEPAGE, pageable")
