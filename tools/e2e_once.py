"""Time the host-buffer path (ph0b_run_host) a few times on one config."""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_2203_02527_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
X = pkg.config_cloud(a.config)
n, d = X.shape
k = n * (n - 1) // 2
ctx = pkg.Context(0)
xin = pkg.PinnedArray(n * d)
xin.array[:] = np.asfortranarray(X).ravel(order="F")
Xh = xin.array.reshape(d, n).T
dg = pkg.PinnedArray(n, np.uint64)
dl = pkg.PinnedArray(n, np.float64)
sc = pkg.PinnedArray(k, np.float64)
for i in range(a.reps):
    t = time.perf_counter()
    nf, ess, ns, tm = ctx.run_host(Xh, dg.array, dl.array, sc.array)
    dt = time.perf_counter() - t
    print(f"rep {i}: {dt*1e3:.1f} ms  {k/dt:.3e} edges/s  D2H {ns*8/1e9:.2f} GB  stages {tm}", flush=True)
