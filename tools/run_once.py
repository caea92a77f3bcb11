"""Run the device-resident pipeline a few times on one config (profiling driver)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_02527_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
X = pkg.config_cloud(a.config, a.n)
n, d = X.shape
ctx = pkg.Context(0)
x = torch.from_numpy(np.asfortranarray(X).ravel(order="F").copy()).cuda()
for i in range(a.reps):
    r = ctx.run_device(x.data_ptr(), n, d)
    t = r.times
    print(f"rep {i}: total {t.total_ms:.2f} ms dist {t.distance_ms:.2f} sort {t.sort_ms:.2f} "
          f"({t.sort_passes} passes) unique {t.unique_ms:.2f} reduce {t.reduce_ms:.2f} "
          f"({t.reduce_rounds} rounds, {t.columns_scanned} cols) collect {t.collect_ms:.2f}",
          flush=True)
