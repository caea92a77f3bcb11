"""A small end-to-end workload for compute-sanitizer (racecheck / synccheck / memcheck, one
tool per run): config C2 (N=2000, d=3, 2e6 edges = 489 sort tiles) through
  * the drop-in entry point (K1, onesweep passes, unique count/scan/write, K4 reduction,
    survivor sort, collect),
  * the bucketed host path (PH0B_OVERLAP_MIN_EDGES=1 forces it: k7 partition count/select/
    scatter, per-bucket sorts, the D2H codec and ring),
  * the in-process multi-GPU path with two virtual ranks (peer-store partition),
  * the reduced-supports and GPU Kruskal kernels,
each checked against the device path's own result (bit for bit) so a run that completes is
also a parity run.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import os
import sys
from pathlib import Path

os.environ.setdefault("PH0B_OVERLAP_MIN_EDGES", "1")
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import paper_2203_02527_b200 as pkg  # noqa: E402


def main():
    X = pkg.config_cloud("C2")
    n, d = X.shape
    bc = pkg.h0_barcode(X)  # K >= 1: takes the bucketed host path under the env above
    ctx = pkg.Context(0)
    dg = np.empty(n, np.uint64)
    dl = np.empty(n)
    sc = np.empty(len(bc.scale))
    nf, ess, ns, _ = ctx.run_host(np.asfortranarray(X), dg, dl, sc)
    assert nf == n - 1 and ns == len(bc.scale)
    assert np.array_equal(dg[:nf], bc.death_grade)
    assert np.array_equal(sc.view(np.uint64), bc.scale.view(np.uint64))
    ctx.close()
    mg = pkg.h0_barcode(X, devices=[0, 0])
    assert np.array_equal(mg.death_grade, bc.death_grade)
    assert np.array_equal(mg.scale.view(np.uint64), bc.scale.view(np.uint64))
    cols, lo, hi = pkg.reduced_supports(X)
    assert len(cols) == n - 1 and np.all(lo < hi)
    kr = pkg.kruskal_barcode(X, return_scale=False)
    assert np.array_equal(kr.death_grade, bc.death_grade)
    pkg.lib().ph0b_release_resources()
    print("sanitize case OK", len(bc.scale), "distinct lengths")


if __name__ == "__main__":
    main()
