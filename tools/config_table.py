"""All five BASELINE configs on one B200 beside the reference's CPU path (tools; run on the
GPU box).  Per config: device-resident time (ph0b_run_device), end-to-end time with pinned
host buffers (ph0b_run_host, D + bars back), the reference's own CPU path timed on one core
on the SAME full config (full path C1-C3, its Kruskal path C4; for C5 the reference's Kruskal
path run recorded with the golden — 366 s and 96 GB on this box's host, too long to repeat per
table), and a bit-exact comparison of D and the ordered bars with the reference's output on
every config.  One JSON line per config."""
import hashlib
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle_bridge as ob  # noqa: E402  (CPU reference: checker + baseline only)
import paper_2203_02527_b200 as pkg  # noqa: E402


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


ctx = pkg.Context(0)
for cfg in sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]:
    X = pkg.config_cloud(cfg)
    n, d = X.shape
    k = n * (n - 1) // 2
    x = torch.from_numpy(np.asfortranarray(X).ravel(order="F").copy()).cuda()
    reps = 10 if k < 1e8 else 5
    ctx.run_device(x.data_ptr(), n, d)
    dev = []
    for _ in range(reps):
        r = ctx.run_device(x.data_ptr(), n, d)
        dev.append(r.times.total_ms)
    xin = pkg.PinnedArray(n * d)
    xin.array[:] = np.asfortranarray(X).ravel(order="F")
    Xh = xin.array.reshape(d, n).T
    dg, dl = pkg.PinnedArray(n, np.uint64), pkg.PinnedArray(n, np.float64)
    sc = pkg.PinnedArray(k, np.float64)
    ctx.run_host(Xh, dg.array, dl.array, sc.array)
    e2e = []
    for _ in range(min(reps, 5)):
        t = time.perf_counter()
        nf, ess, ns, _t = ctx.run_host(Xh, dg.array, dl.array, sc.array)
        e2e.append((time.perf_counter() - t) * 1e3)
    line = {"config": cfg, "n": n, "d": d, "edges": k,
            "device_ms": float(np.median(dev)), "device_edges_per_s": k / np.median(dev) * 1e3,
            "e2e_ms": float(np.median(e2e)), "e2e_edges_per_s": k / np.median(e2e) * 1e3}
    ref = None
    mode = {"C1": 0, "C2": 0, "C3": 0, "C4": 1}.get(cfg)
    if mode is not None and ob.ref_available():
        t = time.perf_counter()
        ref = ob.ref_h0(X, mode=mode, want_scale=True)
        rs = time.perf_counter() - t
        line.update(ref_path="reduce (full)" if mode == 0 else "Kruskal oracle path (full)",
                    ref_s=rs, ref_edges_per_s=k / rs, ref_cores=1,
                    e2e_speedup=rs * 1e3 / np.median(e2e),
                    bitexact_scale=bool(ns == len(ref["scale"]) and
                                        np.array_equal(bits(sc.array[:ns]), bits(ref["scale"]))),
                    bitexact_bars=bool(np.array_equal(dg.array[:nf], ref["death_grade"]) and
                                       np.array_equal(bits(dl.array[:nf]),
                                                      bits(ref["death_length"]))),
                    essential_equal=bool(ess == ref["essential"]))
    else:  # the reference's full-config Kruskal-path run recorded with the golden
        g = np.load(ROOT / "tests" / "golden" / f"ref_kruskal_{cfg}.npz")
        rs = float(g["ref_wall_s"])
        line.update(ref_path="Kruskal oracle path (full; recorded run, tests/golden)",
                    ref_s=rs, ref_edges_per_s=k / rs, ref_cores=1,
                    e2e_speedup=rs * 1e3 / np.median(e2e),
                    bitexact_scale=bool(
                        ns == int(g["n_scale"]) and
                        hashlib.sha256(memoryview(np.ascontiguousarray(bits(sc.array[:ns]))))
                        .digest() == g["scale_sha256"].tobytes()),
                    bitexact_bars=bool(np.array_equal(dg.array[:nf], g["death_grade"]) and
                                       np.array_equal(bits(dl.array[:nf]),
                                                      bits(g["death_length"]))),
                    essential_equal=bool(ess == int(g["essential"])))
    print(json.dumps(line), flush=True)
    for a in (xin, dg, dl, sc):
        a.free()
