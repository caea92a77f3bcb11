import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import oracle_bridge as ob
import paper_2203_02527_b200 as pkg
def bits(a): return np.asarray(a, np.float64).view(np.uint64)
fails = 0
for seed in range(24):
    rng = np.random.default_rng(seed)
    n = int(rng.choice([11600, 12000, 16000]))
    kind = seed % 4
    if kind == 0: X = rng.integers(0, 3, size=(n, 1)).astype(np.float64)
    elif kind == 1: X = rng.integers(0, 2, size=(n, 2)).astype(np.float64)
    elif kind == 2: X = rng.integers(0, 40, size=(n, 2)).astype(np.float64)
    else: X = np.repeat(rng.normal(size=(n // 50, 3)), 50, axis=0)
    base = pkg.h0_barcode(X)  # bucketed host path at this K
    ctx = pkg.Context(0)
    import torch
    xt = torch.from_numpy(np.asfortranarray(X).ravel(order="F").copy()).cuda()
    r = ctx.run_device(xt.data_ptr(), n, X.shape[1])
    nf_dev, ns_dev = int(r.n_finite), int(r.n_scale)
    ctx.close()
    outs = [("multi%d" % k, pkg.h0_barcode(X, devices=[0] * k)) for k in (2, 3, 5, 8)]
    ok = base.scale.size == ns_dev and len(base.death_grade) == nf_dev
    for name, o in outs:
        ok = ok and np.array_equal(o.death_grade, base.death_grade) and np.array_equal(bits(o.scale), bits(base.scale))
    kr = pkg.kruskal_barcode(X, return_scale=False)
    ok = ok and np.array_equal(kr.death_grade, base.death_grade)
    # small-N oracle check on a subsample-free invariant: D strictly increasing, bars count
    ok = ok and np.all(np.diff(bits(base.scale).astype(np.int64)) > 0) and base.essential_count + len(base.death_grade) == n
    print(seed, n, X.shape[1], kind, len(base.scale), "OK" if ok else "MISMATCH", flush=True)
    fails += not ok
    pkg.lib().ph0b_release_resources()
print("fails", fails)
