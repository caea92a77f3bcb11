"""Context-reuse soak: ONE context (and the library's cached drop-in context / multi-GPU
runners) fed a random sequence of clouds — sizes up and down, d across the distance-kernel
paths, tie-heavy and plain — through run_host, run_device, the drop-in call and the
multi-GPU call, each result against the C oracle.  Stale state between calls (buffers grown
for a larger problem, cached plans, look-back epochs, forest labels) would show here.
    python tools/soak_reuse.py [iterations]"""
import sys

import numpy as np

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import oracle_bridge as ob  # noqa: E402
import paper_2203_02527_b200 as pkg  # noqa: E402


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def main():
    import torch
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 120
    rng = np.random.default_rng(2027)
    ctx = pkg.Context(0)
    bad = 0
    for it in range(iters):
        n = int(rng.choice([2, 5, 60, 91, 92, 500, 1200, 2500, 4000, 6000]))
        d = int(rng.choice([1, 2, 3, 8, 9, 16, 33]))
        if rng.random() < 0.4:
            X = rng.integers(0, int(rng.integers(2, 9)), size=(n, d)).astype(np.float64)
        else:
            X = rng.normal(size=(n, d)) * 10.0 ** int(rng.integers(-3, 4))
        ref = ob.oracle_filtration_and_bars(X, reduction_limit=500)
        ok = True
        way = it % 4
        if way == 0:
            dg, dl, sc = np.empty(n, np.uint64), np.empty(n), np.empty(max(len(ref["scale"]), 1))
            nf, ess, ns, _ = ctx.run_host(np.ascontiguousarray(X), dg, dl, sc,
                                          layout=pkg.ph0b.ROW_MAJOR)
            ok = (nf == len(ref["death_grade"]) and ess == ref["essential"] and
                  np.array_equal(dg[:nf], ref["death_grade"]) and
                  np.array_equal(bits(sc[:ns]), bits(ref["scale"])))
        elif way == 1:
            xt = torch.from_numpy(np.asfortranarray(X).ravel(order="F").copy()).cuda()
            r = ctx.run_device(xt.data_ptr(), n, d)
            torch.cuda.synchronize()
            g = torch.as_tensor(type("C", (), {"__cuda_array_interface__": {
                "shape": (int(r.n_finite),), "typestr": "<i8",
                "data": (int(r.d_death_grade), False), "version": 3, "strides": None}})(),
                device="cuda").cpu().numpy().view(np.uint64) if r.n_finite else np.zeros(0, np.uint64)
            ok = (int(r.n_finite) == len(ref["death_grade"]) and
                  int(r.n_scale) == len(ref["scale"]) and np.array_equal(g, ref["death_grade"]))
        elif way == 2:
            bc = pkg.h0_barcode(X)
            ok = (np.array_equal(bc.death_grade, ref["death_grade"]) and
                  np.array_equal(bits(bc.scale), bits(ref["scale"])) and
                  bc.essential_count == ref["essential"])
        else:
            bc = pkg.h0_barcode(X, devices=[0] * int(rng.integers(2, 6)))
            ok = (np.array_equal(bc.death_grade, ref["death_grade"]) and
                  np.array_equal(bits(bc.scale), bits(ref["scale"])))
        if not ok:
            bad += 1
            print("MISMATCH", it, way, n, d, flush=True)
    ctx.close()
    print(f"{iters} calls, {bad} mismatches")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
