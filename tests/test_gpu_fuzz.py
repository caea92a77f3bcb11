"""GPU: seeded random clouds of mixed shapes through every entry point, each against the C
oracle (oracle/ph0_oracle.c, pinned to the reference): the drop-in call, the context host
path, the multi-GPU path (virtual ranks), the reduced supports and the GPU Kruskal barcode.
Shapes mix uniform / clustered / lattice / duplicated / tiny-scale points, N across the sort
and distance tile boundaries, d in 1..20."""
import os

import numpy as np
import pytest

import oracle_bridge as ob
import paper_2203_02527_b200 as pkg

pytestmark = pytest.mark.gpu


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def cloud(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.choice([2, 3, 17, 127, 128, 129, 300, 1000, 2049, 3000]))
    d = int(rng.integers(1, 21))
    kind = seed % 6
    if kind == 0:
        X = rng.uniform(-1, 1, size=(n, d))
    elif kind == 1:
        c = rng.uniform(-10, 10, size=(5, d))
        X = c[rng.integers(0, 5, n)] + 0.1 * rng.normal(size=(n, d))
    elif kind == 2:  # integer lattice values: many exact ties
        X = rng.integers(0, 5, size=(n, d)).astype(np.float64)
    elif kind == 3:  # duplicated points
        base = rng.normal(size=(max(1, n // 4), d))
        X = base[rng.integers(0, len(base), n)]
    elif kind == 4:  # tiny scale (subnormal-adjacent lengths)
        X = rng.normal(size=(n, d)) * 1e-300
    else:  # far-apart groups
        X = rng.normal(size=(n, d)) + 1e6 * (rng.integers(0, 3, size=(n, 1)))
    return X


# PH0B_FUZZ_SEEDS widens the sweep for soak runs (profiles/fuzz_soak_r02.log)
@pytest.mark.parametrize("seed", range(int(os.environ.get("PH0B_FUZZ_SEEDS", "36"))))
def test_random_cloud_all_entry_points(seed):
    X = cloud(seed)
    n = X.shape[0]
    ref = ob.oracle_filtration_and_bars(X, reduction_limit=1000)
    bc = pkg.h0_barcode(X)
    assert bc.essential_count == ref["essential"]
    assert np.array_equal(bc.death_grade, ref["death_grade"])
    assert np.array_equal(bits(bc.death_length), bits(ref["death_length"]))
    assert np.array_equal(bits(bc.scale), bits(ref["scale"]))
    ctx = pkg.Context(0)
    dg, dl, sc = np.empty(n, np.uint64), np.empty(n), np.empty(max(len(ref["scale"]), 1))
    nf, ess, ns, _ = ctx.run_host(np.ascontiguousarray(X), dg, dl, sc, layout=pkg.ph0b.ROW_MAJOR)
    ctx.close()
    assert nf == len(ref["death_grade"]) and ess == ref["essential"]
    assert np.array_equal(dg[:nf], ref["death_grade"])
    assert np.array_equal(bits(sc[:ns]), bits(ref["scale"]))
    ranks = 2 + seed % 3
    mg = pkg.h0_barcode(X, devices=[0] * ranks)
    assert np.array_equal(mg.death_grade, ref["death_grade"])
    assert np.array_equal(bits(mg.scale), bits(ref["scale"]))
    if n >= 2:
        cols, lo, hi = pkg.reduced_supports(X)
        sp = ob.reduce_sparse(ob.filtration(X), stop_at_spanning=True)
        assert np.array_equal(cols, sp["columns"])
        assert np.array_equal(lo, sp["rows_lo"]) and np.array_equal(hi, sp["rows_hi"])
        kr = pkg.kruskal_barcode(X, return_scale=False)
        assert np.array_equal(kr.death_grade, ref["death_grade"])
    pkg.lib().ph0b_release_resources()


@pytest.mark.parametrize("kind", ["lattice3d", "dups", "tiny", "far"])
def test_bucketed_host_path_vs_device_path(kind):
    """K >= 2^26 takes the bucketed host path (partition, per-bucket sorts, packed D stream);
    the device path (one global sort) is its reference here, bit for bit."""
    import torch
    rng = np.random.default_rng(len(kind))
    n = 12000
    if kind == "lattice3d":
        X = rng.integers(0, 23, size=(n, 3)).astype(np.float64)
    elif kind == "dups":
        X = rng.normal(size=(n // 8, 5))[rng.integers(0, n // 8, n)]
    elif kind == "tiny":
        X = rng.normal(size=(n, 2)) * 1e-200
    else:
        X = rng.normal(size=(n, 4)) + 1e8 * rng.integers(0, 4, size=(n, 1))
    ctx = pkg.Context(0)
    xt = torch.from_numpy(np.asfortranarray(X).ravel(order="F").copy()).cuda()
    r = ctx.run_device(xt.data_ptr(), n, X.shape[1])
    cai = {"shape": (int(r.n_scale),), "typestr": "<i8", "data": (int(r.d_scale), False),
           "version": 3, "strides": None}
    D_dev = torch.as_tensor(type("C", (), {"__cuda_array_interface__": cai})(),
                            device="cuda").cpu().numpy().view(np.uint64).copy()
    g_dev = torch.as_tensor(type("C", (), {"__cuda_array_interface__": dict(
        cai, shape=(int(r.n_finite),), data=(int(r.d_death_grade), False))})(),
        device="cuda").cpu().numpy().view(np.uint64).copy()
    dg, dl, sc = np.empty(n, np.uint64), np.empty(n), np.empty(int(r.n_scale))
    nf, ess, ns, _ = ctx.run_host(np.asfortranarray(X), dg, dl, sc)
    ctx.close()
    assert ns == r.n_scale and nf == r.n_finite and ess == r.essential_count
    assert np.array_equal(sc.view(np.uint64), D_dev)
    assert np.array_equal(dg[:nf], g_dev)
    bc = pkg.h0_barcode(X)  # the drop-in call, also bucketed at this size
    assert np.array_equal(bc.scale.view(np.uint64), D_dev)
    assert np.array_equal(bc.death_grade, g_dev)


def edge_cloud(seed):
    """Edge shapes: a handful of coordinates (fewer distinct lengths than ranks), coordinates
    whose differences overflow (lengths of +inf), signed zeros, d beyond the TMA/register
    paths, N at the sort-tile boundaries (K = 4095/4096/4097 ... at N = 91/92)."""
    rng = np.random.default_rng(10_000 + seed)
    kind = seed % 5
    if kind == 0:  # 1..3 coordinate values
        n = int(rng.choice([40, 91, 92, 300, 1500]))
        X = rng.integers(0, 1 + seed % 3, size=(n, int(rng.integers(1, 4)))).astype(np.float64)
    elif kind == 1:  # overflow: some squared differences are +inf
        n = int(rng.choice([50, 200, 700]))
        X = rng.uniform(-1, 1, size=(n, 2)) * 1e154
        X[rng.integers(0, n, max(1, n // 10))] *= 1e154
    elif kind == 2:  # signed zeros and exact duplicates
        n = int(rng.choice([64, 129, 1000]))
        X = rng.choice([-0.0, 0.0, 1.0, -1.0], size=(n, int(rng.integers(1, 5))))
    elif kind == 3:  # high d: shared-memory / generic distance paths
        n = int(rng.choice([91, 92, 257, 1025]))
        X = rng.normal(size=(n, int(rng.integers(21, 65))))
    else:  # N around the tile sizes, mixed scales
        n = int(rng.choice([90, 91, 92, 93, 127, 128, 129, 181, 182, 2897, 2898]))
        X = rng.normal(size=(n, 3)) * 10.0 ** rng.integers(-5, 6, size=(n, 1))
    return X


@pytest.mark.parametrize("seed", range(int(os.environ.get("PH0B_FUZZ_EDGE", "20"))))
def test_edge_clouds_all_entry_points(seed):
    X = edge_cloud(seed)
    n = X.shape[0]
    ref = ob.oracle_filtration_and_bars(X, reduction_limit=1000)
    for bc in (pkg.h0_barcode(X), pkg.h0_barcode(X, devices=[0] * (2 + seed % 7))):
        assert bc.essential_count == ref["essential"]
        assert np.array_equal(bc.death_grade, ref["death_grade"])
        assert np.array_equal(bits(bc.death_length), bits(ref["death_length"]))
        assert np.array_equal(bits(bc.scale), bits(ref["scale"]))
    ctx = pkg.Context(0)
    dg, dl, sc = np.empty(n, np.uint64), np.empty(n), np.empty(max(len(ref["scale"]), 1))
    nf, ess, ns, _ = ctx.run_host(np.ascontiguousarray(X), dg, dl, sc, layout=pkg.ph0b.ROW_MAJOR)
    ctx.close()
    assert nf == len(ref["death_grade"]) and ess == ref["essential"]
    assert np.array_equal(bits(sc[:ns]), bits(ref["scale"]))
    kr = pkg.kruskal_barcode(X, return_scale=False)
    assert np.array_equal(kr.death_grade, ref["death_grade"])
    # the filtration surfaces: u-major lengths, the sorted columns with grades, claimed lows
    f = ob.filtration(X)
    assert np.array_equal(bits(pkg.pairwise_distances(X)), bits(ob.pairwise(X)))
    u, v, g, scale = pkg.build_filtration(X)
    assert np.array_equal(u, f["u"]) and np.array_equal(v, f["v"])
    assert np.array_equal(g, f["grade"]) and np.array_equal(bits(scale), bits(f["scale"]))
    if n >= 2:  # (the claimed low of a surviving column is its reduced support's high row)
        sp = ob.reduce_sparse(f, stop_at_spanning=True)
        assert np.array_equal(pkg.claimed_lows(X), sp["rows_hi"])
    pkg.lib().ph0b_release_resources()


def test_host_path_ring_geometry_switch_same_context():
    """One context, five bucketed host-path calls: the 3rd runs the other D2H ring geometry
    (the ring's slot generations restart at each change), the 5th the faster.  Every call's D
    and bars must be identical."""
    rng = np.random.default_rng(99)
    n = 12000  # K = 7.2e7 >= 2^26: the bucketed, D-streaming path
    X = rng.normal(size=(n, 3)) + 40.0 * rng.integers(0, 3, size=(n, 1))
    ctx = pkg.Context(0)
    first = None
    for _ in range(5):
        dg, dl, sc = np.empty(n, np.uint64), np.empty(n), np.empty(n * (n - 1) // 2)
        nf, ess, ns, _ = ctx.run_host(np.asfortranarray(X), dg, dl, sc)
        cur = (nf, ess, ns, dg[:nf].copy(), dl[:nf].view(np.uint64).copy(),
               sc[:ns].view(np.uint64).copy())
        if first is None:
            first = cur
        else:
            assert cur[:3] == first[:3]
            assert all(np.array_equal(a, b) for a, b in zip(cur[3:], first[3:]))
    ctx.close()
    bc = pkg.h0_barcode(X)
    assert np.array_equal(bc.scale.view(np.uint64), first[5])
    assert np.array_equal(bc.death_grade, first[3])
