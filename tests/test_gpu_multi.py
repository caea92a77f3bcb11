"""GPU: the in-process multi-GPU path behind the drop-in entry point (ph0b_options.n_gpus /
devices, csrc/multi.cpp): row blocks for the distances, a splitter partition whose kernel
stores each part into its destination's receive buffer, local sort/unique, the column
reduction continuing the forest from key range to key range, D slices shipped per rank.
This box has one B200, so the ranks are virtual (the device list repeats ordinal 0); the
results must equal the single-GPU path bit for bit, and at C4 and C5 the reference itself
(tests/golden/ref_kruskal_C*.npz)."""
import hashlib

import numpy as np
import pytest

import oracle_bridge as ob
import paper_2203_02527_b200 as pkg

pytestmark = pytest.mark.gpu


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def same(a, b):
    assert a.essential_count == b.essential_count
    assert np.array_equal(a.death_grade, b.death_grade)
    assert np.array_equal(bits(a.death_length), bits(b.death_length))
    assert len(a.scale) == len(b.scale)
    assert np.array_equal(bits(a.scale), bits(b.scale))


@pytest.mark.parametrize("ranks", [2, 3, 4, 8])
def test_virtual_ranks_equal_single_gpu(ranks):
    rng = np.random.default_rng(ranks)
    clouds = [pkg.config_cloud("C2"), pkg.config_cloud("C3", 3000),
              rng.uniform(0, 1, size=(2500, 3)),
              np.array([[x, y] for x in range(50) for y in range(50)], np.float64),
              rng.integers(0, 8, size=(1500, 2)).astype(np.float64)]  # heavy exact ties
    for X in clouds:
        same(pkg.h0_barcode(X, devices=[0] * ranks), pkg.h0_barcode(X))


def test_far_clusters_forest_continues_across_ranges():
    """Clusters far apart: the spanning forest is completed only by the last key ranges, so
    the reduction must continue the forest rank after rank."""
    rng = np.random.default_rng(7)
    centres = np.array([[0, 0, 0], [100, 0, 0], [0, 300, 0], [0, 0, 1000]], np.float64)
    X = np.concatenate([c + rng.normal(size=(700, 3)) for c in centres])
    for ranks in (2, 4, 8):
        same(pkg.h0_barcode(X, devices=[0] * ranks), pkg.h0_barcode(X))
    ref = ob.oracle_filtration_and_bars(X)
    bc = pkg.h0_barcode(X, devices=[0] * 4)
    assert np.array_equal(bc.death_grade, ref["death_grade"])
    assert np.array_equal(bits(bc.scale), bits(ref["scale"]))


@pytest.mark.parametrize("values,ranks", [(5, 4), (5, 8), (2, 3), (3, 8)])
def test_fewer_lengths_than_ranks(values, ranks):
    """A 1-D lattice with a handful of coordinates has fewer distinct lengths than ranks, so
    some key ranges are empty (the splitters coincide); the forest must continue from the
    last rank that reduced, not from an empty neighbour (fuzz seed 416 found this)."""
    rng = np.random.default_rng(values * 10 + ranks)
    for n in (300, 1000):
        X = rng.integers(0, values, size=(n, 1)).astype(np.float64)
        ref = ob.oracle_filtration_and_bars(X)
        bc = pkg.h0_barcode(X, devices=[0] * ranks)
        assert bc.essential_count == ref["essential"]
        assert np.array_equal(bc.death_grade, ref["death_grade"])
        assert np.array_equal(bits(bc.death_length), bits(ref["death_length"]))
        assert np.array_equal(bits(bc.scale), bits(ref["scale"]))


def test_small_clouds_take_single_gpu_path():
    for n in (0, 1, 2, 5, 40):
        X = np.random.default_rng(n).normal(size=(n, 2))
        same(pkg.h0_barcode(X, devices=[0, 0]), pkg.h0_barcode(X))


@pytest.mark.parametrize("cfg,ranks", [("C4", 2), ("C4", 8), ("C5", 2), ("C5", 4), ("C5", 8)])
def test_multi_vs_reference_full_size(cfg, ranks):
    g = np.load(ob.ROOT / "tests" / "golden" / f"ref_kruskal_{cfg}.npz")
    X = pkg.config_cloud(cfg)
    bc = pkg.h0_barcode(X, devices=[0] * ranks)
    assert len(bc.scale) == int(g["n_scale"])
    assert hashlib.sha256(memoryview(np.ascontiguousarray(bits(bc.scale)))).digest() == \
        g["scale_sha256"].tobytes()
    assert bc.essential_count == int(g["essential"])
    assert np.array_equal(bc.death_grade, g["death_grade"])
    assert np.array_equal(bits(bc.death_length), bits(g["death_length"]))


@pytest.fixture(autouse=True)
def _release_runners():
    yield
    pkg.lib().ph0b_release_resources()  # the virtual ranks' buffers (C5: ~50 GB per list)


def _into(X, devices, capacity):
    import ctypes as C
    from paper_2203_02527_b200 import ph0b
    Xf = np.asfortranarray(X)
    n, d = X.shape
    opt = ph0b._opts(0, 0, 1, True, devices)
    dg = np.empty(n, np.uint64)
    dl = np.empty(n)
    sc = np.empty(max(capacity, 1))
    nf, ess, ns = C.c_uint64(), C.c_uint64(), C.c_uint64()
    rc = pkg.lib().ph0b_h0_barcode_into(C.c_void_p(Xf.ctypes.data), n, d, ph0b.COL_MAJOR,
                                        C.byref(opt), C.c_void_p(dg.ctypes.data),
                                        C.c_void_p(dl.ctypes.data), C.byref(nf), C.byref(ess),
                                        C.c_void_p(sc.ctypes.data), capacity, C.byref(ns), None)
    return rc, pkg.lib().ph0b_last_error().decode(), ns.value, sc


def test_multi_into_capacity_and_bad_device():
    from paper_2203_02527_b200 import ph0b
    X = np.random.default_rng(4).normal(size=(3000, 3))
    ref = pkg.h0_barcode(X)
    rc, msg, ns, sc = _into(X, [0, 0, 0], len(ref.scale))
    assert rc == 0 and ns == len(ref.scale)
    assert np.array_equal(sc[:ns].view(np.uint64), ref.scale.view(np.uint64))
    rc, msg, _, _ = _into(X, [0, 0, 0], len(ref.scale) - 1)
    assert rc == ph0b.PH0B_ERR_CAPACITY and "too small" in msg
    import torch
    bad = torch.cuda.device_count() + 3
    rc, msg, _, _ = _into(X, [0, bad], len(ref.scale))
    assert rc != 0 and msg
