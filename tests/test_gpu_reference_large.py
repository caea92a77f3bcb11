"""GPU parity at the FULL-size configs C4 (N=32768, d=3, 5.4e8 edges) and C5 (N=65536, d=8,
2.1e9 edges — the bench config) against the REFERENCE ITSELF: goldens written by
tests/golden/make_golden_large.py from oracle/_ref (the unmodified reference sources), run
through the reference's Kruskal path (`ph0 oracle`, proj/tools/ph0_cli.cpp:73-80 ->
kruskal_barcode, proj/src/oracle.cpp:32-46), which yields the identical D and ordered
barcode as its reduce path (acceptance.cpp:79-90) and is the only one of its two paths that
fits one host's memory at these sizes.

Bar: |D| equal, sha256 of D's bit patterns equal, the ordered death grades equal, the death
lengths equal as f64 bit patterns, the essential count equal — through the drop-in entry
point (ph0b_h0_barcode), the e2e host path the bench times (ph0b_run_host), and the GPU
Kruskal entry point (ph0b_kruskal_barcode)."""
import hashlib

import numpy as np
import pytest

import oracle_bridge as ob
import paper_2203_02527_b200 as pkg

pytestmark = pytest.mark.gpu

GOLDEN = ob.ROOT / "tests" / "golden"


def golden(cfg):
    p = GOLDEN / f"ref_kruskal_{cfg}.npz"
    assert p.exists(), f"missing reference golden {p.name} (tests/golden/make_golden_large.py)"
    return np.load(p)


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def check_against(g, D, death_grade, death_length, essential):
    assert len(D) == int(g["n_scale"])
    Db = bits(D)
    assert np.array_equal(Db[:64], bits(g["scale_head"]))
    assert np.array_equal(Db[-64:], bits(g["scale_tail"]))
    assert hashlib.sha256(memoryview(np.ascontiguousarray(Db))).digest() == \
        g["scale_sha256"].tobytes(), "D differs from the reference"
    assert int(essential) == int(g["essential"])
    assert np.array_equal(np.asarray(death_grade, np.uint64), g["death_grade"])
    assert np.array_equal(bits(death_length), bits(g["death_length"]))


def cloud(cfg, g):
    X = pkg.config_cloud(cfg)
    assert X.shape == (int(g["n"]), int(g["d"]))
    assert hashlib.sha256(np.asfortranarray(X).tobytes()).digest() == g["X_sha256"].tobytes()
    return X


@pytest.mark.parametrize("cfg", ["C4", "C5"])
def test_dropin_entry_point_vs_reference(cfg):
    """ph0b_h0_barcode (library-allocated D) == the reference at full size."""
    g = golden(cfg)
    X = cloud(cfg, g)
    bc = pkg.h0_barcode(X)
    check_against(g, bc.scale, bc.death_grade, bc.death_length, bc.essential_count)


@pytest.mark.parametrize("cfg", ["C4", "C5"])
def test_host_path_vs_reference(cfg):
    """ph0b_run_host — the bucketed, overlapped path the bench's e2e number times (D shipped
    delta-encoded through the pinned ring) — == the reference at full size."""
    g = golden(cfg)
    X = cloud(cfg, g)
    n, d = X.shape
    ctx = pkg.Context(0)
    xin = pkg.PinnedArray(n * d)
    xin.array[:] = np.asfortranarray(X).ravel(order="F")
    dg = pkg.PinnedArray(n, np.uint64)
    dl = pkg.PinnedArray(n, np.float64)
    sc = pkg.PinnedArray(int(g["n_scale"]), np.float64)
    try:
        nf, ess, ns, _t = ctx.run_host(xin.array.reshape(d, n).T, dg.array, dl.array, sc.array)
        assert nf == n - 1 and ns == int(g["n_scale"])
        check_against(g, sc.array[:ns], dg.array[:nf], dl.array[:nf], ess)
    finally:
        for a in (xin, dg, dl, sc):
            a.free()
        ctx.close()


@pytest.mark.parametrize("cfg", ["C4", "C5"])
def test_gpu_kruskal_vs_reference(cfg):
    """ph0b_kruskal_barcode (the GPU union-find over the GPU filtration) == the reference's
    own Kruskal path: an independent second computation of the bars at full size."""
    g = golden(cfg)
    X = cloud(cfg, g)
    kr = pkg.kruskal_barcode(X, return_scale=False)
    assert kr.essential_count == int(g["essential"])
    assert np.array_equal(kr.death_grade, g["death_grade"])
    assert np.array_equal(bits(kr.death_length), bits(g["death_length"]))


def test_golden_provenance():
    """The goldens record where and how long the reference ran (no GPU needed to read)."""
    for cfg in ("C4", "C5"):
        g = golden(cfg)
        k = int(g["n"]) * (int(g["n"]) - 1) // 2
        assert int(g["k"]) == k
        assert float(g["ref_wall_s"]) > 0 and int(g["host_nproc"]) > 0
        assert len(g["death_grade"]) == int(g["n"]) - 1
