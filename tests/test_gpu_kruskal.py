"""GPU Kruskal barcode (ph0b_kruskal_barcode / PH0B_FLAG_KRUSKAL):
the union-find restatement of the reference oracle (oracle.cpp:32-46) over the GPU
filtration must give the reference's bars bit for bit (acceptance.cpp:79-90: oracle
equivalence), and agree with the column-reduction path on every config where the CPU
cannot follow (C4 here; C4 and C5 against the reference itself in
test_gpu_reference_large.py)."""

import numpy as np
import pytest

import oracle_bridge as ob
import paper_2203_02527_b200 as pkg

pytestmark = pytest.mark.gpu

GOLD = np.load(ob.ROOT / "tests" / "golden" / "ref_small.npz")
CASES = sorted({k.split("/")[0] for k in GOLD.files})
BIG = np.load(ob.ROOT / "tests" / "golden" / "ref_configs.npz")


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def same(a, b):
    assert a.essential_count == b.essential_count
    assert np.array_equal(a.death_grade, b.death_grade)
    assert np.array_equal(bits(a.death_length), bits(b.death_length))


@pytest.mark.parametrize("case", CASES)
def test_kruskal_small_fixtures(case):
    X = GOLD[f"{case}/X"]
    bc = pkg.kruskal_barcode(X)
    assert bc.essential_count == int(GOLD[f"{case}/essential"])
    assert np.array_equal(bc.death_grade, GOLD[f"{case}/death_grade"].astype(np.uint64))
    assert np.array_equal(bits(bc.death_length), bits(GOLD[f"{case}/death_length"]))
    assert np.array_equal(bits(bc.scale), bits(GOLD[f"{case}/scale"]))


@pytest.mark.parametrize("name", ["C1", "C2", "C3_n2048"])
def test_kruskal_config_fixtures(name):
    cfg = name.split("_n")
    X = pkg.config_cloud(cfg[0], int(cfg[1]) if len(cfg) > 1 else None)
    bc = pkg.kruskal_barcode(X, return_scale=False)
    assert bc.essential_count == int(BIG[f"{name}/essential"])
    assert np.array_equal(bc.death_grade, BIG[f"{name}/death_grade"].astype(np.uint64))
    assert np.array_equal(bits(bc.death_length), bits(BIG[f"{name}/death_length"]))


def test_kruskal_flag_equals_entry_point_and_reduction():
    X = pkg.config_cloud("C3", 4096)
    a = pkg.kruskal_barcode(X, return_scale=False)
    b = pkg.h0_barcode(X, return_scale=False, kruskal=True)
    c = pkg.h0_barcode(X, return_scale=False)
    same(a, b)
    same(a, c)


def test_kruskal_degenerate():
    for n in (0, 1):
        bc = pkg.kruskal_barcode(np.zeros((n, 2)))
        assert len(bc.death_grade) == 0 and bc.essential_count == n
    bc = pkg.kruskal_barcode(np.zeros((7, 3)))  # coincident: (0, 0.0, grade 1) bars
    assert np.all(bc.death_grade == 1) and np.all(bc.death_length == 0.0)
    assert bc.essential_count == 1 and len(bc.death_grade) == 6


def test_kruskal_c4_equals_reduction():
    """C4 at full size (5.4e8 edges): two different algorithms on the same filtration."""
    X = pkg.config_cloud("C4")
    same(pkg.kruskal_barcode(X, return_scale=False), pkg.h0_barcode(X, return_scale=False))
