"""GPU: the whole reduced matrix and the reference's option
equivalences, as its acceptance suite checks them (/root/reference/proj/tests/
acceptance.cpp:106-133, test_reduction.cpp:213-255):
  * every surviving column's reduced support {rows_lo, rows_hi = claimed low} and column
    index, in filtration order, equal the reference's reduced matrices (tests/golden/
    ref_reduced.npz, written by oracle/_ref) on its 200 acceptance clouds and the 50
    parallel-determinism clouds (all other columns end empty on both sides);
  * ReductionOptions are result-neutral: workers in {2,3,4,6} and pivoting off give the same
    reduced matrix and barcode (parallel_determinism, pivoting_equivalence);
  * a 96 x 96 integer lattice (9216 points, 4.2e7 edges, ~10^4 sort tiles, massive exact
    ties): the reduced supports equal the literal sparse-column reduction of the C oracle
    — tie order across sort tiles decides which columns survive and what they claim."""
import numpy as np
import pytest

import oracle_bridge as ob
import paper_2203_02527_b200 as pkg

pytestmark = pytest.mark.gpu

RED = np.load(ob.ROOT / "tests" / "golden" / "ref_reduced.npz")
CLOUDS = sorted({k.split("/")[0] for k in RED.files})
ACCEPT = [c for c in CLOUDS if c.startswith("accept_")]
PARDET = [c for c in CLOUDS if c.startswith("pardet_")]


def same_matrix(got, name):
    cols, lo, hi = got
    assert np.array_equal(cols, RED[f"{name}/columns"]), name
    assert np.array_equal(lo, RED[f"{name}/rows_lo"]), name
    assert np.array_equal(hi, RED[f"{name}/rows_hi"]), name


def test_reduced_matrices_vs_reference():
    for name in CLOUDS:
        X = RED[f"{name}/X"]
        got = pkg.reduced_supports(X)
        same_matrix(got, name)
        assert np.array_equal(pkg.claimed_lows(X), RED[f"{name}/rows_hi"]), name


@pytest.mark.parametrize("workers", [2, 3, 4, 6])
def test_parallel_determinism(workers):  # acceptance.cpp:106-122
    for name in PARDET:
        X = RED[f"{name}/X"]
        same_matrix(pkg.reduced_supports(X, workers=workers), name)
        same_matrix(pkg.reduced_supports(X, workers=workers, pivoting=False), name)


def test_pivoting_equivalence():  # acceptance.cpp:124-133, test_reduction.cpp:213-227
    for name in ACCEPT:
        X = RED[f"{name}/X"]
        on = pkg.h0_barcode(X, pivoting=True)
        off = pkg.h0_barcode(X, pivoting=False)
        assert np.array_equal(on.death_grade, off.death_grade), name
        assert np.array_equal(on.death_length.view(np.uint64), off.death_length.view(np.uint64))
        same_matrix(pkg.reduced_supports(X, pivoting=False), name)


def test_workers_zero_rejected():  # reduction.cpp:134
    with pytest.raises(pkg.InvalidArgument, match="worker count must be at least 1"):
        pkg.h0_barcode(RED[f"{ACCEPT[5]}/X"], workers=0)


def test_lattice_reduced_supports_across_many_sort_tiles():
    g = np.array([[x, y] for x in range(96) for y in range(96)], np.float64)
    f = ob.filtration(g)
    ref = ob.reduce_sparse(f, stop_at_spanning=True)
    cols, lo, hi = pkg.reduced_supports(g)
    assert np.array_equal(cols, ref["columns"])
    assert np.array_equal(lo, ref["rows_lo"])
    assert np.array_equal(hi, ref["rows_hi"])
    bc = pkg.h0_barcode(g)
    assert np.array_equal(bc.death_grade, ref["death_grade"])
    assert np.array_equal(bc.scale.view(np.uint64), f["scale"].view(np.uint64))


@pytest.mark.parametrize("name", ["C1", "C2", "C3_n2048"])
def test_config_reduced_supports_vs_oracle(name):
    """The BASELINE configs' reduced matrices: the claimed lows against the reference's own
    (tests/golden/ref_configs.npz), the whole supports against the sparse literal reduction."""
    big = np.load(ob.ROOT / "tests" / "golden" / "ref_configs.npz")
    cfg, _, n = name.partition("_n")
    X = pkg.config_cloud(cfg, int(n) if n else None)
    cols, lo, hi = pkg.reduced_supports(X)
    assert np.array_equal(hi, big[f"{name}/claimed_low"])
    ref = ob.reduce_sparse(ob.filtration(X), stop_at_spanning=True)
    assert np.array_equal(cols, ref["columns"]) and np.array_equal(lo, ref["rows_lo"])
