"""GPU: clouds beyond N = 65536 (the reference allows N <= 2^32-1, filtration.cpp:10-11).
Above 65536 points an edge column travels through the sort as its u-major edge index
instead of u << 16 | v (colcodec.h; K < 2^32 up to N = 92682).  N = 70000, d = 2: K = 2.45e9
edges, more than C5.  No CPU reference completes this size, so the checks are the
size-independent ones: D strictly increasing and holding every sampled length, bars in
filtration order with grades pointing into D, the MST length multiset from an independent
O(N^2) Prim with the reference's exact fold, the reduced supports forming the reference's
pivot forest, and the multi-GPU path (virtual ranks) equal bit for bit."""
import numpy as np
import pytest

import oracle_bridge as ob
import paper_2203_02527_b200 as pkg

pytestmark = pytest.mark.gpu

N = 70000


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def fold_to_all(X, i):
    diff = X[:, 0] - X[i, 0]
    acc = diff * diff
    for k in range(1, X.shape[1]):
        t = X[:, k] - X[i, k]
        acc = acc + t * t
    return np.sqrt(acc)


def prim_lengths(X):
    n = X.shape[0]
    best = np.full(n, np.inf)
    used = np.zeros(n, bool)
    out = np.empty(n - 1)
    cur = 0
    used[0] = True
    for i in range(n - 1):
        np.minimum(best, fold_to_all(X, cur), out=best)
        best[used] = np.inf
        cur = int(np.argmin(best))
        out[i] = best[cur]
        used[cur] = True
    return np.sort(out)


@pytest.fixture(scope="module")
def cloud():
    pkg.lib().ph0b_release_resources()
    return ob.uniform_cloud(N, 2, 70000)  # generate_uniform_cloud (point_cloud.cpp:20-29)


@pytest.fixture(scope="module")
def barcode(cloud):
    return pkg.h0_barcode(cloud)


def test_invariants_and_mst(cloud, barcode):
    bc = barcode
    D = bc.scale
    assert len(bc.death_grade) == N - 1 and bc.essential_count == 1
    Db = bits(D)
    assert np.all(Db[1:] > Db[:-1]), "D must be strictly increasing"
    g = bc.death_grade.astype(np.int64)
    assert g.min() >= 1 and g.max() <= len(D) and np.all(np.diff(g) >= 0)
    assert np.array_equal(Db[g - 1], bits(bc.death_length))
    rng = np.random.default_rng(1)
    for i in rng.integers(0, N, size=6):
        row = np.delete(fold_to_all(cloud, int(i)), int(i))
        pos = np.searchsorted(D, row)
        assert np.array_equal(Db[pos], bits(row)), "every length must appear in D"
    assert np.array_equal(bits(np.sort(bc.death_length)), bits(prim_lengths(cloud)))


def test_reduced_supports_form_the_pivot_forest(cloud, barcode):
    """Each survivor's reduced support {lo, hi} (reduction.cpp:33-49): hi is unclaimed, i.e.
    the minimum vertex of its tree, lo lies in another tree, and the column joins them."""
    cols, lo, hi = pkg.reduced_supports(cloud)
    assert len(cols) == N - 1 and np.all(np.diff(cols.astype(np.int64)) > 0)
    parent = np.arange(N)

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    for a, c in zip(lo.tolist(), hi.tolist()):
        assert a < c
        rc, ra = find(c), find(a)
        assert rc == c, "the claimed low is the minimum vertex of its tree"
        assert ra != rc
        parent[rc] = ra  # ra < c: the merged tree keeps its minimum as the root


def test_multi_gpu_virtual_ranks(cloud, barcode):
    bc = pkg.h0_barcode(cloud, devices=[0, 0, 0, 0])
    pkg.lib().ph0b_release_resources()
    assert bc.essential_count == barcode.essential_count
    assert np.array_equal(bc.death_grade, barcode.death_grade)
    assert np.array_equal(bits(bc.death_length), bits(barcode.death_length))
    assert np.array_equal(bits(bc.scale), bits(barcode.scale))


def test_kruskal_flag_rejected_above_65536(cloud):
    with pytest.raises(pkg.Ph0bError, match="65536"):
        pkg.kruskal_barcode(cloud[:65537], return_scale=False)


def test_just_above_the_packed_limit():
    """N = 65537 (the first edge-id cloud, 1-D so it builds quickly): bars vs the MST."""
    X = ob.uniform_cloud(65537, 1, 3)
    bc = pkg.h0_barcode(X, return_scale=False)
    xs = np.sort(X[:, 0])
    assert np.array_equal(bits(np.sort(bc.death_length)), bits(np.sort(np.diff(xs))))
