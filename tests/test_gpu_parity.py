"""GPU parity: the sm_100a pipeline through the C ABI vs the oracle and the reference's own
outputs (tests/golden, produced by oracle/_ref).  Bar: bit-exact D, bit-exact ordered bars,
identical essential count and claimed lows (integer/byte work and the exact f64 fold)."""
import hashlib
from pathlib import Path

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


def assert_same_barcode(bc, death_grade, death_length, essential, scale=None):
    assert bc.essential_count == int(essential)
    assert np.array_equal(bc.death_grade, np.asarray(death_grade, np.uint64))
    assert np.array_equal(bits(bc.death_length), bits(death_length))
    if scale is not None:
        assert len(bc.scale) == len(scale)
        assert np.array_equal(bits(bc.scale), bits(scale))


@pytest.mark.parametrize("case", CASES)
def test_small_fixtures_bit_exact(case):
    X = GOLD[f"{case}/X"]
    bc = pkg.h0_barcode(X)
    assert_same_barcode(bc, GOLD[f"{case}/death_grade"], GOLD[f"{case}/death_length"],
                        GOLD[f"{case}/essential"], GOLD[f"{case}/scale"])
    if len(X) >= 2:
        lows = pkg.claimed_lows(X)
        assert np.array_equal(lows, GOLD[f"{case}/claimed_low"])


@pytest.mark.parametrize("case", ["collinear3", "ties_1d", "lattice_8x8", "coincident",
                                  "accept_062", "accept_125", "all_same_5"])
def test_filtration_columns_match(case):
    """Column j of M = (u_j, v_j, grade_j) in filtration order (filtration.cpp:20-35)."""
    X = GOLD[f"{case}/X"]
    u, v, g, scale = pkg.build_filtration(X)
    f = ob.filtration(X)
    assert np.array_equal(u, f["u"]) and np.array_equal(v, f["v"])
    assert np.array_equal(g, f["grade"])
    assert np.array_equal(bits(scale), bits(f["scale"]))


def test_pairwise_distances_bitwise():
    rng = np.random.default_rng(11)
    for n, d in ((257, 1), (300, 2), (300, 3), (129, 4), (200, 5), (256, 8), (130, 16),
                 (70, 33), (64, 40)):
        X = rng.normal(size=(n, d)) * 3.7
        got = pkg.pairwise_distances(X)
        assert np.array_equal(bits(got), bits(ob.pairwise(X))), (n, d)


@pytest.mark.parametrize("name", ["C1", "C2", "C3_n2048"])
def test_config_fixtures(name):
    """BASELINE configs C1, C2 and a C3 prefix vs the reference's own full pipeline."""
    cfg = name.split("_n")
    X = pkg.config_cloud(cfg[0], int(cfg[1]) if len(cfg) > 1 else None)
    assert hashlib.sha256(np.asfortranarray(X).tobytes()).digest() == BIG[f"{name}/X_sha256"].tobytes()
    bc = pkg.h0_barcode(X)
    assert len(bc.scale) == int(BIG[f"{name}/n_scale"])
    assert hashlib.sha256(bc.scale.tobytes()).digest() == BIG[f"{name}/scale_sha256"].tobytes()
    assert_same_barcode(bc, BIG[f"{name}/death_grade"], BIG[f"{name}/death_length"],
                        BIG[f"{name}/essential"])
    assert np.array_equal(pkg.claimed_lows(X), BIG[f"{name}/claimed_low"])


def test_c3_full_vs_oracle():
    """C3 (N=8192, d=16, ~3.4e7 edges): D and ordered bars vs the C oracle (Kruskal path)."""
    X = pkg.config_cloud("C3")
    bc = pkg.h0_barcode(X)
    ref = ob.oracle_filtration_and_bars(X)
    assert_same_barcode(bc, ref["death_grade"], ref["death_length"], ref["essential"],
                        ref["scale"])


def test_duplicate_heavy_lattice():
    """A 48x48 integer lattice: massive exact ties in D and in the MST (tie order by (u,v))."""
    g = np.array([[x, y] for x in range(48) for y in range(48)], np.float64)
    bc = pkg.h0_barcode(g)
    ref = ob.oracle_filtration_and_bars(g)
    assert_same_barcode(bc, ref["death_grade"], ref["death_length"], ref["essential"], ref["scale"])
    assert np.array_equal(pkg.claimed_lows(g), ob.reduce_bars(ob.filtration(g))["claimed_low"])


def test_degenerate_sizes():  # acceptance.cpp:98-102, test_reduction.cpp:147-157
    for n, ess in ((0, 0), (1, 1)):
        bc = pkg.h0_barcode(np.zeros((n, 2)))
        assert len(bc.death_grade) == 0 and bc.essential_count == ess and len(bc.scale) == 0
    bc = pkg.h0_barcode(np.array([[0.0, 0.0], [3.0, 4.0]]))
    assert list(bc.death_grade) == [1] and list(bc.death_length) == [5.0]


def test_all_coincident_and_zero_dim():
    bc = pkg.h0_barcode(np.full((300, 3), 0.25))
    assert list(bc.scale) == [0.0] and bc.essential_count == 1
    assert np.all(bc.death_grade == 1) and np.all(bc.death_length == 0.0)
    bc0 = pkg.h0_barcode(np.zeros((5, 0)))
    ref0 = ob.oracle_filtration_and_bars(np.zeros((5, 0)))
    assert_same_barcode(bc0, ref0["death_grade"], ref0["death_length"], ref0["essential"],
                        ref0["scale"])


def test_extreme_magnitudes():
    """Overflow to +inf lengths, subnormal lengths, mixed signs."""
    X = np.array([[1e300, 0.0], [-1e300, 1.0], [0.0, 5e-324], [0.0, 0.0], [1e-310, 2e-310],
                  [3.0, -7.5]])
    bc = pkg.h0_barcode(X)
    ref = ob.oracle_filtration_and_bars(X)
    assert_same_barcode(bc, ref["death_grade"], ref["death_length"], ref["essential"], ref["scale"])


def test_random_sizes_sweep():
    """Ragged sizes around tile (128) and sort-tile (4096) boundaries, d in 1..9."""
    rng = np.random.default_rng(2024)
    for n in (3, 127, 128, 129, 255, 256, 257, 91, 92, 1000):
        d = int(rng.integers(1, 10))
        X = rng.uniform(-2, 2, size=(n, d))
        bc = pkg.h0_barcode(X)
        ref = ob.oracle_filtration_and_bars(X)
        assert_same_barcode(bc, ref["death_grade"], ref["death_length"], ref["essential"],
                            ref["scale"])


@pytest.mark.parametrize("d", [5, 6, 7, 12, 17, 24, 31, 32, 33, 40, 64])
def test_dimension_paths(d):
    """Every distance-kernel path: d in {1,2,3,4,8,16} specialised (other tests), other d <= 32
    through the runtime-d TMA kernel, d > 32 through the global-memory kernel — same fold
    order, bit-exact D and bars."""
    rng = np.random.default_rng(100 + d)
    n = 300 + 7 * d
    X = np.concatenate([rng.normal(0, 1, size=(n // 2, d)),
                        rng.normal(4, 0.5, size=(n - n // 2, d))])
    bc = pkg.h0_barcode(X)
    ref = ob.oracle_filtration_and_bars(X)
    assert_same_barcode(bc, ref["death_grade"], ref["death_length"], ref["essential"],
                        ref["scale"])


def test_quantized_ties_medium():
    """Coordinates on a coarse grid (many equal lengths), N=3000: ties across sort tiles."""
    rng = np.random.default_rng(5)
    X = rng.integers(0, 20, size=(3000, 3)).astype(np.float64)
    bc = pkg.h0_barcode(X)
    ref = ob.oracle_filtration_and_bars(X)
    assert_same_barcode(bc, ref["death_grade"], ref["death_length"], ref["essential"], ref["scale"])


def test_device_context_run_matches_host_api():
    torch = pytest.importorskip("torch")
    X = pkg.config_cloud("C2")
    bc = pkg.h0_barcode(X)
    ctx = pkg.Context(0)
    xt = torch.from_numpy(np.asfortranarray(X).ravel(order="F").copy()).cuda()
    r = ctx.run_device(xt.data_ptr(), X.shape[0], X.shape[1])
    assert r.n_finite == len(bc.death_grade) and r.n_scale == len(bc.scale)
    assert r.essential_count == 1
    # row-major host input through the context (workspace reuse must not matter)
    dg = np.empty(X.shape[0], np.uint64)
    dl = np.empty(X.shape[0])
    sc = np.empty(len(bc.scale))
    nf, ess, ns, t = ctx.run_host(np.ascontiguousarray(X), dg, dl, sc,
                                  layout=pkg.ph0b.ROW_MAJOR)
    assert nf == len(bc.death_grade) and ess == 1 and ns == len(bc.scale)
    assert np.array_equal(dg[:nf], bc.death_grade)
    assert np.array_equal(bits(dl[:nf]), bits(bc.death_length))
    assert np.array_equal(bits(sc), bits(bc.scale))
    ctx.close()


def c_fold_lengths_to_all(X, i):
    """Lengths from point i to all points with the reference's exact sequential fold."""
    diff = X[:, 0] - X[i, 0]
    acc = diff * diff
    for k in range(1, X.shape[1]):
        t = X[:, k] - X[i, k]
        acc = acc + t * t
    return np.sqrt(acc)


def prim_mst_lengths(X):
    n = X.shape[0]
    best = np.full(n, np.inf)
    used = np.zeros(n, bool)
    out = []
    cur = 0
    used[0] = True
    for _ in range(n - 1):
        best = np.minimum(best, c_fold_lengths_to_all(X, cur))
        best[used] = np.inf
        cur = int(np.argmin(best))
        out.append(best[cur])
        used[cur] = True
    return np.sort(np.array(out))


def check_large(X, bc):
    n = X.shape[0]
    D = bc.scale
    assert len(bc.death_grade) == n - 1 and bc.essential_count == 1
    assert np.all(bits(D)[1:] > bits(D)[:-1]), "D must be strictly increasing"
    g = bc.death_grade.astype(np.int64)
    assert g.min() >= 1 and g.max() <= len(D)
    assert np.array_equal(bits(D[g - 1]), bits(bc.death_length))
    assert np.all(np.diff(g) >= 0), "bars must come in filtration order"
    rng = np.random.default_rng(0)
    for i in rng.integers(0, n, size=8):
        row = np.delete(c_fold_lengths_to_all(X, int(i)), int(i))
        pos = np.searchsorted(D, row)
        assert np.array_equal(bits(D[pos]), bits(row)), "every length must appear in D"
    assert np.array_equal(bits(np.sort(bc.death_length)), bits(prim_mst_lengths(X)))


def test_c4_full_size_properties():
    """C4 at full size (N=32768, ~5.4e8 edges): size-independent invariants + the MST length
    multiset from an independent O(N^2) Prim in numpy with the reference's exact fold (the
    bit-exact comparison with the reference itself is in test_gpu_reference_large.py)."""
    X = pkg.config_cloud("C4")
    bc = pkg.h0_barcode(X)
    check_large(X, bc)


def test_overlapped_host_path_matches_device_path():
    """ph0b_run_host on a large cloud takes the bucketed path whose D2H of D overlaps the sort
    (16 key-range buckets, padded segments, per-bucket D slices); it must equal the plain
    path bit for bit (run with PH0B_OVERLAP=0 semantics via the device-result API)."""
    torch = pytest.importorskip("torch")
    X = pkg.config_cloud("C4", 12000)  # K = 7.2e7 >= 2^26: takes the overlapped path
    n, d = X.shape
    ctx = pkg.Context(0)
    xt = torch.from_numpy(np.asfortranarray(X).ravel(order="F").copy()).cuda()
    r = ctx.run_device(xt.data_ptr(), n, d)
    dev_scale = torch.empty(r.n_scale, dtype=torch.float64, device="cuda")
    src = torch.as_tensor(type("C", (), {"__cuda_array_interface__": {
        "shape": (r.n_scale,), "typestr": "<f8", "data": (r.d_scale, False), "version": 3,
        "strides": None}})(), device="cuda")
    dev_scale.copy_(src)
    D_dev = dev_scale.cpu().numpy()
    dg = np.empty(n, np.uint64)
    dl = np.empty(n)
    sc = np.empty(r.n_scale)
    nf, ess, ns, t = ctx.run_host(np.asfortranarray(X), dg, dl, sc)
    assert ns == r.n_scale and nf == n - 1 and ess == 1
    assert np.array_equal(bits(sc), bits(D_dev))
    bc = pkg.h0_barcode(X)  # library-allocated path (not overlapped)
    assert np.array_equal(dg[:nf], bc.death_grade)
    assert np.array_equal(bits(dl[:nf]), bits(bc.death_length))
    assert np.array_equal(bits(sc), bits(bc.scale))
    ctx.close()


def test_overlapped_host_path_separated_clusters():
    """Far-apart clusters: the forest is still disconnected when late buckets are reduced, so
    every padding slot between bucket segments of M is reached by the reduction — they must
    hold the cycle column {0, 0} in whichever buffer M ends up (regression: stale u-major
    columns there produced wrong bars)."""
    rng = np.random.default_rng(5)
    centres = np.array([[0, 0, 0], [100, 0, 0], [0, 100, 0], [0, 0, 100]], np.float64)
    X = np.concatenate([c + rng.normal(size=(3000, 3)) for c in centres])  # N=12000, K>=2^26
    n, d = X.shape
    ctx = pkg.Context(0)
    dg = np.empty(n, np.uint64)
    dl = np.empty(n)
    sc = np.empty(n * (n - 1) // 2)
    nf, ess, ns, t = ctx.run_host(np.asfortranarray(X), dg, dl, sc)
    bc = pkg.h0_barcode(X)
    assert nf == n - 1 and ess == 1 and ns == len(bc.scale)
    assert np.array_equal(dg[:nf], bc.death_grade)
    assert np.array_equal(bits(dl[:nf]), bits(bc.death_length))
    assert np.array_equal(bits(sc[:ns]), bits(bc.scale))
    ctx.close()


@pytest.mark.parametrize("kind", ["identical", "lattice", "line", "two_far"])
def test_pathological_large(kind):
    """~1.3e8 edges with massive ties / a zero span / duplicate lengths: exercises the
    zero-pass plan, the equal-prefix redo (runs longer than the fix-up limit) and the
    overlapped host path at scale; checked by size-independent invariants, the MST length
    multiset (Prim with the reference's fold) and the GPU Kruskal oracle."""
    n = 16384
    if kind == "identical":
        X = np.full((n, 3), 0.25)
    elif kind == "lattice":
        X = np.array([[x, y] for x in range(128) for y in range(128)], np.float64)
    elif kind == "line":
        X = np.arange(n, dtype=np.float64)[:, None] % 1000.0
    else:
        rng = np.random.default_rng(3)
        X = rng.normal(size=(n, 4))
        X[: n // 2] += 1e6
    bc = pkg.h0_barcode(X)
    check_large(X, bc)
    kr = pkg.kruskal_barcode(X, return_scale=False)
    assert np.array_equal(kr.death_grade, bc.death_grade)
    assert np.array_equal(bits(kr.death_length), bits(bc.death_length))
    ctx = pkg.Context(0)
    dg = np.empty(n, np.uint64)
    dl = np.empty(n)
    sc = np.empty(len(bc.scale))
    nf, ess, ns, t = ctx.run_host(np.asfortranarray(X), dg, dl, sc)  # overlapped (K >= 2^26)
    assert nf == n - 1 and ess == 1 and ns == len(bc.scale)
    assert np.array_equal(dg[:nf], bc.death_grade)
    assert np.array_equal(bits(dl[:nf]), bits(bc.death_length))
    assert np.array_equal(bits(sc), bits(bc.scale))
    ctx.close()


@pytest.mark.parametrize("cfg", ["C2", "C3", "C4"])
def test_scale_to_host_matches_device_d(cfg):
    """ph0b_scale_to_host (a device D -> host, compressed through the ring above 2^21 values,
    plain copy below; used for the sharded ranks' slices) reproduces the device D bit for
    bit, including raw (>= 2^32 gap) chunks (C3 is mostly raw)."""
    import ctypes as C
    torch = pytest.importorskip("torch")
    X = pkg.config_cloud(cfg)
    n, d = X.shape
    ctx = pkg.Context(0)
    xt = torch.from_numpy(np.asfortranarray(X).ravel(order="F").copy()).cuda()
    r = ctx.run_device(xt.data_ptr(), n, d)
    dev = torch.as_tensor(type("C", (), {"__cuda_array_interface__": {
        "shape": (r.n_scale,), "typestr": "<i8", "data": (r.d_scale, False), "version": 3,
        "strides": None}})(), device="cuda").cpu().numpy()
    out = pkg.PinnedArray(r.n_scale + 3)
    out.array[:] = -1.0
    moved = C.c_uint64()
    L = pkg.lib()
    L.ph0b_scale_to_host.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64,
                                     C.c_void_p, C.POINTER(C.c_uint64)]
    rc = L.ph0b_scale_to_host(ctx._h, C.c_void_p(r.d_scale), r.n_scale,
                              C.c_void_p(out.array.ctypes.data), out.array.size, None,
                              C.byref(moved))
    assert rc == 0
    assert np.array_equal(out.array[:r.n_scale].view(np.int64), dev)
    assert np.all(out.array[r.n_scale:] == -1.0)
    assert 0 < moved.value <= r.n_scale * 8 + (r.n_scale // 1024 + 1) * 13
    out.free()
    ctx.close()


def test_lattice128_claimed_lows_and_supports():
    """128 x 128 lattice (K = 1.34e8, ties spanning thousands of sort tiles): claimed lows and
    the survivors' reduced supports against the C oracle's sparse reduction
    (tests/golden/make_golden_lattice.py) — they depend on the (u, v) order inside each tie
    group, so an unstable in-warp rank (ATOMS lane order) would show here."""
    G = np.load(Path(__file__).resolve().parent / "golden" / "lattice128_supports.npz")
    X = np.array([[x, y] for x in range(128) for y in range(128)], np.float64)
    assert np.array_equal(pkg.claimed_lows(X), G["rows_hi"])
    cols, lo, hi = pkg.reduced_supports(X)
    assert np.array_equal(cols, G["columns"])
    assert np.array_equal(lo, G["rows_lo"]) and np.array_equal(hi, G["rows_hi"])
    bc = pkg.h0_barcode(X)
    assert np.array_equal(bc.death_grade, G["death_grade"])
    assert len(bc.scale) == int(G["n_scale"])
