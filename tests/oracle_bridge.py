"""TEST INFRASTRUCTURE — ctypes bridge to the CPU oracles (never used by the product path).

* oracle/_build/libph0oracle.so : plain-C restatement of the reference hot path
  (oracle/ph0_oracle.c, each function citing /root/reference/proj file:line), pinned
  against the reference's golden vectors and its shim-built sources.
* oracle/_ref/libph0ref.so      : the reference's own unmodified sources compiled here
  (oracle/Makefile); optional — present when it was built in the build container.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_SO = ROOT / "oracle" / "_build" / "libph0oracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libph0ref.so"
_orc = None
_ref = None

vp, u64, u32 = C.c_void_p, C.c_uint64, C.c_uint32


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else None


def orc() -> C.CDLL:
    global _orc
    if _orc is None:
        if not ORACLE_SO.exists():
            subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "oracle"], check=True)
        L = C.CDLL(str(ORACLE_SO))
        L.orc_mix64.restype = u64
        L.orc_mix64.argtypes = [u64]
        L.orc_splitmix_next.restype = u64
        L.orc_splitmix_next.argtypes = [C.POINTER(u64)]
        L.orc_next_unit_open.restype = C.c_double
        L.orc_next_unit_open.argtypes = [C.POINTER(u64)]
        L.orc_generate_uniform_cloud.restype = C.c_int
        L.orc_generate_uniform_cloud.argtypes = [u64, u64, u64, vp]
        L.orc_pairwise_distances.restype = None
        L.orc_pairwise_distances.argtypes = [vp, u64, u64, vp]
        L.orc_build_filtration.restype = u64
        L.orc_build_filtration.argtypes = [vp, u64, u64, vp, vp, vp, vp, vp]
        L.orc_reduce_barcode.restype = C.c_int64
        L.orc_reduce_barcode.argtypes = [u64, u64, vp, vp, vp, vp, u64, vp, vp, vp,
                                         C.POINTER(u64), C.POINTER(u64)]
        L.orc_generate_cloud.restype = C.c_int
        L.orc_generate_cloud.argtypes = [u32, u64, u64, u64, u32, C.c_double, C.c_double,
                                         C.c_double, u64, vp]
        L.orc_reduce_sparse.restype = C.c_int64
        L.orc_reduce_sparse.argtypes = [u64, u64, vp, vp, vp, vp, u64, vp, vp, vp, vp, vp,
                                        C.POINTER(u64), C.POINTER(u64), C.c_int]
        L.orc_kruskal_barcode.restype = C.c_int64
        L.orc_kruskal_barcode.argtypes = [u64, u64, vp, vp, vp, vp, vp, vp, C.POINTER(u64)]
        _orc = L
    return _orc


def ref_available() -> bool:
    return REF_SO.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        L = C.CDLL(str(REF_SO))
        L.ref_last_error.restype = C.c_char_p
        L.ref_splitmix_next.argtypes = [u64, u64, vp]
        L.ref_generate_uniform_cloud.argtypes = [u64, u64, u64, vp]
        L.ref_pairwise_distances.argtypes = [vp, u64, u64, vp]
        L.ref_build_filtration.argtypes = [vp, u64, u64, vp, vp, vp, vp, C.POINTER(u64)]
        L.ref_h0_barcode.argtypes = [vp, u64, u64, C.c_int, C.c_uint, vp, vp, C.POINTER(u64),
                                     C.POINTER(u64), vp, C.POINTER(u64), vp, vp]
        L.ref_reduced_matrix.argtypes = [vp, u64, u64, C.c_int, C.c_uint, vp, vp, vp,
                                         C.POINTER(u64), vp]
        _ref = L
    return _ref


def colmajor(X) -> tuple[np.ndarray, int, int]:
    X = np.asarray(X, np.float64)
    n, d = X.shape
    return np.asfortranarray(X), n, d


# ---- C restatement --------------------------------------------------------------------------
def splitmix_stream(seed: int, count: int) -> list[int]:
    s = u64(seed)
    return [orc().orc_splitmix_next(C.byref(s)) for _ in range(count)]


def uniform_cloud(n: int, d: int, seed: int) -> np.ndarray:
    buf = np.empty(max(n * d, 1))
    assert orc().orc_generate_uniform_cloud(n, d, seed, _p(buf)) == 0
    return buf[: n * d].reshape(d, n).T


# BASELINE.json configs, restated on the oracle side so fixtures and the
# bench's reference arm build X without the product library.
CONFIGS = {
    "C1": dict(kind=3, n=500, d=2, seed=1, sigma=0.05, lo=0.3, hi=0.7),
    "C2": dict(kind=2, n=2000, d=3, seed=2, sigma=0.05, lo=-1.5, hi=1.5, n_background=400),
    "C3": dict(kind=1, n=8192, d=16, seed=3, clusters=10, sigma=0.5, lo=-5.0, hi=5.0),
    "C4": dict(kind=0, n=32768, d=3, seed=4),
    "C5": dict(kind=1, n=65536, d=8, seed=5, clusters=32, sigma=0.3, lo=-5.0, hi=5.0),
}


def generate_cloud(kind: int, n: int, d: int, seed: int, clusters: int = 0, sigma: float = 0.0,
                   lo: float = 0.0, hi: float = 1.0, n_background: int = 0) -> np.ndarray:
    buf = np.empty(max(n * d, 1))
    rc = orc().orc_generate_cloud(kind, n, d, seed, clusters, sigma, lo, hi, n_background,
                                  _p(buf))
    assert rc == 0, rc
    return buf[: n * d].reshape(d, n).T


def config_cloud(name: str, n: int | None = None) -> np.ndarray:
    cfg = dict(CONFIGS[name])
    if n is not None:
        cfg["n"] = n
    return generate_cloud(**cfg)


def pairwise(X) -> np.ndarray:
    Xf, n, d = colmajor(X)
    k = n * (n - 1) // 2 if n else 0
    out = np.empty(k)
    orc().orc_pairwise_distances(_p(Xf), n, d, _p(out))
    return out


def filtration(X):
    Xf, n, d = colmajor(X)
    k = n * (n - 1) // 2 if n else 0
    u = np.empty(k, np.uint32)
    v = np.empty(k, np.uint32)
    g = np.empty(k, np.uint64)
    ln = np.empty(k)
    sc = np.empty(max(k, 1))
    ns = orc().orc_build_filtration(_p(Xf), n, d, _p(u), _p(v), _p(g), _p(ln), _p(sc))
    return dict(u=u, v=v, grade=g, length=ln, scale=sc[:ns].copy(), n=n, k=k)


def reduce_bars(f: dict):
    """Literal bit-vector column reduction (reduction.cpp:31-51) + extract_barcode."""
    n, k = f["n"], f["k"]
    dg = np.empty(max(n, 1), np.uint64)
    dl = np.empty(max(n, 1))
    lows = np.empty(max(n, 1), np.uint32)
    ess = u64(0)
    adds = u64(0)
    m = orc().orc_reduce_barcode(n, k, _p(f["u"]), _p(f["v"]), _p(f["grade"]), _p(f["scale"]),
                                 len(f["scale"]), _p(dg), _p(dl), _p(lows), C.byref(ess),
                                 C.byref(adds))
    assert m >= 0, m
    return dict(death_grade=dg[:m].copy(), death_length=dl[:m].copy(), claimed_low=lows[:m].copy(),
                essential=ess.value, additions=adds.value)


def reduce_sparse(f: dict, stop_at_spanning: bool = False):
    """The literal column reduction with 2-sparse supports: bars, the survivors' column
    indices and reduced supports {rows_lo, rows_hi}, and the addition count (of the columns
    processed: all of them unless stop_at_spanning)."""
    n, k = f["n"], f["k"]
    dg = np.empty(max(n, 1), np.uint64)
    dl = np.empty(max(n, 1))
    cols = np.empty(max(n, 1), np.uint64)
    lo = np.empty(max(n, 1), np.uint32)
    hi = np.empty(max(n, 1), np.uint32)
    ess, adds = u64(0), u64(0)
    m = orc().orc_reduce_sparse(n, k, _p(f["u"]), _p(f["v"]), _p(f["grade"]), _p(f["scale"]),
                                len(f["scale"]), _p(dg), _p(dl), _p(cols), _p(lo), _p(hi),
                                C.byref(ess), C.byref(adds), int(stop_at_spanning))
    assert m >= 0, m
    return dict(death_grade=dg[:m].copy(), death_length=dl[:m].copy(), columns=cols[:m].copy(),
                rows_lo=lo[:m].copy(), rows_hi=hi[:m].copy(), essential=ess.value,
                additions=adds.value)


def kruskal_bars(f: dict):
    n, k = f["n"], f["k"]
    dg = np.empty(max(n, 1), np.uint64)
    dl = np.empty(max(n, 1))
    ess = u64(0)
    m = orc().orc_kruskal_barcode(n, k, _p(f["u"]), _p(f["v"]), _p(f["grade"]), _p(f["length"]),
                                  _p(dg), _p(dl), C.byref(ess))
    return dict(death_grade=dg[:m].copy(), death_length=dl[:m].copy(), essential=ess.value)


def oracle_filtration_and_bars(X, reduction_limit: int = 3000):
    """Filtration + bars; the literal matrix reduction for n <= reduction_limit (memory
    K*ceil(n/64)*8 B), otherwise the Kruskal oracle (identical ordered bars)."""
    f = filtration(X)
    bars = reduce_bars(f) if f["n"] <= reduction_limit else kruskal_bars(f)
    f.update(bars)
    return f


# ---- shim-built reference -----------------------------------------------------------------
def ref_h0(X, mode: int = 0, workers: int = 1, want_scale: bool = True, want_lows: bool = False):
    Xf, n, d = colmajor(X)
    k = n * (n - 1) // 2 if n else 0
    dg = np.empty(max(n, 1), np.uint64)
    dl = np.empty(max(n, 1))
    nf, ess, ns = u64(0), u64(0), u64(0)
    sc = np.empty(max(k, 1)) if want_scale else None
    st = np.empty(5)
    lows = np.empty(max(n, 1), np.uint32) if want_lows else None
    rc = ref().ref_h0_barcode(_p(Xf), n, d, mode, workers, _p(dg), _p(dl), C.byref(nf),
                              C.byref(ess), _p(sc), C.byref(ns), _p(st), _p(lows))
    if rc != 0:
        raise ValueError(ref().ref_last_error().decode())
    out = dict(death_grade=dg[: nf.value].copy(), death_length=dl[: nf.value].copy(),
               essential=ess.value, n_scale=ns.value, stage_seconds=st.copy())
    if want_scale:
        out["scale"] = sc[: ns.value].copy()
    if want_lows:
        out["claimed_low"] = lows[: nf.value].copy()
    return out


def ref_reduced_matrix(X, pivoting: bool = True, workers: int = 1):
    """The reference's whole reduced matrix: (columns, rows_lo, rows_hi) of the nonzero
    columns, plus ReductionStats (additions, row_ops, probe_ops)."""
    Xf, n, d = colmajor(X)
    cols = np.empty(max(n, 1), np.uint64)
    lo = np.empty(max(n, 1), np.uint32)
    hi = np.empty(max(n, 1), np.uint32)
    m = u64(0)
    st = np.zeros(3, np.uint64)
    rc = ref().ref_reduced_matrix(_p(Xf), n, d, int(pivoting), workers, _p(cols), _p(lo),
                                  _p(hi), C.byref(m), _p(st))
    if rc != 0:
        raise ValueError(ref().ref_last_error().decode())
    k = m.value
    return cols[:k].copy(), lo[:k].copy(), hi[:k].copy(), st


def ref_filtration(X):
    Xf, n, d = colmajor(X)
    k = n * (n - 1) // 2 if n else 0
    u = np.empty(k, np.uint32)
    v = np.empty(k, np.uint32)
    g = np.empty(k, np.uint64)
    sc = np.empty(max(k, 1))
    ns = u64(0)
    rc = ref().ref_build_filtration(_p(Xf), n, d, _p(u), _p(v), _p(g), _p(sc), C.byref(ns))
    if rc != 0:
        raise ValueError(ref().ref_last_error().decode())
    return dict(u=u, v=v, grade=g, scale=sc[: ns.value].copy())
