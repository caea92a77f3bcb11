"""ctypes binding of libph0b.so (include/ph0b.h) — the Python-side caller of the C ABI.

There is no CPU fallback: if the shared object is missing or no sm_100 device is visible the
calls raise.  numpy arrays are the host containers; device runs take raw device pointers
(e.g. ``torch.Tensor.data_ptr()``) so torch is only plumbing for memory and streams.
"""
from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

_LIB_PATH = Path(__file__).resolve().parent / "libph0b.so"
_lib = None

PH0B_OK = 0
PH0B_ERR_INVALID_ARGUMENT = 1
PH0B_ERR_NONFINITE = 2
PH0B_ERR_TOO_LARGE = 3
PH0B_ERR_CUDA = 4
PH0B_ERR_OUT_OF_MEMORY = 5
PH0B_ERR_NO_DEVICE = 6
PH0B_ERR_CAPACITY = 7
COL_MAJOR = 0
ROW_MAJOR = 1
FLAG_NO_SCALE = 1
FLAG_KRUSKAL = 2

EXPORTED_SYMBOLS = [
    "ph0b_h0_barcode", "ph0b_result_free", "ph0b_h0_barcode_into", "ph0b_pairwise_distances",
    "ph0b_build_filtration", "ph0b_claimed_lows", "ph0b_context_create", "ph0b_context_destroy",
    "ph0b_context_reserve", "ph0b_context_workspace_bytes", "ph0b_run_device", "ph0b_run_host",
    "ph0b_last_error", "ph0b_abi_version", "ph0b_host_alloc", "ph0b_host_free",
    "ph0b_last_launch_count", "ph0b_generate_cloud", "ph0b_shard_distances", "ph0b_shard_sample",
    "ph0b_shard_partition", "ph0b_shard_recv", "ph0b_shard_sort_unique", "ph0b_shard_reduce",
    "ph0b_reduce_columns", "ph0b_kruskal_barcode", "ph0b_generate_uniform_cloud_device",
    "ph0b_decode_deltas", "ph0b_decode_packed", "ph0b_scale_to_host",
    "ph0b_shard_partition_count", "ph0b_shard_recv_peer",
    "ph0b_shard_scatter_peers", "ph0b_ipc_get_handle", "ph0b_ipc_open_handle", "ph0b_ipc_close",
    "ph0b_scale_release", "ph0b_host_cache_trim", "ph0b_reduced_supports",
    "ph0b_release_resources", "ph0b_shard_reduce_continue",
]


class Ph0bError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[ph0b error {code}] {msg}")
        self.code = code
        self.msg = msg


class InvalidArgument(Ph0bError, ValueError):
    """Mirrors std::invalid_argument thrown by the reference."""


class Options(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("device", C.c_int32), ("flags", C.c_uint32),
                ("pivoting", C.c_uint32), ("workers", C.c_uint32), ("n_gpus", C.c_uint32),
                ("devices", C.POINTER(C.c_int32))]


class StageTimes(C.Structure):
    _fields_ = [("distance_ms", C.c_float), ("sort_ms", C.c_float), ("unique_ms", C.c_float),
                ("reduce_ms", C.c_float), ("collect_ms", C.c_float), ("total_ms", C.c_float),
                ("sort_passes", C.c_uint32), ("reduce_rounds", C.c_uint32),
                ("columns_scanned", C.c_uint64), ("sort_passes_ms", C.c_float),
                ("reduce_iterations", C.c_uint32), ("d2h_bytes", C.c_uint64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class Result(C.Structure):
    _fields_ = [("n_finite", C.c_uint64), ("death_grade", C.POINTER(C.c_uint64)),
                ("death_length", C.POINTER(C.c_double)), ("essential_count", C.c_uint64),
                ("n_scale", C.c_uint64), ("scale", C.POINTER(C.c_double)), ("times", StageTimes)]


class DeviceResult(C.Structure):
    _fields_ = [("n_finite", C.c_uint64), ("essential_count", C.c_uint64),
                ("n_scale", C.c_uint64), ("d_scale", C.c_void_p), ("d_death_grade", C.c_void_p),
                ("d_death_length", C.c_void_p), ("times", StageTimes)]


def lib() -> C.CDLL:
    """Load libph0b.so (raises if it was not built — no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        raise FileNotFoundError(
            f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(str(_LIB_PATH))
    u64, u32, i32, dp, vp = C.c_uint64, C.c_uint32, C.c_int32, C.POINTER(C.c_double), C.c_void_p
    u64p, u32p = C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)
    sig = {
        "ph0b_h0_barcode": (C.c_int, [vp, u64, u64, u32, C.POINTER(Options), C.POINTER(Result)]),
        "ph0b_result_free": (None, [C.POINTER(Result)]),
        "ph0b_scale_release": (None, [vp]),
        "ph0b_host_cache_trim": (None, []),
        "ph0b_release_resources": (None, []),
        "ph0b_kruskal_barcode": (C.c_int, [vp, u64, u64, u32, C.POINTER(Options),
                                           C.POINTER(Result)]),
        "ph0b_generate_uniform_cloud_device": (C.c_int, [vp, u64, u64, u64, vp, vp]),
        "ph0b_decode_deltas": (C.c_int, [vp, vp, vp, u64, u32, vp]),
        "ph0b_h0_barcode_into": (C.c_int, [vp, u64, u64, u32, C.POINTER(Options), vp, vp, u64p,
                                           u64p, vp, u64, u64p, C.POINTER(StageTimes)]),
        "ph0b_pairwise_distances": (C.c_int, [vp, u64, u64, u32, C.POINTER(Options), vp]),
        "ph0b_build_filtration": (C.c_int, [vp, u64, u64, u32, C.POINTER(Options), vp, vp, vp,
                                            vp, u64p]),
        "ph0b_claimed_lows": (C.c_int, [vp, u64, u64, u32, C.POINTER(Options), vp, u64p]),
        "ph0b_reduced_supports": (C.c_int, [vp, u64, u64, u32, C.POINTER(Options), vp, vp, vp,
                                            u64p]),
        "ph0b_context_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
        "ph0b_context_destroy": (None, [vp]),
        "ph0b_context_reserve": (C.c_int, [vp, u64, u64]),
        "ph0b_context_workspace_bytes": (u64, [vp]),
        "ph0b_run_device": (C.c_int, [vp, vp, u64, u64, u32, vp, C.POINTER(DeviceResult)]),
        "ph0b_run_host": (C.c_int, [vp, vp, u64, u64, u32, vp, vp, vp, u64p, u64p, vp, u64,
                                    u64p, C.POINTER(StageTimes)]),
        "ph0b_last_error": (C.c_char_p, []),
        "ph0b_abi_version": (u32, []),
        "ph0b_host_alloc": (vp, [u64]),
        "ph0b_host_free": (None, [vp]),
        "ph0b_last_launch_count": (u64, []),
        "ph0b_generate_cloud": (C.c_int, [u32, u64, u64, u64, u32, C.c_double, C.c_double,
                                          C.c_double, u64, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _ = (i32, dp, u32p)
    _lib = L
    return L


def _check(rc: int):
    if rc == PH0B_OK:
        return
    msg = lib().ph0b_last_error().decode()
    if rc in (PH0B_ERR_INVALID_ARGUMENT, PH0B_ERR_NONFINITE):
        raise InvalidArgument(rc, msg)
    raise Ph0bError(rc, msg)


def _opts(device: int = 0, flags: int = 0, workers: int = 1, pivoting: bool = True,
          devices=None) -> Options:
    o = Options(C.sizeof(Options), device, flags, int(pivoting), workers)
    if devices is not None and len(devices) > 1:
        arr = (C.c_int32 * len(devices))(*devices)
        o.n_gpus = len(devices)
        o.devices = C.cast(arr, C.POINTER(C.c_int32))
        o._keep = arr  # the array lives as long as the options
    return o


def _as_cloud(X) -> tuple[np.ndarray, int, int]:
    """Column-major f64 copy of an (N, d) cloud (Eigen::MatrixXd storage)."""
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2:
        raise ValueError("point cloud must be a 2-D array (N x d)")
    n, d = X.shape
    return np.asfortranarray(X), n, d


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data) if a.size else None


@dataclass
class Barcode:
    """Mirror of ph0::Barcode (proj/include/ph0/barcode.hpp:17-20) plus D and stage times."""
    death_grade: np.ndarray
    death_length: np.ndarray
    essential_count: int
    scale: np.ndarray | None = None
    times: dict = field(default_factory=dict)

    @property
    def finite(self):
        return [(0.0, int(g), float(x)) for g, x in zip(self.death_grade, self.death_length)]


def _take_scale(res) -> np.ndarray:
    """D of a ph0b_result as a numpy array that takes over the library's buffer (handed back
    with ph0b_scale_release when the array dies) instead of copying it; res.scale is cleared
    so ph0b_result_free leaves it alone."""
    if not res.n_scale:
        return np.zeros(0)
    L = lib()
    ptr = C.cast(res.scale, C.c_void_p).value
    # the finalizer hangs on the ctypes buffer every numpy view of D refers to (numpy collapses
    # view bases to it), so D is released only when no array uses it any more
    buf = (C.c_double * res.n_scale).from_address(ptr)
    weakref.finalize(buf, L.ph0b_scale_release, C.c_void_p(ptr))
    res.scale = None
    return np.frombuffer(buf, dtype=np.float64, count=res.n_scale)


def h0_barcode(X, *, device: int = 0, return_scale: bool = True, workers: int = 1,
               pivoting: bool = True, kruskal: bool = False, devices=None) -> Barcode:
    """pairwise_distances ∘ build_filtration ∘ build_boundary_matrix ∘ reduce ∘ extract_barcode
    (kruskal=True: the union-find barcode of oracle.cpp:32-46 over the same GPU filtration;
    devices=[...]: the in-process multi-GPU path over those ordinals, repeats allowed)."""
    Xf, n, d = _as_cloud(X)
    L = lib()
    res = Result()
    flags = (0 if return_scale else FLAG_NO_SCALE) | (FLAG_KRUSKAL if kruskal else 0)
    opt = _opts(device, flags, workers, pivoting, devices)
    rc = L.ph0b_h0_barcode(_ptr(Xf), n, d, COL_MAJOR, C.byref(opt), C.byref(res))
    _check(rc)
    try:
        m = res.n_finite
        g = np.ctypeslib.as_array(res.death_grade, (m,)).copy() if m else np.zeros(0, np.uint64)
        ln = np.ctypeslib.as_array(res.death_length, (m,)).copy() if m else np.zeros(0)
        sc = _take_scale(res) if return_scale else None
        return Barcode(g, ln, int(res.essential_count), sc, res.times.as_dict())
    finally:
        L.ph0b_result_free(C.byref(res))


def kruskal_barcode(X, *, device: int = 0, return_scale: bool = True) -> Barcode:
    """kruskal_barcode(build_filtration(pairwise_distances(X)), n) (oracle.cpp:32-46) on the
    GPU: the ph0b_kruskal_barcode entry point."""
    Xf, n, d = _as_cloud(X)
    L = lib()
    res = Result()
    opt = _opts(device, 0 if return_scale else FLAG_NO_SCALE)
    _check(L.ph0b_kruskal_barcode(_ptr(Xf), n, d, COL_MAJOR, C.byref(opt), C.byref(res)))
    try:
        m = res.n_finite
        g = np.ctypeslib.as_array(res.death_grade, (m,)).copy() if m else np.zeros(0, np.uint64)
        ln = np.ctypeslib.as_array(res.death_length, (m,)).copy() if m else np.zeros(0)
        sc = _take_scale(res) if return_scale else None
        return Barcode(g, ln, int(res.essential_count), sc, res.times.as_dict())
    finally:
        L.ph0b_result_free(C.byref(res))


def pairwise_distances(X, *, device: int = 0) -> np.ndarray:
    """Lengths of all pairs u < v in u-major order (filtration.cpp:8-18)."""
    Xf, n, d = _as_cloud(X)
    k = n * (n - 1) // 2 if n else 0
    out = np.empty(k, np.float64)
    _check(lib().ph0b_pairwise_distances(_ptr(Xf), n, d, COL_MAJOR, C.byref(_opts(device)),
                                         _ptr(out)))
    return out


def build_filtration(X, *, device: int = 0):
    """(u, v, grade, scale) of the filtration / boundary-matrix columns in filtration order."""
    Xf, n, d = _as_cloud(X)
    k = n * (n - 1) // 2 if n else 0
    u = np.empty(k, np.uint32)
    v = np.empty(k, np.uint32)
    g = np.empty(k, np.uint64)
    scale = np.empty(max(k, 1), np.float64)
    ns = C.c_uint64(0)
    _check(lib().ph0b_build_filtration(_ptr(Xf), n, d, COL_MAJOR, C.byref(_opts(device)),
                                       _ptr(u), _ptr(v), _ptr(g), _ptr(scale), C.byref(ns)))
    return u, v, g, scale[: ns.value].copy()


def claimed_lows(X, *, device: int = 0) -> np.ndarray:
    Xf, n, d = _as_cloud(X)
    out = np.empty(max(n, 1), np.uint32)
    m = C.c_uint64(0)
    _check(lib().ph0b_claimed_lows(_ptr(Xf), n, d, COL_MAJOR, C.byref(_opts(device)), _ptr(out),
                                   C.byref(m)))
    return out[: m.value].copy()


def reduced_supports(X, *, device: int = 0, workers: int = 1, pivoting: bool = True):
    """The reduced matrix of reduce() (reduction.cpp:33-49) as (columns, rows_lo, rows_hi):
    surviving column j = columns[i] ends as {rows_lo[i], rows_hi[i]} (rows_hi = its claimed
    low), every other column ends empty."""
    Xf, n, d = _as_cloud(X)
    cols = np.empty(max(n, 1), np.uint64)
    lo = np.empty(max(n, 1), np.uint32)
    hi = np.empty(max(n, 1), np.uint32)
    m = C.c_uint64(0)
    _check(lib().ph0b_reduced_supports(_ptr(Xf), n, d, COL_MAJOR,
                                       C.byref(_opts(device, 0, workers, pivoting)), _ptr(cols),
                                       _ptr(lo), _ptr(hi), C.byref(m)))
    k = m.value
    return cols[:k].copy(), lo[:k].copy(), hi[:k].copy()


def last_launch_count() -> int:
    return int(lib().ph0b_last_launch_count())


def generate_cloud(kind: int, n: int, d: int, seed: int, clusters: int = 0, sigma: float = 0.0,
                   lo: float = 0.0, hi: float = 1.0, n_background: int = 0) -> np.ndarray:
    """Synthetic cloud (N x d, C-order view of a column-major buffer)."""
    buf = np.empty(max(n * d, 1), np.float64)
    _check(lib().ph0b_generate_cloud(kind, n, d, seed, clusters, sigma, lo, hi, n_background,
                                     _ptr(buf)))
    return buf[: n * d].reshape(d, n).T  # (N, d) view of the col-major storage


# The five BASELINE.json configurations.
CONFIGS = {
    "C1": dict(kind=3, n=500, d=2, seed=1, sigma=0.05, lo=0.3, hi=0.7),
    "C2": dict(kind=2, n=2000, d=3, seed=2, sigma=0.05, lo=-1.5, hi=1.5, n_background=400),
    "C3": dict(kind=1, n=8192, d=16, seed=3, clusters=10, sigma=0.5, lo=-5.0, hi=5.0),
    "C4": dict(kind=0, n=32768, d=3, seed=4),
    "C5": dict(kind=1, n=65536, d=8, seed=5, clusters=32, sigma=0.3, lo=-5.0, hi=5.0),
}


def config_cloud(name: str, n: int | None = None) -> np.ndarray:
    cfg = dict(CONFIGS[name])
    if n is not None:
        cfg["n"] = n
    return generate_cloud(**cfg)


class Context:
    """Device-resident pipeline context (ph0b_context_*): reusable HBM workspace."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        _check(lib().ph0b_context_create(device, C.byref(self._h)))

    def close(self):
        if self._h:
            lib().ph0b_context_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reserve(self, n: int, d: int):
        _check(lib().ph0b_context_reserve(self._h, n, d))

    def generate_uniform_cloud(self, n: int, dim: int, seed: int, d_out_ptr: int,
                               stream: int = 0):
        """generate_uniform_cloud (point_cloud.cpp:20-29) on the device, column-major."""
        _check(lib().ph0b_generate_uniform_cloud_device(self._h, n, dim, seed,
                                                        C.c_void_p(d_out_ptr),
                                                        C.c_void_p(stream or None)))

    @property
    def workspace_bytes(self) -> int:
        return int(lib().ph0b_context_workspace_bytes(self._h))

    def run_device(self, x_ptr: int, n: int, d: int, layout: int = COL_MAJOR,
                   stream: int = 0) -> DeviceResult:
        out = DeviceResult()
        _check(lib().ph0b_run_device(self._h, C.c_void_p(x_ptr), n, d, layout,
                                     C.c_void_p(stream), C.byref(out)))
        return out

    def run_host(self, X: np.ndarray, death_grade: np.ndarray, death_length: np.ndarray,
                 scale: np.ndarray | None, stream: int = 0, layout: int = COL_MAJOR):
        """Host X -> host outputs (buffers may be pinned views from host_alloc)."""
        n, d = X.shape if layout == ROW_MAJOR else (X.shape[0], X.shape[1])
        nf = C.c_uint64(0)
        ess = C.c_uint64(0)
        ns = C.c_uint64(0)
        t = StageTimes()
        _check(lib().ph0b_run_host(self._h, C.c_void_p(X.ctypes.data), n, d, layout,
                                   C.c_void_p(stream), C.c_void_p(death_grade.ctypes.data),
                                   C.c_void_p(death_length.ctypes.data), C.byref(nf),
                                   C.byref(ess), C.c_void_p(scale.ctypes.data) if scale is not None
                                   else None, scale.size if scale is not None else 0, C.byref(ns),
                                   C.byref(t)))
        return int(nf.value), int(ess.value), int(ns.value), t.as_dict()


class PinnedArray:
    """numpy view over pinned host memory from ph0b_host_alloc."""

    def __init__(self, count: int, dtype=np.float64):
        self.dtype = np.dtype(dtype)
        self.nbytes = max(1, count) * self.dtype.itemsize
        self._p = lib().ph0b_host_alloc(self.nbytes)
        if not self._p:
            raise Ph0bError(PH0B_ERR_OUT_OF_MEMORY, f"pinned allocation of {self.nbytes} B failed")
        buf = (C.c_char * self.nbytes).from_address(self._p)
        self.array = np.frombuffer(buf, dtype=self.dtype, count=count)

    def free(self):
        if self._p:
            self.array = None
            lib().ph0b_host_free(self._p)
            self._p = None
