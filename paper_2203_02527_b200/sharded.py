"""Multi-GPU H0 barcode: one process (rank) per GPU, NCCL for the one real
exchange step.

    rank r:  K1 distances of rows [U_r, U_{r+1})      (balanced edge counts, no communication)
             sample lengths -> all-gather -> P-1 splitters (global, on the length key)
             stable partition by splitter -> all-to-all-v (NCCL) of (length, column)
             local radix sort + unique  -> D slice r (D is sharded, contiguous in global order)
             all-gather |D_r| -> grade offsets
             column reduction of the key ranges in order, each continuing the forest the
             earlier ranges left (their tree labels); stops at N-1 survivors -> bars

Exactness: rows are assigned in increasing u and every partition is stable, so what a rank
receives (sources in rank order) is in u-major order and the local stable sort produces the
global (length, u, v) order restricted to its key range; equal lengths never straddle ranks
(splitters are key values).  Reducing the ranges in order, each from the forest the earlier
ranges left, is the reference's left-to-right reduction itself, cut at range boundaries.

`Comm` hides the transport: torch.distributed (NCCL on GPUs, gloo for the CPU tests) or a
thread-based comm that runs P virtual ranks in one process (single-GPU parity tests).
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

import numpy as np

from . import ph0b as _b

SAMPLES_PER_RANK = 4096


def row_ranges(n: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous row ranges [U_r, U_{r+1}) with ~K/parts edges each (row u has n-1-u)."""
    k = n * (n - 1) // 2
    bounds = [0]
    cum = 0
    u = 0
    for r in range(1, parts):
        target = (k * r) // parts
        while u < n and cum + (n - 1 - u) <= target:
            cum += n - 1 - u
            u += 1
        bounds.append(u)
    bounds.append(n)
    return [(bounds[i], bounds[i + 1]) for i in range(parts)]


def choose_splitters(samples: np.ndarray, parts: int) -> np.ndarray:
    s = np.sort(np.asarray(samples, np.uint64))
    if parts <= 1 or len(s) == 0:
        return np.zeros(max(parts - 1, 0), np.uint64)
    idx = [((j + 1) * len(s)) // parts for j in range(parts - 1)]
    return s[np.minimum(idx, len(s) - 1)].astype(np.uint64)


@dataclass
class ShardResult:
    rank: int
    parts: int
    death_grade: np.ndarray | None      # rank 0 only (filtration order)
    death_length: np.ndarray | None
    essential_count: int
    scale_offset: int                   # global index of this rank's first D entry
    n_scale_local: int
    n_scale_total: int
    scale_local: object                 # backend-specific view of the D slice
    edges_local: int


# ---- transports -------------------------------------------------------------------------------
class TorchComm:
    """torch.distributed transport (NCCL for device tensors, gloo for CPU tensors)."""

    same_process = False  # peer buffers are shared through IPC handles

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def allgather_obj(self, obj):
        out = [None] * self.size
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def alltoallv(self, send, send_counts, recv, recv_counts):
        self.dist.all_to_all_single(recv, send, [int(c) for c in recv_counts],
                                    [int(c) for c in send_counts], group=self.group)
        if recv.is_cuda:  # the next stage runs on the ph0b context's own stream
            import torch
            torch.cuda.current_stream(recv.device).synchronize()

    def barrier(self):
        self.dist.barrier(group=self.group)


class ThreadComm:
    """P virtual ranks as threads of one process (single-GPU multi-rank parity tests)."""

    same_process = True  # peer buffers are plain device pointers of this process

    class _Shared:
        def __init__(self, size):
            self.size = size
            self.barrier = threading.Barrier(size)
            self.slots = [None] * size

    def __init__(self, shared: "ThreadComm._Shared", rank: int):
        self.s = shared
        self.rank = rank
        self.size = shared.size

    @classmethod
    def make(cls, size):
        sh = cls._Shared(size)
        return [cls(sh, r) for r in range(size)]

    def allgather_obj(self, obj):
        self.s.barrier.wait()
        self.s.slots[self.rank] = obj
        self.s.barrier.wait()
        out = list(self.s.slots)
        self.s.barrier.wait()
        return out

    def alltoallv(self, send, send_counts, recv, recv_counts):
        import torch
        torch.cuda.synchronize(send.device) if send.is_cuda else None
        peers = self.allgather_obj((send, [int(c) for c in send_counts]))
        pos = 0
        for src in range(self.size):
            sbuf, scounts = peers[src]
            off = sum(scounts[: self.rank])
            cnt = scounts[self.rank]
            if cnt:
                recv[pos:pos + cnt].copy_(sbuf[off:off + cnt])
            pos += cnt
        if recv.is_cuda:
            torch.cuda.synchronize(recv.device)
        self.allgather_obj(None)  # nobody reuses its send buffer before all copies are done

    def barrier(self):
        self.s.barrier.wait()


# ---- device backend (the product path) -----------------------------------------------------
class _CAI:
    def __init__(self, ptr, count, typestr):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


def _dev_view(ptr, count, typestr, device):
    import torch
    if count == 0:
        return torch.empty(0, dtype={"<i8": torch.int64, "<i4": torch.int32,
                                     "<f8": torch.float64}[typestr], device=f"cuda:{device}")
    return torch.as_tensor(_CAI(ptr, count, typestr), device=f"cuda:{device}")


class DeviceBackend:
    """Per-rank stages on the B200 through the C ABI (one ph0b context per rank)."""

    def __init__(self, device: int = 0):
        self.device = device
        self.launches = 0  # kernel launches issued through this backend (evidence counter)
        self.ctx = _b.Context(device)
        self.L = _b.lib()
        h = self.ctx._h
        self.h = h
        L = self.L
        vp, u64, u32 = C.c_void_p, C.c_uint64, C.c_uint32
        u64p = C.POINTER(C.c_uint64)
        for name, res, args in [
            ("ph0b_shard_distances", C.c_int, [vp, vp, u64, u64, u32, u64, u64, vp, u64p, u64p, u64p]),
            ("ph0b_shard_sample", C.c_int, [vp, u64, vp]),
            ("ph0b_shard_partition", C.c_int, [vp, vp, u32, vp, C.POINTER(vp), C.POINTER(vp), vp, vp, vp]),
            ("ph0b_shard_recv", C.c_int, [vp, u64, C.POINTER(vp), C.POINTER(vp)]),
            ("ph0b_shard_sort_unique", C.c_int, [vp, u64, u64, u64, vp, u64p, C.POINTER(vp),
                                                 C.POINTER(C.c_uint32)]),
            ("ph0b_shard_reduce", C.c_int, [vp, u64, u64, u64, vp, u64p, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]),
            ("ph0b_reduce_columns", C.c_int, [vp, vp, u64, u64, vp, vp, u64p]),
            ("ph0b_shard_partition_count", C.c_int, [vp, vp, u32, vp, vp, vp, vp]),
            ("ph0b_shard_recv_peer", C.c_int, [vp, u64, C.POINTER(vp), C.POINTER(vp)]),
            ("ph0b_shard_scatter_peers", C.c_int, [vp, u32, vp, vp, vp, vp]),
            ("ph0b_ipc_get_handle", C.c_int, [vp, vp]),
            ("ph0b_ipc_open_handle", C.c_int, [vp, C.POINTER(vp)]),
            ("ph0b_scale_to_host", C.c_int, [vp, vp, u64, vp, u64, vp, u64p]),
        ]:
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args

    def _count(self):
        self.launches += int(self.L.ph0b_last_launch_count())

    def distances(self, x_ptr, n, d, u_lo, u_hi, layout=_b.COL_MAJOR):
        cnt, lo, hi = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _b._check(self.L.ph0b_shard_distances(self.h, C.c_void_p(x_ptr), n, d, layout, u_lo, u_hi,
                                              None, C.byref(cnt), C.byref(lo), C.byref(hi)))
        self._count()
        return cnt.value, lo.value, hi.value

    def sample(self, s, count):
        s = min(s, count)
        out = np.zeros(s, np.uint64)
        if s:
            _b._check(self.L.ph0b_shard_sample(self.h, s, C.c_void_p(out.ctypes.data)))
        return out

    def partition(self, splitters, parts):
        spl = np.ascontiguousarray(splitters, np.uint64)
        counts = np.zeros(parts, np.uint64)
        pmin = np.zeros(parts, np.uint64)
        pmax = np.zeros(parts, np.uint64)
        kp, vp_ = C.c_void_p(), C.c_void_p()
        _b._check(self.L.ph0b_shard_partition(
            self.h, C.c_void_p(spl.ctypes.data) if spl.size else None, parts, None, C.byref(kp),
            C.byref(vp_), C.c_void_p(counts.ctypes.data), C.c_void_p(pmin.ctypes.data),
            C.c_void_p(pmax.ctypes.data)))
        self._count()
        total = int(counts.sum())
        return (_dev_view(kp.value, total, "<i8", self.device),
                _dev_view(vp_.value, total, "<i4", self.device), counts, pmin, pmax)

    def recv(self, count):
        kp, vp_ = C.c_void_p(), C.c_void_p()
        _b._check(self.L.ph0b_shard_recv(self.h, count, C.byref(kp), C.byref(vp_)))
        return (_dev_view(kp.value, count, "<i8", self.device),
                _dev_view(vp_.value, count, "<i4", self.device))

    def sort_unique(self, count, kmin, kmax):
        import time
        nd, sp, ps = C.c_uint64(), C.c_void_p(), C.c_uint32()
        t0 = time.perf_counter()
        _b._check(self.L.ph0b_shard_sort_unique(self.h, count, kmin, kmax, None, C.byref(nd),
                                                C.byref(sp), C.byref(ps)))
        self.last_sort = (time.perf_counter() - t0, int(ps.value), int(count))
        self._count()
        return nd.value, _dev_view(sp.value, nd.value, "<f8", self.device)

    # ---- exchange over peer memory (NVLink P2P stores; replaces partition + all-to-all-v)
    def partition_count(self, splitters, parts):
        spl = np.ascontiguousarray(splitters, np.uint64)
        counts = np.zeros(parts, np.uint64)
        pmin = np.zeros(parts, np.uint64)
        pmax = np.zeros(parts, np.uint64)
        _b._check(self.L.ph0b_shard_partition_count(
            self.h, C.c_void_p(spl.ctypes.data) if spl.size else None, parts, None,
            C.c_void_p(counts.ctypes.data), C.c_void_p(pmin.ctypes.data),
            C.c_void_p(pmax.ctypes.data)))
        self._count()
        return counts, pmin, pmax

    def recv_peer(self, count, same_process):
        """Receive buffers peers write into; returns what the peers need to reach them."""
        kp, vp_ = C.c_void_p(), C.c_void_p()
        _b._check(self.L.ph0b_shard_recv_peer(self.h, count, C.byref(kp), C.byref(vp_)))
        self._recv = (int(kp.value or 0), int(vp_.value or 0))
        if same_process:
            return self._recv
        hk, hv = (C.c_char * 64)(), (C.c_char * 64)()
        _b._check(self.L.ph0b_ipc_get_handle(C.c_void_p(self._recv[0]), hk))
        _b._check(self.L.ph0b_ipc_get_handle(C.c_void_p(self._recv[1]), hv))
        return (bytes(hk), bytes(hv))

    def open_peer(self, desc, is_self, same_process):
        """Device addresses (in this process) of a peer's receive buffers."""
        if is_self:
            return self._recv
        if same_process:
            return desc
        cache = self.__dict__.setdefault("_ipc", {})
        if desc not in cache:  # buffers are reused across calls: map each handle once
            ptrs = []
            for h in desc:
                p = C.c_void_p()
                _b._check(self.L.ph0b_ipc_open_handle(C.c_char_p(h), C.byref(p)))
                ptrs.append(int(p.value))
            cache[desc] = tuple(ptrs)
        return cache[desc]

    def scatter_peers(self, parts, dst, offsets):
        kd = np.array([d[0] for d in dst], np.uint64)
        vd = np.array([d[1] for d in dst], np.uint64)
        off = np.ascontiguousarray(offsets, np.uint64)
        _b._check(self.L.ph0b_shard_scatter_peers(
            self.h, parts, C.c_void_p(kd.ctypes.data), C.c_void_p(vd.ctypes.data),
            C.c_void_p(off.ctypes.data), None))
        self._count()

    def scale_to_host(self, d_ptr, n, out: np.ndarray) -> int:
        """This rank's D slice (device) -> out (host, ideally pinned), shipped compressed
        through the context's ring like ph0b_run_host; returns the bytes that crossed PCIe."""
        moved = C.c_uint64()
        _b._check(self.L.ph0b_scale_to_host(self.h, C.c_void_p(d_ptr), n,
                                            C.c_void_p(out.ctypes.data), out.size, None,
                                            C.byref(moved)))
        return int(moved.value)

    def reduce_continue(self, n, count, grade_offset, labels, target):
        """Local reduction continuing the forest of the ranges before this one (host labels
        or None); returns the survivors' (uv, grade, length) and this range's final labels."""
        m, up, gp, lp = C.c_uint64(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        lab_in = (np.ascontiguousarray(labels, np.uint32) if labels is not None else None)
        lab_out = np.empty(max(n, 1), np.uint32)
        fn = self.L.ph0b_shard_reduce_continue
        if not fn.argtypes:
            fn.restype = C.c_int
            fn.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint32,
                           C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_void_p),
                           C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_void_p]
        _b._check(fn(self.h, n, count, grade_offset,
                     C.c_void_p(lab_in.ctypes.data) if lab_in is not None else None,
                     max(0, int(target)), None, C.byref(m), C.byref(up), C.byref(gp),
                     C.byref(lp), C.c_void_p(lab_out.ctypes.data)))
        self._count()
        m = m.value
        uv = _dev_view(up.value, m, "<i4", self.device).cpu().numpy().view(np.uint32)
        g = _dev_view(gp.value, m, "<i8", self.device).cpu().numpy().view(np.uint64)
        ln = _dev_view(lp.value, m, "<f8", self.device).cpu().numpy()
        return uv.copy(), g.copy(), ln.copy(), lab_out[:n].copy()

    def reduce(self, n, count, grade_offset):
        m, up, gp, lp = C.c_uint64(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        _b._check(self.L.ph0b_shard_reduce(self.h, n, count, grade_offset, None, C.byref(m),
                                           C.byref(up), C.byref(gp), C.byref(lp)))
        self._count()
        m = m.value
        uv = _dev_view(up.value, m, "<i4", self.device).cpu().numpy().view(np.uint32)
        g = _dev_view(gp.value, m, "<i8", self.device).cpu().numpy().view(np.uint64)
        ln = _dev_view(lp.value, m, "<f8", self.device).cpu().numpy()
        return uv.copy(), g.copy(), ln.copy()

    def reduce_columns(self, uv: np.ndarray, n: int) -> np.ndarray:
        import torch
        uv_dev = torch.from_numpy(np.ascontiguousarray(uv, np.uint32).view(np.int32)).to(
            f"cuda:{self.device}")
        idx = np.zeros(max(len(uv), 1), np.uint32)
        cnt = C.c_uint64()
        _b._check(self.L.ph0b_reduce_columns(self.h, C.c_void_p(uv_dev.data_ptr()), len(uv), n,
                                              None, C.c_void_p(idx.ctypes.data), C.byref(cnt)))
        self._count()
        return idx[: cnt.value].copy()

    def close(self):
        self.ctx.close()


# ---- the SPMD driver -------------------------------------------------------------------------
def exchange_mode(comm, backend) -> str:
    """'peer': one partition kernel stores every part straight into its destination rank's
    receive buffer (peer memory over NVLink); 'collective': partition into a send buffer,
    then all-to-all-v (NCCL).  PH0B_EXCHANGE=collective|peer overrides the default (peer
    when the backend supports it)."""
    import os
    want = os.environ.get("PH0B_EXCHANGE", "peer")
    ok = hasattr(backend, "scatter_peers") and hasattr(comm, "same_process")
    return "peer" if want == "peer" and ok else "collective"


def h0_barcode_sharded(x_ptr, n: int, d: int, comm, backend, layout=_b.COL_MAJOR) -> ShardResult:
    """Run on every rank (same X on every rank: it is <= 4 MiB, replicated)."""
    P, r = comm.size, comm.rank
    lo, hi = row_ranges(n, P)[r]
    count, kmin, kmax = backend.distances(x_ptr, n, d, lo, hi, layout)
    if P > 1:
        samples = np.concatenate(comm.allgather_obj(backend.sample(SAMPLES_PER_RANK, count)))
        spl = choose_splitters(samples, P)
        peer = exchange_mode(comm, backend) == "peer"
        if peer:
            counts, pmin, pmax = backend.partition_count(spl, P)
        else:
            send_k, send_v, counts, pmin, pmax = backend.partition(spl, P)
        allc = np.array(comm.allgather_obj(counts), np.uint64)          # [src][dst]
        allmin = np.array(comm.allgather_obj(pmin), np.uint64)
        allmax = np.array(comm.allgather_obj(pmax), np.uint64)
        recv_counts = allc[:, r]
        total = int(recv_counts.sum())
        have = recv_counts > 0
        kmin = int(allmin[have, r].min()) if have.any() else 0
        kmax = int(allmax[have, r].max()) if have.any() else 0
        if peer:
            # every rank's receive buffer exists before anyone learns where it is; part b of
            # this rank lands after the parts of lower ranks (source-rank order, as the
            # all-to-all-v delivers it, so the received slice is u-major)
            descs = comm.allgather_obj(backend.recv_peer(total, comm.same_process))
            dst = [backend.open_peer(descs[b], b == r, comm.same_process) for b in range(P)]
            offsets = [int(allc[:r, b].sum()) for b in range(P)]
            backend.scatter_peers(P, dst, offsets)
            comm.barrier()  # all stores into every receive buffer are complete
        else:
            recv_k, recv_v = backend.recv(total)
            comm.alltoallv(send_k, counts, recv_k, recv_counts)
            comm.alltoallv(send_v, counts, recv_v, recv_counts)
        count = total
    n_distinct, scale = backend.sort_unique(count, kmin, kmax)
    nds = comm.allgather_obj(int(n_distinct)) if P > 1 else [int(n_distinct)]
    offset = int(sum(nds[:r]))
    # column reduction: the key ranges in filtration order, each continuing the forest the
    # ranges before it left (their final tree labels, N u32) — the reference's left-to-right
    # reduction (reduction.cpp:33-49) cut at range boundaries, so no final re-reduction; it
    # stops as soon as n-1 columns survived (at C5 within the first range)
    labels, found = None, 0
    mine = (np.zeros(0, np.uint32), np.zeros(0, np.uint64), np.zeros(0))
    for turn in range(P):
        if found >= n - 1:
            break
        state = None
        if r == turn:
            uv, grade, length, labels_out = backend.reduce_continue(n, count, offset, labels,
                                                                    n - 1 - found)
            mine = (uv, grade, length)
            state = (len(uv), labels_out)
        if P > 1:
            state = comm.allgather_obj(state)[turn]
        found += state[0]
        labels = state[1]
    parts = comm.allgather_obj(mine) if P > 1 else [mine]
    dg = dl = None
    if r == 0:
        dg = np.concatenate([np.asarray(p_[1], np.uint64) for p_ in parts])
        dl = np.concatenate([np.asarray(p_[2], np.float64) for p_ in parts])
    ess = n - (n - 1 if n >= 1 else 0)
    return ShardResult(rank=r, parts=P, death_grade=dg, death_length=dl, essential_count=ess,
                       scale_offset=offset, n_scale_local=int(n_distinct),
                       n_scale_total=int(sum(nds)), scale_local=scale, edges_local=count)
