"""TEST INFRASTRUCTURE — numpy stand-in for the per-rank device stages of
paper_2203_02527_b200/sharded.py, so the multi-rank orchestration (row split, splitters,
stable partition, all-to-all-v, grade offsets, candidate gather, final reduction) can be
tested with world_size > 1 over gloo on CPU.  Lengths use the reference's exact fold."""
from __future__ import annotations

import numpy as np
import torch


def fold_lengths(X, u, vs):
    acc = (X[u, 0] - X[vs, 0]) * (X[u, 0] - X[vs, 0]) if X.shape[1] else np.zeros(len(vs))
    for k in range(1, X.shape[1]):
        t = X[u, k] - X[vs, k]
        acc = acc + t * t
    return np.sqrt(acc)


def kruskal(uv: np.ndarray, n: int) -> np.ndarray:
    parent = np.arange(n)

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    keep = []
    for i, e in enumerate(uv):
        a, b = find(int(e) >> 16), find(int(e) & 0xFFFF)
        if a != b:
            parent[a] = b
            keep.append(i)
    return np.array(keep, np.int64)


class NumpyBackend:
    def __init__(self, X):
        self.X = np.asarray(X, np.float64)

    def distances(self, x_ptr, n, d, lo, hi, layout=0):
        keys, vals = [], []
        for u in range(lo, hi):
            vs = np.arange(u + 1, n)
            keys.append(fold_lengths(self.X, u, vs).view(np.uint64))
            vals.append(((u << 16) | vs).astype(np.uint32))
        self.keys = np.concatenate(keys) if keys else np.zeros(0, np.uint64)
        self.vals = np.concatenate(vals) if vals else np.zeros(0, np.uint32)
        c = len(self.keys)
        return c, int(self.keys.min()) if c else 0, int(self.keys.max()) if c else 0

    def sample(self, s, count):
        s = min(s, count)
        i = np.arange(s, dtype=np.int64)
        return self.keys[(i * count) // s + (count // s) // 2] if s else np.zeros(0, np.uint64)

    def partition(self, spl, parts):
        b = np.searchsorted(np.asarray(spl, np.uint64), self.keys, side="right")
        order = np.argsort(b, kind="stable")
        counts = np.bincount(b, minlength=parts).astype(np.uint64)
        pmin = np.full(parts, np.iinfo(np.uint64).max, np.uint64)
        pmax = np.zeros(parts, np.uint64)
        for j in range(parts):
            sel = self.keys[b == j]
            if len(sel):
                pmin[j], pmax[j] = sel.min(), sel.max()
        sk = torch.from_numpy(self.keys[order].view(np.int64).copy())
        sv = torch.from_numpy(self.vals[order].view(np.int32).copy())
        return sk, sv, counts, pmin, pmax

    # ---- peer-memory exchange, emulated with POSIX shared memory between rank processes
    def partition_count(self, spl, parts):
        self._part = np.searchsorted(np.asarray(spl, np.uint64), self.keys, side="right")
        counts = np.bincount(self._part, minlength=parts).astype(np.uint64)
        pmin = np.full(parts, np.iinfo(np.uint64).max, np.uint64)
        pmax = np.zeros(parts, np.uint64)
        for j in range(parts):
            sel = self.keys[self._part == j]
            if len(sel):
                pmin[j], pmax[j] = sel.min(), sel.max()
        return counts, pmin, pmax

    def recv_peer(self, count, same_process):
        from multiprocessing import shared_memory
        self._own = [shared_memory.SharedMemory(create=True, size=max(8, 8 * count)),
                     shared_memory.SharedMemory(create=True, size=max(4, 4 * count))]
        self._count_recv = count
        return (self._own[0].name, self._own[1].name)

    def open_peer(self, desc, is_self, same_process):
        from multiprocessing import resource_tracker, shared_memory
        if is_self:
            shms = self._own
        else:
            shms = [shared_memory.SharedMemory(name=nm) for nm in desc]
            for m in shms:  # the owner unlinks it; this process only maps it
                resource_tracker.unregister(m._name, "shared_memory")
            self.__dict__.setdefault("_attached", []).extend(shms)
        return (np.ndarray(shms[0].size // 8, np.uint64, buffer=shms[0].buf),
                np.ndarray(shms[1].size // 4, np.uint32, buffer=shms[1].buf))

    def scatter_peers(self, parts, dst, offsets):
        order = np.argsort(self._part, kind="stable")
        ks, vs, bs = self.keys[order], self.vals[order], self._part[order]
        for b in range(parts):
            sel = bs == b
            c, o = int(sel.sum()), int(offsets[b])
            dst[b][0][o:o + c] = ks[sel]
            dst[b][1][o:o + c] = vs[sel]

    def _take_peer_recv(self):
        n = self._count_recv
        self.keys = np.ndarray(n, np.uint64, buffer=self._own[0].buf).copy()
        self.vals = np.ndarray(n, np.uint32, buffer=self._own[1].buf).copy()
        for m in self.__dict__.pop("_attached", []):
            m.close()
        for m in self._own:
            m.close()
            m.unlink()
        del self._own

    def recv(self, count):
        self.rk = torch.empty(count, dtype=torch.int64)
        self.rv = torch.empty(count, dtype=torch.int32)
        return self.rk, self.rv

    def sort_unique(self, count, kmin, kmax):
        if hasattr(self, "_own"):
            self._take_peer_recv()
        elif hasattr(self, "rk"):
            self.keys = self.rk.numpy().view(np.uint64).copy()
            self.vals = self.rv.numpy().view(np.uint32).copy()
        order = np.argsort(self.keys, kind="stable")
        self.keys, self.vals = self.keys[order], self.vals[order]
        self.D = np.unique(self.keys)
        return len(self.D), self.D.view(np.float64)

    def reduce_continue(self, n, count, offset, labels, target):
        """Kruskal in filtration order from the forest `labels` (root labels; None: singletons),
        stopping after `target` survivors; final labels = each vertex's tree minimum."""
        parent = np.arange(n) if labels is None else np.asarray(labels, np.int64).copy()

        def find(x):
            while parent[x] != x:
                parent[x] = parent[parent[x]]
                x = parent[x]
            return x

        keep = []
        for i, e in enumerate(self.vals):
            if len(keep) >= target:
                break
            a, b = find(int(e) >> 16), find(int(e) & 0xFFFF)
            if a != b:
                lo, hi = min(a, b), max(a, b)
                parent[hi] = lo  # the root stays the tree minimum
                keep.append(i)
        keep = np.array(keep, np.int64)
        g = offset + 1 + np.searchsorted(self.D, self.keys[keep])
        lab = np.array([find(v) for v in range(n)], np.uint32)
        return (self.vals[keep], g.astype(np.uint64), self.keys[keep].view(np.float64), lab)

    def reduce(self, n, count, offset):
        keep = kruskal(self.vals, n)
        g = offset + 1 + np.searchsorted(self.D, self.keys[keep])
        return self.vals[keep], g.astype(np.uint64), self.keys[keep].view(np.float64)

    def reduce_columns(self, uv, n):
        return kruskal(np.asarray(uv, np.uint32), n)
