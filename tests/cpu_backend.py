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

    def recv(self, count):
        self.rk = torch.empty(count, dtype=torch.int64)
        self.rv = torch.empty(count, dtype=torch.int32)
        return self.rk, self.rv

    def sort_unique(self, count, kmin, kmax):
        if hasattr(self, "rk"):
            self.keys = self.rk.numpy().view(np.uint64).copy()
            self.vals = self.rv.numpy().view(np.uint32).copy()
        order = np.argsort(self.keys, kind="stable")
        self.keys, self.vals = self.keys[order], self.vals[order]
        self.D = np.unique(self.keys)
        return len(self.D), self.D.view(np.float64)

    def reduce(self, n, count, offset):
        keep = kruskal(self.vals, n)
        g = offset + 1 + np.searchsorted(self.D, self.keys[keep])
        return self.vals[keep], g.astype(np.uint64), self.keys[keep].view(np.float64)

    def reduce_columns(self, uv, n):
        return kruskal(np.asarray(uv, np.uint32), n)
