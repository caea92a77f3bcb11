"""CPU, world_size 2 and 3 over gloo: the multi-GPU orchestration of sharded.py (row split,
sampled splitters, stable partition + all-to-all-v, grade offsets, candidate gather, final
column reduction) reproduces the oracle's D and ordered bars bit for bit."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, X, out, exchange="peer"):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), PH0B_EXCHANGE=exchange)
    import torch.distributed as dist

    from cpu_backend import NumpyBackend
    from paper_2203_02527_b200.sharded import TorchComm, h0_barcode_sharded

    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = h0_barcode_sharded(0, X.shape[0], X.shape[1], TorchComm(), NumpyBackend(X))
    D = res.scale_local
    out.put((rank, res.scale_offset, np.asarray(D).copy(), res.death_grade, res.death_length,
             res.essential_count, res.edges_local))
    dist.barrier()
    dist.destroy_process_group()


def run_world(X, world, exchange="peer"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, X, q, exchange))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world,exchange", [(2, "peer"), (3, "peer"), (2, "collective"),
                                            (3, "collective")])
def test_sharded_orchestration_matches_oracle(world, exchange):
    """exchange='peer': every rank stores its parts straight into the receive buffers of the
    other ranks (shared memory here, NVLink P2P through CUDA IPC on GPUs); 'collective': send
    buffer + all-to-all-v."""
    import oracle_bridge as ob

    rng = np.random.default_rng(world)
    X = np.vstack([rng.normal(0, 0.1, size=(60, 3)), rng.normal(3, 0.1, size=(50, 3)),
                   rng.integers(0, 4, size=(40, 3)).astype(np.float64)])  # clusters + ties
    res = run_world(X, world, exchange)
    ref = ob.oracle_filtration_and_bars(X)
    D = np.concatenate([r[2] for r in res])
    assert [r[1] for r in res] == list(np.cumsum([0] + [len(r[2]) for r in res])[:-1])
    assert np.array_equal(D.view(np.uint64), ref["scale"].view(np.uint64))
    r0 = res[0]
    assert np.array_equal(r0[3], ref["death_grade"])
    assert np.array_equal(r0[4].view(np.uint64), ref["death_length"].view(np.uint64))
    assert r0[5] == ref["essential"]
    assert sum(r[6] for r in res) == X.shape[0] * (X.shape[0] - 1) // 2


def test_sharded_empty_key_ranges():
    """Two distinct lengths and three ranks: at least one rank's key range is empty, and the
    forest must pass through it unchanged (world_size 3 over gloo)."""
    import oracle_bridge as ob

    X = np.random.default_rng(5).integers(0, 2, size=(80, 1)).astype(np.float64)
    res = run_world(X, 3)
    ref = ob.oracle_filtration_and_bars(X)
    D = np.concatenate([r[2] for r in res])
    assert np.array_equal(D.view(np.uint64), ref["scale"].view(np.uint64))
    assert np.array_equal(res[0][3], ref["death_grade"])
    assert res[0][5] == ref["essential"]
    assert min(len(r[2]) for r in res) == 0  # the case this test is about


def test_row_ranges_balanced():
    from paper_2203_02527_b200.sharded import row_ranges
    for n, p in ((10, 3), (1000, 8), (65536, 8), (5, 8)):
        rr = row_ranges(n, p)
        assert rr[0][0] == 0 and rr[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(rr, rr[1:]))
        cnt = [sum(n - 1 - u for u in range(lo, hi)) for lo, hi in rr] if n < 5000 else None
        if cnt and n >= 100:
            assert max(cnt) - min(cnt) <= 2 * n
