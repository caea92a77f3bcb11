"""GPU: the peer-memory exchange of sharded.py across PROCESSES (CUDA IPC handles), with two
rank processes sharing the single B200 of the tests and gloo carrying the host-side
all-gathers.  Each rank's partition kernel stores its parts straight into the other
process's receive buffer through the IPC mapping; no rank's kernel waits on another's (the
ordering is the host barrier after each scatter).  Bit-exact D and bars vs the oracle."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, X, out):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), PH0B_EXCHANGE="peer")
    import torch
    import torch.distributed as dist

    from paper_2203_02527_b200.sharded import DeviceBackend, TorchComm, h0_barcode_sharded

    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, d = X.shape
    x = torch.from_numpy(np.asfortranarray(X).ravel(order="F").copy()).cuda()
    be = DeviceBackend(0)
    res = h0_barcode_sharded(x.data_ptr(), n, d, TorchComm(), be)
    out.put((rank, res.scale_offset, res.scale_local.cpu().numpy().copy(), res.death_grade,
             res.death_length, res.essential_count))
    dist.barrier()  # nobody unmaps a buffer a peer may still be reading
    be.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ipc_peer_exchange_matches_oracle(world):
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_bridge as ob

    import paper_2203_02527_b200 as pkg
    X = pkg.config_cloud("C2", 1500)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, X, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref = ob.oracle_filtration_and_bars(X)
    D = np.concatenate([r[2] for r in res])
    assert np.array_equal(D.view(np.uint64), ref["scale"].view(np.uint64))
    assert [r[1] for r in res] == list(np.cumsum([0] + [len(r[2]) for r in res])[:-1])
    assert np.array_equal(res[0][3], ref["death_grade"])
    assert np.array_equal(res[0][4].view(np.uint64), ref["death_length"].view(np.uint64))
    assert res[0][5] == ref["essential"]


def test_ipc_peer_exchange_c4_scale():
    """C4 (5.4e8 edges) as 2 rank processes on the one B200: each partition kernel stores
    ~3 GB straight into the other process's receive buffer through the IPC mapping; the
    concatenated D slices and rank 0's bars equal the single-GPU device path bit for bit."""
    import paper_2203_02527_b200 as pkg
    X = pkg.config_cloud("C4")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, X, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    bc = pkg.h0_barcode(X)
    D = np.concatenate([r[2] for r in res])
    assert np.array_equal(D.view(np.uint64), bc.scale.view(np.uint64))
    assert np.array_equal(res[0][3], bc.death_grade)
    assert np.array_equal(res[0][4].view(np.uint64), bc.death_length.view(np.uint64))
    assert res[0][5] == bc.essential_count
