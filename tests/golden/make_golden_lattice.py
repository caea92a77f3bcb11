"""Reduced supports of the 128 x 128 integer lattice (N = 16384, K = 1.34e8 edges, massive
exact ties across thousands of sort tiles) from the C oracle's sparse column reduction
(oracle/ph0_oracle.c orc_reduce_sparse, pinned to the reference's own reduced matrices on its
250 acceptance clouds by tests/test_oracle_cpu.py).  The claimed lows depend on the (u, v)
order inside every tie group, so they expose any instability of the GPU radix sort's ranking.
    make -C oracle && python tests/golden/make_golden_lattice.py
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1] / "tests"))

import oracle_bridge as ob  # noqa: E402


def main():
    X = np.array([[x, y] for x in range(128) for y in range(128)], np.float64)
    f = ob.filtration(X)
    sp = ob.reduce_sparse(f, stop_at_spanning=True)
    assert len(sp["columns"]) == X.shape[0] - 1
    np.savez_compressed(HERE / "lattice128_supports.npz", columns=sp["columns"],
                        rows_lo=sp["rows_lo"], rows_hi=sp["rows_hi"],
                        death_grade=sp["death_grade"], n_scale=np.uint64(len(f["scale"])))
    print("wrote", HERE / "lattice128_supports.npz", len(sp["columns"]), "columns")


if __name__ == "__main__":
    main()
