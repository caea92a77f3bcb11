"""Whole reduced matrices from the REFERENCE ITSELF (oracle/_ref, the unmodified sources) for
the clouds of its acceptance suite, /root/reference/proj/tests/acceptance.cpp:
  * cloud_suite() (:38-47): 200 clouds, N = 2 + i%63, d = 1 + i%3, seed 0xACCE57 + i
    (pivoting_equivalence, :124-133, runs all 200 with pivoting on and off);
  * parallel_determinism() (:106-122): the first 50 of them with seed ^ (0x50D0 << 32),
    reduced with workers in {2, 3, 4, 6} and compared with the sequential reduce.
Per cloud: X and the nonzero columns of the reduced matrix (column index, the two rows) under
the default options, and the reference's ReductionStats.  The script also asserts the
reference's own claim on every cloud — identical reduced matrices for every option set the
acceptance suite uses — so the fixture records one matrix per cloud.

    make -C oracle && python tests/golden/make_golden_reduced.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1] / "tests"))

import oracle_bridge as ob  # noqa: E402

OPTION_SETS = [(True, 1), (False, 1), (True, 2), (True, 3), (True, 4), (True, 6), (False, 3)]


def suite():
    for i in range(200):
        yield f"accept_{i:03d}", 2 + i % 63, 1 + i % 3, 0xACCE57 + i
    for i in range(50):
        yield f"pardet_{i:02d}", 2 + i % 63, 1 + i % 3, (0xACCE57 + i) ^ (0x50D0 << 32)


def main():
    assert ob.ref_available(), "build oracle/_ref first: make -C oracle ref"
    out = {}
    for name, n, d, seed in suite():
        X = ob.uniform_cloud(n, d, seed)
        base = None
        for piv, w in OPTION_SETS:
            cols, lo, hi, st = ob.ref_reduced_matrix(X, piv, w)
            if base is None:
                base = (cols, lo, hi, st)
            else:
                assert all(np.array_equal(a, b) for a, b in zip((cols, lo, hi), base[:3])), \
                    (name, piv, w)
        out[f"{name}/X"] = X
        out[f"{name}/seed"] = np.uint64(seed)
        out[f"{name}/columns"] = base[0]
        out[f"{name}/rows_lo"] = base[1]
        out[f"{name}/rows_hi"] = base[2]
        out[f"{name}/stats"] = base[3]
    np.savez_compressed(HERE / "ref_reduced.npz", **out)
    print("wrote", HERE / "ref_reduced.npz", len(out) // 6, "clouds")


if __name__ == "__main__":
    main()
