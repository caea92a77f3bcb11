"""Subprocess helper for tests/test_gpu_variants.py: runs the GPU path under the knobs set in
the environment (PH0B_MAX_PASSES, PH0B_RANK) and checks bit-exact parity with the oracle."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402

import oracle_bridge as ob  # noqa: E402
import paper_2203_02527_b200 as pkg  # noqa: E402


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def main():
    rng = np.random.default_rng(99)
    clouds = [pkg.config_cloud("C1"), pkg.config_cloud("C2", 1200),
              rng.uniform(0, 1, size=(700, 3)),
              np.array([[x, y] for x in range(30) for y in range(30)], np.float64),
              rng.integers(0, 6, size=(500, 2)).astype(np.float64)]
    for X in clouds:
        bc = pkg.h0_barcode(X)
        ref = ob.oracle_filtration_and_bars(X)
        assert bc.essential_count == ref["essential"]
        assert np.array_equal(bc.death_grade, ref["death_grade"])
        assert np.array_equal(bits(bc.death_length), bits(ref["death_length"]))
        assert np.array_equal(bits(bc.scale), bits(ref["scale"]))
        u, v, g, sc = pkg.build_filtration(X)
        assert np.array_equal(u, ref["u"]) and np.array_equal(v, ref["v"])
        assert np.array_equal(g, ref["grade"])
    # tie order across many sort tiles decides the surviving columns and their supports
    g = np.array([[x, y] for x in range(64) for y in range(64)], np.float64)
    ref = ob.reduce_sparse(ob.filtration(g), stop_at_spanning=True)
    cols, lo, hi = pkg.reduced_supports(g)
    assert np.array_equal(cols, ref["columns"]) and np.array_equal(lo, ref["rows_lo"])
    assert np.array_equal(hi, ref["rows_hi"])
    print("OK")


if __name__ == "__main__":
    main()
