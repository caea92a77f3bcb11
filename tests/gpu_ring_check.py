"""Subprocess helper for tests/test_gpu_variants.py: the host-output paths of ph0b_run_host
(bucketed at K >= 2^26, one compressed slice below) under the D2H knobs set in the environment (ring size / piece size of the
streamed compressed D, or uncompressed D) must equal the library-allocated path bit for bit,
including raw chunks (gaps >= 2^32 between consecutive lengths) and a too-small D buffer."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import paper_2203_02527_b200 as pkg  # noqa: E402


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def main():
    rng = np.random.default_rng(11)
    far = rng.normal(size=(12000, 3))
    far[:6000] += 1e6  # one huge gap in D: a raw chunk
    far_mid = rng.normal(size=(4000, 3))
    far_mid[:2000] += 1e6
    # K >= 2^26: bucketed path; C3 (3.4e7) and far_mid (8e6): one compressed slice after the
    # pipeline
    clouds = [pkg.config_cloud("C4", 12000), far, pkg.config_cloud("C3"), far_mid]
    ctx = pkg.Context(0)
    for X in clouds:
        n = X.shape[0]
        bc = pkg.h0_barcode(X)
        for rep in range(2):  # the ring's slot generations carry over between calls
            dg = np.empty(n, np.uint64)
            dl = np.empty(n)
            sc = pkg.PinnedArray(len(bc.scale) + 7)
            sc.array[:] = -1.0
            nf, ess, ns, t = ctx.run_host(np.asfortranarray(X), dg, dl, sc.array)
            assert nf == n - 1 and ess == 1 and ns == len(bc.scale), (nf, ess, ns)
            assert np.array_equal(dg[:nf], bc.death_grade)
            assert np.array_equal(bits(dl[:nf]), bits(bc.death_length))
            assert np.array_equal(bits(sc.array[:ns]), bits(bc.scale))
            assert np.all(sc.array[ns:] == -1.0)  # nothing written past |D|
            sc.free()
        small = np.empty(len(bc.scale) - 1000)
        try:
            ctx.run_host(np.asfortranarray(X), dg, dl, small)
            raise AssertionError("a D buffer smaller than |D| must be rejected")
        except pkg.Ph0bError as e:
            assert e.code == 7, e  # PH0B_ERR_CAPACITY
    ctx.close()
    print("OK")


if __name__ == "__main__":
    main()
