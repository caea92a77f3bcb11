"""Generate tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref/libph0ref.so, the
unmodified /root/reference/proj sources built by oracle/Makefile).  Run in the build
container (where /root/reference exists):

    make -C oracle ref && python tests/golden/make_golden.py

The fixtures travel with the repo, so GPU parity tests never need /root/reference.
Every case records X, D (scale), the ordered bars, the claimed low of every surviving
column and the essential count.  Large D arrays are stored as sha256 + endpoints.
"""
from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle_bridge as ob  # noqa: E402


def hand_clouds():
    """Hand-built clouds of the reference's own unit tests."""
    return {
        "collinear3": [[0, 0], [1, 0], [3, 0]],              # test_filtration.cpp:29, data/collinear3.txt
        "triangle345": [[0, 0], [3, 4]],                      # test_filtration.cpp:33-39
        "ties_1d": [[0.0], [5.0], [10.0]],                    # test_filtration.cpp:69-82
        "unit_square": [[0, 0], [1, 0], [0, 1], [1, 1]],      # test_reduction.cpp:115-123
        "two_clusters": [[0, 0], [0.1, 0], [10, 0], [10.1, 0]],  # test_reduction.cpp:125-134
        "coincident": [[1, 1], [1, 1], [2, 2]],               # test_reduction.cpp:136-145
        "two_points": [[0, 0], [1, 0]],                       # test_reduction.cpp:95-103
        "single": [[1, 2]],                                   # test_filtration.cpp:61-67
    }


def ref_case(X):
    X = np.asarray(X, np.float64).reshape(len(X), -1) if len(X) else np.zeros((0, 2))
    r = ob.ref_h0(X, mode=0, want_scale=True, want_lows=True)
    return dict(X=X, scale=r["scale"], death_grade=r["death_grade"],
                death_length=r["death_length"], claimed_low=r["claimed_low"],
                essential=np.uint64(r["essential"]))


def main():
    assert ob.ref_available(), "build oracle/_ref first: make -C oracle ref"
    import paper_2203_02527_b200 as pkg

    cases = {}
    for name, pts in hand_clouds().items():
        cases[name] = ref_case(pts)
    cases["empty"] = ref_case(np.zeros((0, 2)))
    # acceptance.cpp:40-48 — 200 clouds, N = 2 + i%63, d = 1 + i%3, seed 0xACCE57 + i
    for i in range(200):
        n, d, seed = 2 + i % 63, 1 + i % 3, 0xACCE57 + i
        X = ob.uniform_cloud(n, d, seed)
        cases[f"accept_{i:03d}"] = ref_case(X)
    # coincident-heavy / lattice clouds (duplicate-distance stress)
    g = np.array([[x, y] for x in range(8) for y in range(8)], np.float64)
    cases["lattice_8x8"] = ref_case(g)
    cases["all_same_5"] = ref_case(np.ones((5, 3)))
    flat = {}
    for name, c in cases.items():
        for k, v in c.items():
            flat[f"{name}/{k}"] = v
    np.savez_compressed(HERE / "ref_small.npz", **flat)

    # configs C1, C2 of BASELINE.json at full size, C3 prefix: bars + lows + D digest
    big = {}
    for name, n in (("C1", None), ("C2", None), ("C3", 2048)):
        X = pkg.config_cloud(name, n)
        r = ob.ref_h0(X, mode=0, want_scale=True, want_lows=True)
        D = r["scale"]
        tag = name if n is None else f"{name}_n{n}"
        big[f"{tag}/n"] = np.uint64(X.shape[0])
        big[f"{tag}/d"] = np.uint64(X.shape[1])
        big[f"{tag}/X_sha256"] = np.frombuffer(
            hashlib.sha256(np.asfortranarray(X).tobytes()).digest(), np.uint8)
        big[f"{tag}/scale_sha256"] = np.frombuffer(hashlib.sha256(D.tobytes()).digest(), np.uint8)
        big[f"{tag}/n_scale"] = np.uint64(len(D))
        big[f"{tag}/scale_head"] = D[:64].copy()
        big[f"{tag}/scale_tail"] = D[-64:].copy()
        big[f"{tag}/death_grade"] = r["death_grade"]
        big[f"{tag}/death_length"] = r["death_length"]
        big[f"{tag}/claimed_low"] = r["claimed_low"]
        big[f"{tag}/essential"] = np.uint64(r["essential"])
        big[f"{tag}/ref_stage_seconds"] = r["stage_seconds"]
        print(tag, "n_scale", len(D), "bars", len(r["death_grade"]), "ref seconds",
              r["stage_seconds"].sum())
    np.savez_compressed(HERE / "ref_configs.npz", **big)
    print("wrote", HERE / "ref_small.npz", HERE / "ref_configs.npz")


if __name__ == "__main__":
    main()
