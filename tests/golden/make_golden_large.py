"""Goldens for the FULL-size configs C4 and C5 from the REFERENCE ITSELF — its Kruskal path
(`ph0 oracle`, /root/reference/proj/tools/ph0_cli.cpp:73-80 -> kruskal_barcode,
/root/reference/proj/src/oracle.cpp:32-46, after the same pairwise_distances and
build_filtration as the reduce path, filtration.cpp:8-35).  That path yields the identical D
and the identical ordered barcode as reduce + extract_barcode (SURVEY.md Finding 4; the
reference's own acceptance.cpp:79-90 asserts the equivalence), and it is the only one of the
reference's two paths whose memory fits a single host at these sizes (48 B/edge).

Runs oracle/_ref/libph0ref.so (the unmodified reference sources, built by oracle/Makefile);
X comes from the oracle's own generator (oracle/ph0_oracle.c: orc_generate_cloud), never from
the product library.

    make -C oracle && python tests/golden/make_golden_large.py C4            # build container
    gpurun -- python tests/golden/make_golden_large.py C5 --out gpurun_out   # needs ~110 GB RAM

Writes <out>/ref_kruskal_<cfg>.npz: X sha256, |D|, sha256 of D's bit patterns, D head/tail,
the full ordered bars (death grades + lengths), the essential count, the reference's stage
seconds and wall time, and the host it ran on (CPU model, nproc, RAM).
"""
from __future__ import annotations

import argparse
import hashlib
import os
import platform
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT / "tests"))

import oracle_bridge as ob  # noqa: E402


def host_info() -> dict:
    cpu = platform.processor()
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    mem_kb = 0
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                mem_kb = int(line.split()[1])
    except OSError:
        pass
    return dict(cpu=cpu, nproc=os.cpu_count(), ram_gb=round(mem_kb / 2**20, 1))


def peak_rss_gb() -> float:
    try:
        for line in open("/proc/self/status"):
            if line.startswith("VmHWM"):
                return int(line.split()[1]) / 2**20
    except OSError:
        pass
    return float("nan")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=sorted(ob.CONFIGS))
    ap.add_argument("--out", default=str(HERE))
    ap.add_argument("--n", type=int, default=None, help="prefix of the config (testing)")
    a = ap.parse_args()
    assert ob.ref_available(), "build oracle/_ref first: make -C oracle ref"
    info = host_info()
    X = ob.config_cloud(a.config, a.n)
    n, d = X.shape
    k = n * (n - 1) // 2
    need_gb = 48 * k / 1e9
    print(f"{a.config}: N={n} d={d} K={k}; host {info}; reference Kruskal path needs "
          f"~{need_gb:.0f} GB", flush=True)
    if need_gb > 0.9 * info["ram_gb"] * 2**30 / 1e9:
        print(f"SKIP: {need_gb:.0f} GB needed > 0.9 x {info['ram_gb']} GiB RAM", flush=True)
        return 2
    t0 = time.perf_counter()
    r = ob.ref_h0(X, mode=1, want_scale=True)
    wall = time.perf_counter() - t0
    D = r["scale"]
    tag = a.config if a.n is None else f"{a.config}_n{a.n}"
    out = {
        "n": np.uint64(n), "d": np.uint64(d), "k": np.uint64(k),
        "X_sha256": np.frombuffer(hashlib.sha256(np.asfortranarray(X).tobytes()).digest(),
                                  np.uint8),
        "n_scale": np.uint64(len(D)),
        "scale_sha256": np.frombuffer(hashlib.sha256(D.tobytes()).digest(), np.uint8),
        "scale_head": D[:64].copy(), "scale_tail": D[-64:].copy(),
        "death_grade": r["death_grade"], "death_length": r["death_length"],
        "essential": np.uint64(r["essential"]),
        "ref_stage_seconds": r["stage_seconds"], "ref_wall_s": np.float64(wall),
        "ref_peak_rss_gb": np.float64(peak_rss_gb()),
        "host_cpu": np.array(info["cpu"]), "host_nproc": np.uint64(info["nproc"] or 0),
        "host_ram_gb": np.float64(info["ram_gb"]),
    }
    path = Path(a.out) / f"ref_kruskal_{tag}.npz"
    np.savez_compressed(path, **out)
    print(f"{tag}: |D|={len(D)} bars={len(r['death_grade'])} essential={r['essential']} "
          f"wall={wall:.1f}s stages={np.round(r['stage_seconds'], 2).tolist()} "
          f"peak_rss={peak_rss_gb():.1f}GB -> {path}", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
