#!/usr/bin/env python
"""Benchmark of the B200 H0 barcode pipeline (BASELINE.json metric: edges/s = K / wall).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]

A step is one full pass of the hot path (pairwise distances -> sort -> unique/D -> boundary
matrix -> column reduction -> barcode collect) over the workload's K = N(N-1)/2 edges.
* value: device time with the cloud already resident in HBM and outputs left in HBM
  (CUDA events on the pipeline stream, barrier + synchronize around the timed region,
  max over ranks).  Inputs (keys/values: 25.8 GB at C5) are far larger than L2.
* e2e:   the same metric through the public C ABI (ph0b_run_host) with host buffers: the
  H2D copy of X from pinned memory and the D2H copy of the bars and of D (|D| doubles)
  into pinned memory are inside the timed region.
* e2e_dropin: the drop-in entry point ph0b_h0_barcode itself (library-allocated result).
* --impl reference: the reference's own CPU implementation (oracle/_ref, the unmodified
  /root/reference sources built here; else the C port in oracle/) on a bounded sample
  of the same workload, rank 0 only; X from the oracle's generator (no product code).
* --gpus N without torchrun: the in-process multi-GPU path of the C ABI (ph0b_options.n_gpus);
  under torchrun (one process per GPU): the sharded pipeline of sharded.py.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "end-to-end H0 barcode time (s) and edges/s vs N at 1/2/4/8 B200 vs CPU ref"
UNIT = "edges/s"
WORKLOADS = {
    "C1": "N=500 d=2 two Gaussian clusters",
    "C2": "N=2000 d=3 noisy circle + uniform background",
    "C3": "N=8192 d=16 mixture of 10 Gaussians",
    "C4": "N=32768 d=3 uniform cube (generate_uniform_cloud seed 4)",
    "C5": "N=65536 d=8 mixture of 32 Gaussians",
}
# Reference arm and cpu_baseline: the reference's full CPU path on the SAME bounded sample
# (the first 3000 points of the workload cloud: 4.5e6 edges, ~3 s of single-core work per
# step).  The full configs are out of reach per step: the reduce path needs
# K*(ceil(N/64)*8+56) B (2.2 TB at C4), and even the reference's Kruskal path takes ~82 s at
# C4 and minutes at C5 (48 B/edge of RAM); those full-config runs are recorded once with the
# goldens (tests/golden/ref_kruskal_C*.npz) and quoted in `reference_full`.
REF_SAMPLE_N = 3000
REF_TIME_CAP_S = 30.0    # per-step cap of the reference arm (stated in the JSON line)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return float(j.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(
                        ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                         "--format=csv,noheader,nounits"], capture_output=True, text=True,
                        timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def host_info():
    cpu, mem_kb = "unknown", 0
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu = line.split(":", 1)[1].strip()
                break
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                mem_kb = int(line.split()[1])
    except OSError:
        pass
    return {"cpu_model": cpu, "nproc": os.cpu_count(), "ram_gb": round(mem_kb / 2**20, 1)}


def reference_full_records():
    """Full-config runs of the reference's Kruskal path (`ph0 oracle`, ph0_cli.cpp:73-80),
    recorded when the goldens were made (tests/golden/make_golden_large.py)."""
    import numpy as np
    out = []
    for cfg in ("C4", "C5"):
        p = ROOT / "tests" / "golden" / f"ref_kruskal_{cfg}.npz"
        if not p.exists():
            continue
        z = np.load(p)
        k = int(z["k"])
        wall = float(z["ref_wall_s"])
        out.append({"config": cfg, "kind": "reference-kruskal-full", "edges": k,
                    "seconds": round(wall, 1), "value": k / wall, "unit": UNIT, "cores": 1,
                    "host": {"cpu_model": str(z["host_cpu"]), "nproc": int(z["host_nproc"]),
                             "ram_gb": float(z["host_ram_gb"])},
                    "stage_seconds": [round(float(x), 2) for x in z["ref_stage_seconds"]]})
    return out


def cpu_reference_sample(cfg_name: str, n_sample: int):
    """The reference's full CPU path (oracle/_ref = the unmodified reference sources; else the
    C port) on the first n_sample points of the config cloud, X built by the oracle's own
    generator.  Returns (seconds, K, kind)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_bridge as ob  # CPU checker / baseline only

    Xs = ob.config_cloud(cfg_name)[:n_sample]
    k = n_sample * (n_sample - 1) // 2
    t0 = time.perf_counter()
    if ob.ref_available():
        ob.ref_h0(Xs, mode=0, want_scale=True)
        kind = "reference"
    else:
        ob.oracle_filtration_and_bars(Xs, reduction_limit=1 << 30)
        kind = "port"
    return time.perf_counter() - t0, k, kind


def cpu_baseline_record(cfg_name, n):
    ns = min(REF_SAMPLE_N, n)
    s, k, kind = cpu_reference_sample(cfg_name, ns)
    return {"value": k / s, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"full reference path (pairwise_distances..extract_barcode, 1 thread) on "
                      f"the first {ns} points of {cfg_name} ({k} edges, {s:.2f} s)",
            "host": host_info(), "reference_full": reference_full_records()}


def run_reference_arm(args, cfg_name):
    """The reference's own CPU implementation only: X from the oracle's generator, the timed
    region calls nothing but oracle/_ref (no product library is loaded in this arm)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_bridge as ob

    n, d = ob.CONFIGS[cfg_name]["n"], ob.CONFIGS[cfg_name]["d"]
    ns = min(REF_SAMPLE_N, n)
    for _ in range(args.warmup):
        cpu_reference_sample(cfg_name, ns)
    secs = []
    kind = "reference"
    k = ns * (ns - 1) // 2
    for _ in range(args.steps):
        s, k, kind = cpu_reference_sample(cfg_name, ns)
        secs.append(s)
    total = sum(secs)
    value = k * len(secs) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(secs),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{cfg_name}: {WORKLOADS[cfg_name]}", "n": n, "d": d,
                   "sample": f"first {ns} points of the workload cloud per step (the full "
                             f"config exceeds the {REF_TIME_CAP_S:.0f} s per-step cap; "
                             f"full-config Kruskal-path runs in cpu_baseline.reference_full)",
                   "parallelism": "cpu, 1 thread (reference path is single-threaded; its "
                                  "reduce_parallel is 25-156x slower)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": kind,
                         "sample": f"full reference path (pairwise_distances..extract_barcode) "
                                   f"on the first {ns} points of {cfg_name}",
                         "host": host_info(), "reference_full": reference_full_records()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def scale_checksum(t):
    """Order-sensitive checksum of D's bit patterns: sum_i bits_i * (2i + 1) mod 2^64
    (int64 wrap-around), in chunks; the same value on a device or a host tensor."""
    import torch
    acc = torch.zeros((), dtype=torch.int64, device=t.device)
    step = 1 << 27
    for a in range(0, t.numel(), step):
        c = t[a:a + step]
        w = torch.arange(a, a + c.numel(), device=t.device, dtype=torch.int64) * 2 + 1
        acc += (c * w).sum()
    return int(acc.item()) & ((1 << 64) - 1)


def load_traffic():
    p = ROOT / "profiles" / "ncu_summary.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:
            return None
    return None


def run_sharded(args, cfg_name):
    """N > 1 (torchrun, one rank per GPU): the sharded pipeline of sharded.py — rows split
    across ranks, splitter partition whose kernel stores each part straight into its
    destination rank's receive buffer over NVLink (CUDA IPC; PH0B_EXCHANGE=collective: send
    buffer + NCCL all-to-all-v instead), D sharded, the column reduction handed from rank to rank.  Total
    work fixed as N grows (strong scaling of the C5 problem)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2203_02527_b200 as pkg
    from paper_2203_02527_b200.sharded import (DeviceBackend, TorchComm, exchange_mode,
                                               h0_barcode_sharded)

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = TorchComm()
    X = pkg.config_cloud(cfg_name)
    n, d = X.shape
    k = n * (n - 1) // 2
    be = DeviceBackend(local)
    xcm = np.asfortranarray(X).ravel(order="F").copy()
    xdev = torch.from_numpy(xcm).to(f"cuda:{local}")

    def sync_all():
        torch.cuda.synchronize(local)
        dist.barrier()

    def timed(fn, steps):
        sync_all()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = None
        for _ in range(steps):
            out = fn()
        torch.cuda.synchronize(local)  # all streams (ph0b contexts, NCCL) drained
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        t = torch.tensor([ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), out

    step = lambda: h0_barcode_sharded(xdev.data_ptr(), n, d, comm, be)  # noqa: E731
    for _ in range(args.warmup):
        step()
    l0 = be.launches
    with ClockSampler(local) as clk:
        ms, res = timed(step, args.steps)
    launches0 = be.launches - l0
    value = k * args.steps / (ms / 1e3)
    sort_s, passes, sort_edges = be.last_sort

    # e2e: pinned host X -> device, sharded pipeline, D slice + bars back to pinned host memory
    xin = pkg.PinnedArray(n * d)
    xin.array[:] = xcm
    dpin = pkg.PinnedArray(max(res.n_scale_local, 1) * 2, np.float64)
    bars = pkg.PinnedArray(2 * n, np.float64)
    xbuf = torch.empty(n * d, dtype=torch.float64, device=f"cuda:{local}")

    moved = [0]

    def e2e_step():
        xbuf.copy_(torch.from_numpy(xin.array), non_blocking=True)
        r = h0_barcode_sharded(xbuf.data_ptr(), n, d, comm, be)
        # the D slice leaves compressed through the ring, as ph0b_run_host ships D
        moved[0] = be.scale_to_host(r.scale_local.data_ptr(), r.n_scale_local, dpin.array)
        if r.death_grade is not None:
            bars.array[: len(r.death_length)] = r.death_length
        return r

    e2e_steps = args.e2e_steps or max(1, min(args.steps, 5))
    e2e_step()
    e2e_ms, r2 = timed(e2e_step, e2e_steps)
    d2h = moved[0] + (16 * (n - 1) if rank == 0 else 0)  # this rank's bytes
    peak, peak_kind = peaks()
    alg = (24 * max(passes, 1) + 16) * sort_edges
    achieved = alg / sort_s / 1e9
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg_name}: {WORKLOADS[cfg_name]}", "n": n, "d": d,
                       "edges": k, "parallelism": f"dp{ws} (row shards + splitter exchange)",
                       "exchange": exchange_mode(comm, be),
                       "l2": "inputs larger than L2", "n_scale": res.n_scale_total,
                       "bars": int(len(res.death_grade))},
            "e2e": {"value": k * e2e_steps / (e2e_ms / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": n * d * 8, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_ms / e2e_steps, "steps": e2e_steps,
                    "api": "sharded.h0_barcode_sharded (pinned host X; D slice per rank to pinned host)"},
            "roofline": {"kernel": "shard sort+unique (rank 0: onesweep passes + unique)",
                         "bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": None,
                         "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                         "alg_bytes_per_launch": alg, "passes": passes},
            "cpu_baseline": None, "clocks": clk.summary(), "gpu_launches": launches0 or None,
        }
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_record(cfg_name, n)
        print(json.dumps(line), flush=True)
    for a in (xin, dpin, bars):
        a.free()
    be.close()
    dist.barrier()
    dist.destroy_process_group()


def run_inproc_multi(args, cfg_name):
    """--gpus N without torchrun: the in-process multi-GPU path behind the C ABI
    (ph0b_options.n_gpus, csrc/multi.cpp) — one process, one host thread and context per GPU,
    the partition kernel storing every part into its destination GPU's receive buffer.
    value: X from the host, bars back, D left on the GPUs (PH0B_FLAG_NO_SCALE); e2e: the
    same call with D streamed into a host buffer.  Host wall clock of the blocking call.
    --virtual: all ranks on GPU 0 (a correctness/overhead run on a one-GPU box, not a
    scaling number)."""
    import ctypes as C

    import numpy as np
    import torch

    import paper_2203_02527_b200 as pkg

    P = args.gpus
    have = torch.cuda.device_count()
    if have < P and not args.virtual:
        raise SystemExit(f"--gpus {P} needs {P} visible GPUs (found {have}); --virtual runs "
                         f"the ranks on GPU 0")
    devices = [0] * P if args.virtual else list(range(P))
    X = pkg.config_cloud(cfg_name)
    n, d = X.shape
    k = n * (n - 1) // 2
    L = pkg.lib()
    Xc = np.asfortranarray(X)
    dg = pkg.PinnedArray(n, np.uint64)
    dl = pkg.PinnedArray(n, np.float64)
    sc = pkg.PinnedArray(k, np.float64)
    nf, ess, ns = C.c_uint64(), C.c_uint64(), C.c_uint64()
    t = pkg.ph0b.StageTimes()

    def call(with_scale):
        opt = pkg.ph0b._opts(0, 0 if with_scale else pkg.ph0b.FLAG_NO_SCALE, 1, True, devices)
        rc = L.ph0b_h0_barcode_into(C.c_void_p(Xc.ctypes.data), n, d, pkg.ph0b.COL_MAJOR,
                                    C.byref(opt), C.c_void_p(dg.array.ctypes.data),
                                    C.c_void_p(dl.array.ctypes.data), C.byref(nf), C.byref(ess),
                                    C.c_void_p(sc.array.ctypes.data) if with_scale else None,
                                    k if with_scale else 0, C.byref(ns), C.byref(t))
        if rc:
            raise RuntimeError(L.ph0b_last_error().decode())

    def timed(with_scale, steps):
        for _ in range(args.warmup):
            call(with_scale)
        t0 = time.perf_counter()
        for _ in range(steps):
            call(with_scale)
        return (time.perf_counter() - t0) * 1e3 / steps

    with ClockSampler(0) as clk:
        ms = timed(False, args.steps)
    e2e_steps = args.e2e_steps or max(1, min(args.steps, 5))
    e2e_ms = timed(True, e2e_steps)
    line = {
        "metric": METRIC, "value": k / (ms / 1e3), "unit": UNIT, "n_gpus": P,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg_name}: {WORKLOADS[cfg_name]}", "n": n, "d": d, "edges": k,
                   "parallelism": f"in-process x{P} ({'virtual ranks on GPU 0' if args.virtual else 'GPUs ' + str(devices)})",
                   "api": "ph0b_h0_barcode_into with ph0b_options.n_gpus/devices",
                   "n_scale": int(ns.value), "bars": int(nf.value)},
        "e2e": {"value": k / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms,
                "steps": e2e_steps, "h2d_bytes_per_step": n * d * 8 * P,
                "d2h_bytes_per_step": int(t.d2h_bytes)},
        "roofline": None, "cpu_baseline": None, "clocks": clk.summary(),
        "gpu_launches": int(L.ph0b_last_launch_count()) or None,
    }
    print(json.dumps(line), flush=True)
    for a in (dg, dl, sc):
        a.free()
    L.ph0b_release_resources()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dropin", action="store_true",
                    help="skip the timing of the drop-in entry point ph0b_h0_barcode")
    ap.add_argument("--sharded", action="store_true",
                    help="use the sharded multi-GPU pipeline even at N=1 (torchrun)")
    ap.add_argument("--virtual", action="store_true",
                    help="--gpus N without torchrun on a box with fewer GPUs: the in-process "
                         "ranks share GPU 0")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: run N independent single-GPU replicas instead of the sharded path")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg_name = args.config

    if args.impl == "reference":
        run_reference_arm(args, cfg_name)
        return

    import numpy as np
    import torch

    import paper_2203_02527_b200 as pkg

    ws, rank, local = dist_env()
    if ws == 1 and args.gpus > 1 and not args.sharded:
        run_inproc_multi(args, cfg_name)
        return
    if (ws > 1 and not args.replicas) or args.sharded:
        run_sharded(args, cfg_name)
        return
    dist = None
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = local if ws > 1 else 0
    torch.cuda.set_device(device)

    X = pkg.config_cloud(cfg_name)
    n, d = X.shape
    k = n * (n - 1) // 2
    ctx = pkg.Context(device)
    ctx.reserve(n, d)
    stream = torch.cuda.Stream(device=device)
    xdev = torch.from_numpy(np.asfortranarray(X).ravel(order="F").copy()).to(f"cuda:{device}")

    def barrier():
        torch.cuda.synchronize(device)
        if dist is not None:
            dist.barrier()

    # ---- device-resident timing (value) ------------------------------------------------------
    for _ in range(args.warmup):
        ctx.run_device(xdev.data_ptr(), n, d, stream=stream.cuda_stream)
    barrier()
    launches = 0
    stage_sums = {}
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(device) as clk:
        start.record(stream)
        for _ in range(args.steps):
            r = ctx.run_device(xdev.data_ptr(), n, d, stream=stream.cuda_stream)
            launches += pkg.last_launch_count()
            for f, _t in r.times._fields_:
                stage_sums[f] = stage_sums.get(f, 0) + getattr(r.times, f)
        end.record(stream)
        barrier()
    ms = start.elapsed_time(end)
    ms_max = ms
    if dist is not None:
        t = torch.tensor([ms], device=f"cuda:{device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    value = ws * k * args.steps / (ms_max / 1e3)
    n_scale = int(r.n_scale)
    n_finite = int(r.n_finite)

    # untimed: the device-path result, to check the e2e result against (bars bit for bit, D by
    # an order-sensitive checksum)
    def dev_tensor(ptr, count, typestr):
        cai = type("CAI", (), {"__cuda_array_interface__": {
            "shape": (int(count),), "typestr": typestr, "data": (int(ptr), False),
            "version": 3, "strides": None}})()
        return torch.as_tensor(cai, device=f"cuda:{device}")

    torch.cuda.synchronize(device)
    dev_dg = dev_tensor(r.d_death_grade, n_finite, "<i8").cpu().numpy().view(np.uint64).copy()
    dev_dl = dev_tensor(r.d_death_length, n_finite, "<f8").cpu().numpy().copy()
    dev_sum = scale_checksum(dev_tensor(r.d_scale, n_scale, "<i8"))

    # ---- end-to-end through the C ABI with host buffers (e2e) --------------------------------
    e2e_steps = args.e2e_steps or max(1, min(args.steps, 5))
    xin = pkg.PinnedArray(n * d)
    xin.array[:] = np.asfortranarray(X).ravel(order="F")
    Xh = xin.array.reshape(d, n).T  # (n, d) view of column-major pinned storage
    dg = pkg.PinnedArray(n, np.uint64)
    dl = pkg.PinnedArray(n, np.float64)
    sc = pkg.PinnedArray(n_scale, np.float64)

    def run_e2e():
        return ctx.run_host(Xh, dg.array, dl.array, sc.array, stream=stream.cuda_stream)

    # W (at least 4) untimed calls: the context also settles its D2H ring geometry here
    # (pipeline.cpp ring_choice(): calls 2-4 time the two geometries)
    for _ in range(max(4, args.warmup)):
        run_e2e()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        nf, ess, ns_, _t = run_e2e()
    e1.record(stream)
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([e2e_ms], device=f"cuda:{device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = ws * k * e2e_steps / (e2e_ms / 1e3)
    h2d = n * d * 8
    # bytes actually moved device -> host per step, as counted by the library (D goes out
    # delta-encoded: a u64 base + 3- or 4-byte deltas per 1024-value chunk; bars 16 B each)
    d2h = int(_t.get("d2h_bytes", 0)) or (ns_ * 8 + nf * 16)
    e2e_check = {
        "bars_equal_device_path": bool(nf == n_finite and
                                       np.array_equal(dg.array[:nf], dev_dg) and
                                       np.array_equal(dl.array[:nf].view(np.uint64),
                                                      dev_dl.view(np.uint64))),
        "scale_equal_device_path": bool(ns_ == n_scale and
                                        scale_checksum(torch.from_numpy(
                                            sc.array[:ns_].view(np.int64))) == dev_sum),
    }
    for a in (xin, dg, dl, sc):
        a.free()

    # ---- the drop-in entry point itself (ph0b_h0_barcode: X from pageable host memory, the
    # library allocates the result — bars and D — and the caller frees it every step; D is
    # streamed into the result buffer while the sort runs, like ph0b_run_host does) -------
    dropin = None
    if not args.no_dropin:
        import ctypes as C
        L = pkg.lib()
        Xc = np.asfortranarray(X)
        opt = pkg.ph0b.Options(C.sizeof(pkg.ph0b.Options), device, 0, 1, 1)

        def dropin_step():
            res = pkg.ph0b.Result()
            rc = L.ph0b_h0_barcode(C.c_void_p(Xc.ctypes.data), n, d, pkg.ph0b.COL_MAJOR,
                                   C.byref(opt), C.byref(res))
            if rc:
                raise RuntimeError(L.ph0b_last_error().decode())
            out = (int(res.n_finite), int(res.n_scale), int(res.essential_count),
                   int(res.times.d2h_bytes))
            ok = out[0] == n_finite and out[1] == n_scale and (
                not out[0] or (res.death_grade[out[0] - 1] == dev_dg[-1] and
                               res.death_length[out[0] - 1] == dev_dl[-1]))
            L.ph0b_result_free(C.byref(res))
            return out, ok

        for _ in range(max(4, args.warmup)):  # warm: sizes the context, faults in the cached
            dropin_step()                     # result buffer once, settles the ring geometry
        t0 = time.perf_counter()
        oks = []
        for _ in range(e2e_steps):
            out, ok = dropin_step()
            oks.append(ok)
        dms = (time.perf_counter() - t0) * 1e3 / e2e_steps
        dropin = {"value": ws * k / (dms / 1e3), "unit": UNIT, "ms_per_step": dms,
                  "steps": e2e_steps, "h2d_bytes_per_step": h2d,
                  "d2h_bytes_per_step": out[3],
                  "api": "ph0b_h0_barcode + ph0b_result_free (pageable X; library-allocated "
                         "result, D streamed while sorting; host wall clock of the blocking call)",
                  "check": {"bars_n_scale_match_device_path": all(oks)}}

    # ---- roofline of the dominant kernel (onesweep digit pass) ------------------------------
    peak, peak_kind = peaks()
    passes = max(1, int(stage_sums.get("sort_passes", 0) / args.steps))
    sort_ms = stage_sums.get("sort_ms", 0.0) / args.steps
    # the passes alone (CUDA events on the pipeline stream around launch_sort_passes; the
    # first-digit histogram kernel before them is excluded)
    pass_ms = (stage_sums.get("sort_passes_ms", 0.0) or stage_sums.get("sort_ms", 0.0)) / args.steps / passes
    alg_bytes = 24 * k  # read key+value (12 B), write key+value (12 B) per edge per pass
    achieved = alg_bytes / (pass_ms / 1e3) / 1e9
    traffic = None
    summ = load_traffic()
    if summ and summ.get("config") == cfg_name:
        traffic = summ.get("onesweep_dram_bytes_per_launch")
    roofline = {"kernel": "k2_onesweep (LSD digit pass)", "bound": "hbm",
                "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                "alg_bytes_per_launch": alg_bytes, "avg_launch_ms": round(pass_ms, 4),
                "passes": passes}

    # K1's FP64 roofline (the second-largest kernel): FP64 instructions per edge counted from
    # the SASS of k1_distance_tma (profiles/fp64_peak_r02.txt: 31.23 at d = 8), against the
    # measured DADD/DMUL issue peak of this pool's B200s (tools/fp64_peak.cu)
    k1 = None
    if d == 8 and stage_sums.get("distance_ms"):
        dms = stage_sums["distance_ms"] / args.steps
        inst = 31.23 * k
        k1 = {"kernel": "k1_distance_tma<8>", "bound": "fp64 (sqrt-sequence latency)",
              "achieved": round(inst / (dms / 1e3) / 1e12, 2), "peak": 18.5,
              "unit": "T FP64 instr/s", "frac": round(inst / (dms / 1e3) / 1e12 / 18.5, 3),
              "inst_per_edge": 31.23, "avg_launch_ms": round(dms, 3),
              "peak_source": "measured, profiles/fp64_peak_r02.txt"}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline_record(cfg_name, n)

    if rank == 0:
        stage_ms = {f: round(stage_sums[f] / args.steps, 3) for f in
                    ("distance_ms", "sort_ms", "sort_passes_ms", "unique_ms", "reduce_ms",
                     "collect_ms", "total_ms")}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            # N = 1: the one C5 problem (the torchrun N > 1 path shards that same problem:
            # strong); --replicas at N > 1: every GPU solves its own copy (weak)
            "scaling": "weak" if ws > 1 else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{cfg_name}: {WORKLOADS[cfg_name]}", "n": n, "d": d,
                       "edges": k, "parallelism": "replicas" if ws > 1 else "single",
                       "l2": "inputs larger than L2 (keys+values 12 B/edge)",
                       "n_scale": n_scale, "bars": n_finite},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms / e2e_steps,
                    "steps": e2e_steps, "api": "ph0b_run_host (pinned host X, D, bars)", "check": e2e_check},
            "e2e_dropin": dropin,
            "roofline": roofline, "roofline_k1": k1, "cpu_baseline": cpu,
            "clocks": clk.summary(), "gpu_launches": launches, "stage_ms": stage_ms,
            "sort_passes": passes,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
