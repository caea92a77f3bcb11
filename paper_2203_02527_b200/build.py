"""In-tree build of libph0b.so (sm_100a CUDA kernels + C++ host + C ABI) with nvcc.

The shared object lands next to this file so it travels with the repo snapshot to the GPU
box (it is git-ignored, not gpurun-ignored).  Objects are cached under build/ and rebuilt
when a source or header is newer.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "libph0b.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", f"-I{ROOT / 'include'}"]
CU_FLAGS = ARCH + COMMON + ["-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))


def _headers():
    return list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "ph0b.h"]


def _compile(src: Path, verbose: bool) -> Path:
    obj = OBJ / (src.name + ".o")
    newest = max([src.stat().st_mtime] + [h.stat().st_mtime for h in _headers()])
    if obj.exists() and obj.stat().st_mtime >= newest:
        return obj
    flags = CU_FLAGS if src.suffix == ".cu" else ARCH + COMMON
    cmd = [NVCC, *flags, "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stdout}\n{res.stderr}")
    if verbose:
        log = OBJ / (src.name + ".ptxas.txt")
        log.write_text(res.stdout + res.stderr)
    return obj


def build_library(verbose: bool = False, force: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    if force:
        for o in OBJ.glob("*.o"):
            o.unlink()
    srcs = _sources()
    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    newest_obj = max(o.stat().st_mtime for o in objs)
    if not LIB.exists() or LIB.stat().st_mtime < newest_obj or force:
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lpthread", "-ldl"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    build_cli()
    return LIB


CLI_SRC = PKG / "cli" / "ph0b_cli.cpp"
CLI_BIN = PKG / "ph0b"


def build_cli() -> Path:
    """The `ph0b` front-end (generate/compute/oracle), linked against libph0b.so."""
    deps = [CLI_SRC, LIB, ROOT / "include" / "ph0b.hpp", ROOT / "include" / "ph0b_io.hpp"]
    if CLI_BIN.exists() and CLI_BIN.stat().st_mtime >= max(p.stat().st_mtime for p in deps):
        return CLI_BIN
    cmd = [os.environ.get("CXX", "g++"), "-std=c++17", "-O2", "-Wall", f"-I{ROOT / 'include'}",
           str(CLI_SRC), "-o", str(CLI_BIN), f"-L{PKG}", "-lph0b", "-Wl,-rpath,$ORIGIN"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"CLI build failed:\n{res.stdout}\n{res.stderr}")
    return CLI_BIN


if __name__ == "__main__":
    try:
        print(build_library(verbose=True, force="--force" in sys.argv))
    except RuntimeError as e:
        print("BUILD FAILED:", e)
        sys.exit(1)
