"""The reference's own hot-path unit tests restated in C++ against the drop-in adapter
include/ph0b.hpp (tests/cpp/test_ref_style.cpp): compiled here (CPU) and run on the B200."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "cpp" / "test_ref_style.cpp"
LIBDIR = ROOT / "paper_2203_02527_b200"


def build(tmp_path) -> Path:
    exe = tmp_path / "test_ref_style"
    cmd = ["g++", "-std=c++17", "-O2", f"-I{ROOT / 'include'}", f"-I{ROOT / 'oracle' / 'shim'}",
           str(SRC), "-o", str(exe), f"-L{LIBDIR}", "-lph0b", f"-Wl,-rpath,{LIBDIR}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_cpp_adapter_compiles(tmp_path):
    assert build(tmp_path).exists()


@pytest.mark.gpu
def test_reference_unit_tests_on_b200(tmp_path):
    exe = build(tmp_path)
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(res.stdout, res.stderr)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "0 failed" in res.stdout
