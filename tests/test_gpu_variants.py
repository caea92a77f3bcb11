"""GPU: the code paths selected by tuning knobs stay bit-exact — truncated radix plans with
the in-place run fix-up and the redo fallback (PH0B_MAX_PASSES), and the ballot ranking used
when the device's ATOMS lane-order self-test fails (PH0B_RANK=2)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

HERE = Path(__file__).resolve().parent
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("env", [{"PH0B_MAX_PASSES": "1"}, {"PH0B_MAX_PASSES": "2"},
                                 {"PH0B_MAX_PASSES": "3"}, {"PH0B_RANK": "2"},
                                 {"PH0B_RANK": "3", "PH0B_MAX_PASSES": "8"},
                                 {"PH0B_RANK": "2", "PH0B_MAX_PASSES": "2"}])
def test_variant_parity(env):
    e = dict(os.environ, **env)
    res = subprocess.run([sys.executable, str(HERE / "gpu_variant_check.py")], env=e,
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0 and "OK" in res.stdout, res.stdout + res.stderr


@pytest.mark.parametrize("env", [{}, {"PH0B_RING_SLOTS": "2", "PH0B_RING_CHUNKS": "1"},
                                 {"PH0B_RING_SLOTS": "3", "PH0B_RING_CHUNKS": "5",
                                  "PH0B_RING_SUBTASKS": "2", "PH0B_RING_STREAMS": "3"},
                                 {"PH0B_D2H_COMPRESS": "0"}])
def test_host_path_d2h_variants(env):
    """The streamed D2H of D (compressed pieces through the pinned ring, slot reuse gated by
    stream memory operations) and the uncompressed fallback, bit-exact at K >= 2^26."""
    e = dict(os.environ, **env)
    res = subprocess.run([sys.executable, str(HERE / "gpu_ring_check.py")], env=e,
                         capture_output=True, text=True, timeout=900)
    assert res.returncode == 0 and "OK" in res.stdout, res.stdout + res.stderr
