"""On-device generate_uniform_cloud (ph0b_generate_uniform_cloud_device, SURVEY.md §8(f)
rank 4) vs the reference generator (point_cloud.cpp:20-29) restated in oracle/ and pinned by
the reference's KATs (test_point_cloud.cpp:21-28, test_splitmix.cpp:7-19)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle_bridge as ob
import paper_2203_02527_b200 as pkg

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def device_cloud(ctx, n, d, seed):
    out = torch.empty(max(n * d, 1), dtype=torch.float64, device="cuda")
    ctx.generate_uniform_cloud(n, d, seed, out.data_ptr())
    torch.cuda.synchronize()
    return out[: n * d].cpu().numpy().reshape(d, n).T  # column-major -> (n, d)


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


@pytest.mark.parametrize("n,d,seed", [(1, 1, 0), (5, 3, 7), (1000, 2, 1), (4097, 3, 4),
                                      (333, 17, 123456789), (32768, 3, 4)])
def test_device_generator_bit_exact(n, d, seed):
    ctx = pkg.Context(0)
    got = device_cloud(ctx, n, d, seed)
    assert np.array_equal(bits(got), bits(ob.uniform_cloud(n, d, seed)))
    ctx.close()


def test_device_generator_kat_and_c4():
    ctx = pkg.Context(0)
    X = device_cloud(ctx, 3, 2, 42)  # test_point_cloud.cpp:21-28: first draws of seed 42
    s = ob.splitmix_stream(42, 6)
    assert np.array_equal(X.ravel(), np.array([(v >> 11) * 2.0 ** -53 for v in s]))
    c4 = device_cloud(ctx, 32768, 3, 4)  # BASELINE C4 = generate_uniform_cloud(32768, 3, 4)
    assert np.array_equal(bits(c4), bits(pkg.config_cloud("C4")))
    ctx.close()


def test_device_generator_errors():
    ctx = pkg.Context(0)
    with pytest.raises(pkg.InvalidArgument, match="point dimension must be at least 1"):
        ctx.generate_uniform_cloud(4, 0, 1, 0)
    ctx.generate_uniform_cloud(0, 0, 1, 0)  # n == 0: nothing to do, no error
    ctx.close()


@pytest.mark.parametrize("zero_at", [0, 7, 29])
def test_zero_draw_rejection_is_exact(zero_at):
    """A zero draw (top 53 bits == 0, p = 2^-53) shifts every later coordinate by one draw
    (next_unit_open's rejection loop).  Forced through the test hook in a subprocess."""
    code = (
        "import sys, numpy as np, torch\n"
        f"sys.path.insert(0, {str(ob.ROOT)!r})\n"
        "import paper_2203_02527_b200 as pkg\n"
        "ctx = pkg.Context(0)\n"
        "out = torch.empty(40, dtype=torch.float64, device='cuda')\n"
        "ctx.generate_uniform_cloud(10, 4, 99, out.data_ptr())\n"
        "print(' '.join(str(int(v)) for v in out.cpu().numpy().view(np.uint64)))\n"
    )
    env = dict(os.environ, PH0B_GEN_FORCE_ZERO=str(zero_at))
    res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         timeout=300)
    assert res.returncode == 0, res.stderr
    got = np.array([int(v) for v in res.stdout.split()], np.uint64)
    draws = [v >> 11 for v in ob.splitmix_stream(99, 41)]
    del draws[zero_at]
    expect = np.array([d * 2.0 ** -53 for d in draws[:40]]).reshape(10, 4)  # row-major (i, j)
    assert np.array_equal(got, bits(expect.T.ravel()))  # column-major storage
