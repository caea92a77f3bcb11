"""CPU: the C-ABI library loads, exports every symbol include/ph0b.h declares, and its
host-side validation reproduces the reference's error behaviour (no GPU needed)."""
import re

import numpy as np
import pytest

import oracle_bridge as ob
import paper_2203_02527_b200 as pkg
from paper_2203_02527_b200 import ph0b

HEADER = ob.ROOT / "include" / "ph0b.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ph0b_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    lib = pkg.lib()
    names = declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(ph0b.EXPORTED_SYMBOLS)


def test_abi_version():
    assert pkg.lib().ph0b_abi_version() == 4


def test_nonfinite_rejected_with_reference_message():  # point_cloud.cpp:15-18
    X = np.array([[1.0, np.inf], [0.0, 0.0]])
    with pytest.raises(ValueError, match="point cloud contains non-finite coordinates"):
        pkg.h0_barcode(X)
    X = np.array([[1.0, np.nan], [0.0, 0.0]])
    with pytest.raises(ValueError, match="non-finite"):
        pkg.pairwise_distances(X)


def test_workers_zero_rejected():  # reduction.cpp:134
    with pytest.raises(ValueError, match="worker count must be at least 1"):
        pkg.h0_barcode(np.zeros((3, 2)), workers=0)


def test_too_large_rejected():
    X = np.zeros((92683, 1))  # K >= 2^32: beyond the 32-bit edge-column codec
    with pytest.raises(pkg.Ph0bError, match="too large"):
        pkg.h0_barcode(X)


def test_generate_uniform_cloud_matches_reference_generator():  # point_cloud.cpp:20-29
    for n, d, seed in ((1, 2, 42), (17, 3, 9), (100, 1, 123)):
        assert np.array_equal(pkg.generate_cloud(0, n, d, seed), ob.uniform_cloud(n, d, seed))
    X = pkg.config_cloud("C4", 1)
    assert X.shape == (1, 3)


def test_config_clouds_deterministic():
    for name in ("C1", "C2"):
        a, b = pkg.config_cloud(name), pkg.config_cloud(name)
        assert np.array_equal(a, b) and np.isfinite(a).all()
    C5 = pkg.config_cloud("C5", 1000)
    assert C5.shape == (1000, 8)


def test_host_delta_decoder_roundtrip():
    """The host half of the compressed D2H (ph0b_decode_deltas): chunked u64 bases + u32
    deltas decode back to the exact bit patterns, at any output alignment, skipping raw
    chunks (which the host path ships uncompressed)."""
    import ctypes as C
    rng = np.random.default_rng(7)
    L = pkg.lib()
    for n, chunk, off in ((1, 4096, 0), (5000, 4096, 1), (20000, 1024, 3), (4096 * 3, 4096, 0),
                          (777, 256, 2)):
        gaps = rng.integers(1, 1 << 31, size=n, dtype=np.uint64)
        seq = np.cumsum(gaps, dtype=np.uint64) + np.uint64(0x3F00000000000000)
        nch = (n + chunk - 1) // chunk
        bases = seq[::chunk].copy()
        deltas = np.zeros(n, np.uint32)
        deltas[1:] = (seq[1:] - seq[:-1]).astype(np.uint32)
        raw = np.zeros(nch, np.uint8)
        if nch > 1:
            raw[1] = 1  # a raw chunk: the decoder must leave it alone
        buf = np.full(n + 8, 0xDEADBEEF, np.uint64)
        out = buf[off:off + n]
        rc = L.ph0b_decode_deltas(C.c_void_p(deltas.ctypes.data), C.c_void_p(bases.ctypes.data),
                                  C.c_void_p(raw.ctypes.data), n, chunk,
                                  C.c_void_p(out.ctypes.data))
        assert rc == 0
        for j in range(nch):
            s, e = j * chunk, min(n, (j + 1) * chunk)
            if raw[j]:
                assert np.all(out[s:e] == 0xDEADBEEF)
            else:
                assert np.array_equal(out[s:e], seq[s:e]), (n, chunk, off, j)
        assert np.all(buf[:off] == 0xDEADBEEF) and np.all(buf[off + n:] == 0xDEADBEEF)


def _pack_stream(seq, chunk, rng):
    """numpy restatement of the device encoder (d2h_codec.cu k9p_*): per chunk the narrowest
    of 3 / 4 bytes holding every delta (0 = raw), chunks concatenated."""
    n = len(seq)
    nch = (n + chunk - 1) // chunk
    bases = seq[::chunk].copy()
    widths = np.zeros(nch, np.uint8)
    offs = np.zeros(nch, np.uint32)
    parts = []
    pos = 0
    for j in range(nch):
        s, e = j * chunk, min(n, (j + 1) * chunk)
        d = np.zeros(e - s, np.uint64)
        d[1:] = seq[s + 1:e] - seq[s:e - 1]
        mx = int(d.max()) if len(d) else 0
        w = 0 if mx >> 32 else (4 if mx >> 24 else 3)
        widths[j], offs[j] = w, pos
        if w:
            b = d.astype("<u4").view(np.uint8).reshape(-1, 4)[:, :w].ravel()
            parts.append(b)
            pos += len(b)
    stream = np.concatenate(parts + [np.zeros(16, np.uint8)])  # + the 8-byte read slack
    return stream, bases, widths, offs


def test_host_packed_decoder_roundtrip():
    """The host half of the streamed D2H (ph0b_decode_packed): 1024-value chunks of 3- or
    4-byte deltas (or raw) decode back to the exact bit patterns, at any output alignment."""
    import ctypes as C
    rng = np.random.default_rng(11)
    L = pkg.lib()
    for n, chunk, off in ((1, 1024, 0), (3000, 1024, 1), (20000, 1024, 3), (1024 * 5, 1024, 0),
                          (777, 256, 2)):
        # gap sizes vary by chunk: some fit 24 bits, some 32, one chunk has a >= 2^32 gap
        hi = np.where((np.arange(n) // chunk) % 3 == 0, 1 << 23, 1 << 31).astype(np.uint64)
        gaps = (rng.random(n) * hi).astype(np.uint64) + np.uint64(1)
        if n > 2 * chunk:
            gaps[2 * chunk + 5] = np.uint64(1 << 40)  # chunk 2 goes raw
        seq = np.cumsum(gaps, dtype=np.uint64) + np.uint64(0x3F00000000000000)
        stream, bases, widths, offs = _pack_stream(seq, chunk, rng)
        assert set(widths.tolist()) <= {0, 3, 4}
        buf = np.full(n + 8, 0xDEADBEEF, np.uint64)
        out = buf[off:off + n]
        rc = L.ph0b_decode_packed(C.c_void_p(stream.ctypes.data), C.c_void_p(bases.ctypes.data),
                                  C.c_void_p(widths.ctypes.data), C.c_void_p(offs.ctypes.data),
                                  n, chunk, C.c_void_p(out.ctypes.data))
        assert rc == 0
        for j in range(len(widths)):
            s, e = j * chunk, min(n, (j + 1) * chunk)
            if widths[j] == 0:
                assert np.all(out[s:e] == 0xDEADBEEF)
            else:
                assert np.array_equal(out[s:e], seq[s:e]), (n, chunk, off, j, widths[j])
        assert np.all(buf[:off] == 0xDEADBEEF) and np.all(buf[off + n:] == 0xDEADBEEF)
    bad = np.array([5], np.uint8)
    one = np.zeros(1, np.uint64)
    rc = L.ph0b_decode_packed(C.c_void_p(one.ctypes.data), C.c_void_p(one.ctypes.data),
                              C.c_void_p(bad.ctypes.data), C.c_void_p(one.ctypes.data), 1, 1024,
                              C.c_void_p(one.ctypes.data))
    assert rc == pkg.ph0b.PH0B_ERR_INVALID_ARGUMENT


def test_abi3_sized_options_still_accepted():
    """An ABI-3 caller's ph0b_options ends at `workers` (20 bytes): still parsed (its
    workers == 0 reaches the reference's message), never read past its end."""
    import ctypes as C
    o = ph0b.Options(20, 0, 0, 1, 0)
    X = np.zeros((3, 2))
    res = ph0b.Result()
    rc = pkg.lib().ph0b_h0_barcode(C.c_void_p(X.ctypes.data), 3, 2, ph0b.COL_MAJOR, C.byref(o),
                                   C.byref(res))
    assert rc == ph0b.PH0B_ERR_INVALID_ARGUMENT
    assert b"worker count must be at least 1" in pkg.lib().ph0b_last_error()
    o.struct_size = 16
    rc = pkg.lib().ph0b_h0_barcode(C.c_void_p(X.ctypes.data), 3, 2, ph0b.COL_MAJOR, C.byref(o),
                                   C.byref(res))
    assert rc == ph0b.PH0B_ERR_INVALID_ARGUMENT
    assert b"struct_size too small" in pkg.lib().ph0b_last_error()


def test_kruskal_flag_limited_to_65536_before_any_device_work():
    X = np.zeros((65537, 1))
    with pytest.raises(pkg.Ph0bError, match="65536"):
        pkg.kruskal_barcode(X)


def test_null_context_rejected():
    import ctypes as C
    L = pkg.lib()
    fn = L.ph0b_run_device
    assert fn(None, None, 0, 0, 0, None, None) == ph0b.PH0B_ERR_INVALID_ARGUMENT
    assert b"null context" in L.ph0b_last_error()
    assert L.ph0b_context_reserve(None, 1, 1) == ph0b.PH0B_ERR_INVALID_ARGUMENT
    assert L.ph0b_context_workspace_bytes(None) == 0
    L.ph0b_shard_sample.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
    assert L.ph0b_shard_sample(None, 4, None) == ph0b.PH0B_ERR_INVALID_ARGUMENT


def test_release_functions_callable_without_gpu():
    L = pkg.lib()
    L.ph0b_host_cache_trim()
    L.ph0b_release_resources()
    L.ph0b_scale_release(None)


def test_null_outputs_rejected_before_any_device_work():
    import ctypes as C
    L = pkg.lib()
    X = np.zeros((3, 2))
    o = ph0b.Options(C.sizeof(ph0b.Options), 0, 0, 1, 1)
    for fn, args in ((L.ph0b_pairwise_distances, (None,)),
                     (L.ph0b_claimed_lows, (None, None)),
                     (L.ph0b_reduced_supports, (None, None, None, None))):
        rc = fn(C.c_void_p(X.ctypes.data), 3, 2, ph0b.COL_MAJOR, C.byref(o), *args)
        assert rc == ph0b.PH0B_ERR_INVALID_ARGUMENT
        assert b"null output" in L.ph0b_last_error()
