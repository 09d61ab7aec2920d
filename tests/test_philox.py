"""Pin oracle/philox.py: Philox4x32-10 against the published Random123 known-answer
vectors (Salmon et al., SC'11; kat_vectors "philox4x32 10"), and the logical-
coordinate mask layout the kernels use (16 bits per element, 8 per Philox call)."""
import numpy as np

from oracle import philox

KAT = [
    ((0, 0, 0, 0), 0, (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, 0xFFFFFFFFFFFFFFFF, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0x299F31D0 << 32) | 0xA4093822,
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


def test_philox_known_answers():
    for ctr, key, want in KAT:
        got = philox.philox4x32_10(*[np.uint32(c) for c in ctr], key)
        assert tuple(int(v) for v in got) == want


def test_mask_layout_and_rate():
    rows = np.arange(64)[:, None]
    cols = np.arange(1024)[None, :]
    u = philox.uniform16(rows, cols, layer=3, site=1, seed=42)
    # 8 consecutive columns share one Philox call: recompute column 13 by hand
    x, y, z, w = philox.philox4x32_10(np.uint32(13 >> 3), np.uint32(5), np.uint32(3), np.uint32(1), 42)
    word = [x, y, z, w][(13 >> 1) & 3]
    assert int(u[5, 13]) == (int(word) >> 16) & 0xFFFF
    keep = philox.keep_mask(rows, cols, 3, 1, 42, 0.1)
    assert abs(keep.mean() - 0.9) < 0.01
    assert philox.threshold(0.1) == 6554 and philox.threshold(0.0) == 0
    # masks are a pure function of logical coordinates
    assert np.array_equal(philox.keep_mask(rows[10:20], cols, 3, 1, 42, 0.1), keep[10:20])


def test_c_restatement_matches_numpy():
    """oracle/philox_grid.c (built by oracle/Makefile) == the numpy restatement, bit for bit,
    including step keys (philox.step_key) and ragged column counts."""
    import pytest
    if philox._clib() is None:
        pytest.skip("oracle/libphilox_grid.so not built (make -C oracle)")
    rows = np.array([0, 1, 7, 12345, 2 ** 31 + 5, 4096 * 24 - 1], dtype=np.int64)
    for n_cols, seed, step, p in ((1024, 7, 0, 0.1), (13, 42, 3, 0.5), (2048, 0, 2 ** 40, 0.25)):
        key = philox.step_key(seed, step)
        a = philox.keep_grid(rows, n_cols, 5, 2, key, p, use_c=True)
        b = philox.keep_grid(rows, n_cols, 5, 2, key, p, use_c=False)
        assert np.array_equal(a, b)


def test_step_key():
    assert philox.step_key(7, 0) == 7
    assert philox.step_key(7, 1) == (7 + 0x9E3779B97F4A7C15) % 2 ** 64
    assert philox.step_key(2 ** 64 - 1, 1) == (0x9E3779B97F4A7C15 - 1)
