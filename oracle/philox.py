"""Philox4x32-10 and logical-coordinate dropout masks (numpy, bit-exact).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The GPU kernels (csrc/smpk_common.cuh: philox4x32_10 / dropout_keep) draw every
dropout decision from Philox4x32-10 keyed by the 64-bit seed and countered by
*logical* coordinates, never by buffer offsets (SURVEY.md Appendix C.2 "Dropout
RNG rule"), so masks are invariant to the TP degree and the oracle reproduces
them exactly:

    counter = (col >> 3, row, layer, site);  word = output[(col >> 1) & 3]
    u16     = (word >> (16 * (col & 1))) & 0xffff
    keep    = u16 >= rint(p * 65536)            (16 random bits per element)

Sites: 0 = attention probabilities (row = (global_sample*nh + global_head)*s_q + q,
col = key position), 1 = attention-output hidden dropout, 2 = MLP-output hidden
dropout (row = global token index = global_sample*s + t, col = channel).
The SPEC disables dropout in equivalence tests; masks are
exercised separately for bit-exactness.
"""
from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = np.uint32(0x9E3779B9)
W1 = np.uint32(0xBB67AE85)
MASK32 = np.uint64(0xFFFFFFFF)

GOLDEN64 = 0x9E3779B97F4A7C15


def step_key(seed: int, step: int) -> int:
    """Philox key of training step `step` (csrc/smpk_common.cuh philox_key): the device-resident
    step word snapshotted per top-level forward is folded into the 64-bit key."""
    return (int(seed) + int(step) * GOLDEN64) % (1 << 64)


SITE_ATTN_PROB = 0
SITE_ATTN_OUT = 1
SITE_MLP_OUT = 2


def philox4x32_10(c0, c1, c2, c3, seed: int):
    """Vectorised Philox4x32-10. c* are uint32 arrays (broadcastable); returns 4 uint32 arrays."""
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint32) for c in (c0, c1, c2, c3))
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    x, y, z, w = (a.astype(np.uint32).copy() for a in (c0, c1, c2, c3))
    k0 = np.uint32(seed & 0xFFFFFFFF)
    k1 = np.uint32((seed >> 32) & 0xFFFFFFFF)
    with np.errstate(over="ignore"):
        for _ in range(10):
            p0 = M0 * x.astype(np.uint64)
            p1 = M1 * z.astype(np.uint64)
            hi0 = (p0 >> np.uint64(32)).astype(np.uint32)
            lo0 = (p0 & MASK32).astype(np.uint32)
            hi1 = (p1 >> np.uint64(32)).astype(np.uint32)
            lo1 = (p1 & MASK32).astype(np.uint32)
            x, y, z, w = hi1 ^ y ^ k0, lo1, hi0 ^ w ^ k1, lo0
            k0 = np.uint32((int(k0) + int(W0)) & 0xFFFFFFFF)
            k1 = np.uint32((int(k1) + int(W1)) & 0xFFFFFFFF)
    return x, y, z, w


def uniform16(rows: np.ndarray, cols: np.ndarray, layer: int, site: int, seed: int) -> np.ndarray:
    """The 16-bit draw of element (row, col): one Philox call per 8 columns,
    word = out[(col >> 1) & 3], low half for even col, high half for odd."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    rows, cols = np.broadcast_arrays(rows, cols)
    x, y, z, w = philox4x32_10((cols >> 3).astype(np.uint32), rows.astype(np.uint32),
                               np.uint32(layer), np.uint32(site), seed)
    lane = (cols >> 1) & 3
    word = np.where(lane == 0, x, np.where(lane == 1, y, np.where(lane == 2, z, w))).astype(np.uint32)
    return np.where((cols & 1) == 0, word & np.uint32(0xFFFF), word >> np.uint32(16)).astype(np.uint32)


def threshold(p: float) -> int:
    """rint(p * 65536) in fp32 (csrc/smpk_common.cuh dropout_threshold)."""
    return int(np.rint(np.float32(p) * np.float32(65536.0)))


def keep_mask(rows, cols, layer: int, site: int, seed: int, p: float) -> np.ndarray:
    """Boolean keep mask: keep iff u16 >= rint(p * 65536)."""
    return uniform16(rows, cols, layer, site, seed) >= np.uint32(threshold(p))


_CLIB = None


def _clib():
    """oracle/libphilox_grid.so (oracle/philox_grid.c, built by oracle/Makefile), or None."""
    global _CLIB
    if _CLIB is None:
        import ctypes
        import os
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libphilox_grid.so")
        _CLIB = False
        if os.path.exists(path):
            lib = ctypes.CDLL(path)
            lib.philox_keep_grid.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint32,
                                             ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p]
            lib.philox_keep_grid.restype = None
            _CLIB = lib
    return _CLIB or None


def keep_grid(rows, n_cols: int, layer: int, site: int, seed: int, p: float, use_c: bool = True) -> np.ndarray:
    """[len(rows), n_cols] keep mask of logical rows `rows` x columns 0..n_cols-1 (the C
    restatement when built, else numpy; tests/test_philox.py checks they agree)."""
    r = np.ascontiguousarray(np.asarray(rows, dtype=np.int64).reshape(-1))
    lib = _clib() if use_c else None
    if lib is None:
        return keep_mask(r[:, None], np.arange(n_cols, dtype=np.int64)[None, :], layer, site, seed, p)
    out = np.empty((r.size, n_cols), dtype=np.uint8)
    lib.philox_keep_grid(r.ctypes.data, r.size, int(n_cols), int(layer) & 0xFFFFFFFF, int(site) & 0xFFFFFFFF,
                         int(seed) % (1 << 64), threshold(p), out.ctypes.data)
    return out.astype(bool)


def hidden_mask(global_rows: np.ndarray, n_cols: int, layer: int, site: int, seed: int, p: float) -> np.ndarray:
    """[len(rows), n_cols] keep mask for a hidden-dropout site."""
    if _clib() is not None:
        return keep_grid(global_rows, n_cols, layer, site, seed, p)
    r = np.asarray(global_rows, dtype=np.int64)[:, None]
    c = np.arange(n_cols, dtype=np.int64)[None, :]
    return keep_mask(r, c, layer, site, seed, p)


def attn_prob_mask(global_samples, global_heads, s_q: int, s_k: int, nh_global: int, layer: int, seed: int,
                   p: float) -> np.ndarray:
    """[len(samples), len(heads), s_q, s_k] keep mask for attention-probability dropout."""
    gs = np.asarray(global_samples, dtype=np.int64)[:, None, None, None]
    gh = np.asarray(global_heads, dtype=np.int64)[None, :, None, None]
    q = np.arange(s_q, dtype=np.int64)[None, None, :, None]
    k = np.arange(s_k, dtype=np.int64)[None, None, None, :]
    rows = (gs * nh_global + gh) * s_q + q
    if _clib() is not None:
        return keep_grid(rows, s_k, layer, SITE_ATTN_PROB, seed, p).reshape(rows.shape[:3] + (s_k,))
    return keep_mask(rows, k, layer, SITE_ATTN_PROB, seed, p)
