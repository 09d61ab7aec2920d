"""ctypes binding of libsmpk.so (the C ABI declared in include/smpk.h).

There is deliberately no fallback: if the library is missing or the device is
not an sm_100 part, every op raises.  ``declare()`` is the single place where
argument types are registered; ``call()`` checks the return code and raises
the SPEC's exception classes (see errors.py).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import raise_for

LIB_PATH = Path(os.environ.get("SMPK_LIB", Path(__file__).resolve().parent / "libsmpk.so"))

_lib: C.CDLL | None = None

P = C.c_void_p
I = C.c_int
L = C.c_int64
F = C.c_float

# symbol -> argtypes (restype is always c_int except smpk_last_error)
SIGNATURES: dict[str, list] = {
    "smpk_version": [],
    "smpk_device_info": [C.POINTER(I), C.POINTER(I), C.POINTER(I)],
    "smpk_gemm": [P, I, L, L, L, P, I, L, L, L, P, I, L, L, L, I, I, I, I, I, F, F, I, I, P, P, L, P],
    "smpk_gemm_ex": [P, I, L, L, L, P, I, L, L, L, P, I, L, L, L, I, I, I, I, I, F, F, I, I, P, P, L, P, L, P],
    "smpk_gemm_ex2": [P, I, L, L, L, P, I, L, L, L, P, I, L, L, L, I, I, I, I, I, F, F, I, I, P, P, L, P, L, P, P],
    "smpk_colsum_partials": [P, I, I, P, I, P],
    "smpk_bdr_ln_fwd": [P, P, P, P, P, P, P, P, P, I, I, F, F, C.c_uint64, P, I, I, L, P],
    "smpk_ln_bwd": [P, P, P, P, P, P, P, P, P, P, P, I, I, I, I, F, C.c_uint64, P, I, I, L, P, L, P],
    "smpk_softmax_fwd": [P, P, P, P, I, I, I, I, F, I, F, C.c_uint64, P, I, L, I, I, P],
    "smpk_softmax_bwd": [P, P, P, I, I, I, I, F, F, C.c_uint64, P, I, L, I, I, P],
    "smpk_colsum": [P, I, I, L, P, I, I, P, L, P],
    "smpk_embed_fwd": [P, L, P, L, L, L, L, I, P, L, P, L, I, P, P],
    "smpk_embed_bwd": [P, L, P, L, L, L, I, P, L, I, I, L, P],
    "smpk_vocab_ce_fwd_local": [P, L, L, I, L, L, P, L, P, P],
    "smpk_vocab_ce_combine": [P, I, L, P, L, P, P, P],
    "smpk_vocab_ce_bwd": [P, L, L, I, L, L, P, L, P, P, F, P, L, P],
    "smpk_flash_attn_fwd": [P, L, I, I, I, I, P, L, P, P, F, I, F, P, P],
    "smpk_attn_dropout_bits": [I, I, I, I, F, C.c_uint64, P, I, L, I, I, P, I, P],
    "smpk_attn_dropout_bits_blocked": [I, I, I, I, F, C.c_uint64, P, I, L, I, L, I, I, P, I, P],
    "smpk_flash_attn_bwd": [P, L, P, L, P, L, P, I, I, I, I, P, P, F, I, F, P, P, L, P],
    "smpk_gemm_rs": [P, I, L, P, I, L, P, I, L, L, L, I, I, I, P],
    "smpk_bdr_ln_fwd_ex": [P, I, L, P, P, P, P, P, P, P, P, P, I, L, I, I, F, F, C.c_uint64, P, I, I, L, P, P, L, P],
    "smpk_bdr_ln_fwd_dist": [P, P, P, P, P, P, P, P, P, I, I, F, F, C.c_uint64, P, I, I, L, L, P, P, I, P],
    "smpk_ln_bwd_dist": [P, P, P, P, P, P, P, P, P, P, P, I, I, I, F, C.c_uint64, P, I, I, L, L, P, P, I, P, L, P],
    "smpk_bias_act_fwd": [P, P, I, I, I, P, P, P],
    "smpk_act_bwd": [P, P, I, I, I, P, P],
    "smpk_copy_async": [P, P, L, P],
    "smpk_stream_flag": [P, C.c_uint32, I, P],
    "smpk_peer_put": [P, I, P, I, P, C.c_double, P],
    "smpk_flag_wait": [P, P, I, C.c_uint32, C.c_double, P],
    "smpk_flag_set": [P, I, C.c_uint32, P],
    "smpk_rng_next": [P, P, P],
    "smpk_gemm_grouped": [P, I, P],
    "smpk_embed_bwd_sorted": [P, L, P, L, L, L, I, P, L, I, I, L, P, L, P],
    "smpk_adam_step": [P, P, P, P, P, L, F, F, F, F, F, I, F, P],
    "smpk_debug_fa_trace": [P, I],
    "smpk_debug_fb_trace": [P, I],
    "smpk_debug_gemm_trace": [P, I],
    "smpk_ln_bwd_ex": [P, I, L, P, P, P, P, P, P, P, P, I, L, P, P, P, I, I, I, I, F, C.c_uint64, P, I, I, L, P, P, L, P,
                       L, P],
    "smpk_symm_export": [P, P, C.POINTER(L)],
    "smpk_symm_barrier": [P, P, I, I, C.c_double, P],
    "smpk_symm_timeout_peer": [],
    "smpk_p2p_alloc": [L, C.POINTER(P)],
    "smpk_p2p_free": [P],
    "smpk_p2p_export": [P, P],
    "smpk_p2p_import": [P, C.POINTER(P)],
    "smpk_p2p_close": [P],
    "smpk_p2p_send": [P, P, L, P, P, C.c_uint32, C.c_uint32, P],
    "smpk_p2p_recv": [P, P, L, P, P, C.c_uint32, P],
}

# functions returning int64 (sizes) rather than a status code
SIZE_FUNCS: dict[str, list] = {
    "smpk_ln_bwd_workspace": [I, I],
    "smpk_colsum_workspace": [I, I],
    "smpk_gemm_workspace": [I, I, I, I, I],
    "smpk_set_sm_limits": [I, I],
    "smpk_gemm_colsum_rows": [I],
    "smpk_flash_attn_bwd_workspace": [I, I, I, I],
    "smpk_embed_bwd_sorted_workspace": [L, L, I],
}


def extra_signatures(sigs: dict[str, list]) -> None:
    """Register more symbols (used by the op modules at import)."""
    SIGNATURES.update(sigs)
    if _lib is not None:
        _declare(_lib)


def _declare(lib: C.CDLL) -> None:
    lib.smpk_last_error.restype = C.c_char_p
    lib.smpk_last_error.argtypes = []
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    for name, args in SIZE_FUNCS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int64


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"libsmpk.so not found at {LIB_PATH}; build it with "
                "`python -m paper_2111_05972_b200.build` (there is no CPU fallback)")
        _lib = C.CDLL(str(LIB_PATH))
        _declare(_lib)
    return _lib


# kernels launched by each entry point (for bench.py's gpu_launches count)
LAUNCHES_PER_CALL = {"smpk_copy_async": 0, "smpk_stream_flag": 0, "smpk_set_sm_limits": 0, "smpk_ln_bwd": 2, "smpk_ln_bwd_ex": 2, "smpk_ln_bwd_dist": 2, "smpk_colsum": 2, "smpk_flash_attn_bwd": 3}
launch_count = 0


def call(name: str, *args, launches: int | None = None) -> None:
    """Invoke an ABI entry point; launches overrides the per-entry kernel count it adds to
    launch_count (entries whose second reduction kernel is conditional)."""
    global launch_count
    launch_count += LAUNCHES_PER_CALL.get(name, 1) if launches is None else launches
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        raise_for(rc, lib().smpk_last_error().decode(errors="replace"))


def size(name: str, *args) -> int:
    return int(getattr(lib(), name)(*args))


def exported_symbols() -> list[str]:
    """Every entry point this binding declares (checked against include/smpk.h by the tests)."""
    return ["smpk_last_error", *SIGNATURES, *SIZE_FUNCS]


def last_error() -> str:
    return lib().smpk_last_error().decode(errors="replace")


_SMS: dict = {}


def device_sms() -> int:
    """SM count of the current CUDA device (smpk_device_info, cached)."""
    import torch
    dev = torch.cuda.current_device()
    if dev not in _SMS:
        n, a, b = C.c_int(0), C.c_int(0), C.c_int(0)
        call("smpk_device_info", C.byref(n), C.byref(a), C.byref(b), launches=0)
        _SMS[dev] = n.value
    return _SMS[dev]
