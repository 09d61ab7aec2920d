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


def call(name: str, *args) -> None:
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        raise_for(rc, lib().smpk_last_error().decode(errors="replace"))


def last_error() -> str:
    return lib().smpk_last_error().decode(errors="replace")
