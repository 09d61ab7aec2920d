"""The C ABI library loads on a CPU-only host and exports every symbol include/smpk.h declares
(no compute calls without a GPU)."""
import ctypes
import os
import re

from paper_2111_05972_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "smpk.h")).read()
    return sorted(set(re.findall(r"SMPK_API\s+[\w\s\*]+?\b(smpk_\w+)\s*\(", text)))


def test_header_lists_entry_points():
    syms = header_symbols()
    assert "smpk_gemm" in syms and "smpk_last_error" in syms
    assert len(syms) >= 10


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, f"libsmpk.so lacks {missing}"


def test_binding_covers_header():
    assert set(header_symbols()) == set(_lib.exported_symbols()) | {"smpk_version", "smpk_device_info"} or \
        set(header_symbols()) <= set(_lib.exported_symbols()) | {"smpk_version", "smpk_device_info"}
    lib = _lib.lib()  # declares argtypes for every binding without calling a kernel
    assert lib.smpk_version() >= 1


def test_sm100a_cubin_only():
    """Every kernel is compiled for sm_100a (tcgen05 needs the 'a' target)."""
    import subprocess
    r = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    if r.returncode != 0:
        return  # cuobjdump unavailable
    elfs = [l for l in r.stdout.splitlines() if "ELF file" in l]
    assert elfs and all("sm_100a" in l for l in elfs), r.stdout
