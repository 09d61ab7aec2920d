"""Per-unit timeline of the persistent GEMM (SMPK_GEMM_TRACE=1): main-loop start/end on the MMA warp,
accumulator-ready and epilogue-done on epilogue warp 4 (dev tool).  usage: gemm_trace.py [variant]"""
import os
import sys

os.environ["SMPK_GEMM_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2111_05972_b200 import _lib  # noqa: E402
from paper_2111_05972_b200 import kernels as K  # noqa: E402

M, N, Kd = 4096, 4096, 1024
x, w, b = (torch.randn(M, Kd, device="cuda").bfloat16(), torch.randn(N, Kd, device="cuda").bfloat16(),
           torch.randn(N, device="cuda").bfloat16())
dy, w2 = torch.randn(M, Kd, device="cuda").bfloat16(), torch.randn(Kd, N, device="cuda").bfloat16()
z = torch.randn(M, N, device="cuda").bfloat16()
variants = {"plain": lambda: K.linear(x, w), "bias_gelu": lambda: K.linear(x, w, b, act="gelu"),
            "dgelu_colsum": lambda: K.matmul_nn(dy, w2, epi=K.EPI_DACT, act="gelu", aux=z, want_colsum=True)}
for name in (sys.argv[1:] or list(variants)):
    for _ in range(3):
        variants[name]()
    torch.cuda.synchronize()
    buf = np.zeros(148 * 40, dtype=np.uint64)
    _lib.call("smpk_debug_gemm_trace", buf.ctypes.data, 148)
    t = buf.reshape(148, 40).astype(np.int64)
    t0 = t[:, 0].min()
    rel = lambda c: (t[:, c] - t0) / 1000.0  # noqa: E731
    print(f"== {name}: kernel start spread {np.ptp(t[:, 0]) / 1000:.2f} us")
    for k in range(4):
        ms, me, ar, ed = rel(1 + 4 * k), rel(2 + 4 * k), rel(3 + 4 * k), rel(4 + 4 * k)
        ok = t[:, 1 + 4 * k] > 0
        if not ok.any():
            break
        sel = lambda v: np.median(v[ok])  # noqa: E731
        print(f"  unit {k}: mainloop {sel(ms):6.2f} -> {sel(me):6.2f} (med {sel(me - ms):5.2f})  acc ready "
              f"{sel(ar):6.2f}  epilogue done {sel(ed):6.2f} (med epi {sel(ed - ar):5.2f})")
