"""Timeline of the fused attention backward (SMPK_FA_TRACE=1): per-CTA phase times (dev tool)."""
import os
import sys

os.environ.setdefault("SMPK_FA_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2111_05972_b200 import _lib, ops

a = sys.argv[1:]
B, nh, s, dh = (int(v) for v in (a[:4] if a else (8, 16, 512, 64)))
causal = bool(int(a[4])) if len(a) > 4 else False
qkv = torch.randn(B * s, 3 * nh * dh, device="cuda").bfloat16()
dctx = torch.randn(B * s, nh * dh, device="cuda").bfloat16()
bits = ops.attn_dropout_bits(B, nh, s, s, p=0.1, seed=1)
ctx, lse = ops.flash_attn_fwd(qkv, B, s, nh, dh, p=0.1, keep_bits=bits, causal=causal)
for _ in range(5):
    ops.flash_attn_bwd(dctx, qkv, ctx, lse, B, s, nh, dh, p=0.1, keep_bits=bits, causal=causal)
torch.cuda.synchronize()
n = (s // 128) * nh * B
buf = np.zeros(n * 64, dtype=np.uint64)
_lib.call("smpk_debug_fb_trace", buf.ctypes.data, n)
t = buf.reshape(n, 64).astype(np.int64)
t0 = t[:, 0].min()
rel = (t[:, :44] - t0) / 1000.0
print(f"kernel span {rel[:, 26].max():.2f} us, CTAs {n}")
d = rel[:, 26] - rel[:, 0]
print(f"CTA duration   min {d.min():7.2f} med {np.median(d):7.2f} max {d.max():7.2f}")
print(f"K/V landed after start: med {np.median(rel[:, 1] - rel[:, 0]):.2f}")
for tt in range(4):  # (first 4 tiles of each CTA)
    med = lambda c: np.median(rel[:, c + tt] - rel[:, 0])
    print(f"tile {tt}: S^T {med(2):6.2f}  P stored {med(6):6.2f}  dP^T {med(10):6.2f}  dS stored {med(14):6.2f}  "
          f"dQ ready {med(18):6.2f}  dQ drained {med(22):6.2f} | S loaded {med(32):6.2f} pdt_free {med(36):6.2f} "
          f"computed {med(40):6.2f}")
print("end", np.median(rel[:, 26] - rel[:, 0]))

