"""Timeline of the fused attention forward (SMPK_FA_TRACE=1): per-CTA phase times (dev tool)."""
import ctypes
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
bits = ops.attn_dropout_bits(B, nh, s, s, p=0.1, seed=1)
for _ in range(5):
    ops.flash_attn_fwd(qkv, B, s, nh, dh, p=0.1, keep_bits=bits, causal=causal)
torch.cuda.synchronize()
n = (s // 256) * nh * B
buf = np.zeros(n * 20, dtype=np.uint64)
_lib.call("smpk_debug_fa_trace", buf.ctypes.data, n)
t = buf.reshape(n, 20).astype(np.int64)
t0 = t[:, 0].min()
rel = (t[:, :19] - t0) / 1000.0
print(f"kernel span {rel[:, 18].max():.2f} us, CTAs {n}")
for name, col in [("start", 0), ("Q landed", 1)] + [(f"S{j} ready", 2 + j) for j in range(4)] + \
        [(f"P{j} stored", 10 + j) for j in range(4)] + [("epilogue done", 18)]:
    v = rel[:, col]
    print(f"{name:14s} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f}")
d = rel[:, 18] - rel[:, 0]
print(f"CTA duration   min {d.min():7.2f} med {np.median(d):7.2f} max {d.max():7.2f}")
for j in range(4):
    print(f"softmax {j}: S ready -> P stored med {np.median(rel[:, 10 + j] - rel[:, 2 + j]):.2f} us; "
          f"wait for S{j} after P{j-1}: {np.median(rel[:, 2 + j] - (rel[:, 9 + j] if j else rel[:, 1])):.2f} us")
first = np.argsort(rel[:, 0])
print("start times of CTAs sorted (us):", np.round(np.sort(rel[:, 0])[::16], 2))
