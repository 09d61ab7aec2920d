"""One fused attention fwd + bwd at the BERT-large bench shape (ncu target; dev tool).
usage: python scripts/attn_once.py [B nh s dh causal p]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2111_05972_b200 import ops

a = sys.argv[1:]
B, nh, s, dh = (int(v) for v in (a[:4] if a else (8, 16, 512, 64)))
causal = bool(int(a[4])) if len(a) > 4 else False
p = float(a[5]) if len(a) > 5 else 0.1
qkv = torch.randn(B * s, 3 * nh * dh, device="cuda").bfloat16()
dctx = torch.randn(B * s, nh * dh, device="cuda").bfloat16()
bits = ops.attn_dropout_bits(B, nh, s, s, p=p, seed=1)
for _ in range(3):
    ctx, lse = ops.flash_attn_fwd(qkv, B, s, nh, dh, causal=causal, p=p, keep_bits=bits)
    ops.flash_attn_bwd(dctx, qkv, ctx, lse, B, s, nh, dh, causal=causal, p=p, keep_bits=bits)
torch.cuda.synchronize()
print("ok")
