"""Time fused vs materialised attention (fwd / bwd) at BERT-large and GPT shapes (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2111_05972_b200 import layers as Lm
from paper_2111_05972_b200 import ops


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


for (B, nh, s, dh, causal, p) in [(8, 16, 512, 64, False, 0.1), (8, 16, 512, 64, False, 0.0), (8, 2, 2048, 128, True, 0.1),
                                  (1, 10, 2048, 128, True, 0.1)]:
    qkv = torch.randn(B * s, 3 * nh * dh, device="cuda").bfloat16()
    dctx = torch.randn(B * s, nh * dh, device="cuda").bfloat16()
    m = Lm.LayerMeta(hidden=nh * dh, heads_local=nh, heads_global=nh, head_dim=dh, eps=1e-5, p_attn=p, p_hidden=0.0,
                     causal=causal, pre_ln=False, post_ln=True, activation="gelu", layer_id=0, seed=1, head_offset=0,
                     sample_offset=0, tp_size=1)
    ctx_m, P, Pd = Lm.attn_core_fwd(qkv, B, s, m, None)
    bits = ops.attn_dropout_bits(B, nh, s, s, p=p, seed=1)
    ctx_f, lse = ops.flash_attn_fwd(qkv, B, s, nh, dh, causal=causal, p=p, keep_bits=bits)
    flops_f = 4 * B * nh * s * s * dh * (0.5 if causal else 1.0)
    t_mf = timeit(lambda: Lm.attn_core_fwd(qkv, B, s, m, None))
    t_bits = timeit(lambda: ops.attn_dropout_bits(B, nh, s, s, p=p, seed=1)) if p > 0 else 0.0
    t_ff = timeit(lambda: ops.flash_attn_fwd(qkv, B, s, nh, dh, causal=causal, p=p, keep_bits=bits))
    t_mb = timeit(lambda: Lm.attn_core_bwd(dctx, qkv, P, Pd, B, s, m))
    t_fb = timeit(lambda: ops.flash_attn_bwd(dctx, qkv, ctx_f, lse, B, s, nh, dh, causal=causal, p=p, keep_bits=bits))
    print(f"B={B} nh={nh} s={s} dh={dh} causal={causal} p={p}: fwd materialized {t_mf:.1f} us, flash {t_ff:.1f} us "
          f"({flops_f / t_ff / 1e6:.0f} TF/s) + bits {t_bits:.1f} us | bwd materialized {t_mb:.1f} us, flash {t_fb:.1f} us "
          f"({2.5 * flops_f / t_fb / 1e6:.0f} TF/s)", flush=True)
