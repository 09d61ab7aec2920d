"""Fused (flash) attention on tcgen05 vs the fp64 oracle attention core, same bf16 inputs,
same Philox dropout masks (oracle/philox.py)."""
import math

import numpy as np
import pytest
import torch

from oracle import philox, tp

pytestmark = pytest.mark.gpu


def keep_bits(ops, B, nh, s, p, seed, layer, soff, hoff, nhg):
    return ops.attn_dropout_bits(B, nh, s, s, p=p, seed=seed, layer=layer, sample_offset=soff, head_offset=hoff,
                                 nh_global=nhg, device="cuda")


def rel(a, b):
    a, b = a.double().cpu(), b.double().cpu()
    return ((a - b).norm() / max(b.norm().item(), 1e-30)).item()


CASES = [
    # B, nh, s, dh, causal, masked, p
    (2, 4, 256, 64, False, False, 0.0),
    (2, 4, 512, 64, False, True, 0.0),
    (2, 2, 384, 64, True, False, 0.0),
    (1, 2, 256, 128, True, False, 0.0),
    (2, 3, 256, 128, False, True, 0.0),
    (2, 4, 256, 64, False, True, 0.1),
    (1, 2, 512, 128, True, False, 0.1),
]


@pytest.mark.parametrize("case", CASES, ids=[str(c) for c in CASES])
def test_flash_fwd_vs_oracle(case):
    from paper_2111_05972_b200 import ops
    B, nh, s, dh, causal, masked, p = case
    g = torch.Generator().manual_seed(s + dh)
    H = nh * dh
    qkv = (torch.randn(B * s, 3 * H, generator=g)).to(torch.bfloat16)
    mask = None
    if masked:
        mask = torch.zeros(B, s)
        mask[0, -37:] = -10000.0
        mask[-1, :5] = -10000.0
    seed, layer, soff, hoff, nhg = 77, 3, 5, 2, nh + 4
    ctx, lse = ops.flash_attn_fwd(qkv.cuda(), B, s, nh, dh, mask_add=None if mask is None else mask.cuda(),
                                  causal=causal, p=p,
                                  keep_bits=keep_bits(ops, B, nh, s, p, seed, layer, soff, hoff, nhg))
    q, k, v = qkv.double().split(H, -1)
    ref = tp.attention_core(q.reshape(B, s, nh, dh), k.reshape(B, s, nh, dh), v.reshape(B, s, nh, dh),
                            None if mask is None else mask.double(), causal,
                            tp.DropoutCtx(seed=seed, layer=layer, sample_offset=soff) if p > 0 else None, p, hoff, nhg)
    assert rel(ctx.reshape(B, s, H), ref) < 1e-2
    # log-sum-exp (log2 domain) of the scaled masked scores
    sc = tp.attention_scores_mask((q.reshape(B, s, nh, dh).permute(0, 2, 1, 3) @
                                   k.reshape(B, s, nh, dh).permute(0, 2, 3, 1)) / math.sqrt(dh),
                                  None if mask is None else mask.double(), causal)
    lse_ref = torch.logsumexp(sc, -1) / math.log(2.0)
    assert (lse.cpu().double() - lse_ref).abs().max().item() < 2e-2


@pytest.mark.parametrize("case", CASES, ids=[str(c) for c in CASES])
def test_flash_bwd_vs_oracle(case):
    from paper_2111_05972_b200 import ops
    B, nh, s, dh, causal, masked, p = case
    g = torch.Generator().manual_seed(2 * s + dh)
    H = nh * dh
    qkv = torch.randn(B * s, 3 * H, generator=g).to(torch.bfloat16)
    dctx = torch.randn(B * s, H, generator=g).to(torch.bfloat16)
    mask = None
    if masked:
        mask = torch.zeros(B, s)
        mask[0, -37:] = -10000.0
    seed, layer, soff, hoff, nhg = 31, 1, 2, 1, nh + 2
    kw = dict(mask_add=None if mask is None else mask.cuda(), causal=causal, p=p,
              keep_bits=keep_bits(ops, B, nh, s, p, seed, layer, soff, hoff, nhg))
    ctx, lse = ops.flash_attn_fwd(qkv.cuda(), B, s, nh, dh, **kw)
    dqkv = ops.flash_attn_bwd(dctx.cuda(), qkv.cuda(), ctx, lse, B, s, nh, dh, **kw)
    x = qkv.double().requires_grad_(True)
    q, k, v = x.split(H, -1)
    ref = tp.attention_core(q.reshape(B, s, nh, dh), k.reshape(B, s, nh, dh), v.reshape(B, s, nh, dh),
                            None if mask is None else mask.double(), causal,
                            tp.DropoutCtx(seed=seed, layer=layer, sample_offset=soff) if p > 0 else None, p, hoff, nhg)
    ref.backward(dctx.double().reshape(B, s, H))
    gq, gk, gv = x.grad.split(H, -1)
    dq, dk, dv = dqkv.cpu().split(H, -1)
    errs = {"dq": rel(dq, gq), "dk": rel(dk, gk), "dv": rel(dv, gv)}
    assert all(e < 2e-2 for e in errs.values()), errs


def test_flash_matches_materialized_path():
    """The fused kernel and the GEMM + softmax + GEMM path give the same context."""
    from paper_2111_05972_b200 import layers as Lm
    from paper_2111_05972_b200 import ops
    B, nh, s, dh = 2, 4, 512, 64
    qkv = torch.randn(B * s, 3 * nh * dh, device="cuda").bfloat16()
    m = Lm.LayerMeta(hidden=nh * dh, heads_local=nh, heads_global=nh, head_dim=dh, eps=1e-5, p_attn=0.1,
                     p_hidden=0.0, causal=False, pre_ln=False, post_ln=True, activation="gelu", layer_id=4, seed=9,
                     head_offset=0, sample_offset=0, tp_size=1)
    ctx_ref, _, _ = Lm.attn_core_fwd(qkv, B, s, m, None)
    ctx, _ = ops.flash_attn_fwd(qkv, B, s, nh, dh, p=0.1, keep_bits=keep_bits(ops, B, nh, s, 0.1, 9, 4, 0, 0, nh))
    assert rel(ctx, ctx_ref) < 1e-2


@pytest.mark.parametrize("shape", [(2, 3, 128, 256, 5, 1, 7), (1, 2, 512, 512, 0, 0, 2)])
def test_dropout_bits_bit_exact(shape):
    """smpk_attn_dropout_bits == oracle/philox.py attn_prob_mask, bit for bit."""
    from paper_2111_05972_b200 import ops
    B, nh, sq, sk, soff, hoff, nhg = shape
    p, seed, layer = 0.15, 123456789012, 6
    bits = ops.attn_dropout_bits(B, nh, sq, sk, p=p, seed=seed, layer=layer, sample_offset=soff, head_offset=hoff,
                                 nh_global=nhg, device="cuda").cpu().numpy().view(np.uint32)
    got = ((bits[..., None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(B, nh, sq, sk).astype(bool)
    ref = philox.attn_prob_mask(np.arange(B) + soff, np.arange(nh) + hoff, sq, sk, nhg, layer, seed, p)
    assert np.array_equal(got, ref)


def test_causal_keep_bits_cover_lower_triangle():
    """causal=True writes exactly the words the causal kernels read (key tile <= query tile) and
    they equal the full generation's."""
    from paper_2111_05972_b200 import ops
    B, nh, s = 2, 3, 512
    full = ops.attn_dropout_bits(B, nh, s, s, p=0.1, seed=5, layer=2)
    part = torch.zeros_like(full)
    ops.attn_dropout_bits(B, nh, s, s, p=0.1, seed=5, layer=2, out=part, causal=True)
    q = torch.arange(s, device=full.device)[:, None] // 128
    w = torch.arange(s // 32, device=full.device)[None, :] // 4
    need = (w <= q).expand(B, nh, s, s // 32)
    assert torch.equal(part[need], full[need])
    assert int(part[~need].abs().sum()) == 0


def test_blocked_keep_bits_equal_whole_batch_slices():
    """The overlapped micro-batch's bits (blocks of b samples, one per rank, stride = the rank's
    batch) are exactly the corresponding samples of the whole gathered batch's bits."""
    from paper_2111_05972_b200 import ops
    T, Bfull, nh, s = 3, 4, 2, 128
    b = Bfull // 2
    whole = ops.attn_dropout_bits(T * Bfull, nh, s, s, p=0.1, seed=9, layer=4, sample_offset=8)
    for mb in (0, 1):
        got = ops.attn_dropout_bits(T * b, nh, s, s, p=0.1, seed=9, layer=4, sample_offset=8 + mb * b,
                                    sample_block=b, block_stride=Bfull)
        want = torch.cat([whole[j * Bfull + mb * b:j * Bfull + (mb + 1) * b] for j in range(T)], 0)
        assert torch.equal(got, want)
