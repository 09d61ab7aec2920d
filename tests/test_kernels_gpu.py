"""Row kernels (LayerNorm, bias-dropout-residual, softmax, colsum) vs the CPU oracle.

Inputs are bf16-rounded and fed identically to the sm_100a kernel and to the
fp64 oracle; dropout masks come from oracle/philox.py and must match bit-exactly
(a single flipped keep bit would show as an O(1) error on that element).
Tolerances: rel-Frobenius <= 1e-2 for single bf16 ops."""
import math

import numpy as np
import pytest
import torch

from oracle import philox, tp

pytestmark = pytest.mark.gpu
TOL = 1e-2


def rel(a, b):
    a, b = a.double().cpu(), b.double().cpu()
    return ((a - b).norm() / max(b.norm().item(), 1e-30)).item()


def bf(t):
    return t.to(torch.bfloat16)


@pytest.fixture(scope="module")
def ops():
    from paper_2111_05972_b200 import ops
    return ops


@pytest.mark.parametrize("H", [128, 256, 384, 1024, 2048, 5120])
@pytest.mark.parametrize("p", [0.0, 0.1])
def test_bdr_ln_fwd(ops, H, p):
    g = torch.Generator().manual_seed(H)
    M = 300
    x, res = bf(torch.randn(M, H, generator=g)), bf(torch.randn(M, H, generator=g))
    bias, gam, bet = bf(torch.randn(H, generator=g)), bf(1 + 0.1 * torch.randn(H, generator=g)), bf(
        torch.randn(H, generator=g))
    seed, layer, site, off = 1234, 3, ops.SITE_ATTN_OUT, 77
    r, y, mean, rstd = ops.bdr_ln(x.cuda(), bias=bias.cuda(), residual=res.cuda(), gamma=gam.cuda(),
                                  beta=bet.cuda(), eps=1e-5, p=p, seed=seed, layer=layer, site=site, row_offset=off)
    v = x.double() + bias.double()
    if p > 0:
        keep = philox.hidden_mask(np.arange(M) + off, H, layer, site, seed, p)
        v = v * torch.from_numpy(keep).double() / (1 - p)
    v = v + res.double()
    assert rel(r, v) < TOL
    ref = tp.layer_norm(bf(v).double(), gam.double(), bet.double(), 1e-5)
    assert rel(y, ref) < TOL
    if p > 0:  # dropped positions must be exactly the residual
        dropped = torch.from_numpy(~keep)
        assert torch.equal(r.cpu()[dropped], bf(res.double())[dropped])


@pytest.mark.parametrize("H", [128, 256, 384, 1024, 2048])
@pytest.mark.parametrize("p", [0.0, 0.2])
@pytest.mark.parametrize("with_ln", [True, False])
def test_ln_bwd(ops, H, p, with_ln):
    g = torch.Generator().manual_seed(H + 1)
    M = 257
    r = bf(torch.randn(M, H, generator=g) * 2)
    gam, bet = bf(1 + 0.1 * torch.randn(H, generator=g)), bf(torch.randn(H, generator=g))
    dy, dres = bf(torch.randn(M, H, generator=g)), bf(torch.randn(M, H, generator=g))
    seed, layer, site = 99, 1, ops.SITE_MLP_OUT
    rc = r.cuda()
    if with_ln:
        _, _, mean, rstd = ops.bdr_ln(rc, gamma=gam.cuda(), beta=bet.cuda(), want_r=False)
    else:
        mean = rstd = None
    dr, dsub, dgw, dgb, dbias = ops.ln_bwd(dy.cuda(), rc, mean, rstd, gam.cuda() if with_ln else None,
                                           dres=dres.cuda(), p=p, seed=seed, layer=layer, site=site,
                                           grads_f32=True)
    rr = r.double().requires_grad_(True)
    gw, gb = gam.double().requires_grad_(True), bet.double().requires_grad_(True)
    y = tp.layer_norm(rr, gw, gb, 1e-5) if with_ln else rr
    (y * dy.double()).sum().backward()
    ref_dr = rr.grad + dres.double()
    assert rel(dr, ref_dr) < TOL
    keep = torch.from_numpy(philox.hidden_mask(np.arange(M), H, layer, site, seed, p)).double() if p > 0 else 1.0
    ref_dsub = ref_dr * keep / (1 - p)
    assert rel(dsub, ref_dsub) < TOL
    assert rel(dbias, ref_dsub.sum(0)) < TOL
    if with_ln:
        assert rel(dgw, gw.grad) < TOL and rel(dgb, gb.grad) < TOL


@pytest.mark.parametrize("sk", [128, 512, 2048])
@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("p", [0.0, 0.1])
def test_softmax(ops, sk, causal, p):
    g = torch.Generator().manual_seed(sk)
    B, nh, sq = 2, 3, sk
    S = bf(torch.randn(B, nh, sq, sk, generator=g) * 4)
    mask = torch.zeros(B, sk)
    mask[1, -5:] = -10000.0
    scale = 1 / math.sqrt(64)
    seed, layer, soff, hoff, nhg = 5, 2, 10, 3, 12
    P, Pd = ops.softmax_fwd(S.cuda(), scale=scale, mask_add=mask.cuda(), causal=causal, p=p, seed=seed, layer=layer,
                            sample_offset=soff, head_offset=hoff, nh_global=nhg)
    sc = tp.attention_scores_mask(S.double() * scale, mask.double(), causal)
    Pr = tp.safe_softmax(sc)
    assert rel(P, Pr) < TOL
    keep = None
    if p > 0:
        keep = torch.from_numpy(philox.attn_prob_mask(np.arange(B) + soff, np.arange(nh) + hoff, sq, sk, nhg, layer,
                                                      seed, p))
        Pdr = Pr * keep.double() / (1 - p)
        assert rel(Pd, Pdr) < TOL
        assert torch.equal(Pd.cpu() == 0, (~keep) | (Pr == 0) | (bf(Pr) == 0))
    dPd = bf(torch.randn(B, nh, sq, sk, generator=g))
    dS = ops.softmax_bwd(P, dPd.cuda(), scale=scale, p=p, seed=seed, layer=layer, sample_offset=soff,
                         head_offset=hoff, nh_global=nhg)
    s_ = sc.clone().requires_grad_(True)
    pr = tp.safe_softmax(s_)
    if p > 0:
        pr = pr * keep.double() / (1 - p)
    (pr * dPd.double()).sum().backward()
    ref = s_.grad * scale
    ref = torch.nan_to_num(ref)
    assert rel(dS, ref) < TOL


def test_colsum(ops):
    g = torch.Generator().manual_seed(0)
    x = bf(torch.randn(1000, 384, generator=g))
    out = ops.colsum(x.cuda(), out_dtype=torch.float32)
    assert rel(out, x.double().sum(0)) < 1e-5
    out2 = ops.colsum(x.cuda(), out_dtype=torch.float32)
    assert torch.equal(out, out2)  # deterministic


def test_bdr_ln_deterministic(ops):
    x = torch.randn(4096, 1024, device="cuda").bfloat16()
    gam = torch.ones(1024, device="cuda").bfloat16()
    bet = torch.zeros(1024, device="cuda").bfloat16()
    a = ops.bdr_ln(x, gamma=gam, beta=bet, p=0.1, seed=3)
    b = ops.bdr_ln(x, gamma=gam, beta=bet, p=0.1, seed=3)
    for u, v in zip(a, b):
        assert torch.equal(u, v)


def test_hidden_keep_bytes_roundtrip(ops):
    """bdr_ln stores the hidden-dropout keep bits it draws; ln_bwd reading them is bit-identical
    to re-drawing the Philox stream, and the bits equal oracle/philox.py's mask."""
    M, H, p, seed, layer, site, row0 = 640, 1024, 0.2, 77, 5, ops.SITE_MLP_OUT, 4096
    g = torch.Generator().manual_seed(3)
    x = bf(torch.randn(M, H, generator=g)).cuda()
    res = bf(torch.randn(M, H, generator=g)).cuda()
    gam = bf(1 + 0.1 * torch.randn(H, generator=g)).cuda()
    bet = bf(0.1 * torch.randn(H, generator=g)).cuda()
    kb = ops.keep_bytes(M, H, "cuda")
    r, y, mean, rstd = ops.bdr_ln(x, residual=res, gamma=gam, beta=bet, p=p, seed=seed, layer=layer, site=site,
                                  row_offset=row0, keep_out=kb)
    bits = np.unpackbits(kb.cpu().numpy(), axis=1, bitorder="little").astype(bool)
    ref = philox.hidden_mask(np.arange(M) + row0, H, layer, site, seed, p)
    assert np.array_equal(bits, ref.reshape(M, H))
    dy = bf(torch.randn(M, H, generator=g)).cuda()
    kw = dict(p=p, seed=seed, layer=layer, site=site, row_offset=row0)
    a = ops.ln_bwd(dy, r, mean, rstd, gam, **kw)
    b = ops.ln_bwd(dy, r, mean, rstd, gam, keep_in=kb, **kw)
    for u, v in zip(a, b):
        if u is not None:
            assert torch.equal(u, v)


@pytest.mark.parametrize("H", [1024, 2048])
def test_bdr_ln_fast_path_bits(ops, H):
    """The local fast path (bias + residual + LayerNorm, whole 256-column chunks): keep bytes equal
    oracle/philox.py bit for bit, r equals the fp32 emulation of (x + bias) * keep / (1 - p) +
    residual rounded to bf16 bit for bit, and y matches the fp64 LayerNorm."""
    M, p, seed, layer, site, row0 = 517, 0.1, 11, 2, ops.SITE_ATTN_OUT, 300
    g = torch.Generator().manual_seed(H + 1)
    x, res = bf(torch.randn(M, H, generator=g)), bf(torch.randn(M, H, generator=g))
    bias, gam, bet = bf(torch.randn(H, generator=g)), bf(1 + 0.1 * torch.randn(H, generator=g)), bf(
        torch.randn(H, generator=g))
    kb = ops.keep_bytes(M, H, "cuda")
    r, y, mean, rstd = ops.bdr_ln(x.cuda(), bias=bias.cuda(), residual=res.cuda(), gamma=gam.cuda(), beta=bet.cuda(),
                                  eps=1e-5, p=p, seed=seed, layer=layer, site=site, row_offset=row0, keep_out=kb)
    keep = philox.hidden_mask(np.arange(M) + row0, H, layer, site, seed, p).reshape(M, H)
    bits = np.unpackbits(kb.cpu().numpy(), axis=1, bitorder="little").astype(bool)
    assert np.array_equal(bits, keep)
    ik = np.float32(1.0) / (np.float32(1.0) - np.float32(p))
    v = (x.float() + bias.float()) * torch.tensor(ik)
    v = torch.where(torch.from_numpy(keep), v, torch.zeros_like(v)) + res.float()
    assert torch.equal(r.cpu(), v.to(torch.bfloat16))
    ref = tp.layer_norm(r.cpu().double(), gam.double(), bet.double(), 1e-5)
    assert rel(y, ref) < TOL


@pytest.mark.parametrize("H", [1024, 2048])
def test_bdr_ln_fast_path_variants(ops, H):
    """The pre-LN layers' two row calls on the fast path: r = residual + dropout(x + bias) without a
    LayerNorm (keep bytes and r bit-exact), and a LayerNorm of x alone (vs the fp64 LayerNorm)."""
    M, p, seed, layer, site, row0 = 389, 0.1, 4, 1, ops.SITE_MLP_OUT, 17
    g = torch.Generator().manual_seed(H + 2)
    x, res = bf(torch.randn(M, H, generator=g)), bf(torch.randn(M, H, generator=g))
    bias, gam, bet = bf(torch.randn(H, generator=g)), bf(1 + 0.1 * torch.randn(H, generator=g)), bf(
        torch.randn(H, generator=g))
    kb = ops.keep_bytes(M, H, "cuda")
    r, y, mean, rstd = ops.bdr_ln(x.cuda(), bias=bias.cuda(), residual=res.cuda(), p=p, seed=seed, layer=layer,
                                  site=site, row_offset=row0, keep_out=kb)
    assert y is None and mean is None
    keep = philox.hidden_mask(np.arange(M) + row0, H, layer, site, seed, p).reshape(M, H)
    assert np.array_equal(np.unpackbits(kb.cpu().numpy(), axis=1, bitorder="little").astype(bool), keep)
    ik = np.float32(1.0) / (np.float32(1.0) - np.float32(p))
    v = torch.where(torch.from_numpy(keep), (x.float() + bias.float()) * torch.tensor(ik), torch.zeros(M, H)) + res.float()
    assert torch.equal(r.cpu(), v.to(torch.bfloat16))
    y2, mean2, rstd2 = ops.layer_norm(x.cuda(), gam.cuda(), bet.cuda(), 1e-5)
    ref = tp.layer_norm(x.double(), gam.double(), bet.double(), 1e-5)
    assert rel(y2, ref) < TOL
    assert rel(mean2, x.double().mean(1)) < 1e-5
