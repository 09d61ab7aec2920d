"""Torch-tensor wrappers of the row kernels (LayerNorm, softmax, dropout, colsum).

Same contract as kernels.py: CUDA tensors only, outputs from the torch caching
allocator, launches on the current stream, no CPU path.
"""
from __future__ import annotations

import torch

from . import _lib
from .kernels import _check_cuda, _ptr, _stream

SITE_ATTN_PROB, SITE_ATTN_OUT, SITE_MLP_OUT = 0, 1, 2


def rng_next(counter: torch.Tensor) -> torch.Tensor:
    """Snapshot the device step counter into a new 1-element tensor and increment the counter
    (smpk_rng_next, on the current stream; CUDA-graph capturable)."""
    _check_cuda(counter)
    snap = torch.empty(1, dtype=torch.int64, device=counter.device)
    _lib.call("smpk_rng_next", _ptr(counter), _ptr(snap), _stream())
    return snap


def _f32(t):
    return None if t is None else t


def bdr_ln(x: torch.Tensor, *, bias=None, residual=None, gamma=None, beta=None, eps=1e-5, p=0.0, seed=0, rng=None,
           layer=0, site=SITE_ATTN_OUT, row_offset=0, want_r=True, want_y=True, nslots=1, slot_stride=0,
           out_peers=None, peer_off=0, rows=None, cols=None, keep_out=None, x_peers=None, x_peer_off=0):
    """r = residual + dropout(x + bias); y = LN(r). Returns (r, y, mean, rstd) (None where not computed).

    nslots > 1: x is the ascending-rank sum of nslots partial slots slot_stride elements apart
    (reduce-scatter consumer); out_peers (device table of peer addresses): the output is also
    stored to every peer at element offset peer_off (allgather producer); keep_out ([M, H/8]
    uint8) receives the hidden-dropout keep bits for the backward."""
    _check_cuda(x, bias, residual, gamma, beta)
    M, H = (rows, cols) if rows is not None else x.shape
    r = torch.empty(M, H, dtype=torch.bfloat16, device=x.device) if want_r else None
    y = mean = rstd = None
    if gamma is not None:
        y = torch.empty(M, H, dtype=torch.bfloat16, device=x.device) if want_y else None
        mean = torch.empty(M, dtype=torch.float32, device=x.device)
        rstd = torch.empty(M, dtype=torch.float32, device=x.device)
    npeers = 0 if out_peers is None else out_peers.numel()
    _lib.call("smpk_bdr_ln_fwd_ex", _ptr(x), int(nslots), int(slot_stride), _ptr(bias), _ptr(residual), _ptr(r),
              _ptr(gamma), _ptr(beta), _ptr(y), _ptr(mean), _ptr(rstd), _ptr(out_peers), npeers, int(peer_off), M, H,
              float(eps), float(p), int(seed) & (2 ** 64 - 1), _ptr(rng), int(layer), int(site), int(row_offset),
              _ptr(keep_out if p > 0 else None), _ptr(x_peers), int(x_peer_off), _stream())
    return r, y, mean, rstd


def layer_norm(x: torch.Tensor, gamma, beta, eps=1e-5):
    _, y, mean, rstd = bdr_ln(x, gamma=gamma, beta=beta, eps=eps, want_r=False)
    return y, mean, rstd


def keep_bytes(M: int, H: int, device) -> torch.Tensor:
    """Buffer for the hidden-dropout keep bits of an [M, H] activation ([M, H/8] bytes)."""
    return torch.empty(M, (H + 7) // 8, dtype=torch.uint8, device=device)


def add(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """a + b through the row kernel (bf16 round once)."""
    r, _, _, _ = bdr_ln(a, residual=b)
    return r


def ln_bwd(dy, r, mean, rstd, gamma, *, dres=None, p=0.0, seed=0, rng=None, layer=0, site=SITE_ATTN_OUT, row_offset=0,
           want_dgamma=True, want_dbias=True, grads_f32=False, want_dr=True, nslots=1, slot_stride=0,
           out_peers=None, peer_off=0, rows=None, cols=None, keep_in=None, x_peers=None, x_peer_off=0,
           param_grads_out=None):
    """Backward of bdr_ln. Returns (dr, dsub, dgamma, dbeta, dbias); dsub is dr when p == 0.
    param_grads_out: one contiguous [n, H] buffer receiving the rows (dgamma, dbeta) [+ dbias].

    gamma None = no-LayerNorm mode (d = dy + dres).  nslots / out_peers as in bdr_ln (dy read as a
    slot sum; dsub also stored to every peer)."""
    _check_cuda(dy, r, gamma, dres)
    M, H = (rows, cols) if rows is not None else dy.shape
    dev = dy.device
    dr = torch.empty(M, H, dtype=torch.bfloat16, device=dev) if want_dr else None
    dsub = torch.empty(M, H, dtype=torch.bfloat16, device=dev) if p > 0 else None
    gdt = torch.float32 if grads_f32 else torch.bfloat16
    dgamma = torch.empty(H, dtype=gdt, device=dev) if (want_dgamma and gamma is not None) else None
    dbeta = torch.empty(H, dtype=gdt, device=dev) if (want_dgamma and gamma is not None) else None
    dbias = torch.empty(H, dtype=gdt, device=dev) if want_dbias else None
    if param_grads_out is not None:  # rows: [dgamma, dbeta,] [dbias]
        k = 0
        if dgamma is not None:
            dgamma, dbeta, k = param_grads_out[0], param_grads_out[1], 2
        if dbias is not None:
            dbias = param_grads_out[k]
    ws_bytes = _lib.size("smpk_ln_bwd_workspace", M, H)
    ws = torch.empty(max(ws_bytes, 4) // 4, dtype=torch.float32, device=dev)
    npeers = 0 if out_peers is None else out_peers.numel()
    _lib.call("smpk_ln_bwd_ex", _ptr(dy), int(nslots), int(slot_stride), _ptr(r), _ptr(mean), _ptr(rstd),
              _ptr(gamma), _ptr(dres), _ptr(dr), _ptr(dsub), _ptr(out_peers), npeers, int(peer_off), _ptr(dgamma),
              _ptr(dbeta), _ptr(dbias), int(grads_f32), 0, M, H, float(p), int(seed) & (2 ** 64 - 1), _ptr(rng), int(layer),
              int(site), int(row_offset), _ptr(keep_in if p > 0 else None), _ptr(x_peers), int(x_peer_off), _ptr(ws),
              int(ws_bytes), _stream(),
              launches=2 if (dgamma is not None or dbeta is not None or dbias is not None) else 1)
    if dsub is None:
        dsub = dr if dr is not None else (dy if nslots == 1 else None)
    return dr, dsub, dgamma, dbeta, dbias


def softmax_fwd(scores: torch.Tensor, *, scale: float, mask_add=None, causal=False, p=0.0, seed=0, rng=None, layer=0,
                sample_offset=0, head_offset=0, nh_global=None):
    """scores [B, nh, sq, sk] -> (P, Pd) with Pd = P when p == 0."""
    _check_cuda(scores, mask_add)
    B, nh, sq, sk = scores.shape
    P = torch.empty_like(scores)
    Pd = torch.empty_like(scores) if p > 0 else None
    if mask_add is not None:
        mask_add = mask_add.reshape(B, sk).to(torch.float32).contiguous()
    _lib.call("smpk_softmax_fwd", _ptr(scores), _ptr(P), _ptr(Pd), _ptr(mask_add), B, nh, sq, sk, float(scale),
              int(bool(causal)), float(p), int(seed) & (2 ** 64 - 1), _ptr(rng), int(layer), int(sample_offset), int(head_offset),
              int(nh_global if nh_global is not None else nh), _stream())
    return P, (Pd if Pd is not None else P)


def softmax_bwd(P: torch.Tensor, dPd: torch.Tensor, *, scale: float, p=0.0, seed=0, rng=None, layer=0, sample_offset=0,
                head_offset=0, nh_global=None, out=None):
    _check_cuda(P, dPd)
    B, nh, sq, sk = P.shape
    dS = out if out is not None else torch.empty_like(P)
    _lib.call("smpk_softmax_bwd", _ptr(P), _ptr(dPd), _ptr(dS), B, nh, sq, sk, float(scale), float(p),
              int(seed) & (2 ** 64 - 1), _ptr(rng), int(layer), int(sample_offset), int(head_offset),
              int(nh_global if nh_global is not None else nh), _stream())
    return dS


def colsum(x: torch.Tensor, *, out_dtype=None) -> torch.Tensor:
    """Column sums of a row-major [M, N] bf16 matrix (bias gradient)."""
    _check_cuda(x)
    M, N = x.shape
    out = torch.empty(N, dtype=out_dtype or x.dtype, device=x.device)
    ws_bytes = _lib.size("smpk_colsum_workspace", M, N)
    ws = torch.empty(max(ws_bytes, 4) // 4, dtype=torch.float32, device=x.device)
    _lib.call("smpk_colsum", _ptr(x), M, N, x.stride(0), _ptr(out), int(out.dtype == torch.float32), 0, _ptr(ws),
              int(ws_bytes), _stream())
    return out


def attn_dropout_bits(B: int, nh: int, sq: int, sk: int, *, p: float, seed=0, rng=None, layer=0, sample_offset=0,
                      head_offset=0, nh_global=None, device=None, out=None, causal=False, sample_block=None,
                      block_stride=0) -> torch.Tensor | None:
    """Keep bits [B, nh, sq, sk/32] (uint32 words as int32) of the attention-probability dropout;
    None when p == 0.  Generated once per layer and shared by the forward and the backward.
    sample_block / block_stride: the B samples are blocks of sample_block consecutive global
    samples block_stride apart (an overlapped micro-batch's gathered samples)."""
    if p <= 0.0:
        return None
    bits = out if out is not None else torch.empty(B, nh, sq, sk // 32, dtype=torch.int32,
                                                   device=device or torch.cuda.current_device())
    _check_cuda(bits)
    if sample_block is None:
        _lib.call("smpk_attn_dropout_bits", B, nh, sq, sk, float(p), int(seed) & (2 ** 64 - 1), _ptr(rng),
                  int(layer), int(sample_offset), int(head_offset), int(nh_global if nh_global is not None else nh),
                  _ptr(bits), int(bool(causal)), _stream())
    else:
        _lib.call("smpk_attn_dropout_bits_blocked", B, nh, sq, sk, float(p), int(seed) & (2 ** 64 - 1), _ptr(rng),
                  int(layer), int(sample_offset), int(sample_block), int(block_stride), int(head_offset),
                  int(nh_global if nh_global is not None else nh), _ptr(bits), int(bool(causal)), _stream())
    return bits


def flash_attn_bwd(dctx: torch.Tensor, qkv: torch.Tensor, ctx: torch.Tensor, lse: torch.Tensor, B: int, s: int,
                   nh: int, dh: int, *, mask_add=None, causal=False, p=0.0, keep_bits=None, dqkv=None):
    """Backward of flash_attn_fwd: returns dqkv [B*s, 3*nh*dh] (dQ | dK | dV blocks)."""
    _check_cuda(dctx, qkv, ctx, lse, mask_add, keep_bits)
    if p > 0 and keep_bits is None:
        raise ValueError("flash_attn_bwd: dropout needs the forward's keep bits")
    dctx = dctx.contiguous()
    dqkv = dqkv if dqkv is not None else torch.empty_like(qkv)
    if mask_add is not None:
        mask_add = mask_add.reshape(B, s).to(torch.float32).contiguous()
    ws_bytes = _lib.size("smpk_flash_attn_bwd_workspace", B, nh, s, dh)
    ws = torch.empty(ws_bytes // 4, dtype=torch.float32, device=qkv.device)
    _lib.call("smpk_flash_attn_bwd", _ptr(qkv), qkv.stride(0), _ptr(ctx), ctx.stride(0), _ptr(dctx), dctx.stride(0),
              _ptr(lse), B, nh, s, dh, _ptr(dqkv), _ptr(mask_add), float(1.0 / dh ** 0.5), int(bool(causal)),
              float(p), _ptr(keep_bits if p > 0 else None), _ptr(ws), int(ws_bytes), _stream())
    return dqkv


def flash_attn_fwd(qkv: torch.Tensor, B: int, s: int, nh: int, dh: int, *, mask_add=None, causal=False, p=0.0,
                   keep_bits=None, out=None, lse_out=None):
    """Fused attention on the packed QKV buffer [B*s, 3*nh*dh] (q | k | v blocks, heads inside each).
    Dropout (p > 0) uses keep_bits from attn_dropout_bits.
    Returns (ctx [B*s, nh*dh] bf16, lse [B, nh, s] fp32 log2-domain)."""
    _check_cuda(qkv, mask_add, keep_bits)
    if p > 0 and keep_bits is None:
        raise ValueError("flash_attn_fwd: dropout needs keep bits (ops.attn_dropout_bits)")
    ctx = out if out is not None else torch.empty(B * s, nh * dh, dtype=qkv.dtype, device=qkv.device)
    lse = lse_out if lse_out is not None else torch.empty(B, nh, s, dtype=torch.float32, device=qkv.device)
    if mask_add is not None:
        mask_add = mask_add.reshape(B, s).to(torch.float32).contiguous()
    _lib.call("smpk_flash_attn_fwd", _ptr(qkv), qkv.stride(0), B, nh, s, dh, _ptr(ctx), ctx.stride(0), _ptr(lse),
              _ptr(mask_add), float(1.0 / dh ** 0.5), int(bool(causal)), float(p),
              _ptr(keep_bits if p > 0 else None), _stream())
    return ctx, lse


# ---------------------------------------------------------------------------
# channel-sharded (memory-mode) LayerNorm and the standalone bias + activation
# ---------------------------------------------------------------------------

def bdr_ln_dist(x: torch.Tensor, *, bias=None, residual=None, gamma=None, beta=None, eps=1e-5, p=0.0, seed=0, rng=None, layer=0,
                site=SITE_ATTN_OUT, row_offset=0, col_offset=0, want_r=True, row_sums=False, ext_sums=None,
                h_total=0):
    """smpk_bdr_ln_fwd_dist on the local H/T columns.  row_sums=True also returns the partial
    [M, 2] (sum r, sum r^2); ext_sums (the group's [M, 2] sums) normalises with the full-row
    statistics.  Returns (r, y, mean, rstd, sums)."""
    _check_cuda(x, bias, residual, gamma, beta, ext_sums)
    M, H = x.shape
    dev = x.device
    r = torch.empty(M, H, dtype=torch.bfloat16, device=dev) if want_r else None
    y = mean = rstd = None
    if gamma is not None:
        y = torch.empty(M, H, dtype=torch.bfloat16, device=dev)
        mean = torch.empty(M, dtype=torch.float32, device=dev)
        rstd = torch.empty(M, dtype=torch.float32, device=dev)
    sums = torch.empty(M, 2, dtype=torch.float32, device=dev) if row_sums else None
    _lib.call("smpk_bdr_ln_fwd_dist", _ptr(x), _ptr(bias), _ptr(residual), _ptr(r), _ptr(gamma), _ptr(beta), _ptr(y),
              _ptr(mean), _ptr(rstd), M, H, float(eps), float(p), int(seed) & (2 ** 64 - 1), _ptr(rng), int(layer), int(site),
              int(row_offset), int(col_offset), _ptr(sums), _ptr(ext_sums), int(h_total), _stream())
    return r, y, mean, rstd, sums


def ln_bwd_dist(dy, r, mean, rstd, gamma, *, dres=None, p=0.0, seed=0, rng=None, layer=0, site=SITE_ATTN_OUT, row_offset=0,
                col_offset=0, sums_only=False, ext_sums=None, h_total=0, want_dbias=False):
    """smpk_ln_bwd_dist.  sums_only=True returns the partial [M, 2] (sum g, sum g*xhat); otherwise
    (dr, dsub, dgamma, dbeta, dbias) with the row means taken from ext_sums (gamma None: no LN)."""
    _check_cuda(dy, r, gamma, dres, ext_sums)
    M, H = dy.shape
    dev = dy.device
    ws_bytes = _lib.size("smpk_ln_bwd_workspace", M, H)
    ws = torch.empty(max(ws_bytes, 4) // 4, dtype=torch.float32, device=dev)
    if sums_only:
        sums = torch.empty(M, 2, dtype=torch.float32, device=dev)
        _lib.call("smpk_ln_bwd_dist", _ptr(dy), _ptr(r), _ptr(mean), _ptr(rstd), _ptr(gamma), None, None, None, None,
                  None, None, 0, M, H, float(p), int(seed) & (2 ** 64 - 1), _ptr(rng), int(layer), int(site), int(row_offset),
                  int(col_offset), _ptr(sums), None, 0, _ptr(ws), int(ws_bytes), _stream(), launches=1)
        return sums
    dr = torch.empty(M, H, dtype=torch.bfloat16, device=dev)
    dsub = torch.empty(M, H, dtype=torch.bfloat16, device=dev) if p > 0 else None
    dgamma = torch.empty(H, dtype=torch.bfloat16, device=dev) if gamma is not None else None
    dbeta = torch.empty(H, dtype=torch.bfloat16, device=dev) if gamma is not None else None
    dbias = torch.empty(H, dtype=torch.bfloat16, device=dev) if want_dbias else None
    _lib.call("smpk_ln_bwd_dist", _ptr(dy), _ptr(r), _ptr(mean), _ptr(rstd), _ptr(gamma), _ptr(dres), _ptr(dr),
              _ptr(dsub), _ptr(dgamma), _ptr(dbeta), _ptr(dbias), 0, M, H, float(p), int(seed) & (2 ** 64 - 1), _ptr(rng),
              int(layer), int(site), int(row_offset), int(col_offset), None, _ptr(ext_sums), int(h_total), _ptr(ws),
              int(ws_bytes), _stream(), launches=2 if (dgamma is not None or dbias is not None) else 1)
    return dr, (dsub if dsub is not None else dr), dgamma, dbeta, dbias


def bias_act(x: torch.Tensor, bias: torch.Tensor, act: str):
    """(y, pre): pre = bf16(x + bias), y = act(pre)."""
    from .kernels import ACT
    _check_cuda(x, bias)
    M, N = x.shape
    pre = torch.empty_like(x)
    y = torch.empty_like(x)
    _lib.call("smpk_bias_act_fwd", _ptr(x), _ptr(bias), M, N, ACT[act], _ptr(pre), _ptr(y), _stream())
    return y, pre


def act_bwd(dy: torch.Tensor, pre: torch.Tensor, act: str) -> torch.Tensor:
    from .kernels import ACT
    _check_cuda(dy, pre)
    M, N = dy.shape
    dx = torch.empty_like(dy)
    _lib.call("smpk_act_bwd", _ptr(dy.contiguous()), _ptr(pre), M, N, ACT[act], _ptr(dx), _stream())
    return dx
