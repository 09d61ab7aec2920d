"""Memory-mode TP sub-layers on the GPU ("optimize='memory'", PAPER.md:713-717, 763;
SPEC.md:449-475).

Activations between sub-layers are channel-sharded: every rank of the TP group holds all the
group's token rows and H/T of the hidden channels (stack entry = scatter_and_merge(split
channel, merge batch)).  Every linear is input-split: the local GEMM of the rank's
input channels produces a full-width partial, which is reduce-scattered over output channels
(the output is laid out as T column blocks so block j is contiguous for rank j).  The QKV
weight rows are stored rank-major (q_j | k_j | v_j per rank), so the reduce-scatter slice of
rank j is exactly its heads.  LayerNorms are distributed: local sum x / sum x^2 ->
allreduce of 2 floats per row -> normalise the local channels.  Hidden dropout
uses the global column index (col_offset = j*H/T), so the masks equal the single-rank ones.

The oracle restatement is oracle/tp.py dist_attention_forward_memory / dist_mlp_forward_memory;
tests/mp_tp_check.py checks this path against it at T = 2 / 4.
"""
from __future__ import annotations

import torch

from . import collectives as C
from . import kernels as K
from . import layers as L
from . import ops
from .ops import SITE_ATTN_OUT, SITE_MLP_OUT


def _allreduce_(t: torch.Tensor) -> torch.Tensor:
    return C.all_reduce(t)


class DistLayerNormFn(torch.autograd.Function):
    """LayerNorm over the full hidden size of channel-sharded rows (gamma/beta: local chunks)."""

    @staticmethod
    def forward(ctx, r, gamma, beta, eps, h_total):
        M = r.shape[0]
        r2 = r.reshape(M, -1)
        _, _, _, _, sums = ops.bdr_ln_dist(r2, want_r=False, row_sums=True)
        _allreduce_(sums)
        _, y, mean, rstd, _ = ops.bdr_ln_dist(r2, gamma=gamma, beta=beta, eps=eps, want_r=False, ext_sums=sums,
                                              h_total=h_total)
        ctx.h_total = h_total
        ctx.save_for_backward(r2, mean, rstd, gamma)
        return y.view_as(r)

    @staticmethod
    def backward(ctx, dy):
        r2, mean, rstd, gamma = ctx.saved_tensors
        dy2 = dy.reshape(r2.shape).contiguous()
        sums = ops.ln_bwd_dist(dy2, r2, mean, rstd, gamma, sums_only=True)
        _allreduce_(sums)
        dr, _, dgamma, dbeta, _ = ops.ln_bwd_dist(dy2, r2, mean, rstd, gamma, ext_sums=sums, h_total=ctx.h_total)
        return dr.view_as(dy), dgamma, dbeta, None, None


class BiasDropResidualFn(torch.autograd.Function):
    """r = residual + dropout(x + bias) on the local channels (global dropout columns)."""

    @staticmethod
    def forward(ctx, x, bias, residual, p, seed, layer, site, row_offset, col_offset, rng=None):
        r, _, _, _, _ = ops.bdr_ln_dist(x, bias=bias, residual=residual, p=p, seed=seed, rng=rng, layer=layer, site=site,
                                        row_offset=row_offset, col_offset=col_offset)
        ctx.cfg = (p, seed, layer, site, row_offset, col_offset, rng)
        ctx.has_res = residual is not None
        return r

    @staticmethod
    def backward(ctx, dr):
        p, seed, layer, site, row_offset, col_offset, rng = ctx.cfg
        dr = dr.contiguous()
        _, dsub, _, _, dbias = ops.ln_bwd_dist(dr, None, None, None, None, p=p, seed=seed, rng=rng, layer=layer, site=site,
                                               row_offset=row_offset, col_offset=col_offset, want_dbias=True)
        return dsub, dbias, (dr if ctx.has_res else None), None, None, None, None, None, None, None


class InputSplitLinearRS(torch.autograd.Function):
    """y_j = sum over ranks of x_r W_r^T, column block j (reduce-scatter over output channels).

    x [M, K/T] (local input channels), W [N, K/T] (all output rows, local input columns);
    the partial is computed as T column blocks [T, M, N/T] (one batched tcgen05 GEMM) so the
    NCCL reduce-scatter sends contiguous blocks."""

    @staticmethod
    def forward(ctx, x, W, T):
        M, Kl = x.shape
        N = W.shape[0]
        nb = N // T
        part = torch.empty(T, M, nb, dtype=torch.bfloat16, device=x.device)
        K.gemm_raw(x, 0, Kl, (0, 0), W, 0, Kl, (nb * Kl, 0), part, nb, (M * nb, 0), M, nb, Kl, nb=(T, 1))
        ctx.T = T
        ctx.save_for_backward(x, W)
        return C.reduce_scatter(part.view(T * M, nb), 0)

    @staticmethod
    def backward(ctx, dy):
        x, W = ctx.saved_tensors
        T = ctx.T
        M, Kl = x.shape
        N = W.shape[0]
        nb = N // T
        dfull = C.all_gather(dy.contiguous(), 0).view(T, M, nb)  # block j = dL/d(partial block j)
        dx = torch.empty(M, Kl, dtype=torch.bfloat16, device=x.device)
        for j in range(T):  # dx = sum_j dfull_j W_j   (ascending block order)
            K.matmul_nn(dfull[j], W[j * nb:(j + 1) * nb], out=dx, beta=0.0 if j == 0 else 1.0)
        dW = torch.empty_like(W)
        # dW block j = dfull_j^T x   (batched over the T blocks)
        K.gemm_raw(dfull, 1, nb, (M * nb, 0), x, 1, Kl, (0, 0), dW, Kl, (nb * Kl, 0), nb, Kl, M, nb=(T, 1))
        return dx, dW, None


class BiasActFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, z, bias, act):
        y, pre = ops.bias_act(z, bias, act)
        ctx.act = act
        ctx.save_for_backward(pre)
        return y

    @staticmethod
    def backward(ctx, dy):
        (pre,) = ctx.saved_tensors
        dz = ops.act_bwd(dy, pre, ctx.act)
        return dz, ops.colsum(dz), None


class AttentionCoreFn(torch.autograd.Function):
    """Local-heads attention on the packed [M, 3*nh_l*dh] QKV of this rank's heads."""

    @staticmethod
    def forward(ctx, qkv, mask_add, B, s, m):
        fused = L.use_flash(s, m.head_dim)
        if fused:
            bits, join = L._keep_bits_async(B, s, m, qkv.device)
            join()
            ctxv, lse = ops.flash_attn_fwd(qkv, B, s, m.heads_local, m.head_dim, mask_add=mask_add, causal=m.causal,
                                           p=m.p_attn, keep_bits=bits)
            P, Pd = lse, bits
        else:
            ctxv, P, Pd = L.attn_core_fwd(qkv, B, s, m, mask_add)
        ctx.cfg = (B, s, m, fused)
        ctx.save_for_backward(qkv, ctxv, P, Pd if Pd is not P else None, mask_add)
        return ctxv

    @staticmethod
    def backward(ctx, dctx):
        B, s, m, fused = ctx.cfg
        qkv, ctxv, P, Pd, mask_add = ctx.saved_tensors
        dctx = dctx.contiguous()
        if fused:
            dqkv = ops.flash_attn_bwd(dctx, qkv, ctxv, P, B, s, m.heads_local, m.head_dim, mask_add=mask_add,
                                      causal=m.causal, p=m.p_attn, keep_bits=Pd if m.p_attn > 0 else None)
        else:
            dqkv = L.attn_core_bwd(dctx, qkv, P, Pd if Pd is not None else P, B, s, m)
        return dqkv, None, None, None, None


def attention(X, mod, mask_add, m: L.LayerMeta, j: int):
    """dist_attention_forward, memory mode: X [T*b, s, H/T] -> [T*b, s, H/T]."""
    T = m.tp_size
    Bg, s, hs = X.shape
    M = Bg * s
    H = hs * T
    x2 = X.reshape(M, hs)
    h = DistLayerNormFn.apply(x2, mod.pre_ln_weight, mod.pre_ln_bias, m.eps, H) if m.pre_ln else x2
    qkv = InputSplitLinearRS.apply(h, mod.qkv_weight, T)  # [M, 3H/T]: this rank's heads, q | k | v
    qkv = BiasDropResidualFn.apply(qkv, mod.qkv_bias, None, 0.0, 0, 0, SITE_ATTN_OUT, 0, 0)
    ctxv = AttentionCoreFn.apply(qkv, mask_add, Bg, s, m)
    o = InputSplitLinearRS.apply(ctxv, mod.dense_weight, T)  # [M, H/T]
    r = BiasDropResidualFn.apply(o, mod.dense_bias, x2, m.p_hidden, m.seed, m.layer_id, SITE_ATTN_OUT, m.row_offset,
                                 j * hs, m.rng)
    if m.post_ln:
        r = DistLayerNormFn.apply(r, mod.post_ln_weight, mod.post_ln_bias, m.eps, H)
    return r.view(Bg, s, hs)


def mlp(X, mod, m: L.LayerMeta, j: int):
    """dist_mlp_forward, memory mode."""
    T = m.tp_size
    Bg, s, hs = X.shape
    M = Bg * s
    H = hs * T
    x2 = X.reshape(M, hs)
    h = DistLayerNormFn.apply(x2, mod.pre_ln_weight, mod.pre_ln_bias, m.eps, H) if m.pre_ln else x2
    z = InputSplitLinearRS.apply(h, mod.fc1_weight, T)  # [M, 4H/T]
    a = BiasActFn.apply(z, mod.fc1_bias, m.activation)
    g = InputSplitLinearRS.apply(a, mod.fc2_weight, T)  # [M, H/T]
    r = BiasDropResidualFn.apply(g, mod.fc2_bias, x2, m.p_hidden, m.seed, m.layer_id, SITE_MLP_OUT, m.row_offset,
                                 j * hs, m.rng)
    if m.post_ln:
        r = DistLayerNormFn.apply(r, mod.post_ln_weight, mod.post_ln_bias, m.eps, H)
    return r.view(Bg, s, hs)


class _ChannelSlice(torch.autograd.Function):
    """Prescaled-batch memory entry: the replicated input's channel chunk (backward: allgather)."""

    @staticmethod
    def forward(ctx, x, T, j):
        n = x.shape[-1] // T
        return x[..., j * n:(j + 1) * n].contiguous()

    @staticmethod
    def backward(ctx, g):
        return C.all_gather(g.contiguous(), -1), None, None


def entry(x: torch.Tensor, T: int, j: int, prescaled: bool) -> torch.Tensor:
    """Stack entry (oracle memory_entry): [b, s, H] -> [T*b, s, H/T]."""
    if prescaled:
        return _ChannelSlice.apply(x, T, j)
    return C.scatter_and_merge_for_tp(x, -1, 0)


def exit(X: torch.Tensor, prescaled: bool) -> torch.Tensor:  # noqa: A001
    """Stack exit (oracle memory_exit): [T*b, s, H/T] -> [b, s, H]."""
    if prescaled:
        return C.allgather_replicated(X, -1)
    return C.scatter_and_merge_for_tp(X, 0, -1)
