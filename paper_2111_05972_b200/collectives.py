"""The five tensor-parallel collectives of the paper's custom-module API
(SPEC.md:413-421 tp_collective), as autograd functions over
the TP_GROUP created by smp.init.

  fused_allgather_for_tp(t, dim)              AG along dim      | backward: reduce-scatter along dim
  fwd_allreduce_for_tp(t)                     AR                | backward: identity
  bwd_allreduce_for_tp(t)                     identity          | backward: AR
  scatter_and_merge_for_tp(t, split, merge)   all-to-all        | backward: all-to-all (merge, split)
  reduce_scatter_for_tp(t, dim)               RS along dim      | backward: allgather along dim

Transport: torch.distributed over NCCL (NVLink / NVSwitch on one node), one
process per GPU; reductions are NCCL's (fixed ring/tree order per
communicator, deterministic run to run).  With tp_size()==1 every collective
is the identity.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .errors import NotDivisibleError
from .state import STATE


def _group():
    return STATE.tp_group


def _T() -> int:
    return STATE.tp_size


def _movedim_front(t: torch.Tensor, dim: int) -> torch.Tensor:
    return t.movedim(dim, 0).contiguous() if dim % t.dim() != 0 else t.contiguous()


def all_gather(t: torch.Tensor, dim: int = 0, group=None) -> torch.Tensor:
    T = _T()
    if T == 1:
        return t
    dim = dim % t.dim()
    src = _movedim_front(t, dim)
    out = torch.empty((T * src.shape[0],) + tuple(src.shape[1:]), dtype=t.dtype, device=t.device)
    dist.all_gather_into_tensor(out, src, group=group or _group())
    return out.movedim(0, dim) if dim != 0 else out


def reduce_scatter(t: torch.Tensor, dim: int = 0, group=None) -> torch.Tensor:
    T = _T()
    if T == 1:
        return t
    dim = dim % t.dim()
    if t.shape[dim] % T:
        raise NotDivisibleError(f"reduce_scatter: dim {dim} of size {t.shape[dim]} not divisible by T={T}")
    src = _movedim_front(t, dim)
    out = torch.empty((src.shape[0] // T,) + tuple(src.shape[1:]), dtype=t.dtype, device=t.device)
    dist.reduce_scatter_tensor(out, src, group=group or _group())
    return out.movedim(0, dim).contiguous() if dim != 0 else out


def all_reduce(t: torch.Tensor, group=None) -> torch.Tensor:
    if _T() == 1:
        return t
    dist.all_reduce(t, group=group or _group())
    return t


def all_to_all(t: torch.Tensor, split_dim: int, merge_dim: int, group=None) -> torch.Tensor:
    T = _T()
    if T == 1:
        return t
    split_dim, merge_dim = split_dim % t.dim(), merge_dim % t.dim()
    if t.shape[split_dim] % T:
        raise NotDivisibleError(f"scatter_and_merge: split dim {split_dim} of size {t.shape[split_dim]} "
                                f"not divisible by T={T}")
    chunks = [c.contiguous() for c in torch.chunk(t, T, split_dim)]
    src = torch.stack(chunks, 0)
    out = torch.empty_like(src)
    dist.all_to_all_single(out, src, group=group or _group())
    return torch.cat(list(out.unbind(0)), merge_dim)


class _AllGather(torch.autograd.Function):
    @staticmethod
    def forward(ctx, t, dim):
        ctx.dim = dim
        return all_gather(t, dim)

    @staticmethod
    def backward(ctx, g):
        return reduce_scatter(g.contiguous(), ctx.dim), None


class _FwdAllReduce(torch.autograd.Function):
    @staticmethod
    def forward(ctx, t):
        return all_reduce(t.clone())

    @staticmethod
    def backward(ctx, g):
        return g


class _BwdAllReduce(torch.autograd.Function):
    @staticmethod
    def forward(ctx, t):
        return t.view_as(t)

    @staticmethod
    def backward(ctx, g):
        return all_reduce(g.contiguous().clone())


class _ScatterAndMerge(torch.autograd.Function):
    @staticmethod
    def forward(ctx, t, split_dim, merge_dim):
        ctx.dims = (split_dim, merge_dim)
        return all_to_all(t, split_dim, merge_dim)

    @staticmethod
    def backward(ctx, g):
        s, m = ctx.dims
        return all_to_all(g.contiguous(), m, s), None, None


class _ReduceScatter(torch.autograd.Function):
    @staticmethod
    def forward(ctx, t, dim):
        ctx.dim = dim
        return reduce_scatter(t, dim)

    @staticmethod
    def backward(ctx, g):
        return all_gather(g.contiguous(), ctx.dim), None


class _TpDpEntry(torch.autograd.Function):
    """TP-across-DP module entry: gather every peer's samples along the batch.
    Backward: the gathered gradient is TP-replicated (the sub-layer's input-gradient
    allreduce made it so), so each rank keeps its own block."""

    @staticmethod
    def forward(ctx, t):
        ctx.b = t.shape[0]
        return all_gather(t.contiguous(), 0)

    @staticmethod
    def backward(ctx, g):
        i = STATE.tp_rank
        return g[i * ctx.b:(i + 1) * ctx.b].contiguous()


class _TpDpExit(torch.autograd.Function):
    """TP-across-DP module exit: return each sample to the rank it originated from.
    Backward: allgather the per-rank output gradients (replicated full gradient)."""

    @staticmethod
    def forward(ctx, t):
        T, i = STATE.tp_size, STATE.tp_rank
        b = t.shape[0] // T
        return t[i * b:(i + 1) * b].contiguous()

    @staticmethod
    def backward(ctx, g):
        return all_gather(g.contiguous(), 0)


class _AllGatherReplicated(torch.autograd.Function):
    """Allgather of per-rank slices of a TP-replicated result (prescaled batch):
    every rank computes the same loss, so the backward keeps the local slice (no comm)."""

    @staticmethod
    def forward(ctx, t, dim):
        ctx.dim, ctx.n = dim, t.shape[dim]
        return all_gather(t.contiguous(), dim)

    @staticmethod
    def backward(ctx, g):
        i = STATE.tp_rank
        return g.narrow(ctx.dim, i * ctx.n, ctx.n).contiguous(), None


def allgather_replicated(t: torch.Tensor, dim: int) -> torch.Tensor:
    return t if STATE.tp_size == 1 else _AllGatherReplicated.apply(t, dim)


def tp_dp_entry(t: torch.Tensor) -> torch.Tensor:
    return t if STATE.tp_size == 1 else _TpDpEntry.apply(t)


def tp_dp_exit(t: torch.Tensor) -> torch.Tensor:
    return t if STATE.tp_size == 1 else _TpDpExit.apply(t)


def fused_allgather_for_tp(tensor: torch.Tensor, dim: int) -> torch.Tensor:
    """Allgather across TP_GROUP, concatenated along dim."""
    return _AllGather.apply(tensor, dim)


def fwd_allreduce_for_tp(tensor: torch.Tensor) -> torch.Tensor:
    """Allreduce across TP_GROUP in forward; identity in backward."""
    return _FwdAllReduce.apply(tensor)


def bwd_allreduce_for_tp(tensor: torch.Tensor) -> torch.Tensor:
    """Identity in forward; allreduce across TP_GROUP in backward."""
    return _BwdAllReduce.apply(tensor)


def scatter_and_merge_for_tp(tensor: torch.Tensor, split_dim: int, merge_dim: int) -> torch.Tensor:
    """Slice along split_dim into T slices, all-to-all, concatenate along merge_dim."""
    return _ScatterAndMerge.apply(tensor, split_dim, merge_dim)


def reduce_scatter_for_tp(tensor: torch.Tensor, dim: int) -> torch.Tensor:
    """Slice along dim and reduce-scatter the slices across TP_GROUP."""
    return _ReduceScatter.apply(tensor, dim)
