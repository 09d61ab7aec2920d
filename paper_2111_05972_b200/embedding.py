"""Embeddings, the LM head and the vocab-parallel cross-entropy on libsmpk.

* ``DistributedEmbedding`` — the paper's module:
  the table is sharded along the EMBEDDING dimension; indices are allgathered, each
  rank looks up its D/T slice for every gathered index, and scatter_and_merge
  (split batch, merge embedding) returns full-width rows to the originating rank.
  Prescaled batch: no gather; the a2a becomes an allgather along emb.
* ``VocabParallelEmbedding`` — builder-defined extension for the north_star's
  "vocab-parallel embedding": rank j owns rows
  [j*Vp/T, (j+1)*Vp/T) of the Vp-padded vocabulary; masked lookup + allreduce
  (prescaled) or reduce-scatter over the batch (TP across DP).
* ``vocab_parallel_cross_entropy`` — per-token softmax CE over a vocab-sharded logits
  tensor: local (max, sum-exp, target logit) -> allgather of
  3 floats per row -> rank-ordered combine.
"""
from __future__ import annotations

import math

import torch
from torch import nn

from . import _lib
from . import collectives as C
from . import kernels as K
from .errors import IndexOutOfRangeError, NotDivisibleError
from .kernels import _check_cuda, _ptr, _stream
from .state import STATE

IGNORE_INDEX = -100
U64_MAX = 2 ** 64 - 1


def vocab_padded(V: int, T: int, multiple: int = 128) -> int:
    q = T * multiple
    return (V + q - 1) // q * q


# ---------------------------------------------------------------------------
# raw kernels
# ---------------------------------------------------------------------------

def embed_lookup(ids: torch.Tensor, table: torch.Tensor, *, row_offset: int, vocab: int, pos_table=None,
                 seq: int = 1, check: bool = False) -> torch.Tensor:
    _check_cuda(ids, table, pos_table)
    ids = ids.reshape(-1).to(torch.int64).contiguous()
    n, D = ids.numel(), table.shape[1]
    out = torch.empty(n, D, dtype=table.dtype, device=table.device)
    err = None
    if check:
        err = torch.full((1,), -1, dtype=torch.int64, device=table.device)  # == UINT64_MAX
    _lib.call("smpk_embed_fwd", _ptr(ids), n, _ptr(table), table.stride(0), int(row_offset), table.shape[0],
              int(vocab), D, _ptr(out), out.stride(0), _ptr(pos_table),
              pos_table.stride(0) if pos_table is not None else 0, int(seq), _ptr(err), _stream())
    if check and not torch.cuda.is_current_stream_capturing():
        pos = int(err.item())
        if pos != -1:
            bad = int(ids[pos].item())
            raise IndexOutOfRangeError(f"embedding index {bad} out of range [0, {vocab}) at position {pos}", pos)
    return out


def embed_grad(ids: torch.Tensor, dy: torch.Tensor, *, rows: int, row_offset: int, padding_idx=None,
               out_dtype=torch.bfloat16, out=None, accumulate=False, method: str = "auto") -> torch.Tensor:
    """Deterministic scatter-add of dy rows into the rows of a (local) table.

    method "sort" (default for 8-aligned widths): radix sort by row + fixed-order segmented sums,
    O(n log rows) -- the NCF-scale path; "scan": the owner-computes kernel that scans the token
    list once per 8-row block, O(rows * n), summing strictly in token order (small vocabularies,
    odd widths).  out / accumulate: add into an existing gradient buffer (fp32 or bf16)."""
    _check_cuda(ids, dy, out)
    ids = ids.reshape(-1).to(torch.int64).contiguous()
    dy = dy.reshape(ids.numel(), -1).contiguous()
    D = dy.shape[1]
    g = out if out is not None else torch.empty(rows, D, dtype=out_dtype, device=dy.device)
    f32 = int(g.dtype == torch.float32)
    pad = int(-1 if padding_idx is None else padding_idx)
    sortable = D % 8 == 0 and g.stride(0) % 8 == 0 and D <= 8192
    if method == "sort" or (method == "auto" and sortable):
        n = ids.numel()
        ws_bytes = _lib.size("smpk_embed_bwd_sorted_workspace", n, rows, D)
        ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=dy.device)
        _lib.call("smpk_embed_bwd_sorted", _ptr(ids), n, _ptr(dy), dy.stride(0), int(row_offset), rows, D, _ptr(g),
                  g.stride(0), f32, int(bool(accumulate)), pad, _ptr(ws), ws.numel(), _stream(),
                  launches=4 + 4 * max(1, (max(rows, 1).bit_length() + 7) // 8))
        return g
    _lib.call("smpk_embed_bwd", _ptr(ids), ids.numel(), _ptr(dy), dy.stride(0), int(row_offset), rows, D, _ptr(g),
              g.stride(0), f32, int(bool(accumulate)), pad, _stream())
    return g


# ---------------------------------------------------------------------------
# autograd functions
# ---------------------------------------------------------------------------

class _LookupFn(torch.autograd.Function):
    """Local (masked) lookup of the rank's table slice; backward = deterministic scatter-add."""

    @staticmethod
    def forward(ctx, ids, table, row_offset, vocab, padding_idx, pos_table, seq, check):
        out = embed_lookup(ids, table, row_offset=row_offset, vocab=vocab, pos_table=pos_table, seq=seq,
                           check=check)
        ctx.save_for_backward(ids)
        ctx.meta = (table.shape[0], row_offset, padding_idx, pos_table is not None, seq)
        return out

    @staticmethod
    def backward(ctx, dy):
        (ids,) = ctx.saved_tensors
        rows, off, pad, has_pos, seq = ctx.meta
        dt = embed_grad(ids, dy, rows=rows, row_offset=off, padding_idx=pad)
        dpos = None
        if has_pos and ctx.needs_input_grad[5]:
            n = ids.numel()
            pos_ids = torch.arange(n, device=dy.device) % seq
            dpos = embed_grad(pos_ids, dy, rows=seq, row_offset=0)
        return None, dt, None, None, None, dpos, None, None


class VocabParallelCrossEntropy(torch.autograd.Function):
    @staticmethod
    def forward(ctx, logits, targets, vocab, col_offset, ignore_index):
        _check_cuda(logits, targets)
        logits = logits.contiguous()
        N, v_local = logits.shape
        targets = targets.reshape(-1).to(torch.int64).contiguous()
        stats = torch.empty(N, 4, dtype=torch.float32, device=logits.device)
        _lib.call("smpk_vocab_ce_fwd_local", _ptr(logits), logits.stride(0), N, v_local, int(col_offset), int(vocab),
                  _ptr(targets), int(ignore_index), _ptr(stats), _stream())
        stats_all = C.all_gather(stats.reshape(1, N, 4), 0)  # [T, N, 4], rank order
        T = stats_all.shape[0]
        loss = torch.empty(N, dtype=torch.float32, device=logits.device)
        ms = torch.empty(N, 2, dtype=torch.float32, device=logits.device)
        _lib.call("smpk_vocab_ce_combine", _ptr(stats_all), T, N, _ptr(targets), int(ignore_index), _ptr(loss),
                  _ptr(ms), _stream())
        ctx.save_for_backward(logits, targets, ms)
        ctx.meta = (vocab, col_offset, ignore_index)
        return loss

    @staticmethod
    def backward(ctx, gloss):
        logits, targets, ms = ctx.saved_tensors
        vocab, col_offset, ignore_index = ctx.meta
        N, v_local = logits.shape
        g = gloss.reshape(-1).to(torch.float32).contiguous()
        dl = torch.empty_like(logits)
        _lib.call("smpk_vocab_ce_bwd", _ptr(logits), logits.stride(0), N, v_local, int(col_offset), int(vocab),
                  _ptr(targets), int(ignore_index), _ptr(ms), _ptr(g), 1.0, _ptr(dl), dl.stride(0), _stream())
        return dl, None, None, None, None


def vocab_parallel_cross_entropy(logits_shard: torch.Tensor, targets: torch.Tensor, vocab_size: int,
                                 ignore_index: int = IGNORE_INDEX) -> torch.Tensor:
    """Per-token CE [N] (fp32) for logits sharded over the vocabulary across TP_GROUP.

    logits_shard: [N, Vp/T] bf16, rank j holding global columns [j*Vp/T, (j+1)*Vp/T)."""
    N, v_local = logits_shard.reshape(-1, logits_shard.shape[-1]).shape
    return VocabParallelCrossEntropy.apply(logits_shard.reshape(N, v_local), targets, vocab_size,
                                           STATE.tp_rank * v_local, ignore_index)


# ---------------------------------------------------------------------------
# modules
# ---------------------------------------------------------------------------

def _dev():
    return torch.device("cuda", torch.cuda.current_device())


class VocabParallelEmbedding(nn.Module):
    """Vocab-parallel embedding (rows sharded over tp_rank; builder-defined)."""

    def __init__(self, num_embeddings, embedding_dim, padding_idx=None, initializer_range=0.02, pad_multiple=128,
                 check_indices=False):
        super().__init__()
        T = STATE.tp_size
        self.num_embeddings, self.embedding_dim, self.padding_idx = num_embeddings, embedding_dim, padding_idx
        self.vocab_padded = vocab_padded(num_embeddings, T, pad_multiple)
        self.rows_local = self.vocab_padded // T
        self.row_offset = STATE.tp_rank * self.rows_local
        g = torch.Generator(device=_dev()).manual_seed(STATE.seed * 31 + 17 + STATE.tp_rank)
        w = torch.randn(self.rows_local, embedding_dim, generator=g, device=_dev()) * initializer_range
        real = torch.arange(self.row_offset, self.row_offset + self.rows_local, device=_dev()) < num_embeddings
        self.weight = nn.Parameter((w * real[:, None]).to(torch.bfloat16))
        self.check_indices = check_indices

    @torch.no_grad()
    def load_full(self, E: torch.Tensor):
        """E: [Vp or V, D] full table."""
        full = torch.zeros(self.vocab_padded, self.embedding_dim, dtype=torch.bfloat16, device=_dev())
        full[:E.shape[0]] = E.to(torch.bfloat16)
        self.weight.copy_(full[self.row_offset:self.row_offset + self.rows_local])

    def forward(self, input_ids, pos_table=None, seq=1):
        b = input_ids.shape[0]
        if STATE.prescaled or STATE.tp_size == 1:
            ids = input_ids
        else:
            ids = C.all_gather(input_ids.reshape(b, -1).contiguous(), 0)
        pt = pos_table if STATE.tp_rank == 0 else None
        y = _LookupFn.apply(ids, self.weight, self.row_offset, self.num_embeddings, self.padding_idx, pt, seq,
                            self.check_indices)
        y = y.reshape(*ids.shape, self.embedding_dim)
        if STATE.tp_size == 1:
            return y
        if STATE.prescaled:
            return C.fwd_allreduce_for_tp(y)
        return C.reduce_scatter_for_tp(y, 0)


class DistributedEmbedding(nn.Module):
    """smp.nn.DistributedEmbedding: sharded along the embedding dimension."""

    def __init__(self, num_embeddings, embedding_dim, padding_idx=None, max_norm=None, norm_type=2.0,
                 scale_grad_by_freq=False, sparse=False, _weight=None, initializer_range=0.02,
                 _skip_allgather=False, _skip_scatter_and_merge=False, check_indices=True):
        super().__init__()
        T = STATE.tp_size
        if embedding_dim % T:
            raise NotDivisibleError(f"embedding_dim {embedding_dim} not divisible by tensor_parallel_degree {T}")
        if max_norm is not None or scale_grad_by_freq or sparse:
            raise NotImplementedError("max_norm / scale_grad_by_freq / sparse are not on the TP hot path")
        self.num_embeddings, self.embedding_dim, self.padding_idx = num_embeddings, embedding_dim, padding_idx
        self.d_local = embedding_dim // T
        self._skip_allgather, self._skip_scatter_and_merge = _skip_allgather, _skip_scatter_and_merge
        self.check_indices = check_indices
        if _weight is not None:
            w = _weight.to(_dev(), torch.bfloat16)[:, STATE.tp_rank * self.d_local:(STATE.tp_rank + 1) * self.d_local]
        else:
            g = torch.Generator(device=_dev()).manual_seed(STATE.seed * 29 + 5 + STATE.tp_rank)
            w = (torch.randn(num_embeddings, self.d_local, generator=g, device=_dev()) * initializer_range)
            if padding_idx is not None:
                w[padding_idx] = 0
        self.weight = nn.Parameter(w.to(torch.bfloat16).contiguous())

    @torch.no_grad()
    def load_full(self, E: torch.Tensor):
        j = STATE.tp_rank
        self.weight.copy_(E[:, j * self.d_local:(j + 1) * self.d_local].to(torch.bfloat16))

    def forward(self, input_ids):
        shape = input_ids.shape
        T = STATE.tp_size
        gather = not (STATE.prescaled or self._skip_allgather) and T > 1
        ids = C.all_gather(input_ids.reshape(shape[0], -1).contiguous(), 0) if gather else input_ids
        y = _LookupFn.apply(ids, self.weight, 0, self.num_embeddings, self.padding_idx, None, 1,
                            self.check_indices)
        y = y.reshape(*ids.shape, self.d_local)
        if T == 1 or self._skip_scatter_and_merge:
            return y
        if gather:
            return C.scatter_and_merge_for_tp(y, 0, -1)  # split batch, merge embedding
        return C.allgather_replicated(y, -1)  # prescaled: AG along emb, backward = local slice


class _LMHeadFn(torch.autograd.Function):
    """logits_j = h @ E_j^T on the TP-replicated hidden state; backward: dE_j, and dh summed
    over the vocab shards (allreduce = bwd_allreduce_for_tp), unless the caller's allgather
    already reduces it (its backward is a reduce-scatter)."""

    @staticmethod
    def forward(ctx, h, E, reduce_grad):
        ctx.save_for_backward(h, E)
        ctx.reduce_grad = reduce_grad
        return K.matmul_nt(h, E)

    @staticmethod
    def backward(ctx, dl):
        h, E = ctx.saved_tensors
        dl = dl.contiguous()
        dh = K.matmul_nn(dl, E)
        if ctx.reduce_grad:
            C.all_reduce(dh)
        dE = K.matmul_tn(dl, h)
        return dh, dE, None


def lm_head_logits(h: torch.Tensor, E_local: torch.Tensor, reduce_grad: bool = True) -> torch.Tensor:
    """Vocab-sharded logits of the tied LM head: [N, H] x [Vp/T, H]^T -> [N, Vp/T]."""
    return _LMHeadFn.apply(h.reshape(-1, h.shape[-1]).contiguous(), E_local, reduce_grad)
