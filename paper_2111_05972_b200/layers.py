"""Fused forward/backward of the transformer sub-layers on one TP rank (speed mode).

``AttentionFn`` and ``MlpFn`` are torch.autograd.Functions whose forward and
backward issue the sm_100a kernels of libsmpk directly (tcgen05 GEMMs with fused
epilogues, fused softmax/dropout, fused bias-dropout-residual-LayerNorm), with
the row-parallel partial-sum allreduce of the forward and the column-parallel
input-gradient allreduce of the backward ("two allreduces during
forward, and two allreduces during backward") issued over the TP group.

Per-rank dataflow:
  attention: [pre-LN] -> QKV_j (+b) -> per local head softmax(QK^T/sqrt(dh) + mask)
             -> dropout -> .V -> ctx_j @ Wo_j^T -> AR -> +bo -> dropout -> +x -> [post-LN]
  mlp:       [pre-LN] -> FC1_j (+b, act) -> FC2_j -> AR -> +b2 -> dropout -> +x -> [post-LN]
Between sub-layers the activation is either TP-replicated (prescaled batch, AR) or
row-sharded by owning rank (TP across DP: AG in, RS out); weights are the rank's
shards in the Megatron layout (oracle/tp.py shard_layer_params_speed).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import collectives as C
from . import kernels as K
from . import ops
from .ops import SITE_ATTN_OUT, SITE_MLP_OUT
from .exchange import AGB, AGF, RSB, RSF, chunk_order, mbkind, publish_order
from .state import STATE, get_pool


@dataclass
class LayerMeta:
    hidden: int
    heads_local: int
    heads_global: int
    head_dim: int
    eps: float
    p_attn: float
    p_hidden: float
    causal: bool
    pre_ln: bool
    post_ln: bool
    activation: str
    layer_id: int
    seed: int
    head_offset: int
    sample_offset: int  # global id of the first sample the attention sees (gathered batch)
    tp_size: int
    row_offset: int = 0  # global token row of this rank's first activation row (hidden dropout)
    shard_rows: bool = False  # activations row-sharded between sub-layers (AG in / RS out)
    comm: str = "peer"  # "peer": fused NVLink peer-store collectives; "nccl": torch.distributed
    push_next: bool = False  # the next sub-layer gathers this output unnormalised: push it from the epilogue
    grad: bool = True  # grad mode was on at the sub-layer call (Function.forward always runs without it)
    rng: object = None  # device step snapshot of this forward (ops.rng_next): Philox key = seed + step * golden
    mb: int = -1  # overlapped micro-batch (tp_exchange="overlap"): 0 / 1, -1 = the whole batch
    mb_batch: int = 0  # with mb >= 0: this rank's full batch (samples), the micro-batch is its half mb


class LinearFn(torch.autograd.Function):
    """y = x @ W^T (+ b) on the tcgen05 GEMM; backward dX = dY W, dW = dY^T X, db = colsum(dY)."""

    @staticmethod
    def forward(ctx, x, W, b):
        ctx.save_for_backward(x, W)
        ctx.has_b = b is not None
        return K.linear(x, W, b)

    @staticmethod
    def backward(ctx, dy):
        x, W = ctx.saved_tensors
        dy = dy.contiguous()
        dx = K.matmul_nn(dy, W) if ctx.needs_input_grad[0] else None
        dW = K.matmul_tn(dy, x)
        db = ops.colsum(dy) if ctx.has_b else None
        return dx, dW, db


class LayerNormFn(torch.autograd.Function):
    """Replicated LayerNorm over the last dim (speed mode) on the row kernels."""

    @staticmethod
    def forward(ctx, x, w, b, eps):
        shape = x.shape
        x2 = x.reshape(-1, shape[-1]).contiguous()
        y, mean, rstd = ops.layer_norm(x2, w, b, eps)
        ctx.save_for_backward(x2, mean, rstd, w)
        ctx.shape = shape
        return y.view(shape)

    @staticmethod
    def backward(ctx, dy):
        x2, mean, rstd, w = ctx.saved_tensors
        dx, _, dw, db, _ = ops.ln_bwd(dy.reshape(x2.shape).contiguous(), x2, mean, rstd, w, want_dbias=False)
        return dx.view(ctx.shape), dw, db, None


# ---------------------------------------------------------------------------
# attention core: qkv [B*s, 3*hl*dh] -> ctx [B*s, hl*dh]
# ---------------------------------------------------------------------------

def attn_core_fwd(qkv: torch.Tensor, B: int, s: int, m: LayerMeta, mask_add):
    hl, dh = m.heads_local, m.head_dim
    hd = hl * dh
    ld = 3 * hd
    S = torch.empty(B, hl, s, s, dtype=qkv.dtype, device=qkv.device)
    K.gemm_raw(qkv, 0, ld, (dh, s * ld), qkv[:, hd:], 0, ld, (dh, s * ld), S, s, (s * s, hl * s * s),
               s, s, dh, nb=(hl, B))
    P, Pd = ops.softmax_fwd(S, scale=1.0 / math.sqrt(dh), mask_add=mask_add, causal=m.causal, p=m.p_attn,
                            seed=m.seed, rng=m.rng, layer=m.layer_id, sample_offset=m.sample_offset, head_offset=m.head_offset,
                            nh_global=m.heads_global)
    del S
    ctx = torch.empty(B * s, hd, dtype=qkv.dtype, device=qkv.device)
    K.gemm_raw(Pd, 0, s, (s * s, hl * s * s), qkv[:, 2 * hd:], 1, ld, (dh, s * ld), ctx, hd, (dh, s * hd),
               s, dh, s, nb=(hl, B))
    return ctx, P, Pd


def attn_core_bwd(dctx: torch.Tensor, qkv: torch.Tensor, P, Pd, B: int, s: int, m: LayerMeta):
    hl, dh = m.heads_local, m.head_dim
    hd = hl * dh
    ld = 3 * hd
    dqkv = torch.empty_like(qkv)
    # dPd = dctx V^T
    dP = torch.empty(B, hl, s, s, dtype=qkv.dtype, device=qkv.device)
    K.gemm_raw(dctx, 0, hd, (dh, s * hd), qkv[:, 2 * hd:], 0, ld, (dh, s * ld), dP, s, (s * s, hl * s * s),
               s, s, dh, nb=(hl, B))
    # dV = Pd^T dctx
    K.gemm_raw(Pd, 1, s, (s * s, hl * s * s), dctx, 1, hd, (dh, s * hd), dqkv[:, 2 * hd:], ld, (dh, s * ld),
               s, dh, s, nb=(hl, B))
    dS = ops.softmax_bwd(P, dP, scale=1.0 / math.sqrt(dh), p=m.p_attn, seed=m.seed, rng=m.rng, layer=m.layer_id,
                         sample_offset=m.sample_offset, head_offset=m.head_offset, nh_global=m.heads_global, out=dP)
    # dQ = dS K ; dK = dS^T Q
    K.gemm_raw(dS, 0, s, (s * s, hl * s * s), qkv[:, hd:], 1, ld, (dh, s * ld), dqkv, ld, (dh, s * ld),
               s, dh, s, nb=(hl, B))
    K.gemm_raw(dS, 1, s, (s * s, hl * s * s), qkv, 1, ld, (dh, s * ld), dqkv[:, hd:], ld, (dh, s * ld),
               s, dh, s, nb=(hl, B))
    return dqkv


FLASH = {"enabled": True, "min_seq": 128}


def use_flash(s: int, head_dim: int) -> bool:
    """Fused tcgen05 attention (csrc/flash_attn*.cu) whenever its shape constraints hold; the
    materialised path (tcgen05 batched GEMMs + fused softmax kernels) covers the rest and is the
    A/B reference (scripts/attn_bench.py: 36 + 122 us vs 115 + 155 us at BERT-large s=512)."""
    return FLASH["enabled"] and s % 128 == 0 and head_dim in (64, 128) and s >= FLASH["min_seq"]


_SIDE: dict = {}


def _side_stream() -> torch.cuda.Stream:
    """Per-device side stream for data-independent work (attention dropout keep bits) that can
    run concurrently with the GEMM in front of it."""
    dev = torch.cuda.current_device()
    st = _SIDE.get(dev)
    if st is None:
        st = _SIDE[dev] = torch.cuda.Stream(device=dev)
    return st


def _keep_bits_async(B: int, s: int, m: LayerMeta, device):
    """Launch the attention keep-bit generator on the side stream; returns (bits, join) where
    join() makes the current stream wait for it (fork/join is CUDA-graph capturable)."""
    if m.p_attn <= 0:
        return None, (lambda: None)
    main = torch.cuda.current_stream()
    bits = torch.empty(B, m.heads_local, s, s // 32, dtype=torch.int32, device=device)  # main-stream allocation
    side = _side_stream()
    side.wait_stream(main)
    with torch.cuda.stream(side):
        if m.mb < 0:
            ops.attn_dropout_bits(B, m.heads_local, s, s, p=m.p_attn, seed=m.seed, rng=m.rng, layer=m.layer_id,
                                  sample_offset=m.sample_offset, head_offset=m.head_offset, nh_global=m.heads_global,
                                  out=bits, causal=m.causal and s % 128 == 0)
        else:  # micro-batch mb: rank j's samples [mb*b, (mb+1)*b) of its mb_batch, rank-major
            b = B // m.tp_size
            ops.attn_dropout_bits(B, m.heads_local, s, s, p=m.p_attn, seed=m.seed, rng=m.rng, layer=m.layer_id,
                                  sample_offset=m.sample_offset + m.mb * b, sample_block=b, block_stride=m.mb_batch,
                                  head_offset=m.head_offset, nh_global=m.heads_global, out=bits,
                                  causal=m.causal and s % 128 == 0)
    return bits, (lambda: main.wait_stream(side))


class _SmLimits:
    """smpk_set_sm_limits for the duration of a with-block (launch-time grid caps)."""

    def __init__(self, gemm_sms: int, row_sms: int):
        self.lim = (int(gemm_sms), int(row_sms))

    def __enter__(self):
        from . import _lib
        _lib.call("smpk_set_sm_limits", *self.lim)

    def __exit__(self, *exc):
        from . import _lib
        _lib.call("smpk_set_sm_limits", 0, 0)


def _overlap_sms(m: LayerMeta) -> int:
    """SMs given to the backward's weight-gradient GEMMs while the input-gradient exchange runs
    next to them (tp_overlap_sms; 0 = serial).  Only with the peer-memory exchange at T > 1."""
    if m.tp_size == 1 or STATE.config.get("tp_comm", "peer") != "peer":
        return 0
    return int(STATE.config.get("tp_overlap_sms", 0))


def _wgrad_async(m: LayerMeta, jobs):
    """Run the weight-gradient GEMMs `jobs` (no data dependence on the exchange that follows) on
    the side stream with a capped grid; returns (join, row_sms) — the exchange kernels launched
    before join() should cap their grids at row_sms so both streams fit on the GPU at once.
    The fork / join is CUDA-graph capturable.  Output tensors must be allocated by the caller on
    the main stream."""
    gs = _overlap_sms(m)
    if gs <= 0:
        for f in jobs:
            f()
        return (lambda: None), 0
    from . import _lib
    nsm = _lib.device_sms()
    main = torch.cuda.current_stream()
    side = _side_stream()
    side.wait_stream(main)
    with torch.cuda.stream(side), _SmLimits(gs, 0):
        for f in jobs:
            f()
    return (lambda: main.wait_stream(side)), max(nsm - gs, 8)


def _ln_in(x2, w, b, m: LayerMeta):
    y, mean, rstd = ops.layer_norm(x2, w, b, m.eps)
    return y, mean, rstd


def _residual_bwd_out(dh: torch.Tensor, dr: torch.Tensor | None, x2, ln_w, mean, rstd, m: LayerMeta):
    """Gradient wrt the sub-layer input x given dh (through the branch) and dr (through the residual)."""
    if m.pre_ln:
        dx, _, dgw, dgb, _ = ops.ln_bwd(dh, x2, mean, rstd, ln_w, dres=dr, want_dbias=False)
        return dx, dgw, dgb
    return ops.add(dh, dr), None, None


# Row-sharded activations (TP across DP ranks, the default for tp_size > 1): every rank keeps
# the rows of ITS OWN samples between sub-layers ([b*s, H]); the column-parallel GEMM input is
# allgathered over the TP group and the row-parallel partial sums are reduce-scattered back
# to the owning rank (AG + RS = the paper's allreduce, same bytes).  Bias / dropout / residual /
# LayerNorm then run once per row instead of T times, and the stack needs no entry gather or exit
# slice ("returns the combined data samples to their respective GPUs").
# Replicated parameters (LayerNorms, row-parallel biases) see only their rank's rows, so their
# gradients are allreduced once per sub-layer (one flat bucket).

def _gather_rows(t, m: LayerMeta):
    return C.all_gather(t.contiguous(), 0) if m.shard_rows else t


def _combine_rows(partial, m: LayerMeta):
    """Row-parallel partial sums -> own rows (RS) or replicated rows (AR)."""
    if m.shard_rows:
        return C.reduce_scatter(partial, 0)
    return C.all_reduce(partial)


def _sync_replicated(grads, m: LayerMeta, keep=None):
    """Allreduce the partial gradients of TP-replicated parameters in one bucket (row-sharded mode).
    keep: (post-LN weight, bias) gradients already summed over the peer pool (slots 0, 1)."""
    if keep is not None:
        grads = list(grads)
        grads[0], grads[1] = keep
        synced = grads[:2]
        rest = _sync_replicated([None, None] + grads[2:], m)
        return synced + rest[2:]
    if not m.shard_rows:
        return grads
    live = [g for g in grads if g is not None]
    if not live:
        return grads
    flat = torch.cat([g.float().reshape(-1) for g in live])
    C.all_reduce(flat)
    out, off = [], 0
    for g in grads:
        if g is None:
            out.append(None)
            continue
        n = g.numel()
        out.append(flat[off:off + n].view_as(g).to(g.dtype))
        off += n
    return out


# With tp_comm == "peer" the AG / RS above are fused into the producing kernels over the TP
# group's symmetric peer-mapped pool (symm.py, csrc/symm.cu): the row kernel that produces a
# sub-layer input stores it into every peer's gather region, the row-parallel GEMM epilogue
# stores its partial tiles into the owning rank's slot region (NVLink peer stores overlapped
# with the MMA main loop), and the consuming row kernel sums the T slots in ascending rank
# order.  One epoch barrier orders each exchange.

def _peer(m: LayerMeta, R: int) -> bool:
    """Peer-store collectives need whole 128-row GEMM tiles per owner; otherwise NCCL."""
    return m.shard_rows and m.comm == "peer" and R % 128 == 0


# (data_ptr, numel) of a sub-layer output -> the pool region its producer already stored it
# into on every rank (the previous sub-layer's epilogue did the allgather's peer stores)
_PUSHED: dict = {}


def _push_target(m: LayerMeta, R: int, H: int):
    """Gather region the sub-layer epilogue stores its output into (push_next), or None."""
    if not (m.push_next and _peer(m, R)):
        return None, {}
    pool = get_pool()
    G = pool.alloc(m.tp_size * R * H * 2)
    tbl, off = pool.peers(G, pool.me * R * H)
    return G, dict(out_peers=tbl, peer_off=off)


# tp_exchange == "chunks" (default with peer comm): the sub-layer runs as T per-owner chunks, own
# rows first; gathers and reduce-scatters move on the copy engines through the mailboxes of
# exchange.py while the SMs compute the next chunk.  The saved tensors are the same as the
# barrier path's (full gathered input, qkv / ctx / lse / f / z over all T*b samples), so the
# backward is shared.

def _chunked(m: LayerMeta, R: int) -> bool:
    return m.tp_size > 1 and _peer(m, R) and STATE.config.get("tp_exchange", "barrier") == "chunks"


def _publish(G: int, R: int, H: int, m: LayerMeta) -> None:
    """Send this rank's rows of gather region G (already in G[me]) to every peer's G[me]."""
    pool = get_pool()
    xch = pool.exchange()
    off = G + pool.me * R * H * 2
    src = pool.view(off, (R, H))
    xch.put(AGF, [(j, [(off, src)]) for j in publish_order(pool.me, m.tp_size)], ack=False)


def _chunk_gather_in(x2, m: LayerMeta, ln=None):
    """Gather region of the sub-layer input for the chunk loop: published by the previous
    sub-layer's consumer, or (stack entry / pre-LN) written here and published now.
    Returns (hf [T*R, H] view, mean, rstd, region)."""
    R, H = x2.shape
    pool = get_pool()
    G = _PUSHED.pop((x2.data_ptr(), x2.numel()), None) if ln is None else None
    mean = rstd = None
    if G is None:
        if STATE.xch_fresh:  # step entry: every rank is done with the previous step's regions
            pool.barrier()
            STATE.xch_fresh = False
        G = pool.alloc(m.tp_size * R * H * 2)
        off = G // 2 + pool.me * R * H
        if ln is not None:
            _, _, mean, rstd = ops.bdr_ln(x2, gamma=ln[0], beta=ln[1], eps=m.eps, want_r=False, want_y=False,
                                          out_peers=pool.self_table, peer_off=off)
        else:
            ops.bdr_ln(x2, want_r=False, out_peers=pool.self_table, peer_off=off)
        _publish(G, R, H, m)
    return pool.view(G, (m.tp_size * R, H)), mean, rstd, G


def _chunk_rs_slots(m: LayerMeta, R: int, N: int):
    """This rank's reduce-scatter slots [T, R, N] (slot j = rank j's partial of my rows)."""
    pool = get_pool()
    P = pool.scratch("rsf_slots", m.tp_size * R * N * 2)
    return P, pool.view(P, (m.tp_size, R, N))


def _chunk_partial_out(c: int, P: int, slots, R: int, N: int):
    """Output buffer of chunk c's row-parallel product: my own slot, or a staging buffer."""
    pool = get_pool()
    return slots[pool.me] if c == pool.me else pool.exchange().staging("rsf", c, (R, N))


def _chunk_partial_send(c: int, P: int, dst, R: int, N: int) -> None:
    pool = get_pool()
    if c != pool.me:
        pool.exchange().send(RSF, c, P + pool.me * R * N * 2, dst, ack=True, stage_tag="rsf")


def _chunk_consume(m: LayerMeta, R: int, H: int, P: int, consume):
    """Await the T-1 partial slots, run consume(slot kwargs, push kwargs) (the fused sum +
    bias + dropout + residual + LayerNorm), release the slots, publish the output rows.
    Returns (consume's result, next gather region or None)."""
    pool = get_pool()
    xch = pool.exchange()
    T = m.tp_size
    xch.await_all(RSF, chunk_order(pool.me, T)[1:])
    Gn = pool.alloc(T * R * H * 2) if m.push_next else None
    pkw = dict(out_peers=pool.self_table, peer_off=Gn // 2 + pool.me * R * H) if Gn is not None else {}
    res = consume(dict(nslots=T, slot_stride=R * H), pkw)
    xch.release_all([RSF], chunk_order(pool.me, T)[1:])
    xch.join()  # this sub-layer's partial copies (done: the peers consumed theirs) and older publishes
    if Gn is not None:
        _publish(Gn, R, H, m)
    return res, Gn


def _chunk_grad_publish(dy2, r, mean, rstd, m: LayerMeta, site: int, keep=None):
    """Backward of the sub-layer epilogue on own rows (chunked exchange): the branch gradient goes
    into this rank's slot of the site's gather region and the fp32 [nv, H] replicated-parameter
    gradient partials into its slot of the vector region; both are published to every peer.
    Returns (dr, gather region, vector region, nv)."""
    R, H = dy2.shape
    pool = get_pool()
    xch = pool.exchange()
    T, me = m.tp_size, pool.me
    has_ln = m._post_w is not None
    nv = 3 if has_ln else 1  # [dgamma, dbeta,] dbias
    dG = pool.scratch(f"agb{site}", T * R * H * 2)
    V = pool.scratch(f"vecb{nv}", T * nv * H * 4)
    pg = pool.view(V + me * nv * H * 4, (nv, H), dtype=torch.float32)
    kw = dict(p=m.p_hidden, seed=m.seed, rng=m.rng, layer=m.layer_id, site=site, row_offset=m.row_offset,
              want_dr=m.post_ln, keep_in=keep)
    dr, _, _, _, _ = ops.ln_bwd(dy2, r, mean, rstd, m._post_w, out_peers=pool.self_table,
                                peer_off=dG // 2 + me * R * H, param_grads_out=pg, want_dbias=True,
                                grads_f32=True, **kw)
    mine = pool.view(dG + me * R * H * 2, (R, H))
    xch.put(AGB, [(j, [(dG + me * R * H * 2, mine), (V + me * nv * H * 4, pg)]) for j in publish_order(me, T)],
            ack=True)
    return dr, dG, V, nv


def _chunk_grad_finish(m: LayerMeta, R: int, H: int, Pb: int, bslots, dr, x2, pre_w, mu1, rs1, V: int, nv: int):
    """Await the input-gradient partial slots, reduce them into dx (+ pre-LN backward), sum the
    replicated-parameter gradient slots in ascending rank order (fp32, rounded once), release
    every slot.  Returns (dx, dpre_w, dpre_b, dpost_w, dpost_b, dbias_out)."""
    pool = get_pool()
    xch = pool.exchange()
    T = m.tp_size
    xch.await_all(RSB, chunk_order(pool.me, T)[1:])
    dx, dpre_w, dpre_b = _input_grad(bslots[0], dict(nslots=T, slot_stride=R * H), dr, x2, pre_w, mu1, rs1, m, R, H)
    slots = pool.view(V, (T, nv, H), dtype=torch.float32)
    tot = slots.sum(0).to(torch.bfloat16)  # one reduction over the T slots (rank order), one rounding
    xch.release_all([RSB, AGB], chunk_order(pool.me, T)[1:])
    xch.join()
    if nv == 3:
        m._post_synced = True
        return dx, dpre_w, dpre_b, tot[0], tot[1], tot[2]
    return dx, dpre_w, dpre_b, None, None, tot[0]


# tp_exchange == "overlap": the same whole-sub-layer GEMMs as the barrier exchange, but every
# transfer is a copy-engine copy through the mailboxes of exchange.py (no barrier kernel, no SM
# spent on NVLink), and DistributedTransformer runs the batch as two micro-batches on two streams,
# so one micro-batch's exchange overlaps the other's compute.

def _overlap(m: LayerMeta, R: int) -> bool:
    return m.tp_size > 1 and _peer(m, R) and STATE.config.get("tp_exchange", "barrier") == "overlap"


def _ov_publish(G: int, R: int, H: int, m: LayerMeta) -> None:
    pool = get_pool()
    xch = pool.exchange()
    off = G + pool.me * R * H * 2
    src = pool.view(off, (R, H))
    xch.put(mbkind(AGF, m.mb), [(j, [(off, src)]) for j in publish_order(pool.me, m.tp_size)], ack=False,
            mb=m.mb)


def _ov_gather_in(x2, m: LayerMeta, ln=None):
    """Gather region of the sub-layer input: this rank's rows (published by the previous
    sub-layer's consumer, or written and published here), then every peer's rows awaited."""
    R, H = x2.shape
    pool = get_pool()
    xch = pool.exchange()
    G = _PUSHED.pop((x2.data_ptr(), x2.numel()), None) if ln is None else None
    mean = rstd = None
    if G is None:
        if STATE.xch_fresh:  # step entry: every rank is done with the previous step's regions
            pool.barrier()
            STATE.xch_fresh = False
        G = pool.alloc(m.tp_size * R * H * 2)
        off = G // 2 + pool.me * R * H
        if ln is not None:
            _, _, mean, rstd = ops.bdr_ln(x2, gamma=ln[0], beta=ln[1], eps=m.eps, want_r=False, want_y=False,
                                          out_peers=pool.self_table, peer_off=off)
        else:
            ops.bdr_ln(x2, want_r=False, out_peers=pool.self_table, peer_off=off)
        _ov_publish(G, R, H, m)
    xch.await_all(mbkind(AGF, m.mb), chunk_order(pool.me, m.tp_size)[1:])
    return pool.view(G, (m.tp_size * R, H)), mean, rstd, G


def _ov_rs(a, w, w_mn: bool, m: LayerMeta, R: int, N: int, kind: int, extra=()):
    """Row-parallel product into this micro-batch's partial region; every owner's row block
    leaves on the copy engines for its slot on the owner, the own block stays.  Returns
    (consumer slot kwargs: the T slots as a table of local addresses, partial view)."""
    pool = get_pool()
    xch = pool.exchange()
    T, me = m.tp_size, pool.me
    k = mbkind(kind, m.mb)
    Pp = pool.scratch(f"ovp{k}", T * R * N * 2)
    S = pool.scratch(f"ovs{k}", T * R * N * 2)
    P = pool.view(Pp, (T * R, N))
    xch.reuse(("ovp", k), [c for c in range(T) if c != me])  # last round's copies out of P have left
    _product(a, w, w_mn, out=P, extra=extra)
    xch.put(k, [(c, [(S + me * R * N * 2, P[c * R:(c + 1) * R])]) for c in publish_order(me, T)], ack=True,
            stage_tag=("ovp", k), mb=m.mb)
    xch.await_all(k, chunk_order(me, T)[1:])
    base = pool.bases[me]
    tbl = xch.table(("ovslots", k, R, N), [base + (Pp + me * R * N * 2 if j == me else S + j * R * N * 2)
                                           for j in range(T)])
    return dict(nslots=T, x_peers=tbl, x_peer_off=0), P


def _ov_release(m: LayerMeta, *kinds) -> None:
    pool = get_pool()
    xch = pool.exchange()
    xch.release_all([mbkind(kind, m.mb) for kind in kinds], chunk_order(pool.me, m.tp_size)[1:])
    xch.join(m.mb)


def _ov_grad_publish(dy2, r, mean, rstd, m: LayerMeta, site: int, keep=None):
    """Backward of the sub-layer epilogue on own rows; the branch gradient and the fp32
    replicated-parameter partials are published to every peer and the peers' awaited.
    Returns (dr, branch gradient of all T*R rows, vector region, nv)."""
    R, H = dy2.shape
    pool = get_pool()
    xch = pool.exchange()
    T, me = m.tp_size, pool.me
    k = mbkind(AGB, m.mb)
    has_ln = m._post_w is not None
    nv = 3 if has_ln else 1
    dG = pool.scratch(f"ovg{site}_{k}", T * R * H * 2)
    V = pool.scratch(f"ovv{nv}_{k}", T * nv * H * 4)
    pg = pool.view(V + me * nv * H * 4, (nv, H), dtype=torch.float32)
    kw = dict(p=m.p_hidden, seed=m.seed, rng=m.rng, layer=m.layer_id, site=site, row_offset=m.row_offset,
              want_dr=m.post_ln, keep_in=keep)
    dr, _, _, _, _ = ops.ln_bwd(dy2, r, mean, rstd, m._post_w, out_peers=pool.self_table,
                                peer_off=dG // 2 + me * R * H, param_grads_out=pg, want_dbias=True,
                                grads_f32=True, **kw)
    mine = pool.view(dG + me * R * H * 2, (R, H))
    xch.put(k, [(j, [(dG + me * R * H * 2, mine), (V + me * nv * H * 4, pg)]) for j in publish_order(me, T)],
            ack=True, mb=m.mb)
    xch.await_all(k, chunk_order(me, T)[1:])
    return dr, pool.view(dG, (T * R, H)), V, nv


def _ov_vec_sums(m: LayerMeta, V: int, nv: int, H: int):
    """Replicated-parameter gradient slots summed in ascending rank order (fp32, rounded once):
    (dpost_w, dpost_b, dbias) -- the first two None without a post-LN."""
    pool = get_pool()
    slots = pool.view(V, (m.tp_size, nv, H), dtype=torch.float32)
    tot = slots.sum(0).to(torch.bfloat16)  # one reduction over the T slots (rank order), one rounding
    if nv == 3:
        m._post_synced = True
        return tot[0], tot[1], tot[2]
    return None, None, tot[0]


def _gather_in(x2, m: LayerMeta, ln=None):
    """Column-parallel GEMM input: [pre-LN](own rows) gathered over the group.
    Returns (hf, mean, rstd, pool region or None)."""
    R, H = x2.shape
    if _peer(m, R):
        pool = get_pool()
        G = _PUSHED.pop((x2.data_ptr(), x2.numel()), None) if ln is None else None
        if G is not None:  # rows already stored into every rank's region by the producer
            pool.barrier()
            return pool.view(G, (m.tp_size * R, H)), None, None, G
        G = pool.alloc(m.tp_size * R * H * 2)
        tbl, off = pool.peers(G, pool.me * R * H)
        mean = rstd = None
        if ln is not None:
            _, _, mean, rstd = ops.bdr_ln(x2, gamma=ln[0], beta=ln[1], eps=m.eps, want_r=False, want_y=False,
                                          out_peers=tbl, peer_off=off)
        else:
            ops.bdr_ln(x2, want_r=False, out_peers=tbl, peer_off=off)
        pool.barrier()
        return pool.view(G, (m.tp_size * R, H)), mean, rstd, G
    if ln is not None:
        h, mean, rstd = ops.layer_norm(x2, ln[0], ln[1], m.eps)
    else:
        h, mean, rstd = x2, None, None
    return _gather_rows(h, m), mean, rstd, None


def _product(a, w, w_mn: bool, out=None, extra=()):
    """a @ w (w_mn: w given [K, N]) or a @ w^T; `extra` GEMM thunks (independent weight gradients)
    are launched together with it in one grouped persistent grid (kernels.grouped)."""
    if not extra:
        return K.matmul_nn(a, w, out=out) if w_mn else K.linear(a, w, out=out)
    with K.grouped():
        for f in extra:
            f()
        y = K.matmul_nn(a, w, out=out) if w_mn else K.linear(a, w, out=out)
    return y


def _rs_out(a, w, w_mn: bool, m: LayerMeta, R: int, N: int, extra=()):
    """Row-parallel product combined over the group -> (x, slot kwargs, region).

    Peer mode, "pull" (default): every rank writes its full partial product into its own
    symmetric-pool region with a local TMA-store epilogue; after one epoch barrier the consumer
    row kernel reads its rows from all T ranks' regions over NVLink and sums them in ascending
    rank order (the slot kwargs carry the peer table and offset).  "push": the GEMM epilogue
    stores each output box straight into the owner's slot (smpk_gemm_rs).  Otherwise NCCL.
    extra: independent GEMM thunks fused into the same launch (backward weight gradients)."""
    if _peer(m, R):
        pool = get_pool()
        T = m.tp_size
        if STATE.config.get("tp_rs", "pull") == "pull":
            P = pool.scratch("rs_out", T * R * N * 2)
            out = pool.view(P, (T * R, N))
            _product(a, w, w_mn, out=out, extra=extra)
            pool.barrier()
            return out, dict(nslots=T, x_peers=pool.base_table, x_peer_off=P // 2 + pool.me * R * N), None
        for f in extra:
            f()
        P = pool.scratch("partials", T * R * N * 2)
        peers, off = pool.host_peers(P, pool.me * R * N)
        K.gemm_rs(a, w, w_mn, peers, ldc=N, rows_per_owner=R, slot_off=off)
        pool.barrier()
        return pool.view(P, (T * R, N)), dict(nslots=T, slot_stride=R * N), None
    y = _product(a, w, w_mn, extra=extra)
    return _combine_rows(y, m), {}, None


def _gather_grad(dy2, r, mean, rstd, m: LayerMeta, site: int, keep=None):
    """Backward of the sub-layer epilogue on own rows; the branch gradient is gathered for the
    column/row-parallel GEMMs.  keep: the forward's hidden-dropout keep bytes.
    Returns (dr, dbranch_full, dgamma, dbeta, dbias, region); dbias (the sub-layer output bias
    gradient, column sums of the branch gradient over all rows of the group) is None when the
    caller has to reduce it itself."""
    R, H = dy2.shape
    has_ln = m._post_w is not None
    kw = dict(p=m.p_hidden, seed=m.seed, rng=m.rng, layer=m.layer_id, site=site, row_offset=m.row_offset,
              want_dr=m.post_ln, keep_in=keep)
    if _peer(m, R):
        pool = get_pool()
        T = m.tp_size
        # one gather region per site: the weight-gradient GEMMs of this sub-layer may still read it
        # on the side stream (tp_overlap_sms) when the next sub-layer's exchange starts; peers write
        # the same site's region again only two exchanges later, after this rank's side-stream join
        # has been ordered before a barrier they wait on (cross-rank write-after-read)
        G = pool.scratch(f"grad_gather{site}", T * R * H * 2)
        tbl, off = pool.peers(G, pool.me * R * H)
        nv = 3 if has_ln else 1  # [dgamma, dbeta,] dbias: this rank's partial sums over its own rows
        pg = torch.empty(nv, H, dtype=torch.float32, device=dy2.device)
        dr, _, dgw, dgb, dbias = ops.ln_bwd(dy2, r, mean, rstd, m._post_w, out_peers=tbl, peer_off=off,
                                            param_grads_out=pg, want_dbias=True, grads_f32=True, **kw)
        # the replicated-parameter gradients ride the same barrier: copy this rank's fp32 [nv, H]
        # partial into every peer's slot, then sum the T slots in ascending rank order in fp32 and
        # round once (the same precision as the NCCL path's fp32 allreduce, _sync_replicated)
        L = pool.scratch(f"vec_grads{nv}", T * nv * H * 4)
        pool.push_copy(pg, L + pool.me * nv * H * 4)
        pool.barrier()
        slots = pool.view(L, (T, nv, H), dtype=torch.float32)
        tot = slots.sum(0).to(torch.bfloat16)  # one reduction over the T slots (rank order), one rounding
        if has_ln:
            dgw, dgb = tot[0], tot[1]
            m._post_synced = True
        return dr, pool.view(G, (T * R, H)), dgw, dgb, tot[nv - 1], None
    dr, d, dgw, dgb, dbias = ops.ln_bwd(dy2, r, mean, rstd, m._post_w, want_dbias=not m.shard_rows, **kw)
    return dr, _gather_rows(d, m), dgw, dgb, dbias, None


def _input_grad(dhx, skw, dr, x2, pre_w, mu1, rs1, m: LayerMeta, R: int, H: int):
    """dx = [pre-LN backward](sum of dh slots) + residual gradient dr."""
    if m.pre_ln:
        dx, _, dgw, dgb, _ = ops.ln_bwd(dhx, x2, mu1, rs1, pre_w, dres=dr, want_dbias=False, rows=R, cols=H,
                                        **skw)
        return dx, dgw, dgb
    dx, _, _, _ = ops.bdr_ln(dhx, residual=dr, rows=R, cols=H, **skw)
    return dx, None, None


def _free(*regions):
    if any(r is not None for r in regions):
        pool = get_pool()
        for r in regions:
            if r is not None:
                pool.free(r)


# ---------------------------------------------------------------------------
# attention sub-layer
# ---------------------------------------------------------------------------

class AttentionFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, wqkv, bqkv, wo, bo, pre_w, pre_b, post_w, post_b, mask_add, m: LayerMeta):
        b, s, H = x.shape
        R = b * s
        x2 = x.reshape(R, H)
        fused = use_flash(s, m.head_dim)
        B = b * (m.tp_size if m.shard_rows else 1)  # T*b samples when row-sharded
        if fused:  # keep bits depend only on (seed, layer, coordinates): overlap them with the QKV GEMM
            bits, join = _keep_bits_async(B, s, m, x.device)
        kb = ops.keep_bytes(R, H, x.device) if m.p_hidden > 0 else None  # reused by the backward

        def epilogue(ox, skw, pkw):  # bias + dropout + residual [+ LayerNorm] of this rank's rows
            return ops.bdr_ln(ox, bias=bo, residual=x2, gamma=post_w if m.post_ln else None,
                              beta=post_b if m.post_ln else None, eps=m.eps, p=m.p_hidden, seed=m.seed, rng=m.rng,
                              layer=m.layer_id, site=SITE_ATTN_OUT, row_offset=m.row_offset, rows=R, cols=H,
                              keep_out=kb, **skw, **pkw)

        if fused and _chunked(m, R):  # per-owner chunks, copy-engine exchanges (exchange.py)
            hf, mu1, rs1, G = _chunk_gather_in(x2, m, (pre_w, pre_b) if m.pre_ln else None)
            pool = get_pool()
            qkv = torch.empty(B * s, wqkv.shape[0], dtype=x.dtype, device=x.device)
            ctxv = torch.empty(B * s, m.heads_local * m.head_dim, dtype=x.dtype, device=x.device)
            lse = torch.empty(B, m.heads_local, s, dtype=torch.float32, device=x.device)
            Pr, slots = _chunk_rs_slots(m, R, H)
            mk = mask_add.reshape(B, s) if mask_add is not None else None
            for i, c in enumerate(chunk_order(pool.me, m.tp_size)):
                if c != pool.me:
                    pool.exchange().await_(AGF, c)
                rows, smp = slice(c * R, (c + 1) * R), slice(c * b, (c + 1) * b)
                K.linear(hf[rows], wqkv, bqkv, out=qkv[rows])
                if i == 0:
                    join()
                ops.flash_attn_fwd(qkv[rows], b, s, m.heads_local, m.head_dim, mask_add=None if mk is None else mk[smp],
                                   causal=m.causal, p=m.p_attn, keep_bits=None if bits is None else bits[smp],
                                   out=ctxv[rows], lse_out=lse[smp])
                dst = _chunk_partial_out(c, Pr, slots, R, H)
                K.linear(ctxv[rows], wo, out=dst)
                _chunk_partial_send(c, Pr, dst, R, H)
            P, Pd = lse, bits
            (r, y, mu2, rs2), Gn = _chunk_consume(m, R, H, Pr, lambda skw, pkw: epilogue(slots[0], skw, pkw))
            PR = None
        elif fused and _overlap(m, R):  # copy-engine exchanges, overlapped micro-batches
            hf, mu1, rs1, G = _ov_gather_in(x2, m, (pre_w, pre_b) if m.pre_ln else None)
            qkv = K.linear(hf, wqkv, bqkv)
            join()
            ctxv, lse = ops.flash_attn_fwd(qkv, B, s, m.heads_local, m.head_dim, mask_add=mask_add,
                                           causal=m.causal, p=m.p_attn, keep_bits=bits)
            P, Pd = lse, bits
            skw, Pv = _ov_rs(ctxv, wo, False, m, R, H, RSF)
            pool = get_pool()
            Gn = pool.alloc(m.tp_size * R * H * 2) if m.push_next else None
            pkw = dict(out_peers=pool.self_table, peer_off=Gn // 2 + pool.me * R * H) if Gn is not None else {}
            r, y, mu2, rs2 = epilogue(Pv, skw, pkw)
            _ov_release(m, RSF)
            if Gn is not None:
                _ov_publish(Gn, R, H, m)
            PR = None
        else:
            hf, mu1, rs1, G = _gather_in(x2, m, (pre_w, pre_b) if m.pre_ln else None)
            assert hf.shape[0] == B * s
            qkv = K.linear(hf, wqkv, bqkv)
            if fused:
                join()
                ctxv, lse = ops.flash_attn_fwd(qkv, B, s, m.heads_local, m.head_dim, mask_add=mask_add,
                                               causal=m.causal, p=m.p_attn, keep_bits=bits)
                P, Pd = lse, bits  # the backward re-reads the same keep bits
            else:
                ctxv, P, Pd = attn_core_fwd(qkv, B, s, m, mask_add)
            ox, skw, PR = _rs_out(ctxv, wo, False, m, R, H)
            Gn, pkw = _push_target(m, R, H)
            r, y, mu2, rs2 = epilogue(ox, skw, pkw)
        ctx.kb = kb
        _free(PR)
        if not (m.grad and any(ctx.needs_input_grad)):  # no backward will run: release the gather now
            _free(G)
            G = None
        ctx.m, ctx.shape, ctx.fused, ctx.B, ctx.G = m, (b, s, H), fused, B, G
        ctx.save_for_backward(x2, hf, mu1, rs1, qkv, P, Pd if Pd is not P else None, ctxv, r, mu2, rs2, wqkv, wo,
                              pre_w, post_w, mask_add)
        out = y if m.post_ln else r
        if Gn is not None:
            _PUSHED[(out.data_ptr(), out.numel())] = Gn
        return out.view(b, s, H)

    @staticmethod
    def backward(ctx, dy):
        m: LayerMeta = ctx.m
        b, s, H = ctx.shape
        R, B = b * s, ctx.B
        x2, hf, mu1, rs1, qkv, P, Pd, ctxv, r, mu2, rs2, wqkv, wo, pre_w, post_w, mask_add = ctx.saved_tensors
        if Pd is None:
            Pd = P
        dy2 = dy.reshape(R, H).contiguous()
        m._post_w = post_w if m.post_ln else None
        if ctx.fused and _overlap(m, R):  # copy-engine exchanges, overlapped micro-batches
            dr, dof, V, nv = _ov_grad_publish(dy2, r, mu2, rs2, m, SITE_ATTN_OUT, ctx.kb)
            if not m.post_ln:
                dr = dy2
            dwo, dwqkv = torch.empty_like(wo), torch.empty_like(wqkv)
            with K.grouped():  # dWo and dctx read the same dof
                K.matmul_tn(dof, ctxv, out=dwo)
                dctx = K.matmul_nn(dof, wo)
            dqkv = ops.flash_attn_bwd(dctx, qkv, ctxv, P, B, s, m.heads_local, m.head_dim, mask_add=mask_add,
                                      causal=m.causal, p=m.p_attn, keep_bits=Pd if m.p_attn > 0 else None)
            dbqkv = ops.colsum(dqkv)
            skw, Pv = _ov_rs(dqkv, wqkv, True, m, R, H, RSB, extra=(lambda: K.matmul_tn(dqkv, hf, out=dwqkv),))
            dx, dpre_w, dpre_b = _input_grad(Pv, skw, dr, x2, pre_w, mu1, rs1, m, R, H)
            dpost_w, dpost_b, dbo = _ov_vec_sums(m, V, nv, H)
            _ov_release(m, RSB, AGB)
            _free(ctx.G)
            dpost_w, dpost_b, dpre_w, dpre_b = _sync_replicated(
                [None, None, dpre_w, dpre_b] if nv == 3 else [dpost_w, dpost_b, dpre_w, dpre_b], m,
                keep=(dpost_w, dpost_b) if nv == 3 else None)
            return (dx.view(b, s, H), dwqkv, dbqkv, dwo, dbo, dpre_w, dpre_b, dpost_w, dpost_b, None, None)
        if ctx.fused and _chunked(m, R):  # per-owner chunks, copy-engine exchanges (exchange.py)
            pool = get_pool()
            T, me = m.tp_size, pool.me
            dr, dG, V, nv = _chunk_grad_publish(dy2, r, mu2, rs2, m, SITE_ATTN_OUT, ctx.kb)
            if not m.post_ln:
                dr = dy2
            dof = pool.view(dG, (T * R, H))
            dctx = torch.empty_like(ctxv)
            dqkv = torch.empty_like(qkv)
            Pb = pool.scratch("rsb_slots", T * R * H * 2)
            bslots = pool.view(Pb, (T, R, H))
            for c in chunk_order(me, T):
                if c != me:
                    pool.exchange().await_(AGB, c)
                rows, smp = slice(c * R, (c + 1) * R), slice(c * b, (c + 1) * b)
                K.matmul_nn(dof[rows], wo, out=dctx[rows])
                ops.flash_attn_bwd(dctx[rows], qkv[rows], ctxv[rows], P[smp], b, s, m.heads_local, m.head_dim,
                                   mask_add=None if mask_add is None else mask_add.reshape(B, s)[smp],
                                   causal=m.causal, p=m.p_attn, keep_bits=Pd[smp] if m.p_attn > 0 else None,
                                   dqkv=dqkv[rows])
                dst = bslots[me] if c == me else pool.exchange().staging("rsb", c, (R, H))
                K.matmul_nn(dqkv[rows], wqkv, out=dst)
                if c != me:
                    pool.exchange().send(RSB, c, Pb + me * R * H * 2, dst, ack=True, stage_tag="rsb")
            dwo, dwqkv = torch.empty_like(wo), torch.empty_like(wqkv)
            with K.grouped():  # the weight gradients hide the last partial's copy
                K.matmul_tn(dof, ctxv, out=dwo)
                K.matmul_tn(dqkv, hf, out=dwqkv)
            dbqkv = ops.colsum(dqkv)
            dx, dpre_w, dpre_b, dpost_w, dpost_b, dbo = _chunk_grad_finish(m, R, H, Pb, bslots, dr, x2, pre_w, mu1,
                                                                           rs1, V, nv)
            _free(ctx.G)
            dpost_w, dpost_b, dpre_w, dpre_b = _sync_replicated(
                [None, None, dpre_w, dpre_b] if nv == 3 else [dpost_w, dpost_b, dpre_w, dpre_b], m,
                keep=(dpost_w, dpost_b) if nv == 3 else None)
            return (dx.view(b, s, H), dwqkv, dbqkv, dwo, dbo, dpre_w, dpre_b, dpost_w, dpost_b, None, None)
        dr, dof, dpost_w, dpost_b, dbo, G2 = _gather_grad(dy2, r, mu2, rs2, m, SITE_ATTN_OUT, ctx.kb)
        if not m.post_ln:
            dr = dy2
        if dbo is None:
            dbo = ops.colsum(dof)  # over all rows of the group: complete on every rank
        ov = _overlap_sms(m) > 0 and not (m.tp_size == 1 and not m.pre_ln)
        dwo = torch.empty_like(wo)
        if ov:
            dctx = K.matmul_nn(dof, wo)
        else:  # dWo and dctx read the same dof: one grouped launch
            with K.grouped():
                K.matmul_tn(dof, ctxv, out=dwo)
                dctx = K.matmul_nn(dof, wo)
        if ctx.fused:
            dqkv = ops.flash_attn_bwd(dctx, qkv, ctxv, P, B, s, m.heads_local, m.head_dim, mask_add=mask_add,
                                      causal=m.causal, p=m.p_attn, keep_bits=Pd if m.p_attn > 0 else None)
        else:
            dqkv = attn_core_bwd(dctx, qkv, P, Pd, B, s, m)
        dwqkv = torch.empty_like(wqkv)
        wq_thunk = (lambda: K.matmul_tn(dqkv, hf, out=dwqkv))
        dbqkv = ops.colsum(dqkv)
        if m.tp_size == 1 and not m.pre_ln:
            with K.grouped():  # dWqkv and dx read the same dqkv
                wq_thunk()
                dx = K.matmul_nn(dqkv, wqkv, epi=K.EPI_ADD, aux=dr)
            dpre_w = dpre_b = None
        else:
            dhx, skw, PR = _rs_out(dqkv, wqkv, True, m, R, H, extra=() if ov else (wq_thunk,))
            join, rsm = (lambda: None), 0
            if ov:  # weight gradients on the side stream, next to the reduce-scatter consumer
                join, rsm = _wgrad_async(m, [lambda: K.matmul_tn(dof, ctxv, out=dwo),
                                             lambda: K.matmul_tn(dqkv, hf, out=dwqkv)])
            with _SmLimits(0, rsm):
                dx, dpre_w, dpre_b = _input_grad(dhx, skw, dr, x2, pre_w, mu1, rs1, m, R, H)
            join()
            _free(PR)
        _free(G2, ctx.G)
        dpost_w, dpost_b, dpre_w, dpre_b = _sync_replicated(
            [None, None, dpre_w, dpre_b] if getattr(m, "_post_synced", False) else [dpost_w, dpost_b, dpre_w, dpre_b],
            m, keep=(dpost_w, dpost_b) if getattr(m, "_post_synced", False) else None)
        return (dx.view(b, s, H), dwqkv, dbqkv, dwo, dbo, dpre_w, dpre_b, dpost_w, dpost_b, None, None)


# ---------------------------------------------------------------------------
# MLP sub-layer
# ---------------------------------------------------------------------------

class MlpFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w1, b1, w2, b2, pre_w, pre_b, post_w, post_b, m: LayerMeta):
        b, s, H = x.shape
        R = b * s
        x2 = x.reshape(R, H)
        kb = ops.keep_bytes(R, H, x.device) if m.p_hidden > 0 else None  # reused by the backward

        def epilogue(gx, skw, pkw):  # bias + dropout + residual [+ LayerNorm] of this rank's rows
            return ops.bdr_ln(gx, bias=b2, residual=x2, gamma=post_w if m.post_ln else None,
                              beta=post_b if m.post_ln else None, eps=m.eps, p=m.p_hidden, seed=m.seed, rng=m.rng,
                              layer=m.layer_id, site=SITE_MLP_OUT, row_offset=m.row_offset, rows=R, cols=H,
                              keep_out=kb, **skw, **pkw)

        if _chunked(m, R):  # per-owner chunks, copy-engine exchanges (exchange.py)
            hf, mu1, rs1, G = _chunk_gather_in(x2, m, (pre_w, pre_b) if m.pre_ln else None)
            pool = get_pool()
            TR = m.tp_size * R
            f = torch.empty(TR, w1.shape[0], dtype=x.dtype, device=x.device)
            z = torch.empty_like(f) if m.activation != "none" else None
            Pr, slots = _chunk_rs_slots(m, R, H)
            for c in chunk_order(pool.me, m.tp_size):
                if c != pool.me:
                    pool.exchange().await_(AGF, c)
                rows = slice(c * R, (c + 1) * R)
                K.linear(hf[rows], w1, b1, act=m.activation, out=f[rows],
                         aux_out=None if z is None else z[rows])
                dst = _chunk_partial_out(c, Pr, slots, R, H)
                K.linear(f[rows], w2, out=dst)
                _chunk_partial_send(c, Pr, dst, R, H)
            (r, y, mu2, rs2), Gn = _chunk_consume(m, R, H, Pr, lambda skw, pkw: epilogue(slots[0], skw, pkw))
            PR = None
        elif _overlap(m, R):  # copy-engine exchanges, overlapped micro-batches
            hf, mu1, rs1, G = _ov_gather_in(x2, m, (pre_w, pre_b) if m.pre_ln else None)
            f, z = K.linear(hf, w1, b1, act=m.activation)
            skw, Pv = _ov_rs(f, w2, False, m, R, H, RSF)
            pool = get_pool()
            Gn = pool.alloc(m.tp_size * R * H * 2) if m.push_next else None
            pkw = dict(out_peers=pool.self_table, peer_off=Gn // 2 + pool.me * R * H) if Gn is not None else {}
            r, y, mu2, rs2 = epilogue(Pv, skw, pkw)
            _ov_release(m, RSF)
            if Gn is not None:
                _ov_publish(Gn, R, H, m)
            PR = None
        else:
            hf, mu1, rs1, G = _gather_in(x2, m, (pre_w, pre_b) if m.pre_ln else None)
            f, z = K.linear(hf, w1, b1, act=m.activation)
            gx, skw, PR = _rs_out(f, w2, False, m, R, H)
            Gn, pkw = _push_target(m, R, H)
            r, y, mu2, rs2 = epilogue(gx, skw, pkw)
        ctx.kb = kb
        _free(PR)
        if not (m.grad and any(ctx.needs_input_grad)):  # no backward will run: release the gather now
            _free(G)
            G = None
        ctx.m, ctx.shape, ctx.G = m, (b, s, H), G
        ctx.save_for_backward(x2, hf, mu1, rs1, f, z, r, mu2, rs2, w1, w2, pre_w, post_w)
        out = y if m.post_ln else r
        if Gn is not None:
            _PUSHED[(out.data_ptr(), out.numel())] = Gn
        return out.view(b, s, H)

    @staticmethod
    def backward(ctx, dy):
        m: LayerMeta = ctx.m
        b, s, H = ctx.shape
        R = b * s
        x2, hf, mu1, rs1, f, z, r, mu2, rs2, w1, w2, pre_w, post_w = ctx.saved_tensors
        dy2 = dy.reshape(R, H).contiguous()
        m._post_w = post_w if m.post_ln else None
        if _overlap(m, R):  # copy-engine exchanges, overlapped micro-batches
            dr, dgf, V, nv = _ov_grad_publish(dy2, r, mu2, rs2, m, SITE_MLP_OUT, ctx.kb)
            if not m.post_ln:
                dr = dy2
            dw1, dw2 = torch.empty_like(w1), torch.empty_like(w2)
            with K.grouped():  # dW2 and dz read the same dgf
                K.matmul_tn(dgf, f, out=dw2)
                dz, db1 = K.matmul_nn(dgf, w2, epi=K.EPI_DACT, act=m.activation, aux=z, want_colsum=True)
            skw, Pv = _ov_rs(dz, w1, True, m, R, H, RSB, extra=(lambda: K.matmul_tn(dz, hf, out=dw1),))
            dx, dpre_w, dpre_b = _input_grad(Pv, skw, dr, x2, pre_w, mu1, rs1, m, R, H)
            dpost_w, dpost_b, db2 = _ov_vec_sums(m, V, nv, H)
            _ov_release(m, RSB, AGB)
            _free(ctx.G)
            dpost_w, dpost_b, dpre_w, dpre_b = _sync_replicated(
                [None, None, dpre_w, dpre_b] if nv == 3 else [dpost_w, dpost_b, dpre_w, dpre_b], m,
                keep=(dpost_w, dpost_b) if nv == 3 else None)
            return (dx.view(b, s, H), dw1, db1, dw2, db2, dpre_w, dpre_b, dpost_w, dpost_b, None)
        if _chunked(m, R):  # per-owner chunks, copy-engine exchanges (exchange.py)
            pool = get_pool()
            T, me = m.tp_size, pool.me
            dr, dG, V, nv = _chunk_grad_publish(dy2, r, mu2, rs2, m, SITE_MLP_OUT, ctx.kb)
            if not m.post_ln:
                dr = dy2
            dgf = pool.view(dG, (T * R, H))
            dz = torch.empty_like(z)
            cr = K.colsum_rows(R)
            part = torch.empty(T * cr, z.shape[1], dtype=torch.float32, device=z.device)
            Pb = pool.scratch("rsb_slots", T * R * H * 2)
            bslots = pool.view(Pb, (T, R, H))
            for c in chunk_order(me, T):
                if c != me:
                    pool.exchange().await_(AGB, c)
                rows = slice(c * R, (c + 1) * R)
                K.matmul_nn(dgf[rows], w2, epi=K.EPI_DACT, act=m.activation, aux=z[rows], out=dz[rows],
                            colsum_part=part[c * cr:(c + 1) * cr])
                dst = bslots[me] if c == me else pool.exchange().staging("rsb", c, (R, H))
                K.matmul_nn(dz[rows], w1, out=dst)
                if c != me:
                    pool.exchange().send(RSB, c, Pb + me * R * H * 2, dst, ack=True, stage_tag="rsb")
            dw1, dw2 = torch.empty_like(w1), torch.empty_like(w2)
            with K.grouped():  # the weight gradients hide the last partial's copy
                K.matmul_tn(dgf, f, out=dw2)
                K.matmul_tn(dz, hf, out=dw1)
            db1 = K.colsum_reduce(part, torch.empty(z.shape[1], dtype=z.dtype, device=z.device))
            dx, dpre_w, dpre_b, dpost_w, dpost_b, db2 = _chunk_grad_finish(m, R, H, Pb, bslots, dr, x2, pre_w, mu1,
                                                                           rs1, V, nv)
            _free(ctx.G)
            dpost_w, dpost_b, dpre_w, dpre_b = _sync_replicated(
                [None, None, dpre_w, dpre_b] if nv == 3 else [dpost_w, dpost_b, dpre_w, dpre_b], m,
                keep=(dpost_w, dpost_b) if nv == 3 else None)
            return (dx.view(b, s, H), dw1, db1, dw2, db2, dpre_w, dpre_b, dpost_w, dpost_b, None)
        dr, dgf, dpost_w, dpost_b, db2, G2 = _gather_grad(dy2, r, mu2, rs2, m, SITE_MLP_OUT, ctx.kb)
        if not m.post_ln:
            dr = dy2
        if db2 is None:
            db2 = ops.colsum(dgf)
        ov = _overlap_sms(m) > 0 and not (m.tp_size == 1 and not m.pre_ln)
        dw2 = torch.empty_like(w2)
        if ov:
            dz, db1 = K.matmul_nn(dgf, w2, epi=K.EPI_DACT, act=m.activation, aux=z, want_colsum=True)
        else:  # dW2 and dz read the same dgf: one grouped launch (dz's dGeLU epilogue behind dW2's tiles)
            with K.grouped():
                K.matmul_tn(dgf, f, out=dw2)
                dz, db1 = K.matmul_nn(dgf, w2, epi=K.EPI_DACT, act=m.activation, aux=z, want_colsum=True)
        dw1 = torch.empty_like(w1)
        w1_thunk = (lambda: K.matmul_tn(dz, hf, out=dw1))
        if m.tp_size == 1 and not m.pre_ln:
            with K.grouped():  # dW1 and dx read the same dz
                w1_thunk()
                dx = K.matmul_nn(dz, w1, epi=K.EPI_ADD, aux=dr)
            dpre_w = dpre_b = None
        else:
            dhx, skw, PR = _rs_out(dz, w1, True, m, R, H, extra=() if ov else (w1_thunk,))
            join, rsm = (lambda: None), 0
            if ov:  # weight gradients on the side stream, next to the reduce-scatter consumer
                join, rsm = _wgrad_async(m, [lambda: K.matmul_tn(dgf, f, out=dw2),
                                             lambda: K.matmul_tn(dz, hf, out=dw1)])
            with _SmLimits(0, rsm):
                dx, dpre_w, dpre_b = _input_grad(dhx, skw, dr, x2, pre_w, mu1, rs1, m, R, H)
            join()
            _free(PR)
        _free(G2, ctx.G)
        dpost_w, dpost_b, dpre_w, dpre_b = _sync_replicated(
            [None, None, dpre_w, dpre_b] if getattr(m, "_post_synced", False) else [dpost_w, dpost_b, dpre_w, dpre_b],
            m, keep=(dpost_w, dpost_b) if getattr(m, "_post_synced", False) else None)
        return (dx.view(b, s, H), dw1, db1, dw2, db2, dpre_w, dpre_b, dpost_w, dpost_b, None)
