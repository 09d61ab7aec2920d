"""fp64 CPU restatement of the SPEC's tensor_parallel module — TEST INFRASTRUCTURE ONLY.

Follows SPEC.md:390-516 (types, operations, invariants, design decisions) and
the paper's mechanics (Fig 5 / DistributedEmbedding,
PAPER.md:699-717 speed and memory distributions, PAPER.md:873-893 collective
primitives), with the per-rank dataflow spelled out in SURVEY.md Appendix C.

Simulated ranks are Python lists indexed by tp_rank and are always processed in
ascending order; every reduction sums peers in ascending tp_rank order
(SPEC.md:499, 509).  Tensors are torch CPU tensors; the SPEC's parity oracle is
fp64, fp32 is used only to time the CPU baseline.

Numerics choices the GPU kernels mirror:
  * gelu = erf form ("gelu"), tanh form ("gelu_tanh"), or relu;
  * attention mask: additive float [B, s_k] plus optional causal (-inf above the
    diagonal); scale 1/sqrt(d_h) applied before the mask; a row whose scores are
    all -inf produces zero probabilities;
  * LayerNorm with eps inside the sqrt, biased variance;
  * dropout from oracle.philox masks keyed by logical coordinates.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import philox

# ---------------------------------------------------------------------------
# types
# ---------------------------------------------------------------------------


class OracleError(ValueError):
    pass


@dataclass
class LayerConfig:
    """TransformerLayerConfig (PAPER.md:818 argument list)."""
    num_attention_heads: int
    attention_head_size: int
    hidden_size: int
    intermediate_size: int
    attention_dropout_prob: float = 0.0
    hidden_dropout_prob: float = 0.0
    activation: str = "gelu"
    layernorm_epsilon: float = 1e-5
    causal_mask_size: int | None = None
    pre_layernorm: bool = False
    post_layernorm: bool = True
    optimize: str = "speed"

    def validate(self, T: int = 1) -> None:
        if self.hidden_size != self.num_attention_heads * self.attention_head_size:
            raise OracleError("hidden_size must equal num_attention_heads * attention_head_size")
        if self.optimize == "speed" and self.num_attention_heads % T:
            raise OracleError(f"num_attention_heads {self.num_attention_heads} not divisible by T={T}")
        if self.optimize == "memory" and (self.hidden_size % T or self.intermediate_size % T):
            raise OracleError(f"hidden/intermediate not divisible by T={T}")
        if self.intermediate_size % T:
            raise OracleError(f"intermediate_size {self.intermediate_size} not divisible by T={T}")


@dataclass
class DropoutCtx:
    """Logical coordinates for dropout masks (oracle/philox.py)."""
    seed: int = 0
    layer: int = 0
    sample_offset: int = 0  # global id of sample 0 of the tensor the op sees
    step: int = 0  # training step (device step word snapshot); key = philox.step_key(seed, step)
    # timing-only mode (bench.py CPU baseline): draw masks with torch's CPU RNG instead
    # of the bit-exact numpy Philox, which would dominate a CPU timing
    torch_rng: bool = False


# ---------------------------------------------------------------------------
# collectives over simulated ranks
# ---------------------------------------------------------------------------

def _check_group(xs: list[torch.Tensor]) -> int:
    if not xs:
        raise OracleError("empty TP group")
    shp = xs[0].shape
    for x in xs:
        if x.shape != shp:
            raise OracleError(f"shape mismatch in TP group: {tuple(x.shape)} vs {tuple(shp)}")
    return len(xs)


def allgather(xs: list[torch.Tensor], dim: int) -> list[torch.Tensor]:
    """fused_allgather_for_tp: concatenation along dim, identical on all ranks."""
    _check_group(xs)
    full = torch.cat(xs, dim)
    return [full.clone() for _ in xs]


def fwd_allreduce(xs: list[torch.Tensor]) -> list[torch.Tensor]:
    """fwd_allreduce_for_tp: elementwise sum (ascending rank) on all ranks."""
    _check_group(xs)
    acc = xs[0].clone()
    for x in xs[1:]:
        acc = acc + x
    return [acc.clone() for _ in xs]


def bwd_allreduce(xs: list[torch.Tensor]) -> list[torch.Tensor]:
    """bwd_allreduce_for_tp: identity in forward (sum in backward)."""
    _check_group(xs)
    return [x.clone() for x in xs]


def scatter_and_merge(xs: list[torch.Tensor], split_dim: int, merge_dim: int) -> list[torch.Tensor]:
    """Slice along split_dim into T parts, all-to-all, concatenate received parts along merge_dim."""
    T = _check_group(xs)
    if xs[0].shape[split_dim] % T:
        raise OracleError(f"split dim {split_dim} of size {xs[0].shape[split_dim]} not divisible by T={T}")
    parts = [list(torch.chunk(x, T, split_dim)) for x in xs]
    return [torch.cat([parts[i][j] for i in range(T)], merge_dim) for j in range(T)]


def reduce_scatter(xs: list[torch.Tensor], dim: int) -> list[torch.Tensor]:
    """Slice along dim; rank i receives the ascending-rank sum of slice i."""
    T = _check_group(xs)
    if xs[0].shape[dim] % T:
        raise OracleError(f"dim {dim} of size {xs[0].shape[dim]} not divisible by T={T}")
    parts = [list(torch.chunk(x, T, dim)) for x in xs]
    out = []
    for i in range(T):
        acc = parts[0][i].clone()
        for r in range(1, T):
            acc = acc + parts[r][i]
        out.append(acc)
    return out


def tp_collective(kind: str, xs: list[torch.Tensor], dim: int | None = None, split_dim: int | None = None,
                  merge_dim: int | None = None) -> list[torch.Tensor]:
    """tp_collective(kind, inputs, dims)."""
    if kind == "allgather":
        return allgather(xs, dim)
    if kind == "fwd_allreduce":
        return fwd_allreduce(xs)
    if kind == "bwd_allreduce":
        return bwd_allreduce(xs)
    if kind == "scatter_and_merge":
        return scatter_and_merge(xs, split_dim, merge_dim)
    if kind == "reduce_scatter":
        return reduce_scatter(xs, dim)
    raise OracleError(f"unknown collective {kind!r}")


# ---------------------------------------------------------------------------
# DistributedLinear (Fig 5)
# ---------------------------------------------------------------------------

def shard_linear(W: torch.Tensor, b: torch.Tensor | None, T: int):
    """DistLinearParams: W = [W_1 ... W_T] column-wise, bias on rank 0 only."""
    out_f, in_f = W.shape
    if in_f % T:
        raise OracleError(f"in_features {in_f} not divisible by T={T}")
    Ws = [w.clone() for w in torch.chunk(W, T, 1)]
    bs = [b.clone() if (j == 0 and b is not None) else None for j in range(T)]
    return Ws, bs


def dist_linear_forward(xs: list[torch.Tensor], Ws: list[torch.Tensor], bs: list[torch.Tensor | None],
                        prescaled: bool = False):
    """Per-rank y^(i) = sum_j W_j x_j^(i) + b.

    TP-across-DP: a2a (split features, merge batch) -> local [T*b, in/T] GEMM (+b iff j=0)
    -> reduce-scatter over batch blocks.  Prescaled: feature slice -> partial -> allreduce.
    Returns (ys, saved) where saved feeds dist_linear_backward."""
    T = _check_group(xs)
    if xs[0].shape[-1] % T:
        raise OracleError(f"input feature dim {xs[0].shape[-1]} not divisible by T={T}")
    if prescaled:
        Xs = [xs[0][..., j * (xs[0].shape[-1] // T):(j + 1) * (xs[0].shape[-1] // T)] for j in range(T)]
    else:
        Xs = scatter_and_merge(xs, split_dim=-1, merge_dim=0)
    partial = []
    for j in range(T):
        y = Xs[j] @ Ws[j].t()
        if bs[j] is not None:
            y = y + bs[j]
        partial.append(y)
    ys = fwd_allreduce(partial) if prescaled else reduce_scatter(partial, 0)
    return ys, {"X": Xs, "prescaled": prescaled}


def dist_linear_backward(dys: list[torch.Tensor], Ws: list[torch.Tensor], saved: dict | None):
    """Duals of the forward collectives: RS <-> AG(batch), a2a self-dual.

    Returns (dxs, dWs, db) with db on rank 0 = sum over the gathered batch."""
    if saved is None:
        raise OracleError("dist_linear_backward called before forward")
    T = _check_group(dys)
    Xs = saved["X"]
    if saved["prescaled"]:
        dY = [dys[0]] * T  # identical on every rank; AR dual is identity
    else:
        dY = allgather(dys, 0)
    dXj = [dY[j] @ Ws[j] for j in range(T)]
    dWs = [dY[j].reshape(-1, dY[j].shape[-1]).t() @ Xs[j].reshape(-1, Xs[j].shape[-1]) for j in range(T)]
    db = dY[0].reshape(-1, dY[0].shape[-1]).sum(0)
    if saved["prescaled"]:
        dxs = allgather(dXj, -1)
    else:
        dxs = scatter_and_merge(dXj, split_dim=0, merge_dim=-1)
    return dxs, dWs, db


# ---------------------------------------------------------------------------
# DistributedEmbedding, embedding-dim sharded
# ---------------------------------------------------------------------------

def check_indices(idx: torch.Tensor, V: int) -> None:
    bad = ((idx < 0) | (idx >= V)).reshape(-1).nonzero()
    if bad.numel():
        pos = int(bad[0])
        raise IndexError(f"embedding index {int(idx.reshape(-1)[pos])} out of range [0, {V}) at position {pos}")


def dist_embedding_forward(idxs: list[torch.Tensor], Es: list[torch.Tensor], prescaled: bool = False):
    """AG(indices) -> local lookup of the D/T slice -> scatter_and_merge(batch -> emb).

    Prescaled: skip the gather, lookup, allgather along emb."""
    T = _check_group(Es)
    V = Es[0].shape[0]
    for i in idxs:
        check_indices(i, V)
    if prescaled:
        Ys = [Es[j][idxs[0]] for j in range(T)]
        return allgather(Ys, -1)
    I = torch.cat(idxs, 0)  # AG batch, rank-major
    Ys = [Es[j][I] for j in range(T)]
    return scatter_and_merge(Ys, split_dim=0, merge_dim=-1)


def embedding_gather_routing(idxs: list[torch.Tensor]) -> torch.Tensor:
    """Integer routing of the dim-sharded embedding: gathered order is rank-major."""
    return torch.cat(idxs, 0)


# ---------------------------------------------------------------------------
# vocab-parallel embedding + cross-entropy (builder-defined)
# ---------------------------------------------------------------------------

def vocab_padded(V: int, T: int, multiple: int = 128) -> int:
    q = T * multiple
    return (V + q - 1) // q * q


def vocab_owner(ids: torch.Tensor, Vp: int, T: int):
    """owner(id) = id // (Vp/T), local = id - owner*(Vp/T) (bit-exact integer routing)."""
    per = Vp // T
    owner = torch.div(ids, per, rounding_mode="floor")
    return owner, ids - owner * per


def vocab_embedding_forward(idxs: list[torch.Tensor], Es: list[torch.Tensor], prescaled: bool = True):
    """Rank j owns rows [j*Vp/T, (j+1)*Vp/T).  Masked lookup; RS(batch) or AR (prescaled)."""
    T = _check_group(Es)
    per = Es[0].shape[0]
    I = idxs[0] if prescaled else torch.cat(idxs, 0)
    partial = []
    for j in range(T):
        loc = I - j * per
        own = (loc >= 0) & (loc < per)
        y = Es[j][loc.clamp(0, per - 1)] * own.unsqueeze(-1).to(Es[j].dtype)
        partial.append(y)
    return fwd_allreduce(partial) if prescaled else reduce_scatter(partial, 0)


def cross_entropy_ref(logits: torch.Tensor, targets: torch.Tensor, V: int, ignore_index: int = -100):
    """Single-rank reference: per-row loss = logsumexp(l[:V]) - l[target]; ignored rows -> 0."""
    l = logits[..., :V]
    lse = torch.logsumexp(l, -1)
    valid = targets != ignore_index
    t = torch.where(valid, targets, torch.zeros_like(targets))
    tgt = l.gather(-1, t.unsqueeze(-1)).squeeze(-1)
    return torch.where(valid, lse - tgt, torch.zeros_like(lse))


def vocab_parallel_ce_forward(logit_shards: list[torch.Tensor], targets: torch.Tensor, V: int,
                              ignore_index: int = -100):
    """Per shard: local max m_j, S_j = sum exp(l - m_j) over real columns, target logit if owned.

    AG of (m_j, S_j, l_tgt*[owned]) combined in rank order: m = max m_j,
    S = sum_j S_j e^{m_j - m}, loss = log S + m - l_tgt.  Padded columns (>= V) are -inf."""
    T = _check_group(logit_shards)
    per = logit_shards[0].shape[-1]
    ms, Ss, tl = [], [], []
    valid = targets != ignore_index
    for j in range(T):
        l = logit_shards[j]
        col = torch.arange(j * per, (j + 1) * per)
        l = torch.where(col < V, l, torch.full_like(l, -math.inf))
        m = l.max(-1).values
        m_safe = torch.where(torch.isinf(m), torch.zeros_like(m), m)
        S = torch.exp(l - m_safe.unsqueeze(-1)).sum(-1)
        loc = targets - j * per
        own = valid & (loc >= 0) & (loc < per)
        t = l.gather(-1, loc.clamp(0, per - 1).unsqueeze(-1)).squeeze(-1)
        ms.append(m)
        Ss.append(S)
        tl.append(torch.where(own, t, torch.zeros_like(t)))
    m = ms[0]
    for j in range(1, T):
        m = torch.maximum(m, ms[j])
    S = torch.zeros_like(m)
    tgt = torch.zeros_like(m)
    for j in range(T):
        S = S + torch.where(torch.isinf(ms[j]), torch.zeros_like(S), Ss[j] * torch.exp(ms[j] - m))
        tgt = tgt + tl[j]
    loss = torch.log(S) + m - tgt
    return torch.where(valid, loss, torch.zeros_like(loss)), (m, S)


def vocab_parallel_ce_backward(logit_shards, targets, V, stats, grad_loss, ignore_index: int = -100):
    """dlogits_j = (softmax - onehot_j) * g on the local shard."""
    m, S = stats
    per = logit_shards[0].shape[-1]
    valid = targets != ignore_index
    g = torch.where(valid, grad_loss, torch.zeros_like(grad_loss))
    out = []
    for j, l in enumerate(logit_shards):
        col = torch.arange(j * per, (j + 1) * per)
        p = torch.exp(l - m.unsqueeze(-1)) / S.unsqueeze(-1)
        p = torch.where(col < V, p, torch.zeros_like(p))
        onehot = (col.unsqueeze(0) == targets.reshape(-1, 1)).reshape(p.shape).to(p.dtype)
        out.append((p - onehot) * g.unsqueeze(-1))
    return out


# ---------------------------------------------------------------------------
# LayerNorm
# ---------------------------------------------------------------------------

def layer_norm(x: torch.Tensor, w: torch.Tensor | None, b: torch.Tensor | None, eps: float) -> torch.Tensor:
    mu = x.mean(-1, keepdim=True)
    var = ((x - mu) ** 2).mean(-1, keepdim=True)
    y = (x - mu) / torch.sqrt(var + eps)
    if w is not None:
        y = y * w
    if b is not None:
        y = y + b
    return y


def dist_layernorm_forward(xs: list[torch.Tensor], ws: list[torch.Tensor] | None, bs: list[torch.Tensor] | None,
                           eps: float, n_total: int | None = None) -> list[torch.Tensor]:
    """Local sum x, sum x^2 -> scalar allreduce -> global mean/var -> ApplyLayerNorm on the shard."""
    T = _check_group(xs)
    n = n_total if n_total is not None else sum(x.shape[-1] for x in xs)
    if n == 0:
        raise OracleError("zero channels")
    s1 = fwd_allreduce([x.sum(-1, keepdim=True) for x in xs])[0]
    s2 = fwd_allreduce([(x * x).sum(-1, keepdim=True) for x in xs])[0]
    mean = s1 / n
    var = (s2 / n - mean * mean).clamp_min(0.0)
    out = []
    for j in range(T):
        y = (xs[j] - mean) / torch.sqrt(var + eps)
        if ws is not None:
            y = y * ws[j]
        if bs is not None:
            y = y + bs[j]
        out.append(y)
    return out


# ---------------------------------------------------------------------------
# single-rank reference transformer layer ("reference")
# ---------------------------------------------------------------------------

def activation(name: str, z: torch.Tensor) -> torch.Tensor:
    if name in ("gelu", "gelu_erf"):
        return 0.5 * z * (1.0 + torch.erf(z / math.sqrt(2.0)))
    if name == "gelu_tanh":
        return 0.5 * z * (1.0 + torch.tanh(math.sqrt(2.0 / math.pi) * (z + 0.044715 * z ** 3)))
    if name == "relu":
        return torch.relu(z)
    raise OracleError(f"unknown activation {name!r}")


def init_layer_params(cfg: LayerConfig, seed: int, dtype=torch.float64, std: float = 0.02) -> dict:
    """Full (unsharded) parameters: weights N(0, std) (initializer_range);
    biases N(0, std) so bias paths are exercised; LN gamma ~ 1 + N(0, std), beta ~ N(0, std)."""
    g = torch.Generator().manual_seed(seed)
    H, I = cfg.hidden_size, cfg.intermediate_size

    def n(*shape):
        return (torch.randn(*shape, generator=g, dtype=torch.float64) * std).to(dtype)

    p = {
        "wqkv": n(3 * H, H), "bqkv": n(3 * H),
        "wo": n(H, H), "bo": n(H),
        "w1": n(I, H), "b1": n(I),
        "w2": n(H, I), "b2": n(H),
    }
    for blk in ("attn", "mlp"):
        for where in ("pre", "post"):
            if (where == "pre" and cfg.pre_layernorm) or (where == "post" and cfg.post_layernorm):
                p[f"{blk}_{where}_ln_w"] = (1.0 + n(H)).to(dtype)
                p[f"{blk}_{where}_ln_b"] = n(H)
    return p


def _dropout(x: torch.Tensor, keep: np.ndarray | None, p: float) -> torch.Tensor:
    if keep is None or p == 0.0:
        return x
    return x * torch.from_numpy(keep).to(x.dtype) / (1.0 - p)


def attention_scores_mask(scores: torch.Tensor, mask_add: torch.Tensor | None, causal: bool) -> torch.Tensor:
    # scores [B, nh, sq, sk]
    if mask_add is not None:
        scores = scores + mask_add[:, None, None, :].to(scores.dtype)
    if causal:
        sq, sk = scores.shape[-2:]
        cm = torch.ones(sq, sk, dtype=torch.bool).triu(1 + sk - sq)
        scores = scores.masked_fill(cm, -math.inf)
    return scores


def safe_softmax(scores: torch.Tensor) -> torch.Tensor:
    m = scores.max(-1, keepdim=True).values
    m = torch.where(torch.isinf(m), torch.zeros_like(m), m)
    e = torch.exp(scores - m)
    s = e.sum(-1, keepdim=True)
    return torch.where(s > 0, e / torch.where(s > 0, s, torch.ones_like(s)), torch.zeros_like(e))


def attention_core(q, k, v, mask_add, causal, dctx: DropoutCtx | None, p_attn: float, head_offset: int,
                   nh_global: int):
    """q,k,v [B, s, nh_local, dh] -> ctx [B, s, nh_local*dh]; probs dropout keyed by global heads."""
    B, s, nh, dh = q.shape
    qh, kh, vh = (t.permute(0, 2, 1, 3) for t in (q, k, v))
    scores = (qh @ kh.transpose(-1, -2)) * (1.0 / math.sqrt(dh))
    scores = attention_scores_mask(scores, mask_add, causal)
    probs = safe_softmax(scores)
    if dctx is not None and p_attn > 0 and dctx.torch_rng:
        probs = probs * (torch.rand(probs.shape, dtype=probs.dtype) >= p_attn) / (1.0 - p_attn)
    elif dctx is not None and p_attn > 0:
        keep = philox.attn_prob_mask(np.arange(B) + dctx.sample_offset, np.arange(nh) + head_offset,
                                     s, s, nh_global, dctx.layer, philox.step_key(dctx.seed, dctx.step), p_attn)
        probs = _dropout(probs, keep, p_attn)
    ctx = probs @ vh
    return ctx.permute(0, 2, 1, 3).reshape(B, s, nh * dh)


def _hidden_keep(dctx, B, s, H, site, p, col_offset=0, n_cols=None):
    if dctx is None or p == 0:
        return None
    if dctx.torch_rng:
        return (torch.rand(B, s, n_cols if n_cols is not None else H) >= p).numpy()
    rows = np.arange(B * s) + dctx.sample_offset * s
    cols = np.arange(n_cols if n_cols is not None else H) + col_offset
    keep = philox.keep_mask(rows[:, None], cols[None, :], dctx.layer, site, philox.step_key(dctx.seed, dctx.step), p)
    return keep.reshape(B, s, -1)


def attention_layer_ref(x, p, cfg: LayerConfig, mask_add=None, dctx: DropoutCtx | None = None):
    """DistributedAttentionLayer reference: [pre-LN] -> MHA -> out-proj -> dropout -> +x -> [post-LN]."""
    B, s, H = x.shape
    nh, dh, eps = cfg.num_attention_heads, cfg.attention_head_size, cfg.layernorm_epsilon
    h = layer_norm(x, p["attn_pre_ln_w"], p["attn_pre_ln_b"], eps) if cfg.pre_layernorm else x
    qkv = h @ p["wqkv"].t() + p["bqkv"]
    q, k, v = qkv.split(H, -1)
    ctx = attention_core(q.reshape(B, s, nh, dh), k.reshape(B, s, nh, dh), v.reshape(B, s, nh, dh),
                         mask_add, cfg.causal_mask_size is not None, dctx, cfg.attention_dropout_prob, 0, nh)
    o = ctx @ p["wo"].t() + p["bo"]
    o = _dropout(o, _hidden_keep(dctx, B, s, H, philox.SITE_ATTN_OUT, cfg.hidden_dropout_prob),
                 cfg.hidden_dropout_prob)
    r = x + o
    return layer_norm(r, p["attn_post_ln_w"], p["attn_post_ln_b"], eps) if cfg.post_layernorm else r


def mlp_layer_ref(x, p, cfg: LayerConfig, dctx: DropoutCtx | None = None):
    """DistributedTransformerOutputLayer reference: [pre-LN] -> FC1 -> act -> FC2 -> dropout -> +x -> [post-LN]."""
    B, s, H = x.shape
    eps = cfg.layernorm_epsilon
    h = layer_norm(x, p["mlp_pre_ln_w"], p["mlp_pre_ln_b"], eps) if cfg.pre_layernorm else x
    a = activation(cfg.activation, h @ p["w1"].t() + p["b1"])
    g = a @ p["w2"].t() + p["b2"]
    g = _dropout(g, _hidden_keep(dctx, B, s, H, philox.SITE_MLP_OUT, cfg.hidden_dropout_prob),
                 cfg.hidden_dropout_prob)
    r = x + g
    return layer_norm(r, p["mlp_post_ln_w"], p["mlp_post_ln_b"], eps) if cfg.post_layernorm else r


def transformer_layer_ref(x, p, cfg: LayerConfig, mask_add=None, dctx: DropoutCtx | None = None):
    """attention -> residual -> norm -> MLP -> residual -> norm, honouring pre/post flags."""
    return mlp_layer_ref(attention_layer_ref(x, p, cfg, mask_add, dctx), p, cfg, dctx)


def transformer_ref(x, params: list[dict], cfg: LayerConfig, mask_add=None, seed: int = 0, sample_offset: int = 0):
    """DistributedTransformer: a stack of layers; layer l uses dropout layer id l."""
    for l, p in enumerate(params):
        x = transformer_layer_ref(x, p, cfg, mask_add, DropoutCtx(seed, l, sample_offset))
    return x


# ---------------------------------------------------------------------------
# sharding of layer parameters (speed mode: Megatron layout)
# ---------------------------------------------------------------------------

def shard_layer_params_speed(p: dict, cfg: LayerConfig, T: int) -> list[dict]:
    """Rank j: QKV rows of its heads (q_j; k_j; v_j) [3H/T, H]; Wo[:, j]; W1 rows j; W2[:, j].
    Row-parallel biases (bo, b2) and LayerNorms are replicated."""
    H, I = cfg.hidden_size, cfg.intermediate_size
    hs, ins = H // T, I // T
    wq, wk, wv = p["wqkv"].split(H, 0)
    bq, bk, bv = p["bqkv"].split(H, 0)
    out = []
    for j in range(T):
        sl = slice(j * hs, (j + 1) * hs)
        d = {
            "wqkv": torch.cat([wq[sl], wk[sl], wv[sl]], 0).clone(),
            "bqkv": torch.cat([bq[sl], bk[sl], bv[sl]], 0).clone(),
            "wo": p["wo"][:, sl].clone(), "bo": p["bo"].clone(),
            "w1": p["w1"][j * ins:(j + 1) * ins].clone(), "b1": p["b1"][j * ins:(j + 1) * ins].clone(),
            "w2": p["w2"][:, j * ins:(j + 1) * ins].clone(), "b2": p["b2"].clone(),
        }
        for key in p:
            if "_ln_" in key:
                d[key] = p[key].clone()
        out.append(d)
    return out


def _entry(xs, prescaled):
    return xs[0] if prescaled else torch.cat(xs, 0)


def _exit(X, T, prescaled):
    return [X.clone() for _ in range(T)] if prescaled else list(torch.chunk(X, T, 0))


def dist_attention_forward_speed(xs, shards, cfg: LayerConfig, mask_add=None, prescaled=False,
                                 dctx: DropoutCtx | None = None, keep_entry_exit=True):
    """Speed mode: heads column-parallel, out-proj row-parallel + fwd allreduce."""
    T = len(shards)
    cfg.validate(T)
    X = _entry(xs, prescaled) if keep_entry_exit else xs
    B, s, H = X.shape
    nh, dh, eps = cfg.num_attention_heads, cfg.attention_head_size, cfg.layernorm_epsilon
    nh_l = nh // T
    partial = []
    for j in range(T):
        pj = shards[j]
        h = layer_norm(X, pj["attn_pre_ln_w"], pj["attn_pre_ln_b"], eps) if cfg.pre_layernorm else X
        qkv = h @ pj["wqkv"].t() + pj["bqkv"]
        q, k, v = qkv.split(H // T, -1)
        ctx = attention_core(q.reshape(B, s, nh_l, dh), k.reshape(B, s, nh_l, dh), v.reshape(B, s, nh_l, dh),
                             mask_add, cfg.causal_mask_size is not None, dctx, cfg.attention_dropout_prob,
                             j * nh_l, nh)
        partial.append(ctx @ pj["wo"].t())
    o = fwd_allreduce(partial)[0] + shards[0]["bo"]
    o = _dropout(o, _hidden_keep(dctx, B, s, H, philox.SITE_ATTN_OUT, cfg.hidden_dropout_prob),
                 cfg.hidden_dropout_prob)
    r = X + o
    y = layer_norm(r, shards[0]["attn_post_ln_w"], shards[0]["attn_post_ln_b"], eps) if cfg.post_layernorm else r
    return _exit(y, T, prescaled) if keep_entry_exit else y


def dist_mlp_forward_speed(xs, shards, cfg: LayerConfig, prescaled=False, dctx: DropoutCtx | None = None,
                           keep_entry_exit=True):
    """Speed mode MLP: FC1 output-split -> act -> FC2 input-split -> fwd allreduce."""
    T = len(shards)
    X = _entry(xs, prescaled) if keep_entry_exit else xs
    B, s, H = X.shape
    eps = cfg.layernorm_epsilon
    partial = []
    for j in range(T):
        pj = shards[j]
        h = layer_norm(X, pj["mlp_pre_ln_w"], pj["mlp_pre_ln_b"], eps) if cfg.pre_layernorm else X
        a = activation(cfg.activation, h @ pj["w1"].t() + pj["b1"])
        partial.append(a @ pj["w2"].t())
    g = fwd_allreduce(partial)[0] + shards[0]["b2"]
    g = _dropout(g, _hidden_keep(dctx, B, s, H, philox.SITE_MLP_OUT, cfg.hidden_dropout_prob),
                 cfg.hidden_dropout_prob)
    r = X + g
    y = layer_norm(r, shards[0]["mlp_post_ln_w"], shards[0]["mlp_post_ln_b"], eps) if cfg.post_layernorm else r
    return _exit(y, T, prescaled) if keep_entry_exit else y


def dist_transformer_layer_forward_speed(xs, shards, cfg, mask_add=None, prescaled=False, dctx=None):
    T = len(shards)
    X = _entry(xs, prescaled)
    X = dist_attention_forward_speed(X, shards, cfg, mask_add, prescaled, dctx, keep_entry_exit=False)
    X = dist_mlp_forward_speed(X, shards, cfg, prescaled, dctx, keep_entry_exit=False)
    return _exit(X, T, prescaled)


# ---------------------------------------------------------------------------
# memory mode
# ---------------------------------------------------------------------------

def _chan(t: torch.Tensor, T: int, j: int) -> torch.Tensor:
    n = t.shape[-1] // T
    return t[..., j * n:(j + 1) * n]


def _dist_ln(Xs, p, key, cfg, T):
    H = cfg.hidden_size
    ws = [_chan(p[f"{key}_w"], T, j) for j in range(T)]
    bs = [_chan(p[f"{key}_b"], T, j) for j in range(T)]
    return dist_layernorm_forward(Xs, ws, bs, cfg.layernorm_epsilon, n_total=H)


def dist_attention_forward_memory(Xs, p, cfg: LayerConfig, mask_add=None, dctx: DropoutCtx | None = None):
    """Memory mode on channel-sharded activations Xs[j] [B, s, H/T] (full params p, sliced here).

    Every linear is input-split + reduce-scatter over channels; QKV output rows are
    permuted rank-major so the RS slice j is exactly rank j's heads."""
    T = len(Xs)
    cfg.validate(T)
    H = cfg.hidden_size
    nh, dh = cfg.num_attention_heads, cfg.attention_head_size
    nh_l, hs = nh // T, H // T
    B, s, _ = Xs[0].shape
    hX = _dist_ln(Xs, p, "attn_pre_ln", cfg, T) if cfg.pre_layernorm else Xs
    wq, wk, wv = p["wqkv"].split(H, 0)
    bq, bk, bv = p["bqkv"].split(H, 0)
    perm_w = torch.cat([torch.cat([w[j * hs:(j + 1) * hs] for w in (wq, wk, wv)], 0) for j in range(T)], 0)
    perm_b = torch.cat([torch.cat([b[j * hs:(j + 1) * hs] for b in (bq, bk, bv)], 0) for j in range(T)], 0)
    qkv_partial = [hX[j] @ _chan(perm_w, T, j).t() for j in range(T)]
    qkv = reduce_scatter(qkv_partial, -1)
    ctxs = []
    for j in range(T):
        t = qkv[j] + perm_b[j * 3 * hs:(j + 1) * 3 * hs]
        q, k, v = t.split(hs, -1)
        ctxs.append(attention_core(q.reshape(B, s, nh_l, dh), k.reshape(B, s, nh_l, dh),
                                   v.reshape(B, s, nh_l, dh), mask_add, cfg.causal_mask_size is not None,
                                   dctx, cfg.attention_dropout_prob, j * nh_l, nh))
    o = reduce_scatter([ctxs[j] @ _chan(p["wo"], T, j).t() for j in range(T)], -1)
    out = []
    for j in range(T):
        oj = o[j] + _chan(p["bo"], T, j)
        keep = _hidden_keep(dctx, B, s, H, philox.SITE_ATTN_OUT, cfg.hidden_dropout_prob, col_offset=j * hs,
                            n_cols=hs)
        out.append(Xs[j] + _dropout(oj, keep, cfg.hidden_dropout_prob))
    return _dist_ln(out, p, "attn_post_ln", cfg, T) if cfg.post_layernorm else out


def dist_mlp_forward_memory(Xs, p, cfg: LayerConfig, dctx: DropoutCtx | None = None):
    T = len(Xs)
    H, I = cfg.hidden_size, cfg.intermediate_size
    hs = H // T
    B, s, _ = Xs[0].shape
    hX = _dist_ln(Xs, p, "mlp_pre_ln", cfg, T) if cfg.pre_layernorm else Xs
    z = reduce_scatter([hX[j] @ _chan(p["w1"], T, j).t() for j in range(T)], -1)
    a = [activation(cfg.activation, z[j] + _chan(p["b1"], T, j)) for j in range(T)]
    g = reduce_scatter([a[j] @ _chan(p["w2"], T, j).t() for j in range(T)], -1)
    out = []
    for j in range(T):
        gj = g[j] + _chan(p["b2"], T, j)
        keep = _hidden_keep(dctx, B, s, H, philox.SITE_MLP_OUT, cfg.hidden_dropout_prob, col_offset=j * hs,
                            n_cols=hs)
        out.append(Xs[j] + _dropout(gj, keep, cfg.hidden_dropout_prob))
    return _dist_ln(out, p, "mlp_post_ln", cfg, T) if cfg.post_layernorm else out


def memory_entry(xs, T, prescaled):
    """Stack entry: scatter_and_merge(split channel, merge batch); prescaled: channel slice."""
    if prescaled:
        return [_chan(xs[0], T, j) for j in range(T)]
    return scatter_and_merge(xs, split_dim=-1, merge_dim=0)


def memory_exit(Xs, prescaled):
    if prescaled:
        return allgather(Xs, -1)
    return scatter_and_merge(Xs, split_dim=0, merge_dim=-1)


def dist_attention_forward(xs, p, cfg: LayerConfig, mask_add=None, prescaled=False, dctx=None):
    """dist_attention_forward in cfg.optimize mode; full params p."""
    T = len(xs)
    if cfg.optimize == "memory":
        return memory_exit(dist_attention_forward_memory(memory_entry(xs, T, prescaled), p, cfg, mask_add, dctx),
                           prescaled)
    return dist_attention_forward_speed(xs, shard_layer_params_speed(p, cfg, T), cfg, mask_add, prescaled, dctx)


def dist_mlp_forward(xs, p, cfg: LayerConfig, prescaled=False, dctx=None):
    """dist_mlp_forward."""
    T = len(xs)
    if cfg.optimize == "memory":
        return memory_exit(dist_mlp_forward_memory(memory_entry(xs, T, prescaled), p, cfg, dctx), prescaled)
    return dist_mlp_forward_speed(xs, shard_layer_params_speed(p, cfg, T), cfg, prescaled, dctx)


def dist_transformer_layer_forward(xs, p, cfg: LayerConfig, mask_add=None, prescaled=False, dctx=None):
    """dist_transformer_layer_forward."""
    T = len(xs)
    if cfg.optimize == "memory":
        Xs = memory_entry(xs, T, prescaled)
        Xs = dist_attention_forward_memory(Xs, p, cfg, mask_add, dctx)
        Xs = dist_mlp_forward_memory(Xs, p, cfg, dctx)
        return memory_exit(Xs, prescaled)
    return dist_transformer_layer_forward_speed(xs, shard_layer_params_speed(p, cfg, T), cfg, mask_add, prescaled,
                                                dctx)


# ---------------------------------------------------------------------------
# plan_replacement
# ---------------------------------------------------------------------------

def plan_replacement(spec, registry: dict, tp_marks: set) -> set:
    """Replace a module iff (1) registry has its kind, (2) it is enabled directly or via an
    enabled ancestor, (3) no ancestor is replaced, (4) it shares no parameter with a module
    outside its subtree.  Deterministic top-down (preorder, trace-ordered children) scan.

    ``spec`` is an mpsim.model_graph.ModelSpec (or anything with root_id / children /
    module / subtree)."""
    users: dict[str, set] = {}
    for m in spec.modules:
        for pid in m.param_ids:
            users.setdefault(pid, set()).add(m.id)
    replaced: set = set()

    def visit(mid: str, enabled: bool, under_replaced: bool) -> None:
        m = spec.module(mid)
        en = enabled or mid in tp_marks
        take = False
        if not under_replaced and en and m.kind is not None and m.kind in registry:
            sub = set(spec.subtree(mid))
            shared = any(not users[pid] <= sub for s in sub for pid in spec.module(s).param_ids)
            take = not shared
        if take:
            replaced.add(mid)
        for c in spec.children(mid):
            visit(c, en, under_replaced or take)

    visit(spec.root_id, False, False)
    return replaced


# ---------------------------------------------------------------------------
# AdamW (PAPER.md:765 optimizer state sharding; csrc/runtime.cu smpk_adam_step restated)
# ---------------------------------------------------------------------------

def adamw_ref(master, param_out, grad, m, v, *, lr, betas, eps, weight_decay, step, grad_scale):
    """In-place AdamW on fp32 torch tensors (same update order as smpk_adam_step)."""
    b1, b2 = betas
    g = grad.float() * grad_scale
    m.mul_(b1).add_((1.0 - b1) * g)
    v.mul_(b2).add_((1.0 - b2) * g * g)
    bc1, bc2 = 1.0 - b1 ** step, 1.0 - b2 ** step
    upd = (m / bc1) / ((v / bc2).sqrt() + eps)
    master.sub_(lr * (upd + weight_decay * master))
    param_out.copy_(master.to(param_out.dtype))
