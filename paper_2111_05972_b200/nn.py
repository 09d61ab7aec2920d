"""smp.nn — distributed modules of the tensor-parallel hot path.

Signatures follow the paper's API: DistributedLinear,
DistributedEmbedding, DistributedTransformerLayer, DistributedTransformer,
DistributedTransformerLMHead, plus the DistributedAttentionLayer /
DistributedTransformerOutputLayer children and
DistributedLayerNorm.  Parameters live on the current CUDA device
in bf16, sharded by tp_rank; forward/backward run in libsmpk (no CPU path).
"""
from __future__ import annotations

import math

import torch
from torch import nn

from . import collectives as C
from . import layers as L
from . import memory_mode as MM
from .errors import NotDivisibleError, ShapeMismatchError
from .state import STATE, begin_forward, get_pool, next_layer_id

DTYPE = torch.bfloat16


class DistributedModule(nn.Module):
    """Base class of every smp.nn module."""

    @property
    def tp_size(self) -> int:
        return STATE.tp_size

    @property
    def tp_rank(self) -> int:
        return STATE.tp_rank


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("smp.nn modules need a CUDA device (libsmpk has no CPU path)")
    return torch.device("cuda", torch.cuda.current_device())


def _param(shape, std, gen, zero=False, one=False):
    dev = _device()
    if zero:
        t = torch.zeros(shape, dtype=DTYPE, device=dev)
    elif one:
        t = torch.ones(shape, dtype=DTYPE, device=dev)
    else:
        t = (torch.randn(shape, generator=gen, dtype=torch.float32, device=dev) * std).to(DTYPE)
    return nn.Parameter(t)


def _gen(layer_id: int, salt: int):
    g = torch.Generator(device=_device())
    g.manual_seed((STATE.seed * 1000003 + layer_id * 7919 + salt * 104729 + STATE.tp_rank) % (2 ** 63))
    return g


def _mask_2d(attention_mask, B, s):
    """Accept an additive mask [B, s] or HF-extended [B, 1, 1, s]; returns fp32 [B, s] or None."""
    if attention_mask is None:
        return None
    m = attention_mask.reshape(B, -1)
    if m.shape[1] != s:
        raise ShapeMismatchError(f"attention_mask must have {s} key positions, got {tuple(attention_mask.shape)}")
    return m.to(torch.float32).contiguous()


# ---------------------------------------------------------------------------
# DistributedLinear (Fig 5, 802)
# ---------------------------------------------------------------------------

class _SliceFeatures(torch.autograd.Function):
    """Prescaled input split: keep feature slice j; backward = allgather along features."""

    @staticmethod
    def forward(ctx, x, j, T):
        n = x.shape[-1] // T
        return x[..., j * n:(j + 1) * n]

    @staticmethod
    def backward(ctx, g):
        return C.all_gather(g.contiguous(), -1), None, None


class DistributedLinear(DistributedModule):
    """smp.nn.DistributedLinear(in_features, out_features): W = [W_1 ... W_T] split column-wise
    (over input features), bias only on tp_rank 0.  Each rank slices its input rows by
    feature, all-to-all delivers slice j of every peer's samples to rank j, rank j applies
    W_j to the gathered [T*b, in/T] block (+ b iff j == 0), and a reduce-scatter over the
    batch returns y^(i) = sum_j W_j x_j^(i) (+ b) to rank i.  Prescaled batch: feature slice
    -> partial product -> allreduce."""

    def __init__(self, in_features, out_features, bias=True, initializer_range=0.02):
        super().__init__()
        T = STATE.tp_size
        if in_features % T:
            raise NotDivisibleError(f"in_features {in_features} not divisible by tensor_parallel_degree {T}")
        self.in_features, self.out_features = in_features, out_features
        g = _gen(next_layer_id(), 3)
        self.weight = _param((out_features, in_features // T), initializer_range, g)
        self.bias = _param((out_features,), 0, None, zero=True) if (bias and STATE.tp_rank == 0) else None

    @torch.no_grad()
    def load_full(self, W: torch.Tensor, b: torch.Tensor | None = None):
        n = self.in_features // STATE.tp_size
        j = STATE.tp_rank
        self.weight.copy_(W[:, j * n:(j + 1) * n])
        if self.bias is not None and b is not None:
            self.bias.copy_(b)

    def forward(self, x):
        T, j = STATE.tp_size, STATE.tp_rank
        lead = x.shape[:-1]
        x2 = x.reshape(-1, self.in_features).to(DTYPE)
        if T == 1:
            y = L.LinearFn.apply(x2.contiguous(), self.weight, self.bias)
        elif STATE.prescaled:
            y = C.fwd_allreduce_for_tp(L.LinearFn.apply(_SliceFeatures.apply(x2, j, T), self.weight, self.bias))
        else:
            Xj = C.scatter_and_merge_for_tp(x2.contiguous(), -1, 0)  # [T*b, in/T]
            y = C.reduce_scatter_for_tp(L.LinearFn.apply(Xj, self.weight, self.bias), 0)
        return y.reshape(*lead, self.out_features)


# ---------------------------------------------------------------------------
# transformer (speed mode)
# ---------------------------------------------------------------------------

class _LayerBase(DistributedModule):
    def __init__(self, num_attention_heads, attention_head_size, hidden_size, intermediate_size,
                 attention_dropout_prob, hidden_dropout_prob, activation, layernorm_epsilon, initializer_range,
                 use_normal_initialization, causal_mask_size, add_cross_attention, pre_layernorm, post_layernorm,
                 layer_id=None):
        super().__init__()
        if hidden_size != num_attention_heads * attention_head_size:
            raise ShapeMismatchError("hidden_size must equal num_attention_heads * attention_head_size")
        T = STATE.tp_size
        if num_attention_heads % T:
            raise NotDivisibleError(f"num_attention_heads {num_attention_heads} not divisible by "
                                    f"tensor_parallel_degree {T}")
        if intermediate_size % T:
            raise NotDivisibleError(f"intermediate_size {intermediate_size} not divisible by {T}")
        if add_cross_attention:
            raise NotImplementedError("add_cross_attention: only self-attention is on the hot path "
                                      "(SPEC.md:513 non-goal)")
        if activation not in ("gelu", "gelu_erf", "gelu_tanh", "relu"):
            raise ValueError(f"activation must be gelu | gelu_tanh | relu, got {activation!r}")
        self.num_attention_heads = num_attention_heads
        self.attention_head_size = attention_head_size
        self.hidden_size = hidden_size
        self.intermediate_size = intermediate_size
        self.attention_dropout_prob = attention_dropout_prob
        self.hidden_dropout_prob = hidden_dropout_prob
        self.activation = activation
        self.layernorm_epsilon = layernorm_epsilon
        self.initializer_range = initializer_range
        self.causal_mask_size = causal_mask_size
        self.pre_layernorm = pre_layernorm
        self.post_layernorm = post_layernorm
        self.layer_id = next_layer_id() if layer_id is None else layer_id

    @property
    def _memory(self) -> bool:
        """Memory mode: channel-sharded activations, input-split linears."""
        return STATE.optimize == "memory" and STATE.tp_size > 1

    def _meta(self, rc) -> L.LayerMeta:
        """rc = (attention sample offset, own first global token row, row-sharded?[, micro-batch,
        full per-rank batch]) -- the last two for the overlapped micro-batches of tp_exchange="overlap"."""
        sample_offset, row_offset, shard = rc[:3]
        mb, mb_batch = (rc[3], rc[4]) if len(rc) > 3 else (-1, 0)
        T = STATE.tp_size
        hl = self.num_attention_heads // T
        return L.LayerMeta(hidden=self.hidden_size, heads_local=hl, heads_global=self.num_attention_heads,
                           head_dim=self.attention_head_size, eps=self.layernorm_epsilon,
                           p_attn=self.attention_dropout_prob if self.training else 0.0,
                           p_hidden=self.hidden_dropout_prob if self.training else 0.0,
                           causal=self.causal_mask_size is not None, pre_ln=self.pre_layernorm,
                           post_ln=self.post_layernorm, activation=self.activation, layer_id=self.layer_id,
                           seed=STATE.seed, rng=STATE.rng_cur, grad=torch.is_grad_enabled(), head_offset=STATE.tp_rank * hl,
                           sample_offset=sample_offset, tp_size=T, row_offset=row_offset, shard_rows=shard,
                           comm=STATE.config.get("tp_comm", "peer"), mb=mb, mb_batch=mb_batch)

    def _ln_params(self, prefix):
        H = self.hidden_size // STATE.tp_size if self._memory else self.hidden_size  # memory: channel chunk
        for where, flag in (("pre", self.pre_layernorm), ("post", self.post_layernorm)):
            if flag:
                setattr(self, f"{prefix}{where}_ln_weight", _param((H,), 0, None, one=True))
                setattr(self, f"{prefix}{where}_ln_bias", _param((H,), 0, None, zero=True))
            else:
                setattr(self, f"{prefix}{where}_ln_weight", None)
                setattr(self, f"{prefix}{where}_ln_bias", None)


class DistributedAttentionLayer(_LayerBase):
    """Self-attention sub-layer (speed mode): QKV column-parallel by heads, out-proj row-parallel."""

    def __init__(self, num_attention_heads=32, attention_head_size=32, hidden_size=1024, attention_dropout_prob=0.1,
                 hidden_dropout_prob=0.1, layernorm_epsilon=1e-5, initializer_range=0.02,
                 use_normal_initialization=False, causal_mask_size=None, add_cross_attention=False,
                 pre_layernorm=False, post_layernorm=True, layer_id=None, _standalone=True):
        super().__init__(num_attention_heads, attention_head_size, hidden_size, 4 * hidden_size,
                         attention_dropout_prob, hidden_dropout_prob, "gelu", layernorm_epsilon, initializer_range,
                         use_normal_initialization, causal_mask_size, add_cross_attention, pre_layernorm,
                         post_layernorm, layer_id)
        self._standalone = _standalone
        T, H = STATE.tp_size, hidden_size
        g = _gen(self.layer_id, 1)
        std = initializer_range
        if self._memory:
            # input-split QKV (all 3H output rows, rank-major q_j|k_j|v_j, local input channels)
            self.qkv_weight = _param((3 * H, H // T), std, g)
            self.dense_bias = _param((H // T,), 0, None, zero=True)
        else:
            self.qkv_weight = _param((3 * H // T, H), std, g)
            self.dense_bias = _param((H,), 0, None, zero=True)
        self.qkv_bias = _param((3 * H // T,), 0, None, zero=True)
        self.dense_weight = _param((H, H // T), std, g)
        self._ln_params("")

    def sublayer(self, X, mask, rc, push_next=False):
        m = self._meta(rc)
        m.push_next = push_next
        if self._memory:
            return MM.attention(X, self, mask, m, STATE.tp_rank)
        return L.AttentionFn.apply(X, self.qkv_weight, self.qkv_bias, self.dense_weight, self.dense_bias,
                                   self.pre_ln_weight, self.pre_ln_bias, self.post_ln_weight, self.post_ln_bias,
                                   mask, m)

    def forward(self, hidden_states, attention_mask=None):
        return _run_standalone(self, hidden_states, attention_mask)

    @torch.no_grad()
    def load_full(self, p: dict):
        """Load unsharded parameters (oracle layout: wqkv=[q;k;v] [3H,H], wo [H,H], ...)."""
        T, j, H = STATE.tp_size, STATE.tp_rank, self.hidden_size
        hs = H // T
        sl = slice(j * hs, (j + 1) * hs)
        wq, wk, wv = p["wqkv"].split(H, 0)
        bq, bk, bv = p["bqkv"].split(H, 0)
        self.qkv_bias.copy_(torch.cat([bq[sl], bk[sl], bv[sl]], 0))
        self.dense_weight.copy_(p["wo"][:, sl])
        if self._memory:  # rows rank-major (q_r | k_r | v_r for r = 0..T-1), local input channels
            perm = torch.cat([torch.cat([w[r * hs:(r + 1) * hs] for w in (wq, wk, wv)], 0) for r in range(T)], 0)
            self.qkv_weight.copy_(perm[:, sl])
            self.dense_bias.copy_(p["bo"][sl])
        else:
            self.qkv_weight.copy_(torch.cat([wq[sl], wk[sl], wv[sl]], 0))
            self.dense_bias.copy_(p["bo"])
        ln_sl = sl if self._memory else slice(None)
        for where in ("pre", "post"):
            if getattr(self, f"{where}_ln_weight") is not None:
                getattr(self, f"{where}_ln_weight").copy_(p[f"attn_{where}_ln_w"][ln_sl])
                getattr(self, f"{where}_ln_bias").copy_(p[f"attn_{where}_ln_b"][ln_sl])


class DistributedTransformerOutputLayer(_LayerBase):
    """MLP sub-layer (speed mode): FC1 column-parallel, FC2 row-parallel."""

    def __init__(self, hidden_size=1024, intermediate_size=4096, hidden_dropout_prob=0.1, activation="gelu",
                 layernorm_epsilon=1e-5, initializer_range=0.02, use_normal_initialization=False,
                 pre_layernorm=False, post_layernorm=True, layer_id=None, num_attention_heads=1, _standalone=True):
        super().__init__(num_attention_heads, hidden_size // num_attention_heads, hidden_size, intermediate_size,
                         0.0, hidden_dropout_prob, activation, layernorm_epsilon, initializer_range,
                         use_normal_initialization, None, False, pre_layernorm, post_layernorm, layer_id)
        self._standalone = _standalone
        T, H, I = STATE.tp_size, hidden_size, intermediate_size
        g = _gen(self.layer_id, 2)
        std = initializer_range
        if self._memory:  # input-split FC1 (all 4H rows, local input channels)
            self.fc1_weight = _param((I, H // T), std, g)
            self.fc2_bias = _param((H // T,), 0, None, zero=True)
        else:
            self.fc1_weight = _param((I // T, H), std, g)
            self.fc2_bias = _param((H,), 0, None, zero=True)
        self.fc1_bias = _param((I // T,), 0, None, zero=True)
        self.fc2_weight = _param((H, I // T), std, g)
        self._ln_params("")

    def sublayer(self, X, mask, rc, push_next=False):
        m = self._meta(rc)
        m.push_next = push_next
        if self._memory:
            return MM.mlp(X, self, m, STATE.tp_rank)
        return L.MlpFn.apply(X, self.fc1_weight, self.fc1_bias, self.fc2_weight, self.fc2_bias, self.pre_ln_weight,
                             self.pre_ln_bias, self.post_ln_weight, self.post_ln_bias, m)

    def forward(self, hidden_states, attention_mask=None):
        return _run_standalone(self, hidden_states, None)

    @torch.no_grad()
    def load_full(self, p: dict):
        T, j, I = STATE.tp_size, STATE.tp_rank, self.intermediate_size
        ins = I // T
        sl = slice(j * ins, (j + 1) * ins)
        hs = self.hidden_size // T
        hsl = slice(j * hs, (j + 1) * hs)
        self.fc1_bias.copy_(p["b1"][sl])
        self.fc2_weight.copy_(p["w2"][:, sl])
        if self._memory:
            self.fc1_weight.copy_(p["w1"][:, hsl])
            self.fc2_bias.copy_(p["b2"][hsl])
        else:
            self.fc1_weight.copy_(p["w1"][sl])
            self.fc2_bias.copy_(p["b2"])
        ln_sl = hsl if self._memory else slice(None)
        for where in ("pre", "post"):
            if getattr(self, f"{where}_ln_weight") is not None:
                getattr(self, f"{where}_ln_weight").copy_(p[f"mlp_{where}_ln_w"][ln_sl])
                getattr(self, f"{where}_ln_bias").copy_(p[f"mlp_{where}_ln_b"][ln_sl])


_MB_STREAM: dict = {}


def _microbatch_stream() -> torch.cuda.Stream:
    dev = torch.cuda.current_device()
    if dev not in _MB_STREAM:
        _MB_STREAM[dev] = torch.cuda.Stream(device=dev)
    return _MB_STREAM[dev]


def _memory_mode() -> bool:
    return STATE.optimize == "memory" and STATE.tp_size > 1


def _row_ctx(B: int, s: int):
    """(attention sample offset, own first global token row, row-sharded) for a batch of B own samples.

    TP across DP ranks: activations stay on the owning rank (row-sharded); the
    attention of the local heads sees the whole TP group's samples, starting at global sample
    rdp_rank*T*B.  Prescaled batch / T == 1: activations replicated, samples rdp_rank*B (dp_rank*B)."""
    if STATE.tp_size == 1:
        off = STATE.dp_rank * B
        return (off, off * s, False)
    if _memory_mode():  # channel-sharded activations hold every sample of the group (prescaled: own)
        off = STATE.rdp_rank * B * (1 if STATE.prescaled else STATE.tp_size)
        return (off, off * s, False)
    if STATE.prescaled:
        off = STATE.rdp_rank * B
        return (off, off * s, False)
    return (STATE.rdp_rank * STATE.tp_size * B, STATE.dp_rank * B * s, True)


def _entry(x, attention_mask):
    """Module entry: in row-sharded mode only the attention mask is gathered over the TP group.
    Also snapshots / advances the device dropout step word (state.begin_forward)."""
    begin_forward()
    B, s = x.shape[0], x.shape[1]
    mask = _mask_2d(attention_mask, B, s)
    rc = _row_ctx(B, s)
    if _memory_mode():  # scatter_and_merge(split channel, merge batch) -> [T*b, s, H/T]
        if not STATE.prescaled and mask is not None:
            mask = C.all_gather(mask, 0)
        return MM.entry(x, STATE.tp_size, STATE.tp_rank, STATE.prescaled), mask, rc
    if rc[2] and mask is not None:
        mask = C.all_gather(mask, 0)
    return x, mask, rc


def _exit(Y):
    """Return the rows of this rank's samples from a TP-replicated tensor (backward: allgather)."""
    if STATE.prescaled or STATE.tp_size == 1:
        return Y
    return C.tp_dp_exit(Y)


def _run_standalone(mod, hidden_states, attention_mask):
    x = hidden_states.to(DTYPE).contiguous()
    X, mask, rc = _entry(x, attention_mask)
    Y = mod.sublayer(X, mask, rc)
    return MM.exit(Y, STATE.prescaled) if _memory_mode() else Y


class DistributedTransformerLayer(DistributedModule):
    """smp.nn.DistributedTransformerLayer: attention -> residual -> norm -> MLP ->
    residual -> norm, honouring pre_layernorm / post_layernorm (each sub-layer owns its LNs)."""

    def __init__(self, num_attention_heads=32, attention_head_size=32, hidden_size=1024, intermediate_size=4096,
                 attention_dropout_prob=0.1, hidden_dropout_prob=0.1, activation="gelu", layernorm_epsilon=1e-5,
                 initializer_range=0.02, use_normal_initialization=False, causal_mask_size=None,
                 add_cross_attention=False, pre_layernorm=False, post_layernorm=True, layer_id=None):
        super().__init__()
        lid = next_layer_id() if layer_id is None else layer_id
        self.layer_id = lid
        self.attention = DistributedAttentionLayer(
            num_attention_heads, attention_head_size, hidden_size, attention_dropout_prob, hidden_dropout_prob,
            layernorm_epsilon, initializer_range, use_normal_initialization, causal_mask_size, add_cross_attention,
            pre_layernorm, post_layernorm, layer_id=lid, _standalone=False)
        self.output = DistributedTransformerOutputLayer(
            hidden_size, intermediate_size, hidden_dropout_prob, activation, layernorm_epsilon, initializer_range,
            use_normal_initialization, pre_layernorm, post_layernorm, layer_id=lid,
            num_attention_heads=num_attention_heads, _standalone=False)

    def sublayer(self, X, mask, rc, push_last=False):
        """push_last: a following sub-layer gathers this layer's output (stack-internal)."""
        nopre = not self.output.pre_layernorm
        Y = self.attention.sublayer(X, mask, rc, push_next=nopre)
        return self.output.sublayer(Y, mask, rc, push_next=push_last and not self.attention.pre_layernorm)

    def forward(self, hidden_states, attention_mask=None):
        return _run_standalone(self, hidden_states, attention_mask)

    def load_full(self, p: dict):
        self.attention.load_full(p)
        self.output.load_full(p)


class DistributedTransformer(DistributedModule):
    """smp.nn.DistributedTransformer: num_layers DistributedTransformerLayers; the
    TP-across-DP gather/return happens once at the stack boundary."""

    def __init__(self, num_layers=12, num_attention_heads=32, attention_head_size=32, hidden_size=1024,
                 intermediate_size=4096, attention_dropout_prob=0.1, hidden_dropout_prob=0.1, activation="gelu",
                 layernorm_epsilon=1e-5, initializer_range=0.02, use_normal_initialization=False,
                 causal_mask_size=None, add_cross_attention=False, pre_layernorm=False, post_layernorm=True):
        super().__init__()
        self.num_layers = num_layers
        self.seq_layers = nn.ModuleList([
            DistributedTransformerLayer(num_attention_heads, attention_head_size, hidden_size, intermediate_size,
                                        attention_dropout_prob, hidden_dropout_prob, activation, layernorm_epsilon,
                                        initializer_range, use_normal_initialization, causal_mask_size,
                                        add_cross_attention, pre_layernorm, post_layernorm)
            for _ in range(num_layers)])

    def sublayer(self, X, mask, rc):
        if getattr(self, "_ckpt_groups", None):  # smp.set_activation_checkpointing
            from .checkpointing import run_stack
            return run_stack(self, X, mask, rc)
        if self._split_microbatches(X, rc):
            return self._sublayer_microbatches(X, mask, rc)
        n = len(self.seq_layers)
        for i, layer in enumerate(self.seq_layers):
            X = layer.sublayer(X, mask, rc, push_last=i + 1 < n)
        return X

    def _split_microbatches(self, X, rc) -> bool:
        """tp_exchange="overlap": row-sharded speed mode with an even per-rank batch whose halves
        are whole 128-row GEMM tiles and fused attention."""
        if not (rc[2] and STATE.config.get("tp_exchange", "barrier") == "overlap" and STATE.tp_size > 1
                and STATE.config.get("tp_comm", "peer") == "peer"):
            return False
        B, s = X.shape[0], X.shape[1]
        lay = self.seq_layers[0].attention
        return B % 2 == 0 and (B // 2) * s % 128 == 0 and L.use_flash(s, lay.attention_head_size)

    def _sublayer_microbatches(self, X, mask, rc):
        """The batch as two micro-batches on two streams, layer by layer in lock step: while one
        micro-batch's gathers and reduce-scatters move on the copy engines, the other's GEMMs and
        attention run (PAPER.md:281 TP across DP; exchange.py mailboxes).  Dropout masks and row
        coordinates are those of the whole batch, so the result equals the unsplit stack's."""
        B, s = X.shape[0], X.shape[1]
        b, T = B // 2, STATE.tp_size
        pool = get_pool()
        if STATE.xch_fresh:  # step entry: every rank is done with the previous step's regions
            pool.barrier()
            STATE.xch_fresh = False
        main = torch.cuda.current_stream()
        side = _microbatch_stream()
        side.wait_stream(main)
        xs = [X[:b], X[b:]]
        masks = [None, None] if mask is None else \
            [mask.reshape(T, B, s)[:, h * b:(h + 1) * b].reshape(T * b, s) for h in (0, 1)]
        rcs = [(rc[0], rc[1] + h * b * s, True, h, B) for h in (0, 1)]
        streams = (main, side)
        n = len(self.seq_layers)
        for i, layer in enumerate(self.seq_layers):
            for h in (0, 1):
                with torch.cuda.stream(streams[h]):
                    xs[h] = layer.sublayer(xs[h], masks[h], rcs[h], push_last=i + 1 < n)
        main.wait_stream(side)
        xs[1].record_stream(main)
        return torch.cat(xs, 0)

    def forward(self, hidden_states, attention_mask=None):
        return _run_standalone(self, hidden_states, attention_mask)


# ---------------------------------------------------------------------------
# LayerNorm, embeddings, LM head
# ---------------------------------------------------------------------------

class DistributedLayerNorm(DistributedModule):
    """smp.nn.DistributedLayerNorm.  In speed mode the LayerNorm is replicated
    across the TP group and runs on the fused row kernel."""

    def __init__(self, normalized_shape, eps=1e-5, elementwise_affine=True):
        super().__init__()
        n = normalized_shape if isinstance(normalized_shape, int) else normalized_shape[-1]
        self.normalized_shape, self.eps = n, eps
        self.weight = _param((n,), 0, None, one=True)
        self.bias = _param((n,), 0, None, zero=True)

    def forward(self, x):
        return L.LayerNormFn.apply(x.to(DTYPE), self.weight, self.bias, self.eps)


from .embedding import (DistributedEmbedding, VocabParallelEmbedding, lm_head_logits,  # noqa: E402
                        vocab_parallel_cross_entropy)


class DistributedTransformerLMHead(DistributedModule):
    """smp.nn.DistributedTransformerLMHead: GPT-style LM with a vocab-parallel
    word embedding tied to the LM head, learned position embeddings, a DistributedTransformer
    stack, a final LayerNorm (pre-LN models) and the vocab-parallel cross-entropy.

    forward(input_ids, attention_mask=None, labels=None): with labels returns the per-token
    loss [b, s] (fp32, 0 where labels == -100); otherwise the vocab-sharded logits
    [b, s, Vp/T].  The TP-across-DP gather happens once at the embedding (an allreduce of
    the gathered partial lookups replaces reduce-scatter + the stack's allgather)."""

    def __init__(self, num_layers=12, num_attention_heads=32, attention_head_size=32, hidden_size=1024,
                 intermediate_size=4096, vocab_size=30522, num_positions=1024, attention_dropout_prob=0.1,
                 hidden_dropout_prob=0.1, activation="gelu", layernorm_epsilon=1e-5, num_token_types=0,
                 causal_mask_size=None, add_cross_attention=False, add_lm_head=True, initializer_range=0.02,
                 use_normal_initialization=False, pre_layernorm=False, post_layernorm=True):
        super().__init__()
        if num_token_types:
            raise NotImplementedError("token type embeddings are not on the TP hot path")
        self.vocab_size, self.hidden_size, self.add_lm_head = vocab_size, hidden_size, add_lm_head
        self.word_embedding = VocabParallelEmbedding(vocab_size, hidden_size, initializer_range=initializer_range)
        g = _gen(next_layer_id(), 4)
        self.position_embedding = nn.Parameter(
            (torch.randn(num_positions, hidden_size, generator=g, device=_device()) * initializer_range).to(DTYPE))
        self.transformer = DistributedTransformer(num_layers, num_attention_heads, attention_head_size, hidden_size,
                                                  intermediate_size, attention_dropout_prob, hidden_dropout_prob,
                                                  activation, layernorm_epsilon, initializer_range,
                                                  use_normal_initialization, causal_mask_size, add_cross_attention,
                                                  pre_layernorm, post_layernorm)
        self.final_ln = DistributedLayerNorm(hidden_size, layernorm_epsilon) if pre_layernorm else None

    def forward(self, input_ids, attention_mask=None, labels=None):
        b, s = input_ids.shape
        T = STATE.tp_size
        begin_forward()
        gathered = not (STATE.prescaled or T == 1)
        ids = C.all_gather(input_ids.contiguous(), 0) if gathered else input_ids
        mask = _mask_2d(attention_mask, b, s)
        if gathered and mask is not None:
            mask = C.all_gather(mask, 0)
        rc = _row_ctx(b, s)
        we = self.word_embedding
        from .embedding import _LookupFn
        h = _LookupFn.apply(ids, we.weight, we.row_offset, we.num_embeddings, we.padding_idx,
                            self.position_embedding if STATE.tp_rank == 0 else None, s, False)
        h = h.reshape(ids.shape[0], s, self.hidden_size)
        if gathered:
            h = C.reduce_scatter_for_tp(h, 0)  # partial lookups -> this rank's own rows
        elif T > 1:
            h = C.fwd_allreduce_for_tp(h)
        if _memory_mode():  # channel-sharded stack between the embedding and the LM head
            h = MM.exit(self.transformer.sublayer(MM.entry(h, T, STATE.tp_rank, STATE.prescaled), mask, rc),
                        STATE.prescaled)
        else:
            h = self.transformer.sublayer(h, mask, rc)
        if self.final_ln is not None:
            h = self.final_ln(h)
        if not self.add_lm_head:
            return h
        if gathered:
            h = C.fused_allgather_for_tp(h, 0)  # every rank scores all rows on its vocab shard
        logits = lm_head_logits(h, we.weight, reduce_grad=not gathered)  # [B*s, Vp/T]
        if labels is None:
            out = logits.reshape(ids.shape[0], s, -1)
            return _exit(out) if gathered else out
        lab = C.all_gather(labels.contiguous(), 0) if gathered else labels
        loss = vocab_parallel_cross_entropy(logits, lab.reshape(-1), self.vocab_size)
        loss = loss.reshape(ids.shape[0], s)
        return _exit(loss) if gathered else loss
