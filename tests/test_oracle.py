"""Pin the CPU oracle (oracle/tp.py) against every SPEC worked example and invariant
of the tensor_parallel module (acceptance criteria 9-10 at
SPEC.md:630-631).  The reference ships no tests, so these SPEC pins are the
golden vectors for the TP rows."""
import math
import random

import pytest
import torch

from oracle import tp

D = torch.float64


def rel(a, b):
    return ((a - b).norm() / max(b.norm().item(), 1e-300)).item()


# ---------------------------------------------------------------- collectives
@pytest.mark.parametrize("kind", ["allgather", "fwd_allreduce", "bwd_allreduce", "scatter_and_merge",
                                  "reduce_scatter"])
def test_collective_T1_identity(kind):
    x = torch.randn(4, 6, dtype=D)
    out = tp.tp_collective(kind, [x], dim=0, split_dim=0, merge_dim=1)
    assert torch.equal(out[0], x)


def test_reduce_scatter_golden():
    out = tp.reduce_scatter([torch.tensor([1.0, 2.0], dtype=D), torch.tensor([3.0, 4.0], dtype=D)], 0)
    assert out[0].tolist() == [4.0] and out[1].tolist() == [6.0]


@pytest.mark.parametrize("T", [2, 4])
def test_allgather_of_reduce_scatter_is_allreduce(T):
    xs = [torch.randn(8, 3, dtype=D) for _ in range(T)]
    ag = tp.allgather(tp.reduce_scatter(xs, 0), 0)
    ar = tp.fwd_allreduce(xs)
    for a, b in zip(ag, ar):
        assert torch.allclose(a, b, rtol=0, atol=1e-14)


@pytest.mark.parametrize("T", [2, 4])
def test_scatter_and_merge_self_dual(T):
    xs = [torch.randn(2 * T, 3 * T, dtype=D) for _ in range(T)]
    back = tp.scatter_and_merge(tp.scatter_and_merge(xs, 0, 1), 1, 0)
    for a, b in zip(back, xs):
        assert torch.equal(a, b)


def test_collective_errors():
    with pytest.raises(tp.OracleError):
        tp.reduce_scatter([torch.zeros(3, dtype=D), torch.zeros(3, dtype=D)], 0)
    with pytest.raises(tp.OracleError):
        tp.fwd_allreduce([torch.zeros(3, dtype=D), torch.zeros(4, dtype=D)])


def test_ascending_rank_order_is_bit_stable():
    xs = [torch.randn(64, dtype=D) * 10 ** i for i in range(4)]
    a = tp.fwd_allreduce(xs)[0]
    b = tp.fwd_allreduce(xs)[0]
    assert torch.equal(a, b)
    assert torch.equal(a, ((xs[0] + xs[1]) + xs[2]) + xs[3])


# ---------------------------------------------------------------- DistributedLinear
def test_dist_linear_T1_exact():
    W, b, x = torch.randn(5, 4, dtype=D), torch.randn(5, dtype=D), torch.randn(3, 4, dtype=D)
    Ws, bs = tp.shard_linear(W, b, 1)
    ys, _ = tp.dist_linear_forward([x], Ws, bs)
    assert torch.equal(ys[0], x @ W.t() + b)


def test_dist_linear_identity_golden():
    W = torch.eye(2, dtype=D)
    Ws, bs = tp.shard_linear(W, torch.zeros(2, dtype=D), 2)
    ys, _ = tp.dist_linear_forward([torch.tensor([[3.0, 5.0]], dtype=D), torch.tensor([[1.0, 1.0]], dtype=D)], Ws,
                                   bs)
    assert ys[0].tolist() == [[3.0, 5.0]]


@pytest.mark.parametrize("T", [1, 2, 4])
@pytest.mark.parametrize("prescaled", [False, True])
def test_dist_linear_random(T, prescaled):  # SPEC.md:430, AC9 (<=1e-12)
    g = torch.Generator().manual_seed(T)
    for _ in range(10):
        out_f, in_f, b = random.Random(T).randint(1, 9), 4 * T, 3
        W, bias = torch.randn(out_f, in_f, generator=g, dtype=D), torch.randn(out_f, generator=g, dtype=D)
        xs = [torch.randn(b, in_f, generator=g, dtype=D) for _ in range(T)]
        if prescaled:
            xs = [xs[0]] * T
        Ws, bs = tp.shard_linear(W, bias, T)
        ys, _ = tp.dist_linear_forward(xs, Ws, bs, prescaled=prescaled)
        for i in range(T):
            assert rel(ys[i], xs[i] @ W.t() + bias) <= 1e-12


def test_dist_linear_backward_zero_and_errors():
    W = torch.randn(3, 4, dtype=D)
    Ws, bs = tp.shard_linear(W, torch.zeros(3, dtype=D), 2)
    xs = [torch.randn(2, 4, dtype=D) for _ in range(2)]
    _, saved = tp.dist_linear_forward(xs, Ws, bs)
    dxs, dWs, db = tp.dist_linear_backward([torch.zeros(2, 3, dtype=D)] * 2, Ws, saved)
    assert all(float(t.abs().max()) == 0.0 for t in dxs + dWs + [db])
    with pytest.raises(tp.OracleError):
        tp.dist_linear_backward([torch.zeros(2, 3, dtype=D)] * 2, Ws, None)


@pytest.mark.parametrize("inst", range(20))
def test_dist_linear_backward_finite_difference(inst):  # SPEC.md:439, AC10 (h=1e-5, <=1e-6)
    g = torch.Generator().manual_seed(100 + inst)
    T, b, in_f, out_f = 2, 2, 4, 3
    W = torch.randn(out_f, in_f, generator=g, dtype=D)
    bias = torch.randn(out_f, generator=g, dtype=D)
    xs = [torch.randn(b, in_f, generator=g, dtype=D) for _ in range(T)]
    cs = [torch.randn(b, out_f, generator=g, dtype=D) for _ in range(T)]  # loss = sum_i <c_i, y_i>

    def loss(W_, b_, xs_):
        Ws, bs = tp.shard_linear(W_, b_, T)
        ys, _ = tp.dist_linear_forward(xs_, Ws, bs)
        return sum((c * y).sum() for c, y in zip(cs, ys))

    Ws, bs = tp.shard_linear(W, bias, T)
    _, saved = tp.dist_linear_forward(xs, Ws, bs)
    dxs, dWs, db = tp.dist_linear_backward(cs, Ws, saved)
    dW = torch.cat(dWs, 1)
    h = 1e-5
    worst = 0.0
    for (i, j) in [(i, j) for i in range(out_f) for j in range(in_f)]:
        Wp, Wm = W.clone(), W.clone()
        Wp[i, j] += h
        Wm[i, j] -= h
        fd = (loss(Wp, bias, xs) - loss(Wm, bias, xs)) / (2 * h)
        worst = max(worst, abs(fd - dW[i, j]).item() / max(abs(fd.item()), 1e-8))
    for i in range(out_f):
        bp, bm = bias.clone(), bias.clone()
        bp[i] += h
        bm[i] -= h
        fd = (loss(W, bp, xs) - loss(W, bm, xs)) / (2 * h)
        worst = max(worst, abs(fd - db[i]).item() / max(abs(fd.item()), 1e-8))
    for r in range(T):
        for (i, j) in [(i, j) for i in range(b) for j in range(in_f)]:
            xp = [x.clone() for x in xs]
            xm = [x.clone() for x in xs]
            xp[r][i, j] += h
            xm[r][i, j] -= h
            fd = (loss(W, bias, xp) - loss(W, bias, xm)) / (2 * h)
            worst = max(worst, abs(fd - dxs[r][i, j]).item() / max(abs(fd.item()), 1e-8))
    assert worst <= 1e-6


# ---------------------------------------------------------------- DistributedEmbedding
def test_embedding_golden():
    E = torch.arange(16, dtype=D).reshape(4, 4)
    Es = list(torch.chunk(E, 2, 1))
    out = tp.dist_embedding_forward([torch.tensor([0]), torch.tensor([3])], Es)
    assert torch.equal(out[0], E[[0]]) and torch.equal(out[1], E[[3]])


def test_embedding_oob_names_position():
    E = torch.randn(4, 4, dtype=D)
    with pytest.raises(IndexError, match="position 2"):
        tp.dist_embedding_forward([torch.tensor([0, 1, 4])], [E])


@pytest.mark.parametrize("T", [1, 2, 4])
@pytest.mark.parametrize("prescaled", [False, True])
def test_embedding_random(T, prescaled):
    g = torch.Generator().manual_seed(T)
    V, Dm, b, s = 37, 8 * T, 3, 5
    E = torch.randn(V, Dm, generator=g, dtype=D)
    idxs = [torch.randint(0, V, (b, s), generator=g) for _ in range(T)]
    if prescaled:
        idxs = [idxs[0]] * T
    out = tp.dist_embedding_forward(idxs, list(torch.chunk(E, T, 1)), prescaled)
    for i in range(T):
        assert rel(out[i], E[idxs[i]]) <= 1e-12


# ---------------------------------------------------------------- LayerNorm
def test_layernorm_constant_is_zero():
    xs = [torch.full((3, 4), 2.5, dtype=D), torch.full((3, 4), 2.5, dtype=D)]
    out = tp.dist_layernorm_forward(xs, None, None, 1e-5)
    assert all(float(o.abs().max()) == 0.0 for o in out)


def test_layernorm_8_channels():
    x = torch.randn(5, 8, dtype=D)
    w, b = torch.randn(8, dtype=D), torch.randn(8, dtype=D)
    out = tp.dist_layernorm_forward(list(torch.chunk(x, 2, 1)), list(torch.chunk(w, 2)), list(torch.chunk(b, 2)),
                                    1e-5)
    assert rel(torch.cat(out, 1), tp.layer_norm(x, w, b, 1e-5)) <= 1e-12


# ---------------------------------------------------------------- attention / MLP / layer
def _cfg(T, causal=False, pre=False, post=True, act="gelu", optimize="speed", nh=None):
    nh = nh or 2 * T
    return tp.LayerConfig(num_attention_heads=nh, attention_head_size=4, hidden_size=4 * nh,
                          intermediate_size=8 * T, activation=act, causal_mask_size=(8 if causal else None),
                          pre_layernorm=pre, post_layernorm=post, optimize=optimize)


def _inputs(cfg, T, b=2, s=5, seed=0, prescaled=False):
    g = torch.Generator().manual_seed(seed)
    xs = [torch.randn(b, s, cfg.hidden_size, generator=g, dtype=D) for _ in range(T)]
    if prescaled:
        xs = [xs[0]] * T
    return xs


@pytest.mark.parametrize("T", [1, 2, 4])
@pytest.mark.parametrize("optimize", ["speed", "memory"])
@pytest.mark.parametrize("prescaled", [False, True])
def test_attention_matches_reference(T, optimize, prescaled):  # SPEC.md:464, AC9 (<=1e-10)
    for trial, (causal, pre, post) in enumerate([(False, False, True), (True, True, False), (True, True, True)]):
        cfg = _cfg(T, causal, pre, post, optimize=optimize)
        p = tp.init_layer_params(cfg, seed=trial)
        xs = _inputs(cfg, T, seed=trial, prescaled=prescaled)
        mask = torch.zeros(sum(x.shape[0] for x in (xs if not prescaled else xs[:1])), 5, dtype=D)
        mask[0, -1] = -10000.0
        out = tp.dist_attention_forward(xs, p, cfg, mask, prescaled)
        X = xs[0] if prescaled else torch.cat(xs, 0)
        ref = tp.attention_layer_ref(X, p, cfg, mask)
        got = out[0] if prescaled else torch.cat(out, 0)
        assert rel(got, ref) <= 1e-10


@pytest.mark.parametrize("T", [2, 4])
def test_attention_speed_vs_memory(T):
    for pre in (False, True):
        cs, cm = _cfg(T, pre=pre, optimize="speed"), _cfg(T, pre=pre, optimize="memory")
        p = tp.init_layer_params(cs, seed=3)
        xs = _inputs(cs, T, seed=4)
        a = torch.cat(tp.dist_attention_forward(xs, p, cs), 0)
        b = torch.cat(tp.dist_attention_forward(xs, p, cm), 0)
        assert rel(a, b) <= 1e-10


def test_attention_causal_perturbation():
    cfg = _cfg(2, causal=True, pre=True, post=False)
    p = tp.init_layer_params(cfg, seed=5)
    xs = _inputs(cfg, 2, s=6, seed=6)
    base = tp.dist_attention_forward(xs, p, cfg)
    t = 3
    xs2 = [x.clone() for x in xs]
    for x in xs2:
        x[:, t + 1:] += torch.randn_like(x[:, t + 1:])
    pert = tp.dist_attention_forward(xs2, p, cfg)
    for a, b in zip(base, pert):
        assert torch.equal(a[:, :t + 1], b[:, :t + 1])


@pytest.mark.parametrize("T", [1, 2, 4])
@pytest.mark.parametrize("optimize", ["speed", "memory"])
def test_mlp_matches_reference(T, optimize):
    cfg = _cfg(T, optimize=optimize)
    p = tp.init_layer_params(cfg, seed=7)
    xs = _inputs(cfg, T, seed=8)
    out = tp.dist_mlp_forward(xs, p, cfg)
    assert rel(torch.cat(out, 0), tp.mlp_layer_ref(torch.cat(xs, 0), p, cfg)) <= 1e-10


def test_mlp_relu_zero_pattern():
    T = 2
    cfg = _cfg(T, act="relu")
    p = tp.init_layer_params(cfg, seed=9)
    X = torch.cat(_inputs(cfg, T, seed=10), 0)
    z_full = X @ p["w1"].t() + p["b1"]
    shards = tp.shard_layer_params_speed(p, cfg, T)
    z_loc = torch.cat([tp.activation("relu", X @ s["w1"].t() + s["b1"]) for s in shards], -1)
    assert torch.equal(z_loc == 0, z_full <= 0)
    assert (z_full < 0).any()


@pytest.mark.parametrize("T", [1, 2, 4])
@pytest.mark.parametrize("optimize", ["speed", "memory"])
def test_layer_matches_reference(T, optimize):  # SPEC.md:482-483 (<=1e-9)
    for pre, post in [(True, False), (False, True), (True, True)]:
        cfg = _cfg(T, causal=pre, pre=pre, post=post, optimize=optimize)
        p = tp.init_layer_params(cfg, seed=11)
        xs = _inputs(cfg, T, seed=12)
        out = tp.dist_transformer_layer_forward(xs, p, cfg)
        assert rel(torch.cat(out, 0), tp.transformer_layer_ref(torch.cat(xs, 0), p, cfg)) <= 1e-9


def test_layer_post_ln_toggle_changes_output():
    a, b = _cfg(2, post=True), _cfg(2, post=False)
    p = tp.init_layer_params(a, seed=13)
    xs = _inputs(a, 2, seed=14)
    assert not torch.allclose(torch.cat(tp.dist_transformer_layer_forward(xs, p, a), 0),
                              torch.cat(tp.dist_transformer_layer_forward(xs, p, b), 0))


def test_batch_semantics_invariant():
    cfg = _cfg(2)
    p = tp.init_layer_params(cfg, seed=15)
    xs = _inputs(cfg, 2, seed=16)
    base = tp.dist_transformer_layer_forward(xs, p, cfg)
    xs2 = [xs[0], xs[1] + 1.0]
    pert = tp.dist_transformer_layer_forward(xs2, p, cfg)
    assert torch.equal(base[0], pert[0])
    assert not torch.equal(base[1], pert[1])


def test_dropout_invariant_to_T():
    """Logical-coordinate masks: TP=1 and TP=4 layers agree with dropout on."""
    outs = []
    for T in (1, 2, 4):
        cfg = _cfg(4, causal=True, pre=True, post=False)
        cfg.attention_dropout_prob = cfg.hidden_dropout_prob = 0.25
        p = tp.init_layer_params(cfg, seed=17)
        X = _inputs(cfg, 1, b=4, seed=18)[0]
        xs = list(torch.chunk(X, T, 0))
        o = tp.dist_transformer_layer_forward(xs, p, cfg, dctx=tp.DropoutCtx(seed=99, layer=3))
        outs.append(torch.cat(o, 0))
    assert rel(outs[1], outs[0]) <= 1e-12 and rel(outs[2], outs[0]) <= 1e-12


# ---------------------------------------------------------------- vocab-parallel CE / embedding
@pytest.mark.parametrize("T", [1, 2, 4, 8])
def test_vocab_parallel_ce(T):
    g = torch.Generator().manual_seed(T)
    V, N = 1000, 37
    Vp = tp.vocab_padded(V, T, 16)
    logits = torch.randn(N, Vp, generator=g, dtype=D) * 3
    tgt = torch.randint(0, V, (N,), generator=g)
    tgt[3] = -100
    shards = list(torch.chunk(logits, T, 1))
    loss, stats = tp.vocab_parallel_ce_forward(shards, tgt, V)
    assert rel(loss, tp.cross_entropy_ref(logits, tgt, V)) <= 1e-12
    gl = torch.randn(N, generator=g, dtype=D)
    grads = tp.vocab_parallel_ce_backward(shards, tgt, V, stats, gl)
    lg = logits.clone().requires_grad_(True)
    (tp.cross_entropy_ref(lg, tgt, V) * gl).sum().backward()
    assert rel(torch.cat(grads, 1), lg.grad) <= 1e-12


@pytest.mark.parametrize("T", [1, 2, 4])
@pytest.mark.parametrize("prescaled", [True, False])
def test_vocab_parallel_embedding(T, prescaled):
    g = torch.Generator().manual_seed(T)
    V, Dm = 50, 6
    Vp = tp.vocab_padded(V, T, 4)
    E = torch.randn(Vp, Dm, generator=g, dtype=D)
    idxs = [torch.randint(0, V, (3, 4), generator=g) for _ in range(T)]
    if prescaled:
        idxs = [idxs[0]] * T
    out = tp.vocab_embedding_forward(idxs, list(torch.chunk(E, T, 0)), prescaled)
    if prescaled:
        assert rel(out[0], E[idxs[0]]) <= 1e-12
    else:
        for i in range(T):
            assert rel(out[i], E[idxs[i]]) <= 1e-12
    owner, local = tp.vocab_owner(torch.tensor([0, Vp // T - 1, Vp // T, Vp - 1]), Vp, T)
    assert owner.tolist() == [0, 0, min(1, T - 1) if T > 1 else 1, T - 1] or T == 1
    assert (local >= 0).all() and (local < Vp // T).all()


# ---------------------------------------------------------------- plan_replacement
class _Mod:
    def __init__(self, id, parent, params=(), kind=None):
        self.id, self.parent, self.param_ids, self.kind = id, parent, tuple(params), kind


class _Spec:
    def __init__(self, mods):
        self.modules = mods
        self._by = {m.id: m for m in mods}
        self._kids = {m.id: [] for m in mods}
        for m in mods:
            if m.parent:
                self._kids[m.parent].append(m.id)
        self.root_id = next(m.id for m in mods if m.parent is None)

    def module(self, i):
        return self._by[i]

    def children(self, i):
        return self._kids[i]

    def subtree(self, i):
        out, st = [], [i]
        while st:
            c = st.pop()
            out.append(c)
            st.extend(reversed(self._kids[c]))
        return out


def test_plan_replacement_examples():
    reg = {"transformer": "DistributedTransformer", "linear": "DistributedLinear"}
    spec = _Spec([_Mod("root", None), _Mod("tr", "root", ["p1"], "transformer"), _Mod("lin", "tr", ["p2"], "linear")])
    assert tp.plan_replacement(spec, reg, {"tr"}) == {"tr"}  # parent and child registered -> parent only
    spec2 = _Spec([_Mod("root", None), _Mod("a", "root", ["w"], "linear"), _Mod("b", "root", ["w"], "linear")])
    assert tp.plan_replacement(spec2, reg, {"root"}) == set()  # shares a param with a sibling
    spec3 = _Spec([_Mod("root", None), _Mod("a", "root", ["w"], "linear")])
    assert tp.plan_replacement(spec3, reg, set()) == set()  # registered but not enabled
    assert tp.plan_replacement(spec3, reg, {"a"}) == {"a"}
