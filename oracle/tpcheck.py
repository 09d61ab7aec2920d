"""tpcheck — the SPEC's tensor-parallel invariant suite as a CLI ("External
Interfaces": runs the oracle suite and emits a JSON report {op, T, shape, max_rel_err, pass};
SPEC.md:596-603 cmd_tpcheck: exit 5 on any tolerance violation).  TEST INFRASTRUCTURE (oracle/).

    python -m oracle.tpcheck [--T 1,2,4] [--out report.json] [--gpu] [--inject-fault]

Oracle mode: every distributed op (collectives' AG∘RS == AR, dist_linear fwd/bwd,
dist_embedding, dist_layernorm, attention / MLP / layer in speed and memory mode,
vocab-parallel CE) on T simulated ranks against its single-rank reference, with the SPEC
tolerances (1e-12 linear/embedding/LN, 1e-10 attention/MLP, 1e-9 layer).  --gpu also runs the
sm_100a kernels (libsmpk via smp.nn at T = 1) on the same inputs against the fp64 oracle with
the bf16 tolerances of SURVEY.md §8c (2e-2 per layer).  --inject-fault perturbs one rank's
shard (negative control: the report must fail and the exit code be 5).
"""
from __future__ import annotations

import argparse
import json
import sys

import torch

from . import tp

D = torch.float64


def _rel(a, b) -> float:
    return ((a - b).norm() / max(b.norm().item(), 1e-300)).item()


def _cfg(T, optimize="speed", causal=False, pre=False, post=True, act="gelu"):
    nh = 2 * T
    return tp.LayerConfig(num_attention_heads=nh, attention_head_size=4, hidden_size=4 * nh,
                          intermediate_size=8 * T, activation=act, causal_mask_size=(8 if causal else None),
                          pre_layernorm=pre, post_layernorm=post, optimize=optimize)


def _xs(cfg, T, b=2, s=5, seed=0):
    g = torch.Generator().manual_seed(seed)
    return [torch.randn(b, s, cfg.hidden_size, generator=g, dtype=D) for _ in range(T)]


def oracle_suite(Ts, fault: bool) -> list:
    rep = []

    def add(op, T, shape, err, tol):
        rep.append({"op": op, "T": T, "shape": list(shape), "max_rel_err": err, "tol": tol, "pass": err <= tol})

    for T in Ts:
        g = torch.Generator().manual_seed(100 + T)
        # collectives: AG∘RS == AR, scatter_and_merge self-dual (:497)
        xs = [torch.randn(4 * T, 3, generator=g, dtype=D) for _ in range(T)]
        ar = tp.fwd_allreduce(xs)
        agrs = tp.allgather(tp.reduce_scatter(xs, 0), 0)
        add("allgather(reduce_scatter)==allreduce", T, xs[0].shape, max(_rel(a, b) for a, b in zip(agrs, ar)), 1e-12)
        back = tp.scatter_and_merge(tp.scatter_and_merge(xs, 0, 1), 1, 0)
        add("scatter_and_merge self-dual", T, xs[0].shape, max(_rel(a, b) for a, b in zip(back, xs)), 0.0)
        # DistributedLinear forward / backward
        W, bias = torch.randn(5, 4 * T, generator=g, dtype=D), torch.randn(5, generator=g, dtype=D)
        Ws, bs = tp.shard_linear(W, bias, T)
        if fault:
            Ws[-1] = Ws[-1] + 1e-3
        x = [torch.randn(3, 4 * T, generator=g, dtype=D) for _ in range(T)]
        ys, saved = tp.dist_linear_forward(x, Ws, bs)
        add("dist_linear_forward", T, (3, 4 * T, 5), max(_rel(ys[i], x[i] @ W.t() + bias) for i in range(T)), 1e-12)
        dys = [torch.randn(3, 5, generator=g, dtype=D) for _ in range(T)]
        dxs, dWs, db = tp.dist_linear_backward(dys, Ws, saved)
        dY, X = torch.cat(dys, 0), torch.cat(x, 0)
        err = max(max(_rel(dxs[i], dys[i] @ W) for i in range(T)), _rel(torch.cat(dWs, 1), dY.t() @ X),
                  _rel(db, dY.sum(0)))
        add("dist_linear_backward", T, (3, 4 * T, 5), err, 1e-10)
        # DistributedEmbedding (dim-sharded)
        V = 37
        E = torch.randn(V, 8 * T, generator=g, dtype=D)
        idx = [torch.randint(0, V, (2, 5), generator=g) for _ in range(T)]
        out = tp.dist_embedding_forward(idx, list(torch.chunk(E, T, 1)))
        add("dist_embedding_forward", T, (V, 8 * T), max(_rel(out[i], E[idx[i]]) for i in range(T)), 1e-12)
        # distributed LayerNorm
        xl = torch.randn(6, 8 * T, generator=g, dtype=D)
        w, b = torch.randn(8 * T, generator=g, dtype=D), torch.randn(8 * T, generator=g, dtype=D)
        o = tp.dist_layernorm_forward(list(torch.chunk(xl, T, 1)), list(torch.chunk(w, T)), list(torch.chunk(b, T)),
                                      1e-5)
        add("dist_layernorm_forward", T, xl.shape, _rel(torch.cat(o, 1), tp.layer_norm(xl, w, b, 1e-5)), 1e-12)
        # attention / MLP / layer, both modes
        for optimize in ("speed", "memory"):
            cfg = _cfg(T, optimize=optimize, causal=True, pre=True, post=True)
            p = tp.init_layer_params(cfg, seed=T)
            xs_ = _xs(cfg, T, seed=T)
            X = torch.cat(xs_, 0)
            att = torch.cat(tp.dist_attention_forward(xs_, p, cfg), 0)
            add(f"dist_attention_forward[{optimize}]", T, X.shape, _rel(att, tp.attention_layer_ref(X, p, cfg)), 1e-10)
            mlp = torch.cat(tp.dist_mlp_forward(xs_, p, cfg), 0)
            add(f"dist_mlp_forward[{optimize}]", T, X.shape, _rel(mlp, tp.mlp_layer_ref(X, p, cfg)), 1e-10)
            lay = torch.cat(tp.dist_transformer_layer_forward(xs_, p, cfg), 0)
            add(f"dist_transformer_layer_forward[{optimize}]", T, X.shape,
                _rel(lay, tp.transformer_layer_ref(X, p, cfg)), 1e-9)
        # vocab-parallel cross-entropy
        Vv = 29
        Vp = tp.vocab_padded(Vv, T, multiple=4)
        logits = torch.randn(7, Vp, generator=g, dtype=D)
        logits[:, Vv:] = float("-inf")
        tgt = torch.randint(0, Vv, (7,), generator=g)
        loss, _ = tp.vocab_parallel_ce_forward(list(torch.chunk(logits, T, 1)), tgt, Vv)
        add("vocab_parallel_ce_forward", T, (7, Vp), _rel(loss, tp.cross_entropy_ref(logits[:, :Vv], tgt, Vv)), 1e-12)
    return rep


def gpu_suite() -> list:
    """smp.nn at T = 1 on the GPU vs the fp64 oracle (bf16 tolerances)."""
    import paper_2111_05972_b200 as smp
    rep = []
    smp.init({"tensor_parallel_degree": 1, "optimize": "speed", "seed": 5})
    try:
        for name, (nh, dh, H, I, s, causal, pre, post, act) in {
                "bert_like_post_ln": (4, 64, 256, 1024, 128, False, False, True, "gelu"),
                "gpt_like_pre_ln": (4, 64, 256, 1024, 128, True, True, False, "gelu_tanh")}.items():
            cfg = tp.LayerConfig(num_attention_heads=nh, attention_head_size=dh, hidden_size=H, intermediate_size=I,
                                 activation=act, causal_mask_size=(s if causal else None), pre_layernorm=pre,
                                 post_layernorm=post)
            p = {k: v.to(torch.bfloat16).double() for k, v in tp.init_layer_params(cfg, seed=1).items()}
            g = torch.Generator().manual_seed(0)
            x = torch.randn(2, s, H, generator=g).to(torch.bfloat16)
            dy = torch.randn(2, s, H, generator=g).to(torch.bfloat16)
            layer = smp.nn.DistributedTransformerLayer(
                num_attention_heads=nh, attention_head_size=dh, hidden_size=H, intermediate_size=I,
                attention_dropout_prob=0.0, hidden_dropout_prob=0.0, activation=act,
                causal_mask_size=(s if causal else None), pre_layernorm=pre, post_layernorm=post, layer_id=0)
            layer.load_full({k: v.to(torch.bfloat16) for k, v in p.items()})
            xg = x.cuda().requires_grad_(True)
            y = layer(xg)
            y.backward(dy.cuda())
            xr = x.double().requires_grad_(True)
            yr = tp.transformer_layer_ref(xr, p, cfg)
            yr.backward(dy.double())
            err = max(_rel(y.detach().double().cpu(), yr.detach()), _rel(xg.grad.double().cpu(), xr.grad))
            rep.append({"op": f"gpu:DistributedTransformerLayer[{name}]", "T": 1, "shape": [2, s, H],
                        "max_rel_err": err, "tol": 2e-2, "pass": err <= 2e-2})
    finally:
        smp.reset()
    return rep


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="tpcheck", description=__doc__.split("\n\n")[0])
    ap.add_argument("--T", default="1,2,4", help="comma-separated TP degrees")
    ap.add_argument("--out", default="", help="write the JSON report here (default: stdout)")
    ap.add_argument("--gpu", action="store_true", help="also check the sm_100a kernels against the oracle")
    ap.add_argument("--inject-fault", action="store_true", help="negative control: perturb one rank's shard")
    a = ap.parse_args(argv)
    Ts = [int(t) for t in a.T.split(",") if t]
    rep = oracle_suite(Ts, a.inject_fault)
    if a.gpu:
        rep += gpu_suite()
    text = json.dumps(rep, indent=1)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)
    else:
        print(text)
    return 0 if all(r["pass"] for r in rep) else 5


if __name__ == "__main__":
    sys.exit(main())
