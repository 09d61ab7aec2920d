"""Multi-GPU TP parity check, one process per GPU (torchrun --nproc-per-node T).

Every rank builds smp.nn layers at tensor_parallel_degree = T (speed mode), loads
the shards of the same full parameters, runs forward + backward on its own
samples (TP across DP ranks) or on the shared batch (prescaled), and rank 0
compares every rank's outputs and gradient shards against the fp64 CPU oracle
(oracle/tp.py) on the whole batch.  Exit code 0 = parity holds.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tests/mp_tp_check.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import tp  # noqa: E402

TOL = 2e-2


def rel(a, b):
    a, b = a.double().cpu(), b.double().cpu()
    return ((a - b).norm() / max(b.norm().item(), 1e-30)).item()


def gather_cpu(t):
    T = dist.get_world_size()
    out = [torch.empty_like(t) for _ in range(T)]
    dist.all_gather(out, t.contiguous())
    return [o.cpu() for o in out]


def run_case(smp, name, *, prescaled, causal, pre, post, p, layers=1, act="gelu"):
    T, rank = dist.get_world_size(), dist.get_rank()
    smp.init({"tensor_parallel_degree": T, "optimize": "speed", "_prescaled_batch": prescaled, "seed": 11})
    nh, dh, I, s, B = 2 * T, 64, 512 * T, 128, 2
    H = nh * dh
    cfg = tp.LayerConfig(num_attention_heads=nh, attention_head_size=dh, hidden_size=H, intermediate_size=I,
                         attention_dropout_prob=p, hidden_dropout_prob=p, activation=act,
                         causal_mask_size=(s if causal else None), pre_layernorm=pre, post_layernorm=post)
    params = [{k: v.to(torch.bfloat16).double() for k, v in tp.init_layer_params(cfg, seed=3 + l).items()}
              for l in range(layers)]
    g = torch.Generator().manual_seed(5)
    n_samples = B if prescaled else B * T
    X = torch.randn(n_samples, s, H, generator=g).to(torch.bfloat16)
    DY = torch.randn(n_samples, s, H, generator=g).to(torch.bfloat16)
    mask = torch.zeros(n_samples, s)
    if not causal:
        mask[0, -5:] = -10000.0
    if prescaled:
        x, dy, m = X, DY, mask
    else:
        x, dy, m = X[rank * B:(rank + 1) * B], DY[rank * B:(rank + 1) * B], mask[rank * B:(rank + 1) * B]

    kw = dict(num_attention_heads=nh, attention_head_size=dh, hidden_size=H, intermediate_size=I,
              attention_dropout_prob=p, hidden_dropout_prob=p, activation=act,
              causal_mask_size=(s if causal else None), pre_layernorm=pre, post_layernorm=post)
    if layers == 1:
        mod = smp.nn.DistributedTransformerLayer(layer_id=0, **kw)
        mod.load_full({k: v.to(torch.bfloat16) for k, v in params[0].items()})
        lays = [mod]
    else:
        mod = smp.nn.DistributedTransformer(num_layers=layers, **kw)
        for l, lay in enumerate(mod.seq_layers):
            lay.load_full({k: v.to(torch.bfloat16) for k, v in params[l].items()})
        lays = list(mod.seq_layers)
    xg = x.cuda().requires_grad_(True)
    y = mod(xg, None if causal else m.cuda())
    y.backward(dy.cuda())

    ys, dxs = gather_cpu(y.detach()), gather_cpu(xg.grad)
    shard_grads = []
    for lay in lays:
        a, o = lay.attention, lay.output
        shard_grads.append({k: gather_cpu(t.grad) for k, t in {
            "qkv_w": a.qkv_weight, "qkv_b": a.qkv_bias, "wo": a.dense_weight, "bo": a.dense_bias,
            "w1": o.fc1_weight, "b1": o.fc1_bias, "w2": o.fc2_weight, "b2": o.fc2_bias}.items()})
    ok = True
    if rank == 0:
        xr = X.double().requires_grad_(True)
        pr = [{k: v.clone().requires_grad_(True) for k, v in pl.items()} for pl in params]
        yr = xr
        for l in range(layers):
            yr = tp.transformer_layer_ref(yr, pr[l], cfg, None if causal else mask.double(),
                                          tp.DropoutCtx(seed=11, layer=l, sample_offset=0))
        yr.backward(DY.double())
        errs = {}
        if prescaled:
            errs["y"] = max(rel(yy, yr) for yy in ys)
            errs["dx"] = max(rel(d, xr.grad) for d in dxs)
        else:
            errs["y"] = rel(torch.cat(ys, 0), yr)
            errs["dx"] = rel(torch.cat(dxs, 0), xr.grad)
        hs, ins = H // T, I // T
        for l in range(layers):
            gr = pr[l]
            wq, wk, wv = gr["wqkv"].grad.split(H, 0)
            bq, bk, bv = gr["bqkv"].grad.split(H, 0)
            sg = shard_grads[l]
            for j in range(T):
                sl = slice(j * hs, (j + 1) * hs)
                isl = slice(j * ins, (j + 1) * ins)
                e = {
                    "qkv_w": rel(sg["qkv_w"][j], torch.cat([wq[sl], wk[sl], wv[sl]], 0)),
                    "qkv_b": rel(sg["qkv_b"][j], torch.cat([bq[sl], bk[sl], bv[sl]], 0)),
                    "wo": rel(sg["wo"][j], gr["wo"].grad[:, sl]),
                    "bo": rel(sg["bo"][j], gr["bo"].grad),
                    "w1": rel(sg["w1"][j], gr["w1"].grad[isl]),
                    "b1": rel(sg["b1"][j], gr["b1"].grad[isl]),
                    "w2": rel(sg["w2"][j], gr["w2"].grad[:, isl]),
                    "b2": rel(sg["b2"][j], gr["b2"].grad),
                }
                for k, v in e.items():
                    errs[f"L{l}.r{j}.{k}"] = v
        bad = {k: v for k, v in errs.items() if not v < TOL}
        ok = not bad
        print(f"[{name}] T={T} {'OK' if ok else 'FAIL'} max_err={max(errs.values()):.3e} "
              f"y={errs['y']:.2e} dx={errs['dx']:.2e} {bad if bad else ''}", flush=True)
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.broadcast(flag, 0)
    smp.reset()
    return bool(flag.item())


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2111_05972_b200 as smp
    results = [
        run_case(smp, "tp_across_dp_post_ln", prescaled=False, causal=False, pre=False, post=True, p=0.0),
        run_case(smp, "prescaled_pre_ln_causal", prescaled=True, causal=True, pre=True, post=False, p=0.0),
        run_case(smp, "tp_across_dp_dropout", prescaled=False, causal=True, pre=True, post=False, p=0.1),
        run_case(smp, "stack2_both_ln", prescaled=False, causal=False, pre=True, post=True, p=0.1, layers=2),
    ]
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if all(results) else 1)


if __name__ == "__main__":
    main()
