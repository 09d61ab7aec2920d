"""Pipeline stage send/recv + scheduler on 2 GPUs (torchrun --nproc-per-node 2).

1. StageChannel stress: 11 messages through a 3-slot ring (flow control wraps), both
   directions, payload checked bit-exactly.
2. PP=2 x TP=1 training step of a 4-layer DistributedTransformer split 2+2 with 4
   microbatches under the simple and interleaved policies: per-microbatch losses and every
   parameter gradient vs the fp64 CPU oracle run on the whole model.
Exit code 0 = all checks pass.
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


def channel_stress(rank):
    from paper_2111_05972_b200.pipeline import StageChannel
    ok = True
    shape = (3, 1000)
    fwd = StageChannel(0, 1, 3 * 1000 * 2, slots=3)
    bwd = StageChannel(1, 0, 3 * 1000 * 2, slots=3)
    n = 11
    if rank == 0:
        for i in range(n):
            fwd.send(torch.full(shape, float(i), dtype=torch.bfloat16, device="cuda"))
        got = [bwd.recv(torch.empty(shape, dtype=torch.bfloat16, device="cuda")).clone() for _ in range(n)]
    else:
        got = [fwd.recv(torch.empty(shape, dtype=torch.bfloat16, device="cuda")).clone() for _ in range(n)]
        for i in range(n):
            bwd.send(torch.full(shape, float(100 + i), dtype=torch.bfloat16, device="cuda"))
    torch.cuda.synchronize()
    base = 0 if rank == 1 else 100
    for i, g in enumerate(got):
        ok &= bool((g == base + i).all())
    fwd.close()
    bwd.close()
    print(f"[channel] rank {rank} {'OK' if ok else 'FAIL'}", flush=True)
    return ok


def reference_log(kind, M, P=2):
    """The reference run_step's decision log for a P-stage uniform chain (tests/golden)."""
    import json
    gold = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                                       "reference_golden.json")))["run_step_logs"]
    return [c for c in gold if (c["P"], c["M"], c["kind"], c["forward_only"], c["uniform"]) ==
            (P, M, kind, False, True)][0]["decision_log"]


def pp_step(smp, rank, policy_kind, replay=False):
    from paper_2111_05972_b200.pipeline import PipelineEngine, SchedulePolicy
    smp.init({"tensor_parallel_degree": 1, "pipeline_parallel_degree": 2, "optimize": "speed", "seed": 0})
    L, nh, dh, H, I, s, mb, M = 4, 4, 64, 256, 1024, 128, 2, 4
    cfg = tp.LayerConfig(num_attention_heads=nh, attention_head_size=dh, hidden_size=H, intermediate_size=I,
                         activation="gelu_tanh", causal_mask_size=s, pre_layernorm=True, post_layernorm=False)
    params = [{k: v.to(torch.bfloat16).double() for k, v in tp.init_layer_params(cfg, seed=40 + l).items()}
              for l in range(L)]
    g = torch.Generator().manual_seed(1)
    X = [torch.randn(mb, s, H, generator=g).to(torch.bfloat16) for _ in range(M)]
    Tg = [torch.randn(mb, s, H, generator=g).to(torch.bfloat16) for _ in range(M)]
    stage = smp.nn.DistributedTransformer(num_layers=2, num_attention_heads=nh, attention_head_size=dh,
                                          hidden_size=H, intermediate_size=I, attention_dropout_prob=0.0,
                                          hidden_dropout_prob=0.0, activation="gelu_tanh", causal_mask_size=s,
                                          pre_layernorm=True, post_layernorm=False)
    for j, lay in enumerate(stage.seq_layers):
        lay.load_full({k: v.to(torch.bfloat16) for k, v in params[2 * rank + j].items()})
    ref_log = reference_log(policy_kind, M) if replay else None
    eng = PipelineEngine(stage, pp_rank=rank, pp_size=2, ranks=[0, 1], act_shape=(mb, s, H),
                         policy=SchedulePolicy(policy_kind, M), decision_log=ref_log)
    if replay:  # the engine's decisions are the reference runtime's, action for action
        assert [tuple(e["action"]) for e in eng.log] == [tuple(e["action"]) for e in ref_log]
    inputs = [x.cuda() for x in X] if rank == 0 else None
    tg = [t.cuda() for t in Tg]
    losses = eng.step(inputs, loss_fn=lambda m, y: (y.float() * tg[m].float()).sum())
    torch.cuda.synchronize()
    grads = {}
    for j, lay in enumerate(stage.seq_layers):
        grads[2 * rank + j] = (lay.attention.qkv_weight.grad.cpu(), lay.output.fc2_weight.grad.cpu())
    all_grads = [None, None]
    dist.all_gather_object(all_grads, grads)
    loss_vals = [None, None]
    dist.all_gather_object(loss_vals, [float(l) for l in losses] if losses else None)
    ok = True
    if rank == 0:
        pr = [{k: v.clone().requires_grad_(True) for k, v in p.items()} for p in params]
        ref_losses = []
        for m in range(M):
            h = X[m].double()
            for l in range(L):
                h = tp.transformer_layer_ref(h, pr[l], cfg, None, None)
            lm = (h * Tg[m].double()).sum()
            lm.backward()
            ref_losses.append(lm.item())
        errs = {"loss": max(abs(a - b) / abs(b) for a, b in zip(loss_vals[1], ref_losses))}
        merged = {**all_grads[0], **all_grads[1]}
        for l in range(L):
            wq, wk, wv = pr[l]["wqkv"].grad.split(H, 0)
            errs[f"L{l}.qkv"] = rel(merged[l][0], torch.cat([wq, wk, wv], 0))
            errs[f"L{l}.fc2"] = rel(merged[l][1], pr[l]["w2"].grad)
        bad = {k: v for k, v in errs.items() if not v < TOL}
        ok = not bad
        print(f"[pp2_{policy_kind}{'_replay_reference_log' if replay else ''}] {'OK' if ok else 'FAIL'} schedule={[tuple(e['action']) for e in eng.log]} "
              + " ".join(f"{k}={v:.2e}" for k, v in errs.items()), flush=True)
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.broadcast(flag, 0)
    smp.reset()
    return bool(flag.item())


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2111_05972_b200 as smp
    rank = dist.get_rank()
    res = [channel_stress(rank)]
    res_t = torch.tensor([1 if all(res) else 0], device="cuda")
    dist.all_reduce(res_t, op=dist.ReduceOp.MIN)
    res = [bool(res_t.item())]
    res.append(pp_step(smp, rank, "simple"))
    res.append(pp_step(smp, rank, "interleaved"))
    res.append(pp_step(smp, rank, "interleaved", replay=True))
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if all(res) else 1)


if __name__ == "__main__":
    main()
