"""TP x PP training step on 4 GPUs (torchrun --nproc-per-node 4): BASELINE.json configs[0].

2-layer GPT-style transformer (hidden 256, 4 heads, seq 128, causal, pre-LN, gelu_tanh),
tensor_parallel_degree 2 x pipeline_parallel_degree 2 ("cluster" placement: ranks {0,1} are
stage 0's TP group, {2,3} stage 1's; each tp_rank drives its own chain 0->2 / 1->3), 4
microbatches of 2 sequences per TP rank (TP across DP), simple and interleaved schedules.
The stages exchange activations / gradients over the D2D StageChannels (side streams) while
their TP layers exchange over NVLink peer memory.  Rank 0 checks the per-microbatch losses and
every rank's QKV / FC2 weight-gradient shards against the fp64 oracle run on the whole model
and batch.  Exit code 0 = parity holds.
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


def step(smp, policy_kind):
    from paper_2111_05972_b200.pipeline import PipelineEngine, SchedulePolicy
    st = smp.init({"tensor_parallel_degree": 2, "pipeline_parallel_degree": 2, "optimize": "speed", "seed": 0,
                   "symm_pool_bytes": 256 << 20})
    T, P = 2, 2
    rank, pr, tr = dist.get_rank(), st.pp_rank, st.tp_rank
    L, nh, dh, H, I, s, b, M = 2, 4, 64, 256, 1024, 128, 2, 4
    cfg = tp.LayerConfig(num_attention_heads=nh, attention_head_size=dh, hidden_size=H, intermediate_size=I,
                         activation="gelu_tanh", causal_mask_size=s, pre_layernorm=True, post_layernorm=False)
    params = [{k: v.to(torch.bfloat16).double() for k, v in tp.init_layer_params(cfg, seed=60 + l).items()}
              for l in range(L)]
    g = torch.Generator().manual_seed(2)
    X = [torch.randn(T * b, s, H, generator=g).to(torch.bfloat16) for _ in range(M)]
    Tg = [torch.randn(T * b, s, H, generator=g).to(torch.bfloat16) for _ in range(M)]
    stage = smp.nn.DistributedTransformer(num_layers=1, num_attention_heads=nh, attention_head_size=dh,
                                          hidden_size=H, intermediate_size=I, attention_dropout_prob=0.0,
                                          hidden_dropout_prob=0.0, activation="gelu_tanh", causal_mask_size=s,
                                          pre_layernorm=True, post_layernorm=False)
    stage.seq_layers[0].load_full({k: v.to(torch.bfloat16) for k, v in params[pr].items()})
    eng = PipelineEngine(stage, pp_rank=pr, pp_size=P, ranks=st.pp_group_ranks, act_shape=(b, s, H),
                         policy=SchedulePolicy(policy_kind, M), group=st.pp_group)
    rows = slice(tr * b, (tr + 1) * b)  # this TP rank's samples of every microbatch
    inputs = [x[rows].cuda() for x in X] if pr == 0 else None
    tg = [t[rows].cuda() for t in Tg]
    losses = eng.step(inputs, loss_fn=lambda m, y: (y.float() * tg[m].float()).sum())
    torch.cuda.synchronize()
    lay = stage.seq_layers[0]
    mine = {"pp": pr, "tp": tr, "qkv": lay.attention.qkv_weight.grad.cpu(), "fc2": lay.output.fc2_weight.grad.cpu(),
            "losses": [float(v) for v in losses] if losses else None}
    allg = [None] * dist.get_world_size()
    dist.all_gather_object(allg, mine)
    ok = True
    if rank == 0:
        pr_ = [{k: v.clone().requires_grad_(True) for k, v in p.items()} for p in params]
        ref = []
        for m in range(M):
            h = X[m].double()
            for l in range(L):
                h = tp.transformer_layer_ref(h, pr_[l], cfg, None, None)
            lm = (h * Tg[m].double()).sum()
            lm.backward()
            ref.append(lm.item())
        last = [e for e in allg if e["pp"] == P - 1]
        got = [sum(e["losses"][m] for e in last) for m in range(M)]
        errs = {"loss": max(abs(a - c) / abs(c) for a, c in zip(got, ref))}
        hs, Is = H // T, I // T
        for e in allg:
            l, j = e["pp"], e["tp"]
            wq, wk, wv = pr_[l]["wqkv"].grad.split(H, 0)
            sl = slice(j * hs, (j + 1) * hs)
            errs[f"L{l}t{j}.qkv"] = rel(e["qkv"], torch.cat([wq[sl], wk[sl], wv[sl]], 0))
            errs[f"L{l}t{j}.fc2"] = rel(e["fc2"], pr_[l]["w2"].grad[:, j * Is:(j + 1) * Is])
        bad = {k: v for k, v in errs.items() if not v < TOL}
        ok = not bad
        print(f"[tp2xpp2_{policy_kind}] {'OK' if ok else 'FAIL'} schedule={[tuple(e['action']) for e in eng.log]} "
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
    res = [step(smp, "simple"), step(smp, "interleaved")]
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if all(res) else 1)


if __name__ == "__main__":
    main()
