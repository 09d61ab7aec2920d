"""Data-parallel plumbing (dp.py): RDP gradient buckets and the optimizer-state-sharded AdamW.

CPU (gloo, world size 2 and 4): every rank holds the same parameters and its own gradients; after
GradBuckets.finish the gradients are the rank average, and DistributedAdam with and without
shard_optimizer_state (reduce-scatter -> update own slice -> all-gather) reproduces a
single-process AdamW on the averaged gradients; the sharded optimizer holds 1/|RDP| of the
state (SPEC.md:556 example: ratio exactly 4 at |RDP| = 4).  The update itself is the oracle's
AdamW here (oracle/tp.py adamw_ref); on the GPU the fused smpk_adam_step kernel is checked
against it."""
import os
import socket
import traceback

import pytest
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_plan_buckets():
    from paper_2111_05972_b200.dp import plan_buckets
    assert plan_buckets([3, 3, 3, 3], 6) == [(0, 2), (2, 4)]
    assert plan_buckets([10, 1, 1], 4) == [(0, 1), (1, 3)]
    assert plan_buckets([1, 2, 3], 100) == [(0, 3)]
    assert plan_buckets([], 4) == []


def _params(seed):
    g = torch.Generator().manual_seed(seed)
    return [torch.nn.Parameter(torch.randn(*shape, generator=g).to(torch.bfloat16))
            for shape in ((33, 7), (64,), (5, 5, 3), (130,))]


def _grads(params, rank):
    g = torch.Generator().manual_seed(100 + rank)
    for p in params:
        p.grad = torch.randn(p.shape, generator=g).to(torch.bfloat16)


def _worker(r, W, port, q):
    try:
        os.environ.update(RANK=str(r), WORLD_SIZE=str(W), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import sys
        sys.path.insert(0, ROOT)
        torch.set_num_threads(1)
        import torch.distributed as dist
        dist.init_process_group("gloo")
        from oracle import tp
        from paper_2111_05972_b200.dp import DistributedAdam, GradBuckets
        grp = dist.group.WORLD
        # --- gradient buckets (eager and hook-overlapped)
        for overlap in (False, True):
            ps = _params(1)
            gb = GradBuckets(ps, group=grp, bucket_bytes=400, overlap=overlap)
            if overlap:  # drive the post-accumulate hooks through a real backward
                loss = sum((p.float() * torch.randn(p.shape, generator=torch.Generator().manual_seed(100 + r
                            + 7 * i)).float()).sum() for i, p in enumerate(ps))
                loss.backward()
                want = []
                for i, p in enumerate(ps):
                    acc = torch.zeros(p.shape)
                    for rr in range(W):
                        acc += torch.randn(p.shape, generator=torch.Generator().manual_seed(100 + rr + 7 * i)).float()
                    want.append(acc / W)
            else:
                _grads(ps, r)
                want = []
                for i, p in enumerate(ps):
                    acc = torch.zeros(p.shape)
                    for rr in range(W):
                        q_ = _params(1)
                        _grads(q_, rr)
                        acc += q_[i].grad.float()
                    want.append(acc / W)
            gb.finish()
            gb.remove()
            for p, w in zip(ps, want):
                assert torch.allclose(p.grad.float(), w.to(torch.bfloat16).float(), atol=2e-2), "bucket average"
        # --- optimizer: sharded / unsharded vs single-process reference on the averaged grads
        results = {}
        for shard in (False, True):
            ps = _params(2)
            opt = DistributedAdam(ps, lr=1e-2, weight_decay=0.01, group=grp, shard_optimizer_state=shard,
                                  update_fn=tp.adamw_ref)
            for it in range(3):
                _grads(ps, r + 10 * it)
                opt.step()
            results[shard] = ([p.detach().clone() for p in ps], opt.state_bytes())
        ref = _params(2)
        masters = [p.detach().float().clone() for p in ref]
        ms = [torch.zeros_like(m_) for m_ in masters]
        vs = [torch.zeros_like(m_) for m_ in masters]
        for it in range(3):
            avg = []
            for i, p in enumerate(ref):
                acc = torch.zeros(p.shape)
                for rr in range(W):
                    q_ = _params(2)
                    _grads(q_, rr + 10 * it)
                    acc += q_[i].grad.float()
                avg.append(acc)
            for i, p in enumerate(ref):
                out = torch.empty(p.shape, dtype=torch.bfloat16)
                tp.adamw_ref(masters[i], out, avg[i], ms[i], vs[i], lr=1e-2, betas=(0.9, 0.999), eps=1e-8,
                             weight_decay=0.01, step=it + 1, grad_scale=1.0 / W)
        for shard in (False, True):
            for got, mst in zip(results[shard][0], masters):
                assert torch.allclose(got.float(), mst.to(torch.bfloat16).float(), atol=1e-2, rtol=0), shard
        assert results[False][1] == W * results[True][1], "sharded optimizer state is 1/|RDP|"
        dist.barrier()
        dist.destroy_process_group()
        q.put((r, "ok"))
    except Exception:  # noqa: BLE001
        q.put((r, traceback.format_exc()))


@pytest.mark.parametrize("W", [2, 4])
def test_rdp_buckets_and_sharded_adam_gloo(W):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, W, port, q)) for r in range(W)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    bad = {r: v for r, v in res.items() if v != "ok"}
    assert not bad, "\n".join(f"rank {r}:\n{v}" for r, v in bad.items())


@pytest.mark.gpu
def test_adam_kernel_vs_oracle():
    from oracle import tp
    from paper_2111_05972_b200.dp import adam_step_cuda
    n = 4096 * 3
    g0 = torch.Generator().manual_seed(0)
    master = torch.randn(n, generator=g0)
    m, v = torch.zeros(n), torch.zeros(n)
    mr, vr, masr = m.clone(), v.clone(), master.clone()
    md, vd, masd = m.cuda(), v.cuda(), master.cuda()
    pd = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    pr = torch.empty(n, dtype=torch.bfloat16)
    for step in range(1, 4):
        grad = torch.randn(n, generator=g0)
        kw = dict(lr=1e-3, betas=(0.9, 0.98), eps=1e-6, weight_decay=0.1, step=step, grad_scale=0.5)
        adam_step_cuda(masd, pd, grad.cuda(), md, vd, **kw)
        tp.adamw_ref(masr, pr, grad, mr, vr, **kw)
    torch.cuda.synchronize()
    assert torch.allclose(masd.cpu(), masr, rtol=1e-5, atol=1e-6)
    assert torch.allclose(vd.cpu(), vr, rtol=1e-5, atol=1e-9)
    assert torch.equal(pd.cpu(), masd.cpu().to(torch.bfloat16))
