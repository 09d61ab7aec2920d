"""Single-process 4-GPU probe of the TP reduce-scatter / all-gather row kernel (dev tool).

Every GPU runs the forward sub-layer exchange of BERT-large at T=4 concurrently: pull its 4096
rows from the 4 ranks' [16384, 1024] partials, sum + residual + LayerNorm, push the output rows
into the 4 ranks' gather buffers.  Variants isolate the pull, the push and the local work.

usage: python scripts/nvlink_probe4.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_05972_b200 import ops  # noqa: E402

T = min(4, torch.cuda.device_count())
R, H = 4096, 1024
for a in range(T):
    for b in range(T):
        if a != b:
            with torch.cuda.device(a):
                torch.zeros(1, device=f"cuda:{b}").copy_(torch.zeros(1, device=f"cuda:{a}"))
part = [torch.randn(T * R, H, device=f"cuda:{g}").bfloat16() for g in range(T)]
gath = [torch.zeros(T * R, H, device=f"cuda:{g}").bfloat16() for g in range(T)]
res = [torch.randn(R, H, device=f"cuda:{g}").bfloat16() for g in range(T)]
gam = [torch.ones(H, device=f"cuda:{g}").bfloat16() for g in range(T)]
bet = [torch.zeros(H, device=f"cuda:{g}").bfloat16() for g in range(T)]
xt = [torch.tensor([p.data_ptr() for p in part], dtype=torch.int64, device=f"cuda:{g}") for g in range(T)]
ot = [torch.tensor([q.data_ptr() for q in gath], dtype=torch.int64, device=f"cuda:{g}") for g in range(T)]
for g in range(T):
    torch.cuda.synchronize(g)


def run(g, mode):
    with torch.cuda.device(g):
        if mode == "full":
            ops.bdr_ln(part[g], residual=res[g], gamma=gam[g], beta=bet[g], rows=R, cols=H, nslots=T, x_peers=xt[g],
                       x_peer_off=g * R * H, want_r=True, out_peers=ot[g], peer_off=g * R * H)
        elif mode == "pull":
            ops.bdr_ln(part[g], residual=res[g], gamma=gam[g], beta=bet[g], rows=R, cols=H, nslots=T, x_peers=xt[g],
                       x_peer_off=g * R * H)
        elif mode == "push":
            ops.bdr_ln(res[g], want_r=False, out_peers=ot[g], peer_off=g * R * H)
        elif mode == "local":
            ops.bdr_ln(part[g], residual=res[g], gamma=gam[g], beta=bet[g], rows=R, cols=H, nslots=T,
                       slot_stride=R * H)


def timeit(mode, gpus, it=20):
    """Each GPU replays a CUDA graph of `it` launches; the graphs start back to back so the GPUs
    run concurrently; per-GPU device time from events, max over GPUs."""
    graphs = {}
    for g in gpus:
        with torch.cuda.device(g):
            run(g, mode)
            torch.cuda.synchronize(g)
            gr = torch.cuda.CUDAGraph()
            st = torch.cuda.Stream(device=g)
            with torch.cuda.stream(st):
                with torch.cuda.graph(gr, stream=st):
                    for _ in range(it):
                        run(g, mode)
            graphs[g] = gr
    for g in gpus:
        torch.cuda.synchronize(g)
    ev = {}
    for g in gpus:
        with torch.cuda.device(g):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            graphs[g].replay()
            e1.record()
            ev[g] = (e0, e1)
    for g in gpus:
        torch.cuda.synchronize(g)
    return max(ev[g][0].elapsed_time(ev[g][1]) for g in gpus) * 1e3 / it


remote = (T - 1) * R * H * 2
for mode in ("local", "pull", "push", "full"):
    for gpus in ([0], list(range(T))):
        us = timeit(mode, gpus)
        print(f"{mode:6s} on {len(gpus)} GPU(s): {us:7.1f} us/iter  "
              f"(remote bytes per GPU each way {remote / 1e6:.0f} MB -> {remote / us / 1e3:.0f} GB/s)")
