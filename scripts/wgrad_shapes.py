"""Weight-gradient GEMM shapes of the TP>1 BERT-large backward (dW = dY^T X over all T*b*s gathered
rows): M x N output, K = 4096*T tokens (2048*T per overlapped micro-batch).  Graph-replayed device time per launch (dev tool).
usage: SMPK_GEMM_PAIR_SPLITK=0|1 python scripts/wgrad_shapes.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_05972_b200 import kernels as K  # noqa: E402

H, I = 1024, 4096
for T, Kt in ((1, 4096), (2, 8192), (4, 16384), (8, 32768), (2, 4096), (4, 8192), (8, 16384)):
    shapes = {"dWqkv": (3 * H // T, H), "dWo": (H, H // T), "dW1": (I // T, H), "dW2": (H, I // T)}
    tot_f, tot_t = 0.0, 0.0
    line = []
    for name, (M, N) in shapes.items():
        dy = torch.randn(Kt, M, device="cuda").bfloat16()
        x = torch.randn(Kt, N, device="cuda").bfloat16()
        out = torch.empty(M, N, device="cuda").bfloat16()
        for _ in range(3):
            K.matmul_tn(dy, x, out=out)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(10):
                K.matmul_tn(dy, x, out=out)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 100
        fl = 2 * M * N * Kt
        tot_f += fl
        tot_t += us
        line.append(f"{name} {M}x{N}x{Kt} {us:.1f}us {fl / us / 1e6:.0f}TF/s")
    print(f"T={T}: " + " | ".join(line) + f" || total {tot_t:.1f} us {tot_f / tot_t / 1e6:.0f} TF/s", flush=True)
