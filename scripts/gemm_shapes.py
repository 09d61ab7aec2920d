"""Time the BERT-large layer GEMM shapes (graph-replayed, so no host launch cost) — smpk vs cuBLAS.

usage: python scripts/gemm_shapes.py [--T 1]   (T = TP degree: tokens 4096*T, weight shards / T)
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_05972_b200 import kernels as K  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--T", type=int, default=1)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
T, H, F = a.T, 1024, 4096
tok = 4096 * T


def shapes():
    # (name, kind, M, N, K)   kind: nt = x W^T, nn = dY W, tn = dY^T X
    return [("qkv_fwd", "nt", tok, 3 * H // T, H), ("out_fwd", "nt", tok, H, H // T),
            ("fc1_fwd", "nt", tok, F // T, H), ("fc2_fwd", "nt", tok, H, F // T),
            ("fc2_dgrad", "nn", tok, F // T, H), ("fc1_dgrad", "nn", tok, H, F // T),
            ("out_dgrad", "nn", tok, H // T, H), ("qkv_dgrad", "nn", tok, H, 3 * H // T),
            ("out_wgrad", "tn", H, H // T, tok), ("qkv_wgrad", "tn", 3 * H // T, H, tok),
            ("fc1_wgrad", "tn", F // T, H, tok), ("fc2_wgrad", "tn", H, F // T, tok)]


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


tot_s = tot_c = 0.0
for name, kind, M, N, Kd in shapes():
    if kind == "nt":
        x, w = torch.randn(M, Kd, device="cuda").bfloat16(), torch.randn(N, Kd, device="cuda").bfloat16()
        f_s = lambda: K.linear(x, w)  # noqa: E731
        f_c = lambda: x @ w.t()  # noqa: E731
    elif kind == "nn":
        x, w = torch.randn(M, Kd, device="cuda").bfloat16(), torch.randn(Kd, N, device="cuda").bfloat16()
        f_s = lambda: K.matmul_nn(x, w)  # noqa: E731
        f_c = lambda: x @ w  # noqa: E731
    else:
        x, w = torch.randn(Kd, M, device="cuda").bfloat16(), torch.randn(Kd, N, device="cuda").bfloat16()
        f_s = lambda: K.matmul_tn(x, w)  # noqa: E731
        f_c = lambda: x.t() @ w  # noqa: E731
    us_s, us_c = timed(f_s, a.reps), timed(f_c, a.reps)
    fl = 2.0 * M * N * Kd
    tot_s += us_s
    tot_c += us_c
    ws = K._lib.size("smpk_gemm_workspace", M, N, Kd, 1, 1)
    print(f"{name:10s} {kind} {M:6d}x{N:5d}x{Kd:6d}  smpk {us_s:7.1f} us {fl / us_s / 1e6:6.0f} TF/s   "
          f"cublas {us_c:7.1f} us {fl / us_c / 1e6:6.0f} TF/s   splitk_ws={ws >> 20}MB")
print(f"total smpk {tot_s:.1f} us  cublas {tot_c:.1f} us")
