"""Time the fused-epilogue GEMMs of the BERT-large MLP (graph-replayed): bias+GeLU forward,
dGeLU (+ fused bias-gradient column sums) backward, and the plain GEMM of the same shape."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_05972_b200 import kernels as K  # noqa: E402

M, N, Kd = 4096, 4096, 1024
x, w, b = (torch.randn(M, Kd, device="cuda").bfloat16(), torch.randn(N, Kd, device="cuda").bfloat16(),
           torch.randn(N, device="cuda").bfloat16())
dy, w2 = torch.randn(M, Kd, device="cuda").bfloat16(), torch.randn(Kd, N, device="cuda").bfloat16()
z = torch.randn(M, N, device="cuda").bfloat16()


def timed(fn, reps=20):
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


for name, fn in (("plain", lambda: K.linear(x, w)), ("bias_gelu", lambda: K.linear(x, w, b, act="gelu")),
                 ("dgelu", lambda: K.matmul_nn(dy, w2, epi=K.EPI_DACT, act="gelu", aux=z)),
                 ("dgelu_colsum", lambda: K.matmul_nn(dy, w2, epi=K.EPI_DACT, act="gelu", aux=z, want_colsum=True))):
    us = timed(fn)
    print(f"{name:13s} {M}x{N}x{Kd}: {us:6.1f} us  {2 * M * N * Kd / us / 1e6:6.0f} TF/s")
