"""Run one GEMM configuration a few times (for ncu --set full captures)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2111_05972_b200 import kernels as K

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=4096); ap.add_argument("--N", type=int, default=4096)
ap.add_argument("--K", type=int, default=1024); ap.add_argument("--epi", default="bias_gelu")
ap.add_argument("--iters", type=int, default=5)
a = ap.parse_args()
x = torch.randn(a.M, a.K, device="cuda").bfloat16()
w = torch.randn(a.N, a.K, device="cuda").bfloat16()
b = torch.randn(a.N, device="cuda").bfloat16()
z = torch.randn(a.M, a.N, device="cuda").bfloat16()
wt = torch.randn(a.K, a.N, device="cuda").bfloat16()
for _ in range(a.iters):
    if a.epi == "bias_gelu":
        K.linear(x, w, b, act="gelu")
    elif a.epi == "dgelu":
        K.matmul_nn(x, wt, epi=K.EPI_DACT, act="gelu", aux=z)
    else:
        K.matmul_nt(x, w)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    if a.epi == "bias_gelu":
        K.linear(x, w, b, act="gelu")
    elif a.epi == "dgelu":
        K.matmul_nn(x, wt, epi=K.EPI_DACT, act="gelu", aux=z)
    else:
        K.matmul_nt(x, w)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"{a.epi} {a.M}x{a.N}x{a.K}: {ms*1e3:.1f} us, {2*a.M*a.N*a.K/ms/1e9:.0f} TF/s")
