"""One launch each of the BERT-large MLP GEMM variants (ncu target; dev tool)."""
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
for _ in range(2):
    K.linear(x, w)
    K.linear(x, w, b, act="gelu")
    K.matmul_nn(dy, w2, epi=K.EPI_DACT, act="gelu", aux=z, want_colsum=True)
torch.cuda.synchronize()
print("ok")
