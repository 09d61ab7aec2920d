"""Quick GEMM correctness + speed probe on one GPU (development tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2111_05972_b200 import kernels as K

torch.manual_seed(0)
dev = "cuda"

def rel(a, b):
    return ((a.float() - b.float()).norm() / (b.float().norm() + 1e-30)).item()

def check(name, got, ref, tol=1e-2):
    e = rel(got, ref)
    print(f"{'OK ' if e < tol else 'BAD'} {name}: rel={e:.2e}", flush=True)
    return e < tol

ok = True
for (M, N, Kd) in [(128, 256, 64), (256, 512, 128), (304, 200, 104), (4096, 1024, 1024), (1008, 64, 512), (128, 128, 4096)]:
    a = torch.randn(M, Kd, device=dev).bfloat16()
    w = torch.randn(N, Kd, device=dev).bfloat16()
    ref = a.float() @ w.float().t()
    ok &= check(f"nt {M}x{N}x{Kd}", K.matmul_nt(a, w), ref)
    b = torch.randn(Kd, N, device=dev).bfloat16()
    ok &= check(f"nn {M}x{N}x{Kd}", K.matmul_nn(a, b), a.float() @ b.float())
    at = torch.randn(Kd, M, device=dev).bfloat16()
    ok &= check(f"tn {M}x{N}x{Kd}", K.matmul_tn(at, b), at.float().t() @ b.float())
    ok &= check(f"tn-f32 {M}x{N}x{Kd}", K.matmul_tn(at, b, out_dtype=torch.float32), at.float().t() @ b.float(), 1e-4)
    bias = torch.randn(N, device=dev).bfloat16()
    y, z = K.linear(a, w, bias, act="gelu")
    zr = ref + bias.float()
    ok &= check(f"bias_gelu pre {M}x{N}", z, zr)
    ok &= check(f"bias_gelu act {M}x{N}", y, torch.nn.functional.gelu(z.float()))

# batched, attention-like: qkv [b*s, 3*nh*dh]
b_, s, nh, dh = 2, 256, 4, 64
qkv = torch.randn(b_ * s, 3 * nh * dh, device=dev).bfloat16()
ld = 3 * nh * dh
q = qkv[:, : nh * dh]; k = qkv[:, nh * dh: 2 * nh * dh]; v = qkv[:, 2 * nh * dh:]
S = torch.empty(b_, nh, s, s, device=dev, dtype=torch.bfloat16)
K.gemm_raw(q, 0, ld, (dh, s * ld), k, 0, ld, (dh, s * ld), S, s, (s * s, nh * s * s), s, s, dh, nb=(nh, b_))
qr = q.float().view(b_, s, nh, dh).permute(0, 2, 1, 3); kr = k.float().view(b_, s, nh, dh).permute(0, 2, 1, 3)
vr = v.float().view(b_, s, nh, dh).permute(0, 2, 1, 3)
ok &= check("batched QK^T", S, qr @ kr.transpose(-1, -2))
P = torch.softmax(S.float(), -1).bfloat16()
ctx = torch.empty(b_ * s, nh * dh, device=dev, dtype=torch.bfloat16)
K.gemm_raw(P, 0, s, (s * s, nh * s * s), v, 1, ld, (dh, s * ld), ctx, nh * dh, (dh, s * nh * dh), s, dh, s, nb=(nh, b_))
ok &= check("batched PV", ctx, (P.float() @ vr).permute(0, 2, 1, 3).reshape(b_ * s, nh * dh))

# timing
def bench(fn, flops, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    return ms, flops / ms / 1e9

for (M, N, Kd) in [(8192, 8192, 8192), (4096, 4096, 1024), (4096, 1024, 4096), (4096, 3072, 1024), (32768, 384, 1024)]:
    a = torch.randn(M, Kd, device=dev).bfloat16(); w = torch.randn(N, Kd, device=dev).bfloat16()
    c = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    ms, tf = bench(lambda: K.matmul_nt(a, w, out=c), 2 * M * N * Kd)
    ms2, tf2 = bench(lambda: torch.matmul(a, w.t(), out=c), 2 * M * N * Kd)
    print(f"nt {M}x{N}x{Kd}: smpk {ms:.3f} ms {tf:.0f} TF/s | cublas {ms2:.3f} ms {tf2:.0f} TF/s", flush=True)
    b = torch.randn(Kd, N, device=dev).bfloat16()
    ms, tf = bench(lambda: K.matmul_nn(a, b, out=c), 2 * M * N * Kd)
    print(f"nn {M}x{N}x{Kd}: smpk {ms:.3f} ms {tf:.0f} TF/s", flush=True)
    at = torch.randn(Kd, M, device=dev).bfloat16()
    ms, tf = bench(lambda: K.matmul_tn(at, b, out=c), 2 * M * N * Kd)
    print(f"tn {M}x{N}x{Kd}: smpk {ms:.3f} ms {tf:.0f} TF/s", flush=True)
print("ALL OK" if ok else "FAILURES")
