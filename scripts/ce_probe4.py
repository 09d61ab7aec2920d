"""Single-process T-GPU probe: copy-engine peer copies next to the persistent GEMM (dev tool).

Every GPU pushes an [R, H] bf16 block to each of the T-1 peers with cudaMemcpyAsync (copy engines,
one side stream per peer) -- the all-to-all volume of one TP exchange -- alone, and while the compute
stream runs the BERT-large QKV + FC1 GEMMs of one chunk.  Reports device times (CUDA events).

usage: python scripts/ce_probe4.py [R H]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_05972_b200 import kernels as K  # noqa: E402

T = min(4, torch.cuda.device_count())
R, H = (int(v) for v in sys.argv[1:3]) if len(sys.argv) > 2 else (4096, 1024)
for a in range(T):
    for b in range(T):
        if a != b:
            with torch.cuda.device(a):
                torch.zeros(1, device=f"cuda:{b}").copy_(torch.zeros(1, device=f"cuda:{a}"))
src = [torch.randn(R, H, device=f"cuda:{g}").bfloat16() for g in range(T)]
dst = [[torch.zeros(R, H, device=f"cuda:{g}").bfloat16() for _ in range(T)] for g in range(T)]
x = [torch.randn(R, H, device=f"cuda:{g}").bfloat16() for g in range(T)]
w1 = [torch.randn(4 * H, H, device=f"cuda:{g}").bfloat16() for g in range(T)]
w2 = [torch.randn(3 * H, H, device=f"cuda:{g}").bfloat16() for g in range(T)]
side = [[torch.cuda.Stream(device=g) for _ in range(T)] for g in range(T)]
main = [torch.cuda.Stream(device=g) for g in range(T)]


def copies(g):
    for p in range(T):
        if p == g:
            continue
        s = side[g][p]
        s.wait_stream(main[g])
        with torch.cuda.device(g), torch.cuda.stream(s):
            dst[p][g].copy_(src[g], non_blocking=True)


def gemms(g, n=3):
    with torch.cuda.device(g), torch.cuda.stream(main[g]):
        for _ in range(n):
            K.linear(x[g], w1[g], None)
            K.linear(x[g], w2[g], None)


def join(g):
    for p in range(T):
        if p != g:
            main[g].wait_stream(side[g][p])


def timed(fn, reps=5):
    ev = []
    for g in range(T):
        torch.cuda.synchronize(g)
    for g in range(T):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.device(g):
            e0.record(main[g])
        ev.append((e0, e1))
    for _ in range(reps):
        for g in range(T):
            fn(g)
    for g in range(T):
        with torch.cuda.device(g):
            ev[g][1].record(main[g])
    for g in range(T):
        torch.cuda.synchronize(g)
    return max(e0.elapsed_time(e1) for e0, e1 in ev) / reps * 1e3


def only_copies(g):
    copies(g)
    join(g)


def only_gemm(g):
    gemms(g)


def both(g):
    copies(g)
    gemms(g)
    join(g)


for fn in (only_copies, only_gemm, both):
    fn_t = [timed(fn) for _ in range(3)][-1]
    vol = (T - 1) * R * H * 2
    print(f"T={T} {fn.__name__:12s}: {fn_t:8.1f} us  (per-GPU out volume {vol / 1e6:.1f} MB"
          + (f", {vol / fn_t / 1e3:.0f} GB/s out)" if fn is only_copies else ")"), flush=True)
