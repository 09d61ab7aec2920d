"""Single-process T-GPU probe: copy-engine peer copies, alone and next to the persistent GEMM (dev tool).

Device-timed (CUDA events on the streams that do the work):
  A  one copy of MB megabytes GPU0 -> GPU1 (cudaMemcpyAsync to the peer pointer: copy engine)
  B  GPU0 -> GPU1, GPU2, GPU3 concurrently (3 side streams)
  C  all GPUs -> all peers concurrently (the all-to-all volume of one TP exchange)
  D  a large GEMM on GPU0 alone, and with B running beside it

usage: python scripts/ce_probe4.py [MB]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_05972_b200 import _lib  # noqa: E402
from paper_2111_05972_b200 import kernels as K  # noqa: E402

T = min(4, torch.cuda.device_count())
MB = float(sys.argv[1]) if len(sys.argv) > 1 else 8.0
n = int(MB * (1 << 20))
for a in range(T):
    for b in range(T):
        if a != b:
            with torch.cuda.device(a):
                torch.zeros(1, device=f"cuda:{b}").copy_(torch.zeros(1, device=f"cuda:{a}"))
src = [torch.empty(n, dtype=torch.uint8, device=f"cuda:{g}") for g in range(T)]
dst = [[torch.empty(n, dtype=torch.uint8, device=f"cuda:{g}") for _ in range(T)] for g in range(T)]
side = [[torch.cuda.Stream(device=g) for _ in range(T)] for g in range(T)]


def sync():
    for g in range(T):
        torch.cuda.synchronize(g)


def copy_set(pairs, reps=10):
    """pairs: (src gpu, dst gpu); each on its own stream; returns (per-copy us, span us) on the
    source devices (span = max over source GPUs of first-start .. last-end)."""
    sync()
    evs = []
    for (g, p) in pairs:
        s = side[g][p]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.device(g):
            e0.record(s)
            for _ in range(reps):
                _lib.call("smpk_copy_async", dst[p][g].data_ptr(), src[g].data_ptr(), n, s.cuda_stream)
            e1.record(s)
        evs.append((g, e0, e1))
    sync()
    per = max(e0.elapsed_time(e1) for _, e0, e1 in evs) / reps * 1e3
    return per


x = torch.randn(8192, 4096, device="cuda:0").bfloat16()
w = torch.randn(8192, 4096, device="cuda:0").bfloat16()


def gemm_time(with_copies, reps=5):
    sync()
    main = torch.cuda.current_stream(0)
    with torch.cuda.device(0):
        K.linear(x, w)
        sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if with_copies:
            for p in range(1, T):
                for _ in range(40):
                    _lib.call("smpk_copy_async", dst[p][0].data_ptr(), src[0].data_ptr(), n, side[0][p].cuda_stream)
        e0.record(main)
        for _ in range(reps):
            K.linear(x, w)
        e1.record(main)
    sync()
    return e0.elapsed_time(e1) / reps * 1e3


for _ in range(2):
    a = copy_set([(0, 1)])
    b = copy_set([(0, p) for p in range(1, T)])
    c = copy_set([(g, p) for g in range(T) for p in range(T) if p != g])
print(f"A one copy 0->1 {MB:g} MB: {a:.1f} us = {n / a / 1e3:.0f} GB/s")
print(f"B 0->(1..{T - 1}) concurrent: {b:.1f} us per copy set = {(T - 1) * n / b / 1e3:.0f} GB/s out of GPU0")
print(f"C all-to-all: {c:.1f} us per copy set = {(T - 1) * n / c / 1e3:.0f} GB/s out per GPU")
g0, g1 = gemm_time(False), gemm_time(True)
fl = 2 * 8192 * 8192 * 4096
print(f"D GEMM 8192x8192x4096 alone {g0:.1f} us ({fl / g0 / 1e6:.0f} TF/s); beside GPU0->peers copies {g1:.1f} us "
      f"({fl / g1 / 1e6:.0f} TF/s)")
