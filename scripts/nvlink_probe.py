"""Single-process NVLink probe (2 GPUs, peer access): remote-read / remote-write bandwidth of the
row-kernel access patterns (dev tool; also a target for ncu, which must not wrap multi-rank runs).

usage: python scripts/nvlink_probe.py
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_05972_b200 import _lib, ops  # noqa: E402

assert torch.cuda.device_count() >= 2
cudart = C.CDLL("libcudart.so") if False else None
torch.cuda.set_device(0)
for a, b in ((0, 1), (1, 0)):
    with torch.cuda.device(a):
        try:
            torch.cuda.current_device()
            # torch enables peer access lazily on cross-device copies; force it with a tiny copy
            torch.zeros(1, device=f"cuda:{b}").copy_(torch.zeros(1, device=f"cuda:{a}"))
        except Exception as e:  # noqa: BLE001
            print("peer enable", e)
R, H = 4096, 1024
T = 2
loc = torch.randn(T * R, H, device="cuda:0").bfloat16()
rem = torch.randn(T * R, H, device="cuda:1").bfloat16()
torch.cuda.synchronize(1)
table = torch.tensor([loc.data_ptr(), rem.data_ptr()], dtype=torch.int64, device="cuda:0")
res = torch.randn(R, H, device="cuda:0").bfloat16()


def timeit(fn, it=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / it


# pull: sum of a local slot and a remote slot (R rows each) + residual
us = timeit(lambda: ops.bdr_ln(loc, residual=res, rows=R, cols=H, nslots=2, x_peers=table, x_peer_off=0))
print(f"pull 2 slots (1 remote, {R * H * 2 / 1e6:.1f} MB): {us:.1f} us -> {R * H * 2 / us / 1e3:.0f} GB/s remote")
# push: copy own rows to local + remote (peer stores)
dst = torch.tensor([loc.data_ptr(), rem.data_ptr()], dtype=torch.int64, device="cuda:0")
us = timeit(lambda: ops.bdr_ln(res, want_r=False, out_peers=dst, peer_off=R * H))
print(f"push to 2 (1 remote, {R * H * 2 / 1e6:.1f} MB): {us:.1f} us -> {R * H * 2 / us / 1e3:.0f} GB/s remote")
# copy engine
us = timeit(lambda: _lib.call("smpk_copy_async", rem.data_ptr(), res.data_ptr(), R * H * 2,
                              torch.cuda.current_stream().cuda_stream))
print(f"copy engine {R * H * 2 / 1e6:.1f} MB: {us:.1f} us -> {R * H * 2 / us / 1e3:.0f} GB/s")
# local-only baselines
us = timeit(lambda: ops.bdr_ln(loc, residual=res, rows=R, cols=H, nslots=2, slot_stride=R * H))
print(f"local 2 slots: {us:.1f} us")

# calibration: streaming at these sizes
big = torch.randn(4 * R, H, device="cuda:0").bfloat16()
big2 = torch.empty_like(big)
us = timeit(lambda: big2.copy_(big))
print(f"torch copy {big.numel() * 2 / 1e6:.0f} MB: {us:.1f} us -> {2 * big.numel() * 2 / us / 1e3:.0f} GB/s (r+w)")
small2 = torch.empty_like(res)
us = timeit(lambda: small2.copy_(res))
print(f"torch copy {res.numel() * 2 / 1e6:.0f} MB: {us:.1f} us -> {2 * res.numel() * 2 / us / 1e3:.0f} GB/s (r+w)")
x4 = torch.randn(2 * 4 * R, H, device="cuda:0").bfloat16()
res4 = torch.randn(4 * R, H, device="cuda:0").bfloat16()
us = timeit(lambda: ops.bdr_ln(x4, residual=res4, rows=4 * R, cols=H, nslots=2, slot_stride=4 * R * H))
print(f"local 2 slots x4 rows: {us:.1f} us -> {4 * 4 * R * H * 2 / us / 1e3:.0f} GB/s")
g = torch.ones(H, device="cuda:0").bfloat16(); bb = torch.zeros(H, device="cuda:0").bfloat16()
us = timeit(lambda: ops.bdr_ln(res4, residual=big, gamma=g, beta=bb, p=0.1, seed=1))
print(f"bdr+LN+dropout 16384 rows: {us:.1f} us -> {4 * 4 * R * H * 2 / us / 1e3:.0f} GB/s")
