"""Per-kernel device times of one sort-based embedding backward (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2111_05972_b200 import embedding as E  # noqa: E402

rows, n, D = 100_000_000, 524_288, int(sys.argv[1]) if len(sys.argv) > 1 else 8
rng = np.random.default_rng(0)
grad = torch.zeros(rows, D, dtype=torch.float32, device="cuda")
for dist in ("uniform", "zipf"):
    if dist == "uniform":
        ids = torch.from_numpy(rng.integers(0, rows, n, dtype=np.int64)).cuda()
    else:
        z = rng.zipf(1.05, size=4 * n)
        ids = torch.from_numpy(((z[z <= rows][:n] - 1) * 2654435761) % rows).cuda()
    dy = torch.randn(n, D, device="cuda").bfloat16()
    E.embed_grad(ids, dy, rows=rows, row_offset=0, out=grad, accumulate=True)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        E.embed_grad(ids, dy, rows=rows, row_offset=0, out=grad, accumulate=True)
        torch.cuda.synchronize()
    print("==", dist)
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            print(f"  {ev.device_time_total:8.1f} us  {ev.name[:80]}")
