"""NCCL allreduce / allgather / reduce-scatter bandwidth on this box (torchrun, dev tool)."""
import os

import torch
import torch.distributed as dist

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
T = dist.get_world_size()
for mb in (4, 16, 32, 64, 128):
    n = mb * 2 ** 20 // 2
    x = torch.randn(n, device="cuda").bfloat16()
    for _ in range(3):
        dist.all_reduce(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        dist.all_reduce(x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    busbw = 2 * (T - 1) / T * mb * 2 ** 20 / (ms / 1e3) / 1e9
    out = torch.empty(n * T, device="cuda").bfloat16()
    e0.record()
    for _ in range(10):
        dist.all_gather_into_tensor(out, x)
    e1.record()
    torch.cuda.synchronize()
    ms_ag = e0.elapsed_time(e1) / 10
    if dist.get_rank() == 0:
        print(f"T={T} {mb} MiB: allreduce {ms * 1e3:.0f} us busbw {busbw:.0f} GB/s | allgather(out {mb * T} MiB) "
              f"{ms_ag * 1e3:.0f} us", flush=True)
dist.destroy_process_group()
