"""TP=T reduce-scatter variants for the row-parallel GEMM (dev probe; torchrun --nproc-per-node T)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
import paper_2111_05972_b200 as smp
from paper_2111_05972_b200 import kernels as K, _lib
from paper_2111_05972_b200.state import get_pool

local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
smp.init({"tensor_parallel_degree": dist.get_world_size(), "optimize": "speed", "symm_pool_bytes": 1 << 30})
T, me = dist.get_world_size(), dist.get_rank()
R, N, Kd = 4096, 1024, 1024
pool = get_pool()
a = torch.randn(T * R, Kd, device="cuda").bfloat16()
w = torch.randn(N, Kd, device="cuda").bfloat16()
P = pool.scratch("partials", T * R * N * 2)
loc = torch.empty(T * R, N, device="cuda", dtype=torch.bfloat16)
streams = [torch.cuda.Stream() for _ in range(T)]

def t(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e3

def rs_fused():
    peers, off = pool.host_peers(P, me * R * N)
    K.gemm_rs(a, w, False, peers, ldc=N, rows_per_owner=R, slot_off=off)
    pool.barrier()

def gemm_local():
    K.linear(a, w, out=loc)

def dma(nbytes_rows=R):
    main = torch.cuda.current_stream()
    for j in range(T):
        if j == me: continue
        s = streams[j]; s.wait_stream(main)
        with torch.cuda.stream(s):
            dst = pool.bases[j] + P + (me * R * N) * 2
            _lib.call("smpk_copy_async", dst, loc[j * R:(j + 1) * R].data_ptr(), nbytes_rows * N * 2, s.cuda_stream)
    for j in range(T):
        if j != me: main.wait_stream(streams[j])

def gemm_dma():
    gemm_local(); dma(); pool.barrier()

for name, fn in [("gemm_local", gemm_local), ("rs_fused(peer TMA stores)", rs_fused), ("dma_only", dma),
                 ("gemm+dma", gemm_dma)]:
    us = t(fn)
    if me == 0: print(f"T={T} {name}: {us:.1f} us", flush=True)
dist.barrier(); dist.destroy_process_group()
