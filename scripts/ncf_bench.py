"""NCF embedding microbench (BASELINE.json configs[4]): one TP rank of the
dim-sharded DistributedEmbedding at TP=8 -- item tables 10^8 x {64 (GMF), 512 (MLP)} -> per rank
10^8 x {8, 64} bf16 columns, fp32 gradient tables -- 65,536 lookups per GPU = 524,288 gathered ids
per rank, uniform and Zipf(1.05).  Times the lookup (smpk_embed_fwd) and the sort-based backward
(smpk_embed_bwd_sorted, accumulate into the fp32 gradient), device time with CUDA events over
graph-free launches, and reports GB/s by SURVEY §8d's byte model against MEASURED_PEAKS hbm_gbs:
  forward  per index: D*2 (row read) + D*2 (write) + 8 (id)
  backward per index: D*2 (dy read) + per unique row 2*D*4 (fp32 read-modify-write)
usage: python scripts/ncf_bench.py [rows] [n_lookups]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2111_05972_b200 import embedding as E  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 524_288
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6546.2


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


rng = np.random.default_rng(0)
out = []
for D in (8, 64):
    table = torch.empty(rows, D, dtype=torch.bfloat16, device="cuda").normal_(0, 0.02)
    grad = torch.zeros(rows, D, dtype=torch.float32, device="cuda")
    for dist in ("uniform", "zipf1.05"):
        if dist == "uniform":
            ids = torch.from_numpy(rng.integers(0, rows, n, dtype=np.int64))
        else:
            z = rng.zipf(1.05, size=4 * n)
            z = z[z <= rows][:n] - 1
            ids = torch.from_numpy(rng.permutation(rows)[z]) if rows <= 10_000_000 else torch.from_numpy(
                (z * 2654435761) % rows)
        ids = ids.cuda()
        uniq = int(torch.unique(ids).numel())
        y = E.embed_lookup(ids, table, row_offset=0, vocab=rows)
        dy = torch.randn(n, D, device="cuda").bfloat16()
        t_f = timed(lambda: E.embed_lookup(ids, table, row_offset=0, vocab=rows))
        t_b = timed(lambda: E.embed_grad(ids, dy, rows=rows, row_offset=0, out=grad, accumulate=True))
        bf = n * (4 * D + 8)
        bb = n * 2 * D + uniq * 8 * D
        line = {"table": f"{rows}x{D}", "lookups": n, "ids": dist, "unique_rows": uniq,
                "fwd_us": t_f, "fwd_GBps": bf / t_f / 1e3, "fwd_frac_hbm": bf / t_f / 1e3 / peak,
                "bwd_us": t_b, "bwd_GBps": bb / t_b / 1e3, "bwd_frac_hbm": bb / t_b / 1e3 / peak,
                "lookups_per_s_fwd_bwd": n / ((t_f + t_b) * 1e-6)}
        out.append(line)
        print(json.dumps(line), flush=True)
    del table, grad
    torch.cuda.empty_cache()
