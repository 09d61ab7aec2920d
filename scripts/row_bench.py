"""Row-kernel microbench at the BERT-large and GPT-1.3B bench shapes (dev tool): bias + dropout +
residual + LayerNorm forward (smpk_bdr_ln_fwd) and its backward (smpk_ln_bwd), graph-replayed,
with algorithmic bytes -> GB/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_05972_b200 import ops  # noqa: E402


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


for M, H in ((4096, 1024), (16384, 2048)):
    x, res, dy = (torch.randn(M, H, device="cuda").bfloat16() for _ in range(3))
    b, gam, bet = (torch.randn(H, device="cuda").bfloat16() for _ in range(3))
    kb = ops.keep_bytes(M, H, x.device)
    r, y, mu, rs = ops.bdr_ln(x, bias=b, residual=res, gamma=gam, beta=bet, p=0.1, seed=1, keep_out=kb)
    t_f = timed(lambda: ops.bdr_ln(x, bias=b, residual=res, gamma=gam, beta=bet, p=0.1, seed=1, keep_out=kb))
    t_b = timed(lambda: ops.ln_bwd(dy, r, mu, rs, gam, dres=dy, p=0.1, seed=1, keep_in=kb, want_dbias=True))
    t_bn = timed(lambda: ops.ln_bwd(dy, r, mu, rs, gam, want_dbias=False))
    fb = M * H * 2 * 4 + M * H / 8 + M * 8  # x, res in; r, y out; keep bytes; stats
    bb = M * H * 2 * 5 + M * H / 8 + M * 8  # dy, r, dres in; dr, dsub out; keep; stats
    bn = M * H * 2 * 3 + M * 8
    print(f"M={M} H={H}: bdr_ln_fwd {t_f:.1f} us {fb / t_f / 1e3:.0f} GB/s | ln_bwd(dropout,dres) {t_b:.1f} us "
          f"{bb / t_b / 1e3:.0f} GB/s | ln_bwd(plain) {t_bn:.1f} us {bn / t_bn / 1e3:.0f} GB/s", flush=True)
