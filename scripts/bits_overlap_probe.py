"""Attention keep-bit generator next to the QKV GEMM (dev tool): the generator alone, the GEMM
alone, and both on two streams (generator launched first on a side stream, as in the layer).
SMPK_BITS_CTAS_PER_SM=k selects the persistent k-CTAs-per-SM grid (0: one thread per word).
usage: python scripts/bits_overlap_probe.py [bert|gpt]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2111_05972_b200 import kernels as K  # noqa: E402
from paper_2111_05972_b200 import ops  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "bert"
B, nh, s, H, causal = (8, 16, 512, 1024, False) if wl == "bert" else (8, 16, 2048, 2048, True)
x = torch.randn(B * s, H, device="cuda").bfloat16()
w = torch.randn(3 * H, H, device="cuda").bfloat16()
b = torch.randn(3 * H, device="cuda").bfloat16()
bits = torch.empty(B, nh, s, s // 32, dtype=torch.int32, device="cuda")
side = torch.cuda.Stream()
main = torch.cuda.current_stream()


def gen():
    ops.attn_dropout_bits(B, nh, s, s, p=0.1, seed=1, out=bits, causal=causal)


def gemm():
    K.linear(x, w, b)


def both():
    side.wait_stream(main)
    with torch.cuda.stream(side):
        gen()
    gemm()
    main.wait_stream(side)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


ref = bits.clone()
gen()
torch.cuda.synchronize()
print(f"{wl} per_sm={os.environ.get('SMPK_BITS_CTAS_PER_SM', '0')}: bits {timed(gen):.1f} us, QKV GEMM {timed(gemm):.1f} us, "
      f"both {timed(both):.1f} us", flush=True)
