"""Helper for test_pdl_gpu.py (run as a subprocess, so SMPK_PDL / SMPK_ROW_FAST take effect): a
2-layer BERT-style stack, forward + backward with dropout, eager and CUDA-graph-replayed; prints a
SHA-256 of the output and every gradient."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_05972_b200 as smp  # noqa: E402

smp.init({"tensor_parallel_degree": 1, "optimize": "speed", "seed": 11})
torch.manual_seed(0)
model = smp.nn.DistributedTransformer(num_layers=2, num_attention_heads=16, attention_head_size=64, hidden_size=1024,
                                      intermediate_size=4096, attention_dropout_prob=0.1, hidden_dropout_prob=0.1,
                                      activation="gelu", layernorm_epsilon=1e-5, pre_layernorm=False,
                                      post_layernorm=True)
x = torch.randn(4, 512, 1024, device="cuda", dtype=torch.bfloat16, requires_grad=True)
dy = torch.randn(4, 512, 1024, device="cuda", dtype=torch.bfloat16)
h = hashlib.sha256()


def step():
    for p in model.parameters():
        p.grad = None
    x.grad = None
    y = model(x)
    y.backward(dy)
    return y


smp.set_rng_step(5)
y = step()
torch.cuda.synchronize()
for t in [y, x.grad] + [p.grad for p in model.parameters()]:
    h.update(t.detach().float().cpu().numpy().tobytes())
print(h.hexdigest())
