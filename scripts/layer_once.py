"""Run a few fwd+bwd steps of one BERT-large TP layer (N=1) — target for ncu captures."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_05972_b200 as smp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--batch", type=int, default=8)
a = ap.parse_args()
smp.init({"tensor_parallel_degree": 1, "optimize": "speed", "seed": 5})
layer = smp.nn.DistributedTransformerLayer(num_attention_heads=16, attention_head_size=64, hidden_size=1024,
                                           intermediate_size=4096, attention_dropout_prob=0.1,
                                           hidden_dropout_prob=0.1, activation="gelu", pre_layernorm=False,
                                           post_layernorm=True)
x = torch.randn(a.batch, 512, 1024, device="cuda", dtype=torch.bfloat16, requires_grad=True)
dy = torch.randn_like(x)
for _ in range(a.iters):
    y = layer(x)
    y.backward(dy)
torch.cuda.synchronize()
print("ok")
