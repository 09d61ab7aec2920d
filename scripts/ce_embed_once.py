"""Vocab-parallel cross-entropy fwd+bwd and the vocabulary embedding lookup + sorted backward at
the GPT-1.3B bench shape (16384 tokens, V = 50257 -> 50304, H = 2048), a few times (ncu target;
dev tool).  usage: python scripts/ce_embed_once.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_05972_b200 as smp  # noqa: E402
from paper_2111_05972_b200 import embedding as E  # noqa: E402

smp.init({"tensor_parallel_degree": 1, "seed": 3})
N, V, H = 16384, 50257, 2048
Vp = 50304
logits = (torch.randn(N, Vp, device="cuda") * 2).bfloat16()
logits[:, V:] = float("-inf")
logits.requires_grad_(True)
tgt = torch.randint(0, V, (N,), device="cuda")
emb = E.VocabParallelEmbedding(V, H)
ids = torch.randint(0, V, (8, 2048), device="cuda")
for _ in range(3):
    loss = E.vocab_parallel_cross_entropy(logits, tgt, V)
    loss.sum().backward()
    y = emb(ids)
    y.float().sum().backward()
torch.cuda.synchronize()
print("ok", float(loss.mean()))
