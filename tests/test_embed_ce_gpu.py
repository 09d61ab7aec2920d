"""Embeddings, DistributedLinear, vocab-parallel CE and the LM head on one B200 vs the CPU oracle."""
import math

import pytest
import torch

from oracle import tp

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = a.double().cpu(), b.double().cpu()
    return ((a - b).norm() / max(b.norm().item(), 1e-30)).item()


@pytest.fixture(autouse=True)
def smp1():
    import paper_2111_05972_b200 as smp
    smp.init({"tensor_parallel_degree": 1, "optimize": "speed", "seed": 2})
    yield smp
    smp.reset()


def test_embed_lookup_routing_bit_exact(smp1):
    from paper_2111_05972_b200 import embedding as E
    g = torch.Generator().manual_seed(0)
    V, D = 1000, 96
    table = torch.randn(V, D, generator=g).to(torch.bfloat16)
    ids = torch.randint(0, V, (7, 33), generator=g)
    out = E.embed_lookup(ids.cuda(), table.cuda(), row_offset=0, vocab=V)
    assert torch.equal(out.cpu(), table[ids.reshape(-1)])  # pure routing: bit-exact
    # vocab-parallel masked lookup of rows [300, 600)
    part = E.embed_lookup(ids.cuda(), table[300:600].contiguous().cuda(), row_offset=300, vocab=V)
    own = (ids.reshape(-1) >= 300) & (ids.reshape(-1) < 600)
    ref = torch.where(own[:, None], table[ids.reshape(-1)], torch.zeros(1, D, dtype=torch.bfloat16))
    assert torch.equal(part.cpu(), ref)


def test_embed_oob_reports_position(smp1):
    from paper_2111_05972_b200 import embedding as E
    from paper_2111_05972_b200.errors import IndexOutOfRangeError
    table = torch.zeros(4, 8, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(IndexOutOfRangeError, match="position 2") as ei:
        E.embed_lookup(torch.tensor([0, 3, 4, 1], device="cuda"), table, row_offset=0, vocab=4, check=True)
    assert ei.value.position == 2


@pytest.mark.parametrize("D", [64, 2048, 5120])
def test_embed_grad_deterministic(smp1, D):
    from paper_2111_05972_b200 import embedding as E
    g = torch.Generator().manual_seed(D)
    V, n = 300, 5000
    ids = torch.randint(0, V, (n,), generator=g)
    ids[:50] = 7  # heavy collisions on one row
    dy = torch.randn(n, D, generator=g).to(torch.bfloat16)
    got = E.embed_grad(ids.cuda(), dy.cuda(), rows=V, row_offset=0, padding_idx=3, out_dtype=torch.float32)
    ref = torch.zeros(V, D, dtype=torch.float64).index_add_(0, ids, dy.double())
    ref[3] = 0
    assert rel(got, ref) < 1e-5
    again = E.embed_grad(ids.cuda(), dy.cuda(), rows=V, row_offset=0, padding_idx=3, out_dtype=torch.float32)
    assert torch.equal(got, again)


@pytest.mark.parametrize("case", [
    # rows, D, n, row_offset, padding, hot-row repeats, out dtype, accumulate, method
    (300, 64, 5000, 0, 3, 50, torch.float32, False, "scan"),
    (300, 8, 5000, 0, 3, 3000, torch.float32, False, "sort"),      # one run spanning ~100 windows
    (12000, 64, 70000, 5000, 5123, 9000, torch.float32, True, "sort"),  # vocab shard: ids outside skipped
    (50304, 2048, 16384, 0, None, 700, torch.bfloat16, False, "sort"),  # GPT-1.3B tied table
    (1 << 20, 16, 300000, 0, None, 20000, torch.float32, True, "sort"),  # 3 radix passes
    ((1 << 17) + 3, 8, 200000, 0, None, 5000, torch.float32, False, "sort"),  # 18-bit keys: two 9-bit passes
])
def test_embed_grad_sorted_vs_oracle(smp1, case):
    """Sort-based deterministic scatter-add (csrc/embed_sort.cu) vs an fp64 index_add: vocab-shard
    routing (ids outside [row_offset, row_offset+rows) contribute nothing), padding row, a hot row
    whose run crosses many segment windows, accumulate into an existing buffer, bit-identical
    reruns."""
    from paper_2111_05972_b200 import embedding as E
    rows, D, n, off, pad, hot, odt, acc, method = case
    g = torch.Generator().manual_seed(rows + D)
    ids = torch.randint(0, rows + 2 * off if off else rows, (n,), generator=g)
    ids[torch.randperm(n, generator=g)[:hot]] = off + 7 if rows > 7 else off
    if pad is not None:
        ids[::97] = pad
    dy = torch.randn(n, D, generator=g).to(torch.bfloat16)
    base = torch.randn(rows, D, generator=g).to(odt)
    out = base.clone().cuda() if acc else None
    got = E.embed_grad(ids.cuda(), dy.cuda(), rows=rows, row_offset=off, padding_idx=pad, out_dtype=odt, out=out,
                       accumulate=acc, method=method)
    loc = ids - off
    keep = (loc >= 0) & (loc < rows)
    if pad is not None:
        keep &= ids != pad
    ref = torch.zeros(rows, D, dtype=torch.float64).index_add_(0, loc[keep], dy[keep].double())
    if acc:
        ref += base.double()
    tol = 1e-5 if odt == torch.float32 else 1e-2
    assert rel(got, ref) < tol
    out2 = base.clone().cuda() if acc else None
    again = E.embed_grad(ids.cuda(), dy.cuda(), rows=rows, row_offset=off, padding_idx=pad, out_dtype=odt, out=out2,
                         accumulate=acc, method=method)
    assert torch.equal(got, again)


@pytest.mark.parametrize("V,N", [(4096, 300), (50257, 256), (1000, 37)])
def test_vocab_ce_tp1(smp1, V, N):
    from paper_2111_05972_b200.embedding import vocab_padded, vocab_parallel_cross_entropy
    Vp = vocab_padded(V, 1)
    g = torch.Generator().manual_seed(V)
    logits = (torch.randn(N, Vp, generator=g) * 3).to(torch.bfloat16)
    tgt = torch.randint(0, V, (N,), generator=g)
    tgt[1] = -100
    lg = logits.cuda().requires_grad_(True)
    loss = vocab_parallel_cross_entropy(lg, tgt.cuda(), V)
    gl = torch.randn(N, generator=g)
    loss.backward(gl.cuda())
    lr = logits.double().requires_grad_(True)
    ref = tp.cross_entropy_ref(lr, tgt, V)
    (ref * gl.double()).sum().backward()
    assert rel(loss, ref) < 1e-4
    assert float(loss[1]) == 0.0
    assert rel(lg.grad, lr.grad) < 1e-2


def test_distributed_linear_tp1(smp1):
    smp = smp1
    g = torch.Generator().manual_seed(1)
    W, b = (torch.randn(384, 256, generator=g) * 0.05).to(torch.bfloat16), torch.randn(384, generator=g).to(
        torch.bfloat16)
    x = torch.randn(3, 40, 256, generator=g).to(torch.bfloat16)
    dy = torch.randn(3, 40, 384, generator=g).to(torch.bfloat16)
    lin = smp.nn.DistributedLinear(256, 384)
    lin.load_full(W.cuda(), b.cuda())
    xg = x.cuda().requires_grad_(True)
    y = lin(xg)
    y.backward(dy.cuda())
    Ws, bs = tp.shard_linear(W.double(), b.double(), 1)
    ys, saved = tp.dist_linear_forward([x.double().reshape(-1, 256)], Ws, bs)
    dxs, dWs, db = tp.dist_linear_backward([dy.double().reshape(-1, 384)], Ws, saved)
    assert rel(y.reshape(-1, 384), ys[0]) < 1e-2
    assert rel(xg.grad.reshape(-1, 256), dxs[0]) < 1e-2
    assert rel(lin.weight.grad, dWs[0]) < 1e-2 and rel(lin.bias.grad, db) < 1e-2


def test_distributed_embedding_tp1(smp1):
    smp = smp1
    g = torch.Generator().manual_seed(2)
    E = torch.randn(50, 32, generator=g).to(torch.bfloat16)
    emb = smp.nn.DistributedEmbedding(50, 32)
    emb.load_full(E.cuda())
    ids = torch.randint(0, 50, (4, 9), generator=g)
    out = emb(ids.cuda())
    assert torch.equal(out.cpu(), E[ids])
    out.backward(torch.ones_like(out))
    ref = torch.zeros(50, 32, dtype=torch.float64).index_add_(0, ids.reshape(-1), torch.ones(36, 32, dtype=torch.float64))
    assert rel(emb.weight.grad, ref) < 1e-2


def test_lm_head_gpt_tiny_vs_oracle(smp1):
    """configs[0]-shaped GPT: 2 layers, H=256, 4 heads, s=128, V=4096, pre-LN + final LN, tied LM head."""
    smp = smp1
    L, nh, dh, H, I, V, s, B = 2, 4, 64, 256, 1024, 4096, 128, 2
    model = smp.nn.DistributedTransformerLMHead(num_layers=L, num_attention_heads=nh, attention_head_size=dh,
                                                hidden_size=H, intermediate_size=I, vocab_size=V, num_positions=s,
                                                attention_dropout_prob=0.0, hidden_dropout_prob=0.0,
                                                activation="gelu_tanh", causal_mask_size=s, pre_layernorm=True,
                                                post_layernorm=False)
    cfg = tp.LayerConfig(num_attention_heads=nh, attention_head_size=dh, hidden_size=H, intermediate_size=I,
                         activation="gelu_tanh", causal_mask_size=s, pre_layernorm=True, post_layernorm=False)
    g = torch.Generator().manual_seed(0)
    params = [{k: v.to(torch.bfloat16).double() for k, v in tp.init_layer_params(cfg, seed=10 + l).items()}
              for l in range(L)]
    Emb = (torch.randn(V, H, generator=g) * 0.02).to(torch.bfloat16).double()
    wpe = (torch.randn(s, H, generator=g) * 0.02).to(torch.bfloat16).double()
    for l, lay in enumerate(model.transformer.seq_layers):
        lay.load_full({k: v.to(torch.bfloat16) for k, v in params[l].items()})
    model.word_embedding.load_full(Emb.to(torch.bfloat16).cuda())
    with torch.no_grad():
        model.position_embedding.copy_(wpe.to(torch.bfloat16))
    ids = torch.randint(0, V, (B, s), generator=g)
    labels = torch.roll(ids, -1, 1)
    labels[:, -1] = -100
    loss = model(ids.cuda(), labels=labels.cuda())
    loss.sum().backward()

    pr = [{k: v.clone().requires_grad_(True) for k, v in p.items()} for p in params]
    Er, wr = Emb.clone().requires_grad_(True), wpe.clone().requires_grad_(True)
    h = Er[ids] + wr[None]
    for l in range(L):
        h = tp.transformer_layer_ref(h, pr[l], cfg, None, None)
    h = tp.layer_norm(h, torch.ones(H, dtype=torch.float64), torch.zeros(H, dtype=torch.float64), 1e-5)
    logits = h @ Er.t()
    ref = tp.cross_entropy_ref(logits.reshape(-1, V), labels.reshape(-1), V).reshape(B, s)
    ref.sum().backward()
    assert rel(loss, ref) < 1e-2, rel(loss, ref)
    assert rel(model.word_embedding.weight.grad[:V], Er.grad) < 2e-2
    assert rel(model.position_embedding.grad, wr.grad) < 2e-2
    a = model.transformer.seq_layers[0].attention
    wq, wk, wv = pr[0]["wqkv"].grad.split(H, 0)
    assert rel(a.qkv_weight.grad, torch.cat([wq, wk, wv], 0)) < 2e-2
