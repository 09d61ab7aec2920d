"""Activation checkpointing: the SPEC's grouping rule (bit-exact, CPU) and, on the
GPU, a checkpointed BERT-style stack that reproduces the plain stack's outputs and gradients bit
for bit (recomputation reuses the forward's dropout step snapshot) and matches the oracle."""
import pytest
import torch

from paper_2111_05972_b200.checkpointing import checkpoint_grouping


def test_grouping_spec_examples():
    # [a,b | c,d] on partitions [0,0,1,1], contiguous -> {a,b},{c,d}
    assert checkpoint_grouping(list("abcd"), [0, 0, 1, 1], "contiguous") == [["a", "b"], ["c", "d"]]
    # [a,b] on 0, [c,d,e] on 1, group_3 -> {a,b},{c,d,e}
    assert checkpoint_grouping(list("abcde"), [0, 0, 1, 1, 1], "group_3") == [["a", "b"], ["c", "d", "e"]]
    # each on 3 modules -> 3 singleton groups
    assert checkpoint_grouping(list("abc"), [0, 0, 0], "each") == [["a"], ["b"], ["c"]]


def test_grouping_greedy_blocks_and_errors():
    assert checkpoint_grouping(list("abcdefg"), [0] * 7, "group_2") == [["a", "b"], ["c", "d"], ["e", "f"], ["g"]]
    assert checkpoint_grouping(list("abcde"), [0, 0, 0, 1, 1], "group_2") == [["a", "b"], ["c"], ["d", "e"]]
    assert checkpoint_grouping(list("abc"), [2, 2, 2], "contiguous") == [["a", "b", "c"]]
    for bad in ("group_1", "groups_2", "all"):
        with pytest.raises(ValueError):
            checkpoint_grouping(list("ab"), [0, 0], bad)
    with pytest.raises(ValueError):
        checkpoint_grouping([], [], "each")


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["each", "group_2", "contiguous"])
def test_checkpointed_stack_matches_plain_and_oracle(strategy):
    import paper_2111_05972_b200 as smp
    from oracle import tp
    L, nh, dh, H, I, s = 3, 4, 64, 256, 1024, 128
    cfg = tp.LayerConfig(num_attention_heads=nh, attention_head_size=dh, hidden_size=H, intermediate_size=I,
                         attention_dropout_prob=0.1, hidden_dropout_prob=0.1)
    params = [{k: v.to(torch.bfloat16).double() for k, v in tp.init_layer_params(cfg, seed=30 + l).items()}
              for l in range(L)]
    g = torch.Generator().manual_seed(0)
    x = torch.randn(2, s, H, generator=g).to(torch.bfloat16)
    dy = torch.randn(2, s, H, generator=g).to(torch.bfloat16)
    outs = []
    for ckpt in (False, True):
        smp.init({"tensor_parallel_degree": 1, "optimize": "speed", "seed": 7})
        model = smp.nn.DistributedTransformer(num_layers=L, num_attention_heads=nh, attention_head_size=dh,
                                              hidden_size=H, intermediate_size=I, attention_dropout_prob=0.1,
                                              hidden_dropout_prob=0.1)
        for l, lay in enumerate(model.seq_layers):
            lay.load_full({k: v.to(torch.bfloat16) for k, v in params[l].items()})
        if ckpt:
            groups = smp.set_activation_checkpointing(model, strategy)
            assert groups and sum(len(gr) for gr in groups[0]) == L
        xg = x.cuda().requires_grad_(True)
        y = model(xg)
        y.backward(dy.cuda())
        torch.cuda.synchronize()
        outs.append((y.detach().cpu(), xg.grad.cpu(), model.seq_layers[0].attention.qkv_weight.grad.cpu(),
                     model.seq_layers[-1].output.fc2_weight.grad.cpu()))
        smp.reset()
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    xr = x.double().requires_grad_(True)
    yr = tp.transformer_ref(xr, [{k: v.clone() for k, v in p.items()} for p in params], cfg, None, seed=7)
    yr.backward(dy.double())
    rel = lambda a, b: ((a.double() - b).norm() / b.norm()).item()  # noqa: E731
    assert rel(outs[1][0], yr.detach()) < 2e-2 and rel(outs[1][1], xr.grad) < 2e-2
