"""smp module-replacement rules on torch modules, CPU-only:
the SPEC's three plan_replacement examples plus the tp_register hooks."""
import torch
from torch import nn

import paper_2111_05972_b200 as smp
from paper_2111_05972_b200 import replace as R


class Block(nn.Module):
    def __init__(self, d):
        super().__init__()
        self.inner = nn.Linear(d, d)

    def forward(self, x):
        return self.inner(x)


class DistBlock(nn.Module):
    def __init__(self, d):
        super().__init__()
        self.d = d


def setup_function(_):
    R._REGISTRY.clear()


def test_parent_and_child_registered_only_parent_replaced():
    smp.tp_register_with_module(Block, DistBlock)
    with smp.tensor_parallelism():
        m = nn.Sequential(Block(4))
    assert smp.plan_replacement(m) == ["0"]


def test_shared_parameter_skipped():
    a, b = nn.Linear(4, 4), nn.Linear(4, 4)
    b.weight = a.weight
    m = nn.Sequential(a, b)
    smp.set_tensor_parallelism(m)
    assert smp.plan_replacement(m) == []


def test_registered_not_enabled_skipped():
    m = nn.Sequential(nn.Linear(4, 4))
    assert smp.plan_replacement(m) == []
    smp.set_tensor_parallelism(m[0])
    assert smp.plan_replacement(m) == ["0"]
    smp.set_tensor_parallelism(m[0], False)
    assert smp.plan_replacement(m) == []


def test_tp_register_hooks_record_init_args():
    calls = {}

    def init_hook(d):
        calls["init"] = d
        return (d * 2,), {}

    @smp.tp_register(DistBlock, init_hook=init_hook)
    class MyBlock(nn.Module):
        def __init__(self, d):
            super().__init__()
            self.lin = nn.Linear(d, d)

    with smp.tensor_parallelism():
        mb = MyBlock(3)
    assert mb._smp_init_args == ((3,), {})
    m = nn.Sequential(mb)
    assert smp.plan_replacement(m) == ["0"]
    dm = smp.DistributedModel(m)
    assert isinstance(dm.module[0], DistBlock) and dm.module[0].d == 6 and calls["init"] == 3
