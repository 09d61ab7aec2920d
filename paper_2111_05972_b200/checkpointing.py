"""Activation checkpointing of the TP transformer stack (Appendix H.2 / J.2;
SPEC.md:529-537 checkpoint_grouping).

``checkpoint_grouping`` is the SPEC's grouping rule, bit-exact on module sequences:
  each        -> singleton groups
  contiguous  -> maximal runs of consecutive modules on the same partition (pp_rank)
  group_k     -> greedy left-to-right blocks of k, broken at partition boundaries

``set_activation_checkpointing(model, strategy)`` applies it to a DistributedTransformer
(or any module holding one): each group of consecutive DistributedTransformerLayers runs its
forward without keeping activations, and its backward recomputes the group's forward first
(re-entrant checkpointing).  Only the group-boundary activation is stored.  The recomputation
reproduces the forward bit for bit: it reuses the forward's dropout step snapshot (the
device-resident Philox step word, state.begin_forward), so masks are identical even when other
microbatches' forwards ran in between (pipeline schedules).
"""
from __future__ import annotations

import re

import torch
import torch.utils.checkpoint as tuc

from .state import STATE


def checkpoint_grouping(modules: list, partitions: list, strategy: str) -> list:
    """group consecutive modules for checkpointing.  Returns a list of lists."""
    if not modules:
        raise ValueError("checkpoint_grouping: empty module sequence")
    if len(partitions) != len(modules):
        raise ValueError("checkpoint_grouping: one partition id per module")
    if strategy == "each":
        return [[m] for m in modules]
    k = None
    if strategy != "contiguous":
        mt = re.fullmatch(r"group_(\d+)", strategy)
        if not mt:
            raise ValueError(f"unknown checkpoint strategy {strategy!r} (each | contiguous | group_k)")
        k = int(mt.group(1))
        if k < 2:
            raise ValueError("group_k needs k >= 2")
    groups, cur = [], [modules[0]]
    for m, p, prev in zip(modules[1:], partitions[1:], partitions[:-1]):
        if p != prev or (k is not None and len(cur) == k):
            groups.append(cur)
            cur = [m]
        else:
            cur.append(m)
    groups.append(cur)
    return groups


class _Group(torch.nn.Module):
    """A run of stack-internal layers executed as one checkpointed unit."""

    def __init__(self, layers, last_in_stack: bool):
        super().__init__()
        self.layers = layers
        self.last_in_stack = last_in_stack

    def run(self, X, mask, rc):
        n = len(self.layers)
        # the group's output is gathered by the next group's first sub-layer (peer push from the
        # last epilogue) -- but only in the original forward: the backward's recomputation runs
        # with grad enabled and its output feeds no later forward
        out_push = not self.last_in_stack and not torch.is_grad_enabled()
        for i, layer in enumerate(self.layers):
            X = layer.sublayer(X, mask, rc, push_last=(i + 1 < n) or out_push)
        return X


def _run_checkpointed(group: _Group, X, mask, rc):
    rng = STATE.rng_cur  # the forward's dropout step snapshot, reused by the recomputation

    def fn(x):
        saved = STATE.rng_cur
        STATE.rng_cur = rng
        try:
            return group.run(x, mask, rc)
        finally:
            STATE.rng_cur = saved

    if not X.requires_grad:  # re-entrant checkpointing only backpropagates through grad inputs
        X = X.detach().requires_grad_(True)
    return tuc.checkpoint(fn, X, use_reentrant=True)


def set_activation_checkpointing(model: torch.nn.Module, strategy: str = "each") -> list:
    """Checkpoint the DistributedTransformer stacks inside `model` with the given grouping strategy
    (every layer of one process lives on the same pipeline partition).  Returns the groups (layer
    ids) per stack.  strategy None / "none" removes checkpointing."""
    from .nn import DistributedTransformer
    applied = []
    for mod in model.modules():
        if not isinstance(mod, DistributedTransformer):
            continue
        if strategy in (None, "none"):
            mod._ckpt_groups = None
            continue
        layers = list(mod.seq_layers)
        groups = checkpoint_grouping(layers, [STATE.pp_rank] * len(layers), strategy)
        mod._ckpt_groups = [_Group(g, last_in_stack=(g[-1] is layers[-1])) for g in groups]
        applied.append([[l.layer_id for l in g] for g in groups])
    return applied


def run_stack(stack, X, mask, rc):
    """DistributedTransformer.sublayer with checkpoint groups (used when _ckpt_groups is set)."""
    for g in stack._ckpt_groups:
        if torch.is_grad_enabled():
            X = _run_checkpointed(g, X, mask, rc)
        else:
            X = g.run(X, mask, rc)
    return X
