"""Module replacement: smp.DistributedModel, smp.tp_register, smp.tp_register_with_module,
smp.tensor_parallelism, smp.set_tensor_parallelism.

A module is replaced by its distributed implementation iff (SPEC.md:485-494
plan_replacement):
  (1) a distributed implementation is registered for its class,
  (2) tensor parallelism is enabled for it (directly, or via an enabled ancestor /
      an enclosing ``smp.tensor_parallelism()`` scope at construction),
  (3) no ancestor is already replaced, and
  (4) it shares no parameter with any module outside its own subtree.
The scan is deterministic and top-down (named_children order).  Built-in lookup table:
nn.Linear -> DistributedLinear, nn.Embedding -> DistributedEmbedding.
"""
from __future__ import annotations

import contextlib
import functools
import weakref

import torch
from torch import nn

_REGISTRY: dict = {}  # module class -> (dist class, init_hook, forward_hook, return_hook)
_ENABLED = weakref.WeakSet()
_DISABLED = weakref.WeakSet()
_SCOPE = [False]


def tp_register(dist_module, init_hook=None, forward_hook=None, return_hook=None):
    """Class decorator registering `dist_module` for the decorated class."""

    def deco(cls):
        _wrap_init(cls)
        _REGISTRY[cls] = (dist_module, init_hook, forward_hook, return_hook)
        return cls

    return deco


def tp_register_with_module(module_cls, dist_module, init_hook=None, forward_hook=None, return_hook=None):
    """Register `dist_module` for an existing module class."""
    _wrap_init(module_cls)
    _REGISTRY[module_cls] = (dist_module, init_hook, forward_hook, return_hook)


def _wrap_init(cls):
    if getattr(cls.__init__, "_smp_wrapped", False):
        return
    orig = cls.__init__

    @functools.wraps(orig)
    def init(self, *args, **kwargs):
        orig(self, *args, **kwargs)
        if type(self) is cls:
            self._smp_init_args = (args, kwargs)
        if _SCOPE[0]:
            _ENABLED.add(self)

    init._smp_wrapped = True
    cls.__init__ = init


@contextlib.contextmanager
def tensor_parallelism(enabled: bool = True):
    """Modules constructed inside the scope are marked for tensor parallelism."""
    prev = _SCOPE[0]
    _SCOPE[0] = enabled
    orig = nn.Module.__init__

    def init(self, *a, **k):
        orig(self, *a, **k)
        if _SCOPE[0]:
            _ENABLED.add(self)

    nn.Module.__init__ = init
    try:
        yield
    finally:
        nn.Module.__init__ = orig
        _SCOPE[0] = prev


def set_tensor_parallelism(module: nn.Module, enabled: bool = True) -> None:
    """Mark (or unmark) a module and its subtree for tensor parallelism."""
    (_ENABLED if enabled else _DISABLED).add(module)
    (_DISABLED if enabled else _ENABLED).discard(module)


def _builtin(cls):
    from . import nn as snn
    if cls is nn.Linear:
        return (snn.DistributedLinear, None, None, None)
    if cls is nn.Embedding:
        return (snn.DistributedEmbedding, None, None, None)
    return None


def _lookup(mod):
    for cls in type(mod).__mro__:
        if cls in _REGISTRY:
            return _REGISTRY[cls]
    return _builtin(type(mod))


def plan_replacement(model: nn.Module) -> list:
    """Names (dotted paths) of the modules that will be replaced, in scan order."""
    owners: dict = {}
    for name, m in model.named_modules():
        for p in m.parameters(recurse=False):
            owners.setdefault(id(p), set()).add(name)
    out = []

    def subtree_names(prefix, mod):
        return {prefix + ("." if prefix and n else "") + n for n, _ in mod.named_modules()}

    def visit(name, mod, enabled, under):
        en = (enabled or mod in _ENABLED) and mod not in _DISABLED
        take = False
        if not under and en and _lookup(mod) is not None:
            sub = subtree_names(name, mod)
            shared = any(not owners[id(p)] <= sub for p in mod.parameters())
            take = not shared
        if take:
            out.append(name)
        for cname, child in mod.named_children():
            visit(f"{name}.{cname}" if name else cname, child, en, under or take)

    visit("", model, False, False)
    return out


def _make_dist(mod):
    dist_cls, init_hook, fwd_hook, ret_hook = _lookup(mod)
    if isinstance(mod, nn.Linear):
        d = dist_cls(mod.in_features, mod.out_features, bias=mod.bias is not None)
        d.load_full(mod.weight.detach().to(d.weight.device), None if mod.bias is None else mod.bias.detach().to(
            d.weight.device))
    elif isinstance(mod, nn.Embedding):
        d = dist_cls(mod.num_embeddings, mod.embedding_dim, padding_idx=mod.padding_idx)
        d.load_full(mod.weight.detach().to(d.weight.device))
    else:
        args, kwargs = getattr(mod, "_smp_init_args", ((), {}))
        if init_hook is not None:
            args, kwargs = init_hook(*args, **kwargs)
        d = dist_cls(*args, **kwargs)
    if fwd_hook is not None or ret_hook is not None:
        inner = d.forward

        def forward(*a, **k):
            if fwd_hook is not None:
                a, k = fwd_hook(*a, **k)
            out = inner(*a, **k)
            return ret_hook(out) if ret_hook is not None else out

        d.forward = forward
    return d


class DistributedModel(nn.Module):
    """smp.DistributedModel(model): replace eligible submodules with their distributed versions."""

    def __init__(self, model: nn.Module):
        super().__init__()
        self.replaced = plan_replacement(model)
        for name in self.replaced:
            if name == "":
                model = _make_dist(model)
                continue
            parent_name, _, leaf = name.rpartition(".")
            parent = model.get_submodule(parent_name) if parent_name else model
            setattr(parent, leaf, _make_dist(getattr(parent, leaf)))
        self.module = model

    def forward(self, *args, **kwargs):
        return self.module(*args, **kwargs)
