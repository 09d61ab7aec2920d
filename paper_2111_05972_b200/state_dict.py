"""state_dict / local_state_dict of the TP modules ("local_state_dict ... state_dict";
Appendix J: smp.DistributedModel.state_dict gathers the full model, local_state_dict keeps shards).

``local_state_dict(model)`` is the rank's own shards (torch's state_dict of the smp.nn modules)
plus the TP coordinates needed to reload them.  ``full_state_dict(model)`` all-gathers every
TP-sharded parameter over the TP group and undoes the shard layout, returning the unsharded
tensors in the reference layout that ``load_full`` consumes (wqkv = [q; k; v] [3H, H], wo [H, H],
w1 [I, H], w2 [H, I], vocab tables [V, D], ...), on every rank.  Both TP modes are handled:
speed mode (Megatron column/row shards) and memory mode (input-split linears with rank-major
QKV rows, channel-chunked biases and LayerNorms).
"""
from __future__ import annotations

import torch

from . import collectives as C
from .state import STATE


def _ag(t: torch.Tensor, dim: int) -> torch.Tensor:
    """All-gather a shard over the TP group, concatenated along dim (identity at T == 1)."""
    return C.all_gather(t.detach().contiguous(), dim) if STATE.tp_size > 1 else t.detach().clone()


def _attention_full(a, out: dict) -> None:
    T, H = STATE.tp_size, a.hidden_size
    hs = H // T
    if a._memory:
        # qkv_weight [3H, H/T]: rows rank-major (q_r | k_r | v_r), this rank's input channels
        perm = _ag(a.qkv_weight, 1)  # [3H, H]
        blocks = perm.view(T, 3, hs, H)
        out["wqkv"] = torch.cat([blocks[:, i].reshape(H, H) for i in range(3)], 0)
        out["bo"] = _ag(a.dense_bias, 0)
    else:
        g = _ag(a.qkv_weight, 0).view(T, 3, hs, H)  # rank-major [q_j; k_j; v_j]
        out["wqkv"] = torch.cat([g[:, i].reshape(H, H) for i in range(3)], 0)
        out["bo"] = a.dense_bias.detach().clone()
    gb = _ag(a.qkv_bias, 0).view(T, 3, hs)
    out["bqkv"] = torch.cat([gb[:, i].reshape(H) for i in range(3)], 0)
    out["wo"] = _ag(a.dense_weight, 1)
    for where in ("pre", "post"):
        w = getattr(a, f"{where}_ln_weight")
        if w is not None:
            out[f"attn_{where}_ln_w"] = _ag(w, 0) if a._memory else w.detach().clone()
            out[f"attn_{where}_ln_b"] = (_ag(getattr(a, f"{where}_ln_bias"), 0) if a._memory
                                         else getattr(a, f"{where}_ln_bias").detach().clone())


def _mlp_full(o, out: dict) -> None:
    out["b1"] = _ag(o.fc1_bias, 0)
    out["w2"] = _ag(o.fc2_weight, 1)
    if o._memory:
        out["w1"] = _ag(o.fc1_weight, 1)
        out["b2"] = _ag(o.fc2_bias, 0)
    else:
        out["w1"] = _ag(o.fc1_weight, 0)
        out["b2"] = o.fc2_bias.detach().clone()
    for where in ("pre", "post"):
        w = getattr(o, f"{where}_ln_weight")
        if w is not None:
            out[f"mlp_{where}_ln_w"] = _ag(w, 0) if o._memory else w.detach().clone()
            out[f"mlp_{where}_ln_b"] = (_ag(getattr(o, f"{where}_ln_bias"), 0) if o._memory
                                        else getattr(o, f"{where}_ln_bias").detach().clone())


def full_state_dict(model: torch.nn.Module) -> dict:
    """Unsharded parameters of every smp.nn module inside `model` (collective over the TP group:
    every TP rank must call it).  Keys are '<module path>.<reference name>'."""
    from . import nn as N
    from .embedding import DistributedEmbedding, VocabParallelEmbedding
    out = {}
    for name, mod in model.named_modules():
        pre = f"{name}." if name else ""
        if isinstance(mod, N.DistributedTransformerLayer):
            d = {}
            _attention_full(mod.attention, d)
            _mlp_full(mod.output, d)
            out.update({pre + k: v for k, v in d.items()})
        elif isinstance(mod, N.DistributedLinear):
            out[pre + "weight"] = _ag(mod.weight, 1)
            if STATE.tp_size == 1 or STATE.tp_rank == 0:
                b = mod.bias.detach().clone() if mod.bias is not None else None
            else:
                b = None
            if STATE.tp_size > 1:  # the bias lives on tp_rank 0: broadcast it
                import torch.distributed as dist
                flag = torch.tensor([1 if b is not None else 0], device=mod.weight.device)
                dist.broadcast(flag, STATE.tp_group_ranks[0], group=STATE.tp_group)
                if flag.item():
                    if b is None:
                        b = torch.empty(mod.out_features, dtype=mod.weight.dtype, device=mod.weight.device)
                    dist.broadcast(b, STATE.tp_group_ranks[0], group=STATE.tp_group)
            if b is not None:
                out[pre + "bias"] = b
        elif isinstance(mod, VocabParallelEmbedding):
            out[pre + "weight"] = _ag(mod.weight, 0)[:mod.num_embeddings]
        elif isinstance(mod, DistributedEmbedding):
            out[pre + "weight"] = _ag(mod.weight, 1)
        elif isinstance(mod, N.DistributedLayerNorm):
            out[pre + "weight"] = mod.weight.detach().clone()
            out[pre + "bias"] = mod.bias.detach().clone()
        elif isinstance(mod, N.DistributedTransformerLMHead):
            out[pre + "position_embedding"] = mod.position_embedding.detach().clone()
    return out


def local_state_dict(model: torch.nn.Module) -> dict:
    """This rank's shards (no communication) + the TP coordinates they belong to."""
    sd = {k: v.detach().clone() for k, v in model.state_dict().items()}
    sd["_smp_tp"] = torch.tensor([STATE.tp_rank, STATE.tp_size, STATE.pp_rank, STATE.pp_size])
    return sd


def load_local_state_dict(model: torch.nn.Module, sd: dict) -> None:
    """Reload shards saved by local_state_dict on the same TP / PP coordinates."""
    coords = sd.get("_smp_tp")
    want = [STATE.tp_rank, STATE.tp_size, STATE.pp_rank, STATE.pp_size]
    if coords is not None and coords.tolist() != want:
        raise ValueError(f"local_state_dict was saved at (tp_rank, tp_size, pp_rank, pp_size) = {coords.tolist()}, "
                         f"this rank is {want}")
    model.load_state_dict({k: v for k, v in sd.items() if k != "_smp_tp"})
