"""Data parallelism around the TP path: reduced-data-parallel (RDP) gradient allreduce and the
optimizer-state-sharded AdamW ("gradients ... allreduced across the RDP group",
:765 shard_optimizer_state; SPEC.md:541 MemoryConfig; topology.py:55-59 the RDP group).

The RDP group of a rank is the set of ranks with the same (pp_rank, tp_rank): they hold identical
parameter shards and different samples, so their gradients are averaged.  (TP-replicated
parameters -- LayerNorms, row-parallel biases -- are already summed over the TP group inside the
layers' backward.)

* ``GradBuckets`` flattens the gradients of a parameter list into fixed fp32 buckets (a
  deterministic, size-bounded partition in parameter order) and all-reduces them bucket by
  bucket, optionally launched from post-accumulate-grad hooks so a bucket's NCCL allreduce
  overlaps the rest of the backward (``overlap=True``).
* ``DistributedAdam`` keeps fp32 master weights and Adam moments.  With
  ``shard_optimizer_state`` each RDP rank owns 1/|RDP| of the flattened parameters: the bucket
  gradient is reduce-scattered, the rank updates its slice with the fused ``smpk_adam_step``
  kernel and the bf16 slices are all-gathered back into the model (ZeRO stage 1: no gradient or
  parameter sharding, SPEC.md:565 non-goal).  Without sharding every rank allreduces and updates
  everything.  Collectives run on the RDP process group (NCCL over NVLink on one node).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import _lib
from .kernels import _stream
from .state import STATE

ALIGN = 64  # elements: keeps every rank's slice 256-B aligned


def _world(group) -> int:
    return dist.get_world_size(group) if (group is not None and dist.is_initialized()) else 1


def _rank(group) -> int:
    return dist.get_rank(group) if (group is not None and dist.is_initialized()) else 0


def plan_buckets(numels: list, bucket_elems: int) -> list:
    """Consecutive parameter index ranges whose total size stays <= bucket_elems (a parameter
    larger than a bucket gets its own).  Deterministic: identical on every rank."""
    out, start, acc = [], 0, 0
    for i, n in enumerate(numels):
        if acc and acc + n > bucket_elems:
            out.append((start, i))
            start, acc = i, 0
        acc += n
    if numels:
        out.append((start, len(numels)))
    return out


class GradBuckets:
    """Bucketed gradient allreduce (average) over a process group."""

    def __init__(self, params, group=None, bucket_bytes: int = 64 << 20, overlap: bool = False):
        self.params = [p for p in params if p.requires_grad]
        self.group = group if group is not None else STATE.rdp_group
        self.W = _world(self.group)
        self.buckets = plan_buckets([p.numel() for p in self.params], max(1, bucket_bytes // 4))
        self._pending = []
        self._hooks = []
        if overlap and self.W > 1:
            self._count = [0] * len(self.buckets)
            owner = {}
            for b, (lo, hi) in enumerate(self.buckets):
                for i in range(lo, hi):
                    owner[id(self.params[i])] = b
            for p in self.params:
                self._hooks.append(p.register_post_accumulate_grad_hook(
                    lambda q, b=owner[id(p)]: self._ready(b)))

    def _flat(self, b):
        lo, hi = self.buckets[b]
        ps = self.params[lo:hi]
        return ps, torch.cat([(p.grad if p.grad is not None else torch.zeros_like(p)).float().reshape(-1) for p in ps])

    def _launch(self, b):
        ps, flat = self._flat(b)
        work = dist.all_reduce(flat, group=self.group, async_op=True)
        self._pending.append((ps, flat, work))

    def _ready(self, b):
        self._count[b] += 1
        lo, hi = self.buckets[b]
        if self._count[b] == hi - lo:  # every gradient of the bucket is final: reduce it now
            self._count[b] = 0
            self._launch(b)

    def finish(self):
        """Wait for the launched allreduces (launching any not yet started) and write the averaged
        gradients back.  Call after backward."""
        if self.W == 1:
            return
        if not self._hooks:
            for b in range(len(self.buckets)):
                self._launch(b)
        for ps, flat, work in self._pending:
            work.wait()
            flat.div_(self.W)
            off = 0
            for p in ps:
                n = p.numel()
                if p.grad is None:
                    p.grad = torch.zeros_like(p)
                p.grad.copy_(flat[off:off + n].view_as(p))
                off += n
        self._pending = []

    def remove(self):
        for h in self._hooks:
            h.remove()
        self._hooks = []


def adam_step_cuda(master, param_bf16, grad, m, v, *, lr, betas, eps, weight_decay, step, grad_scale):
    """The fused smpk_adam_step kernel on one contiguous slice."""
    n = master.numel()
    _lib.call("smpk_adam_step", master.data_ptr(), param_bf16.data_ptr(), grad.data_ptr(), m.data_ptr(),
              v.data_ptr(), n, float(lr), float(betas[0]), float(betas[1]), float(eps), float(weight_decay),
              int(step), float(grad_scale), _stream())


class DistributedAdam:
    """AdamW over the RDP group with optional optimizer-state sharding (ZeRO-1)."""

    def __init__(self, params, lr=1e-4, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.0, group=None,
                 shard_optimizer_state: bool | None = None, update_fn=None):
        self.params = [p for p in params if p.requires_grad]
        self.lr, self.betas, self.eps, self.wd = lr, betas, eps, weight_decay
        self.group = group if group is not None else STATE.rdp_group
        self.W, self.r = _world(self.group), _rank(self.group)
        if shard_optimizer_state is None:
            shard_optimizer_state = bool(STATE.config.get("shard_optimizer_state", False))
        self.shard = shard_optimizer_state and self.W > 1
        self.update_fn = update_fn or adam_step_cuda
        self.numels = [p.numel() for p in self.params]
        total = sum(self.numels)
        q = ALIGN * self.W
        self.padded = (total + q - 1) // q * q
        self.per = self.padded // self.W if self.shard else self.padded
        dev = self.params[0].device if self.params else torch.device("cpu")
        flat = torch.zeros(self.padded, dtype=torch.float32, device=dev)
        off = 0
        with torch.no_grad():
            for p, n in zip(self.params, self.numels):
                flat[off:off + n] = p.detach().float().reshape(-1)
                off += n
        lo = self.r * self.per if self.shard else 0
        self.master = flat[lo:lo + self.per].clone()
        self.m = torch.zeros_like(self.master)
        self.v = torch.zeros_like(self.master)
        self.step_count = 0

    def _flat_grads(self):
        g = torch.zeros(self.padded, dtype=torch.float32, device=self.master.device)
        off = 0
        for p, n in zip(self.params, self.numels):
            if p.grad is not None:
                g[off:off + n] = p.grad.float().reshape(-1)
            off += n
        return g

    @torch.no_grad()
    def step(self):
        self.step_count += 1
        g = self._flat_grads()
        if self.W > 1:
            if self.shard:  # each rank keeps the sum of its slice only
                mine = torch.empty(self.per, dtype=torch.float32, device=g.device)
                dist.reduce_scatter_tensor(mine, g, group=self.group)
                g = mine
            else:
                dist.all_reduce(g, group=self.group)
        new_bf16 = torch.empty(self.per, dtype=torch.bfloat16, device=g.device)
        self.update_fn(self.master, new_bf16, g, self.m, self.v, lr=self.lr, betas=self.betas, eps=self.eps,
                       weight_decay=self.wd, step=self.step_count, grad_scale=1.0 / self.W)
        if self.shard:
            full = torch.empty(self.padded, dtype=torch.bfloat16, device=g.device)
            dist.all_gather_into_tensor(full, new_bf16, group=self.group)
        else:
            full = new_bf16
        off = 0
        for p, n in zip(self.params, self.numels):
            p.copy_(full[off:off + n].view_as(p).to(p.dtype))
            off += n

    def zero_grad(self):
        for p in self.params:
            p.grad = None

    def state_bytes(self) -> int:
        """Optimizer bytes held by this rank (master + m + v): 1/|RDP| of the unsharded size when
        sharded (SPEC.md:552-556 memory_report rule)."""
        return 3 * 4 * self.per
