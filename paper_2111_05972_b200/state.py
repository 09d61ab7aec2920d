"""Process-wide smp state: config, topology and the TP / PP process groups.

``smp.init(config)`` accepts the paper's configuration keys (PAPER.md:761-775,
Appendix J.1; SPEC.md:572-575 RunConfig): tensor_parallel_degree,
pipeline_parallel_degree, optimize ("speed" | "memory", default "memory" as in
PAPER.md:763), placement_strategy ("cluster"), _prescaled_batch, microbatches,
plus ``seed`` for the dropout Philox key.  One process per GPU; ranks come from
torch.distributed / the torchrun environment.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from .errors import TopologyError
from .topology import Topology, build_topology

DEFAULTS = {
    "tensor_parallel_degree": 1,
    "pipeline_parallel_degree": 1,
    "microbatches": 1,
    "optimize": "memory",
    "placement_strategy": "cluster",
    "_prescaled_batch": False,
    "fp16_params": False,
    "shard_optimizer_state": False,
    "offload_activations": False,
    "activation_loading_horizon": 4,
    "seed": 0,
    "ddp": True,
    "tp_comm": "peer",  # fused NVLink peer-memory collectives ("nccl": torch.distributed calls)
    "tp_rs": "pull",  # barrier exchange: the consumer pulls the partials ("push": GEMM epilogue stores)
    "tp_exchange": "barrier",  # peer mode: "chunks" = per-owner chunks + copy-engine mailboxes (exchange.py), "barrier"
    "tp_overlap_sms": 0,  # >0: backward weight-gradient GEMMs on this many SMs beside the exchange
    "symm_pool_bytes": None,  # per rank; default min(16 GiB, 10% of HBM): the forward gather regions live
    # until the backward (BERT-L at T=8 ~3.4 GiB, GPT-1.3B at T=4 ~12.3 GiB)
}


@dataclass
class State:
    config: dict = field(default_factory=lambda: dict(DEFAULTS))
    rank: int = 0
    world_size: int = 1
    local_rank: int = 0
    topology: Topology | None = None
    tp_group: object = None
    pp_group: object = None
    rdp_group: object = None
    tp_group_ranks: list = field(default_factory=lambda: [0])
    pp_group_ranks: list = field(default_factory=lambda: [0])
    initialized: bool = False
    layer_counter: int = 0
    step: int = 0  # host mirror: forwards issued eagerly (graph replays advance only the device word)
    rng_counter: object = None  # device int64 step word (one per process), advanced per top-level forward
    rng_cur: object = None  # snapshot of the step word the current forward's dropout kernels read
    xch_fresh: bool = True  # no chunked exchange issued yet in this forward (step-entry barrier due)

    # -- accessors mirroring smp.tp_rank() / smp.tp_size() ...
    @property
    def tp_size(self) -> int:
        return self.topology.tp_degree if self.topology else 1

    @property
    def tp_rank(self) -> int:
        return self.topology.tp_ranks[self.rank] if self.topology else 0

    @property
    def pp_size(self) -> int:
        return self.topology.pp_degree if self.topology else 1

    @property
    def pp_rank(self) -> int:
        return self.topology.pp_ranks[self.rank] if self.topology else 0

    @property
    def rdp_rank(self) -> int:
        return self.topology.rdp_ranks[self.rank] if self.topology else 0

    @property
    def dp_rank(self) -> int:
        return self.topology.dp_rank(self.rank) if self.topology else 0

    @property
    def prescaled(self) -> bool:
        return bool(self.config.get("_prescaled_batch", False))

    @property
    def optimize(self) -> str:
        return self.config.get("optimize", "memory")

    @property
    def seed(self) -> int:
        return int(self.config.get("seed", 0))


STATE = State()


def init(config: dict | None = None, *, backend: str | None = None) -> State:
    """smp.init: parse the config, bootstrap torch.distributed if needed, build TP/PP groups."""
    cfg = dict(DEFAULTS)
    cfg.update(config or {})
    if cfg["optimize"] not in ("speed", "memory"):
        raise ValueError(f"optimize must be 'speed' or 'memory', got {cfg['optimize']!r}")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if dist.is_available() and dist.is_initialized():
        world, rank = dist.get_world_size(), dist.get_rank()
    elif world > 1:
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    tp, pp = int(cfg["tensor_parallel_degree"]), int(cfg["pipeline_parallel_degree"])
    topo = build_topology(world, pp, tp, cfg["placement_strategy"], bool(cfg["_prescaled_batch"]))
    st = STATE
    old_pool = getattr(st, "_pool", None)
    if old_pool is not None:
        old_pool.close()
    st._pool = None
    st.config, st.rank, st.world_size, st.local_rank, st.topology = cfg, rank, world, local, topo
    st.tp_group = st.pp_group = st.rdp_group = None
    st.tp_group_ranks, st.pp_group_ranks = topo.tp_group(rank), topo.pp_group(rank)
    if world > 1:
        # every rank creates every group in the same order (torch.distributed contract)
        for kind in ("tp", "pp", "rdp"):
            for members in topo.groups(kind):
                g = dist.new_group(members) if len(members) < world else dist.group.WORLD
                if rank in members:
                    setattr(st, f"{kind}_group", g)
    st.initialized = True
    st.layer_counter = 0
    st.step = 0
    st.rng_cur = None
    if torch.cuda.is_available():  # created eagerly: a counter first allocated inside a CUDA-graph
        # capture would be re-zeroed by every replay
        st.rng_counter = torch.zeros(1, dtype=torch.int64, device=torch.device("cuda", torch.cuda.current_device()))
    return st


def reset() -> None:
    global STATE
    pool = getattr(STATE, "_pool", None)
    if pool is not None:
        pool.close()
    STATE.__init__()
    STATE._pool = None


def tp_comm() -> str:
    """'peer' (fused NVLink peer-store collectives over the symmetric pool) or 'nccl'."""
    return STATE.config.get("tp_comm", "peer")


def get_pool():
    """The TP group's symmetric peer-mapped pool (created collectively on first use)."""
    pool = getattr(STATE, "_pool", None)
    if pool is None:
        from .symm import SymmPool
        cap = STATE.config.get("symm_pool_bytes")
        if cap is None:
            total = torch.cuda.get_device_properties(torch.cuda.current_device()).total_memory
            cap = min(16 << 30, total // 10)
        cap = int(cap)
        ranks = STATE.tp_group_ranks
        pool = SymmPool(cap, STATE.tp_group, ranks, ranks.index(STATE.rank))
        STATE._pool = pool
    return pool


def begin_forward():
    """Start of a top-level smp forward (module entry): snapshot the device step word and advance
    it, so every training step -- eager or a CUDA-graph replay -- draws fresh dropout masks while
    the backward re-reads the snapshot its forward used."""
    from . import ops
    dev = torch.device("cuda", torch.cuda.current_device())
    if STATE.rng_counter is None or STATE.rng_counter.device != dev:
        if torch.cuda.is_current_stream_capturing():
            raise RuntimeError("smp: the dropout step counter must exist before CUDA-graph capture "
                               "(call smp.init() / run one eager step on this device first)")
        STATE.rng_counter = torch.zeros(1, dtype=torch.int64, device=dev)
    STATE.rng_cur = ops.rng_next(STATE.rng_counter)
    STATE.xch_fresh = True
    from . import layers
    layers._PUSHED.clear()  # push records of an aborted earlier forward can never match a new input
    STATE.step += 1
    return STATE.rng_cur


def rng_step() -> int:
    """Current value of the device step word (synchronising read; tests / checkpoints)."""
    return 0 if STATE.rng_counter is None else int(STATE.rng_counter.item())


def set_rng_step(step: int) -> None:
    """Restore the device step word (resume from a checkpoint)."""
    if STATE.rng_counter is None:
        STATE.rng_counter = torch.zeros(1, dtype=torch.int64, device=torch.device("cuda", torch.cuda.current_device()))
    STATE.rng_counter.fill_(int(step))


def next_layer_id() -> int:
    lid = STATE.layer_counter
    STATE.layer_counter += 1
    return lid


def tp_rank() -> int:
    return STATE.tp_rank


def tp_size() -> int:
    return STATE.tp_size


def pp_rank() -> int:
    return STATE.pp_rank


def pp_size() -> int:
    return STATE.pp_size


def dp_rank() -> int:
    return STATE.dp_rank


def rdp_rank() -> int:
    return STATE.rdp_rank


def rank() -> int:
    return STATE.rank


def size() -> int:
    return STATE.world_size


def get_tp_process_group():
    return STATE.tp_group


def get_pp_process_group():
    return STATE.pp_group


__all__ = ["init", "reset", "STATE", "TopologyError", "tp_rank", "tp_size", "pp_rank", "pp_size", "dp_rank",
           "rdp_rank", "rank", "size"]
