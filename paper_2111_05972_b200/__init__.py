"""smp — B200-native tensor-parallel hot path of the SageMaker model-parallelism design.

Public surface mirrors the paper's ``smp`` API for this path (PAPER.md:131-150,
799-893): ``smp.init(config)``, ``smp.nn.Distributed*`` modules, the ``*_for_tp``
collectives and the pipeline stage send/recv.  Compute runs in libsmpk.so
(hand-written sm_100a kernels, C ABI in include/smpk.h); there is no CPU path.

    import paper_2111_05972_b200 as smp
    smp.init({"tensor_parallel_degree": 8, "optimize": "speed"})
    layer = smp.nn.DistributedTransformerLayer(num_attention_heads=16, attention_head_size=64,
                                               hidden_size=1024, intermediate_size=4096)
"""
from __future__ import annotations

__version__ = "0.1.0"

from . import nn  # noqa: E402
from .collectives import (bwd_allreduce_for_tp, fused_allgather_for_tp, fwd_allreduce_for_tp,  # noqa: E402
                          reduce_scatter_for_tp, scatter_and_merge_for_tp)
from .errors import (IndexOutOfRangeError, NotDivisibleError, PeerTimeoutError, ShapeMismatchError,  # noqa: E402
                     TensorParallelError, TopologyError)
from .symm import synchronize  # noqa: E402
from .state import (STATE, dp_rank, init, pp_rank, pp_size, rank, rdp_rank, reset, rng_step, set_rng_step, size,  # noqa: E402
                    tp_rank, tp_size)
from .topology import Topology, build_topology  # noqa: E402
from .replace import (DistributedModel, plan_replacement, set_tensor_parallelism, tensor_parallelism,  # noqa: E402
                      tp_register, tp_register_with_module)
from . import pipeline  # noqa: E402,F401
from .checkpointing import checkpoint_grouping, set_activation_checkpointing  # noqa: E402
from .state_dict import full_state_dict, load_local_state_dict, local_state_dict  # noqa: E402
from .dp import DistributedAdam, GradBuckets  # noqa: E402
