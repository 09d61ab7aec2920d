"""smp — B200-native tensor-parallel hot path of the SageMaker model-parallelism design.

Public surface mirrors the paper's ``smp`` API for this path (PAPER.md:131-150,
799-893): ``smp.init(config)``, ``smp.nn.Distributed*`` modules, the ``*_for_tp``
collectives and the pipeline stage send/recv.  Compute runs in libsmpk.so
(hand-written sm_100a kernels, C ABI in include/smpk.h).
"""
from __future__ import annotations

__version__ = "0.1.0"
