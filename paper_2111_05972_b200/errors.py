"""Exception classes of the tensor-parallel path.

The SPEC names the error classes of the tensor_parallel module: shape mismatch,
non-divisible dimension, "called before forward"
 and out-of-range embedding index "reported with position"
(SPEC.md:444,448).  The reference code raises ``ValueError`` subclasses for its
own validation errors (model_graph.py:23, topology.py:18, comm.py:28); these
follow the same convention so callers can catch ``ValueError``.
"""
from __future__ import annotations


class TensorParallelError(ValueError):
    """Base class for tensor-parallel errors."""


class ShapeMismatchError(TensorParallelError):
    pass


class NotDivisibleError(TensorParallelError):
    pass


class IndexOutOfRangeError(TensorParallelError, IndexError):
    def __init__(self, msg: str, position: int | None = None):
        super().__init__(msg)
        self.position = position


class BackwardBeforeForwardError(TensorParallelError, RuntimeError):
    pass


class PeerTimeoutError(RuntimeError):
    pass


class KernelError(RuntimeError):
    pass


class TopologyError(ValueError):
    """Invalid world/degree/placement (mirrors mpsim.topology.TopologyError, topology.py:18)."""


# return codes of include/smpk.h
OK, BAD_SHAPE, NOT_DIVISIBLE, OOB_INDEX, PEER_TIMEOUT, CUDA, BAD_ARG, UNSUPPORTED = range(8)


def raise_for(code: int, msg: str) -> None:
    if code == BAD_SHAPE:
        raise ShapeMismatchError(msg)
    if code == NOT_DIVISIBLE:
        raise NotDivisibleError(msg)
    if code == OOB_INDEX:
        raise IndexOutOfRangeError(msg)
    if code == PEER_TIMEOUT:
        raise PeerTimeoutError(msg)
    if code == BAD_ARG:
        raise TensorParallelError(msg)
    raise KernelError(f"smpk error {code}: {msg}")
