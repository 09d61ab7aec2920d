"""Symmetric peer-mapped memory pool of a TP group (csrc/symm.cu).

Each rank allocates one pool (torch allocation) and one flag block, exports CUDA IPC handles
once, and maps every peer's pool — the persistent pre-registered buffers of the paper's D2D
backend, reused here for the tensor-parallel collectives.  Regions are handed
out by a LIFO bump allocator: every rank executes the same sequence of allocations (SPMD),
so the same offset is valid in every peer's pool.  Forward regions that back saved tensors
are released by the backward (reverse order), transient ones right after use.
"""
from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

from . import _lib
from .errors import PeerTimeoutError

ALIGN = 1024


def check_peer_timeout(timeout_s: float | None = None) -> None:
    peer = _lib.lib().smpk_symm_timeout_peer()
    if peer:
        after = f" after {timeout_s:g} s" if timeout_s is not None else ""
        raise PeerTimeoutError(f"symmetric-memory barrier timed out{after} waiting for TP peer {peer - 1}")


def synchronize() -> None:
    """torch.cuda.synchronize() that turns a trapped peer barrier into PeerTimeoutError."""
    try:
        torch.cuda.synchronize()
    except RuntimeError as e:
        check_peer_timeout()
        raise e


class SymmPool:
    def __init__(self, capacity_bytes: int, group, ranks: list, my_index: int, timeout_s: float = 30.0):
        self.T, self.me, self.timeout_s = len(ranks), my_index, timeout_s
        dev = torch.device("cuda", torch.cuda.current_device())
        self.buf = torch.empty(capacity_bytes, dtype=torch.uint8, device=dev)
        self.flags = torch.zeros(64, dtype=torch.int32, device=dev)
        from .exchange import NWORDS
        self.xflags = torch.zeros(NWORDS, dtype=torch.int32, device=dev)  # chunked-exchange mailbox words
        torch.cuda.synchronize()  # zeroed before any peer can map and signal them
        self.capacity = capacity_bytes
        mine = (self._export(self.buf), self._export(self.flags), self._export(self.xflags))
        gathered = [None] * self.T
        dist.all_gather_object(gathered, mine, group=group)
        self._mapped = []
        bases, flag_bases, xflag_bases = [], [], []
        for j, ((hb, ob), (hf, of), (hx, ox)) in enumerate(gathered):
            if j == self.me:
                bases.append(self.buf.data_ptr())
                flag_bases.append(self.flags.data_ptr())
                xflag_bases.append(self.xflags.data_ptr())
                continue
            pb, pf, px = self._import(hb), self._import(hf), self._import(hx)
            self._mapped += [pb, pf, px]
            bases.append(pb + ob)
            flag_bases.append(pf + of)
            xflag_bases.append(px + ox)
        self.bases = bases
        self.xflag_bases = xflag_bases
        self.self_table = torch.tensor([bases[my_index]], dtype=torch.int64, device=dev)
        self._xch = None
        self.flag_table = torch.tensor(flag_bases, dtype=torch.int64, device=dev)
        self.base_table = torch.tensor(bases, dtype=torch.int64, device=dev)
        self.base_array = (C.c_void_p * self.T)(*bases)  # host copy (TMA-store descriptors)
        self.epoch = 0
        self.top = 0
        self.regions: list = []  # [offset, size, live, epoch at release]
        self._scratch: dict = {}
        self._scratch_bottom = capacity_bytes

    @staticmethod
    def _export(t: torch.Tensor):
        h = C.create_string_buffer(64)
        off = C.c_int64()
        _lib.call("smpk_symm_export", t.data_ptr(), h, C.byref(off))
        return h.raw, off.value

    @staticmethod
    def _import(handle: bytes) -> int:
        p = C.c_void_p()
        _lib.call("smpk_p2p_import", C.create_string_buffer(handle, 64), C.byref(p))
        return p.value

    def exchange(self):
        """The chunked-exchange mailboxes of this group (exchange.Exchange), created on first use."""
        if self._xch is None:
            from .exchange import Exchange
            self._xch = Exchange(self)
        return self._xch

    # -- allocation (identical sequence on every rank) -------------------------------
    def alloc(self, nbytes: int) -> int:
        # A freed region becomes reusable only once a barrier has been issued after its release:
        # peers write into a region only after a barrier, and every rank passes a barrier only
        # after the previous readers of that region (on every rank) have finished.
        while self.regions and not self.regions[-1][2] and self.regions[-1][3] != self.epoch:
            self.regions.pop()
        self.top = (self.regions[-1][0] + self.regions[-1][1]) if self.regions else 0
        off = (self.top + ALIGN - 1) // ALIGN * ALIGN
        if off + nbytes > self._scratch_bottom:
            raise RuntimeError(f"symmetric pool exhausted: need {off + nbytes} B of {self._scratch_bottom} B "
                               f"(raise smp config 'symm_pool_bytes')")
        self.top = off + nbytes
        self.regions.append([off, nbytes, True, -1])
        return off

    def free(self, off: int) -> None:
        for r in reversed(self.regions):
            if r[0] == off and r[2]:
                r[2] = False
                r[3] = self.epoch  # released under this epoch; reusable after the next barrier
                return
        raise RuntimeError(f"symmetric pool: free of unknown region {off}")

    def scratch(self, kind: str, nbytes: int) -> int:
        """Permanent transient region per (kind, size), carved from the END of the pool.

        Transient exchanges (row-parallel partial slots, backward gathers) alternate with a
        barrier in between (every reader of one use finishes before any rank passes the barrier
        that precedes the next use's remote writers), so one region per kind suffices."""
        key = (kind, nbytes)
        off = self._scratch.get(key)
        if off is None:
            end = self._scratch_bottom - nbytes
            off = end // ALIGN * ALIGN
            if off < self.top:
                raise RuntimeError("symmetric pool exhausted by scratch regions (raise 'symm_pool_bytes')")
            self._scratch_bottom = off
            self._scratch[key] = off
        return off

    def peers(self, off: int, elem_off: int = 0, elem_size: int = 2):
        """(device table of the T pool bases, element offset of region `off` + elem_off).

        The table is built once at construction, so kernels launched inside a CUDA-graph capture
        never need a host->device copy; the region offset travels as the kernels' int64 offset."""
        assert off % elem_size == 0
        return self.base_table, off // elem_size + elem_off

    def host_peers(self, off: int, elem_off: int = 0, elem_size: int = 2):
        """(host array of the T pool bases, element offset of region `off` + elem_off)."""
        assert off % elem_size == 0
        return self.base_array, off // elem_size + elem_off

    def push_copy(self, src: torch.Tensor, off: int) -> None:
        """Copy the contiguous tensor src to byte offset `off` of every rank's pool (own included),
        on the current stream (copy engine over NVLink; capturable)."""
        st = torch.cuda.current_stream().cuda_stream
        nbytes = src.numel() * src.element_size()
        for j in range(self.T):
            _lib.call("smpk_copy_async", self.bases[j] + off, src.data_ptr(), nbytes, st)

    def view(self, off: int, shape, dtype=torch.bfloat16) -> torch.Tensor:
        n = 1
        for s in shape:
            n *= s
        nbytes = n * torch.tensor([], dtype=dtype).element_size()
        return self.buf[off:off + nbytes].view(dtype).view(*shape)

    def barrier(self) -> None:
        self.epoch = (self.epoch + 1) & 0x7FFFFFFF
        _lib.call("smpk_symm_barrier", self.flag_table.data_ptr(), self.flags.data_ptr(), self.T, self.me,
                  float(self.timeout_s), torch.cuda.current_stream().cuda_stream)

    def check(self) -> None:
        """Raise PeerTimeoutError if a barrier of this process timed out (the barrier kernel traps,
        so the CUDA context is poisoned; the stuck peer is read from mapped host memory)."""
        check_peer_timeout(self.timeout_s)

    def close(self) -> None:
        for p in self._mapped:
            _lib.call("smpk_p2p_close", p)
        self._mapped = []
