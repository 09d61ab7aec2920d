"""Chunked TP exchanges over the symmetric pool: copy-engine mailboxes (tp_exchange="chunks").

The speed-mode sub-layer with TP across DP ranks all-gathers its input rows and
reduce-scatters its output rows.  Instead of one exchange per sub-layer behind a full barrier
(the SMs idle while NVLink moves the whole activation), the sub-layer runs as T chunks — chunk c
is the rows of rank c's samples, own chunk first — and every transfer is a copy-engine copy on a
per-peer side stream, signalled with stream-ordered flag words (csrc/p2p.cu smpk_stream_flag):

  all-gather  : rank j publishes its rows into every peer's gather region; peer r awaits them
                only right before its chunk j (k = (j - r) mod T steps later), so the copy
                overlaps r's chunks before it.
  reduce-scat : rank r's row-parallel partial product of chunk c goes to rank c's slot r while
                r computes chunk c+1; rank c's consumer awaits its T-1 slots at the end.

Mailbox protocol (per kind, per peer pair; EQ-and-reset so fixed values replay in CUDA graphs):
  sender   (side stream S_dst): [wait ack[kind][dst] == 0; write ack = 1]  copy -> dst slot
                                write dst.ready[kind][me] = 1                     (fenced)
  receiver (consuming stream) : wait ready[kind][src] == 1; write ready = 0; consume;
                                [write src.ack[kind][me] = 0]  (slot free again)
Slots that are written once per step (the forward gather regions, which the backward re-reads)
need no ack: the step-entry barrier orders their reuse across steps.
"""
from __future__ import annotations

import torch

from . import _lib

# flag-word kinds (index = kind * 64 + peer)
AGF, RSF, AGB, RSB = 0, 1, 2, 3
_READY, _ACK = 0, 8  # ready words of kind k at k*64, ack words at (k + 8)*64
NWORDS = 16 * 64


class Exchange:
    """Per-TP-group mailbox state on top of a SymmPool (pool.xflag_bases / pool.xflags)."""

    def __init__(self, pool):
        self.pool = pool
        self.T, self.me = pool.T, pool.me
        dev = pool.buf.device
        self.streams = {j: torch.cuda.Stream(device=dev) for j in range(self.T) if j != self.me}
        self.stage_free = {}  # (tag, peer) -> event after the last copy out of that staging buffer
        self._stage = {}

    # -- flag words ----------------------------------------------------------------
    def _word(self, rank: int, kind: int, peer: int, ack: bool) -> int:
        return self.pool.xflag_bases[rank] + 4 * ((kind + (_ACK if ack else _READY)) * 64 + peer)

    @staticmethod
    def _flag(addr: int, value: int, op: int, stream) -> None:
        _lib.call("smpk_stream_flag", addr, value, op, stream.cuda_stream)

    # -- sender ---------------------------------------------------------------------
    def send(self, kind: int, dst: int, dst_off: int, src: torch.Tensor, *, ack: bool, extra=(),
             stage_tag=None) -> None:
        """Copy the contiguous tensor src to byte offset dst_off of rank dst's pool (plus any
        (dst_off, tensor) pairs in extra) on the side stream for dst, after the current stream's
        work so far, then raise dst's ready word.  ack: wait for the previous use's release first."""
        main = torch.cuda.current_stream()
        s = self.streams[dst]
        s.wait_stream(main)
        if ack:
            w = self._word(self.me, kind, dst, True)
            self._flag(w, 0, 0, s)
            self._flag(w, 1, 1, s)
        base = self.pool.bases[dst]
        for off, t in ((dst_off, src),) + tuple(extra):
            _lib.call("smpk_copy_async", base + off, t.data_ptr(), t.numel() * t.element_size(), s.cuda_stream)
            t.record_stream(s)
        self._flag(self._word(dst, kind, self.me, False), 1, 1, s)
        if stage_tag is not None:
            ev = torch.cuda.Event()
            ev.record(s)
            self.stage_free[(stage_tag, dst)] = (ev, torch.cuda.is_current_stream_capturing())

    def staging(self, tag, peer: int, shape, dtype=torch.bfloat16) -> torch.Tensor:
        """Reusable local staging buffer for copies to `peer`; the current stream first waits for
        the previous copy out of it."""
        key = (tag, peer, tuple(shape), dtype)
        t = self._stage.get(key)
        if t is None:
            t = torch.empty(*shape, dtype=dtype, device=self.pool.buf.device)
            self._stage[key] = t
        ev = self.stage_free.get((tag, peer))
        # an event recorded before a CUDA-graph capture began belongs to finished eager work
        if ev is not None and (ev[1] or not torch.cuda.is_current_stream_capturing()):
            torch.cuda.current_stream().wait_event(ev[0])
        return t

    # -- receiver -------------------------------------------------------------------
    def await_(self, kind: int, src: int) -> None:
        """Current stream waits until src's copy of this kind landed, and re-arms the word."""
        w = self._word(self.me, kind, src, False)
        st = torch.cuda.current_stream()
        self._flag(w, 1, 0, st)
        self._flag(w, 0, 1, st)

    def release(self, kind: int, src: int) -> None:
        """After the current stream's consumers of src's slot: tell src the slot is free."""
        self._flag(self._word(src, kind, self.me, True), 0, 1, torch.cuda.current_stream())

    def join(self) -> None:
        """Current stream waits for every side-stream copy issued so far (capture join)."""
        main = torch.cuda.current_stream()
        for s in self.streams.values():
            main.wait_stream(s)


def chunk_order(me: int, T: int) -> list:
    """Chunks (owner ranks) in the order rank `me` processes them: own rows first, then the
    ranks after it -- rank j's rows are needed by rank r at step (j - r) mod T, so every
    publisher serves the peer that needs it soonest first (see publish_order)."""
    return [(me + k) % T for k in range(T)]


def publish_order(me: int, T: int) -> list:
    """Peers in the order rank `me` sends its rows to them (the one that needs them soonest first)."""
    return [(me - k) % T for k in range(1, T)]
