"""Chunked TP exchanges over the symmetric pool: copy-engine mailboxes (tp_exchange="chunks").

The speed-mode sub-layer with TP across DP ranks all-gathers its input rows and
reduce-scatters its output rows.  Instead of one exchange per sub-layer behind a full barrier
(the SMs idle while NVLink moves the whole activation), the sub-layer runs as T chunks — chunk c
is the rows of rank c's samples, own chunk first — and every transfer is a copy-engine copy on a
side stream, signalled with flag words (csrc/symm.cu smpk_peer_put / smpk_flag_wait / smpk_flag_set):

  all-gather  : rank j publishes its rows into every peer's gather region; peer r awaits them
                only right before its chunk j (k = (j - r) mod T steps later), so the copy
                overlaps r's chunks before it.
  reduce-scat : rank r's row-parallel partial product of chunk c goes to rank c's slot r while
                r computes chunk c+1; rank c's consumer awaits its T-1 slots at the end.

Mailbox protocol (per kind, per peer pair; EQ-and-reset so fixed values replay in CUDA graphs):
  sender   (side stream)      : [wait ack[kind][dst] == 0]  copy -> dst slot  [ack = 1]
                                write dst.ready[kind][me] = 1                     (release.sys)
  receiver (consuming stream) : wait ready[kind][src] == 1; write ready = 0; consume;
                                [write src.ack[kind][me] = 0]  (slot free again)
Slots that are written once per step (the forward gather regions, which the backward re-reads)
need no ack: the step-entry barrier orders their reuse across steps.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib

# flag-word kinds (index = kind * 64 + peer); micro-batch mb uses kind + 4 * mb
AGF, RSF, AGB, RSB = 0, 1, 2, 3
_READY, _ACK = 0, 8  # ready words of kind k at k*64, ack words at (k + 8)*64
NWORDS = 16 * 64


def mbkind(kind: int, mb: int) -> int:
    """Flag kind of a micro-batch's mailbox (the two overlapped micro-batches never share words)."""
    return kind + 4 * max(mb, 0)


class _Range(C.Structure):
    _fields_ = [("src", C.c_void_p), ("dst", C.c_void_p), ("bytes", C.c_int64), ("group", C.c_int)]


class _Group(C.Structure):
    _fields_ = [("ready", C.c_void_p), ("ack", C.c_void_p)]


class Exchange:
    """Per-TP-group mailbox state on top of a SymmPool (pool.xflag_bases / pool.xflags).

    Copies are ordinary kernels (smpk_peer_put: vector stores into peer-mapped slots by a few
    CTAs) on one side stream per micro-batch; waits and releases are one-warp kernels
    (smpk_flag_wait / smpk_flag_set).  CUDA-graph memcpy nodes on different branches were
    measured to run one after another, so the copy engines are not used inside the step."""

    def __init__(self, pool):
        self.pool = pool
        self.T, self.me = pool.T, pool.me
        dev = pool.buf.device
        self.dev = dev
        self._streams = {}  # micro-batch -> side stream carrying this rank's copies
        self.stage_free = {}  # (tag, peer) -> event after the last copy out of that buffer
        self._stage = {}
        self._tables = {}
        self.counters = torch.zeros(16 * 8, dtype=torch.int32, device=dev)  # 8 arrival counters per kind

    def stream(self, peer: int = 0, mb: int = -1):
        key = max(mb, 0)
        s = self._streams.get(key)
        if s is None:
            s = self._streams[key] = torch.cuda.Stream(device=self.dev)
        return s

    def table(self, key, ptrs) -> torch.Tensor:
        """Cached device table of absolute addresses (stable across CUDA-graph replays)."""
        t = self._tables.get(key)
        if t is None:
            t = self._tables[key] = torch.tensor(list(ptrs), dtype=torch.int64, device=self.dev)
        return t

    # -- flag words ----------------------------------------------------------------
    def _word(self, rank: int, kind: int, peer: int, ack: bool) -> int:
        return self.pool.xflag_bases[rank] + 4 * ((kind + (_ACK if ack else _READY)) * 64 + peer)

    # -- sender ---------------------------------------------------------------------
    def put(self, kind: int, items, *, ack: bool, stage_tag=None, mb: int = -1) -> None:
        """items: [(dst rank, [(byte offset in dst's pool, contiguous tensor), ...]), ...].  One
        copy kernel on the micro-batch's side stream, after the current stream's work so far;
        each destination's ready word is raised once all of its ranges landed.  ack: wait for the
        previous round's release of each destination first."""
        main = torch.cuda.current_stream()
        s = self.stream(mb=mb)
        s.wait_stream(main)
        ranges, groups = [], []
        for g, (dst, pieces) in enumerate(items):
            groups.append(_Group(self._word(dst, kind, self.me, False),
                                 self._word(self.me, kind, dst, True) if ack else None))
            for off, t in pieces:
                ranges.append(_Range(t.data_ptr(), self.pool.bases[dst] + off, t.numel() * t.element_size(), g))
                t.record_stream(s)
        ra = (_Range * len(ranges))(*ranges)
        ga = (_Group * len(groups))(*groups)
        _lib.call("smpk_peer_put", ra, len(ranges), ga, len(groups), self.counters.data_ptr() + 32 * kind,
                  float(self.pool.timeout_s), s.cuda_stream)
        if stage_tag is not None:
            ev = torch.cuda.Event()
            ev.record(s)
            for dst, _ in items:
                self.stage_free[(stage_tag, dst)] = (ev, torch.cuda.is_current_stream_capturing())

    def send(self, kind: int, dst: int, dst_off: int, src: torch.Tensor, *, ack: bool, extra=(),
             stage_tag=None, mb: int = -1) -> None:
        """put() to one destination: src (plus the (offset, tensor) pairs in extra)."""
        self.put(kind, [(dst, [(dst_off, src)] + list(extra))], ack=ack, stage_tag=stage_tag, mb=mb)

    def staging(self, tag, peer: int, shape, dtype=torch.bfloat16) -> torch.Tensor:
        """Reusable local staging buffer for copies to `peer`; the current stream first waits for
        the previous copy out of it."""
        key = (tag, peer, tuple(shape), dtype)
        t = self._stage.get(key)
        if t is None:
            t = torch.empty(*shape, dtype=dtype, device=self.pool.buf.device)
            self._stage[key] = t
        self.reuse(tag, [peer])
        return t

    def reuse(self, tag, peers) -> None:
        """Current stream waits until the last copies out of the buffer `tag` to `peers` left."""
        capturing = torch.cuda.is_current_stream_capturing()
        seen = set()
        for peer in peers:
            ev = self.stage_free.get((tag, peer))
            # an event recorded before a CUDA-graph capture began belongs to finished eager work
            if ev is not None and id(ev[0]) not in seen and (ev[1] or not capturing):
                seen.add(id(ev[0]))
                torch.cuda.current_stream().wait_event(ev[0])

    # -- receiver -------------------------------------------------------------------
    def await_all(self, kind: int, srcs) -> None:
        """Current stream waits until every src's copy of this kind landed, re-arming the words."""
        srcs = list(srcs)
        if not srcs:
            return
        words = (C.c_void_p * len(srcs))(*[self._word(self.me, kind, j, False) for j in srcs])
        who = (C.c_int * len(srcs))(*srcs)
        _lib.call("smpk_flag_wait", words, who, len(srcs), 1, float(self.pool.timeout_s),
                  torch.cuda.current_stream().cuda_stream)

    def await_(self, kind: int, src: int) -> None:
        self.await_all(kind, [src])

    def release_all(self, kinds, srcs) -> None:
        """After the current stream's consumers of the slots: tell each src its slot is free."""
        words = [self._word(j, kind, self.me, True) for kind in kinds for j in srcs]
        st = torch.cuda.current_stream().cuda_stream
        for i in range(0, len(words), 8):
            w = words[i:i + 8]
            _lib.call("smpk_flag_set", (C.c_void_p * len(w))(*w), len(w), 0, st)

    def release(self, kind: int, src: int) -> None:
        self.release_all([kind], [src])

    def join(self, mb: int = -1) -> None:
        """Current stream waits for every side-stream copy of this micro-batch issued so far
        (capture join)."""
        s = self._streams.get(max(mb, 0))
        if s is not None:
            torch.cuda.current_stream().wait_stream(s)


def chunk_order(me: int, T: int) -> list:
    """Chunks (owner ranks) in the order rank `me` processes them: own rows first, then the
    ranks after it -- rank j's rows are needed by rank r at step (j - r) mod T, so every
    publisher serves the peer that needs it soonest first (see publish_order)."""
    return [(me + k) % T for k in range(T)]


def publish_order(me: int, T: int) -> list:
    """Peers in the order rank `me` sends its rows to them (the one that needs them soonest first)."""
    return [(me - k) % T for k in range(1, T)]
