"""Pipeline parallelism: microbatch scheduler (Python) + D2D stage send/recv (libsmpk).

* ``next_action`` / ``SchedulerState`` / ``SchedulePolicy`` restate the module-server
  scheduler consulted at pp_rank 0 (mpsim pipeline.py:95-165): simple = forwards
  0..M-1 then backwards in order, each gated on its forward; interleaved = a ready
  backward (lowest microbatch) always wins over the next forward.
* ``route`` / ``D2DBuffers`` restate the communication-backend routing rule
  (comm.py:157-225): D2D unless the tensor is on CPU, the pair has
  no NVLink (same node) / RDMA (cross node), or the persistent buffers are full,
  in which case the transfer falls back (here: NCCL send/recv over the PP group).
* ``StageChannel`` is the real D2D transport for one directed peer pair: persistent
  IPC-mapped receive ring on the consumer, copy-engine peer copies on the producer's
  stream, stream-ordered ready/free sequence words (csrc/p2p.cu) — no host sync.
* ``static_schedule`` turns the scheduler decisions into per-stage op lists for a
  chain of P stages (record-and-replay "static mode"), which
  ``PipelineEngine`` executes SPMD (one process per GPU).
* ``check_decision_log`` replays ``next_action`` over a recorded decision log in the reference
  runtime's format {t, ready_backwards, action} (pipeline.py:520-524) and raises
  ``StaticModeViolation`` at the first decision the scheduler would not have taken;
  ``static_schedule(..., replay=log)`` / ``PipelineEngine(..., decision_log=log)`` execute such a
  log's action sequence verbatim (e.g. one recorded by the reference's ``run_step``).

PROVENANCE: the scheduler section (SchedulePolicy, SchedulerState, ready_backwards, next_action) and
the routing section (D2DBuffers, route) are vendored from the reference (mpsim pipeline.py:96-165,
comm.py:157-225) so schedule decisions and D2D routing stay bit-exact with it; they stay in Python
per the north_star.  static_schedule, StageChannel and PipelineEngine are original.
"""
from __future__ import annotations

import ctypes as C
import heapq
from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from . import _lib

FWD = "forward"
BWD = "backward"
MPI = "MPI"
D2D = "D2D"


class StaticModeViolation(RuntimeError):
    """A replayed schedule diverges from what the scheduler decides (pipeline.py:44, :225-246)."""


# ---------------------------------------------------------------------------
# scheduler (pipeline.py:95-165)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class SchedulePolicy:
    kind: str = "interleaved"
    microbatches: int = 1
    forward_only: bool = False

    def __post_init__(self):
        if self.kind not in ("simple", "interleaved"):
            raise ValueError(f"unknown pipeline policy {self.kind!r}")
        if self.microbatches < 1:
            raise ValueError("microbatch count must be >= 1")


@dataclass
class SchedulerState:
    microbatches: int
    issued_fwd: int = 0
    completed_fwd: set = field(default_factory=set)
    issued_bwd: set = field(default_factory=set)
    completed_bwd: int = 0


def ready_backwards(state: SchedulerState) -> list:
    return sorted(m for m in state.completed_fwd if m not in state.issued_bwd)


def next_action(policy: SchedulePolicy, state: SchedulerState):
    """Next (microbatch, direction) to issue at pp_rank 0, or None to wait."""
    M = policy.microbatches
    ready = ready_backwards(state)
    if policy.kind == "interleaved":
        if not policy.forward_only and ready:
            return (ready[0], BWD)
        if state.issued_fwd < M:
            return (state.issued_fwd, FWD)
        return None
    if state.issued_fwd < M:
        return (state.issued_fwd, FWD)
    if policy.forward_only:
        return None
    nb = len(state.issued_bwd)
    if nb < M and nb in state.completed_fwd:
        return (nb, BWD)
    return None


def check_decision_log(policy: SchedulePolicy, log: list) -> list:
    """Replay next_action over a recorded decision log (entries {t, ready_backwards, action},
    the reference runtime's format, pipeline.py:520-524).  The scheduler state before entry i
    is rebuilt from the log itself: issued forwards = the forward actions before i, issued
    backwards = the backward actions before i, completed forwards = ready_backwards(i) plus the
    issued backwards (a backward is only ever issued after its forward completed).  Raises
    StaticModeViolation at the first entry whose action differs from next_action on that state,
    or whose ready set contradicts the issued actions.  Returns the action sequence."""
    M = policy.microbatches
    issued_fwd, issued_bwd, acts = 0, set(), []
    for i, e in enumerate(log):
        ready = [int(m) for m in e["ready_backwards"]]
        if any(m in issued_bwd or m >= issued_fwd for m in ready) or ready != sorted(set(ready)):
            raise StaticModeViolation(f"decision {i}: ready_backwards {ready} inconsistent with the issued actions "
                                      f"(forwards issued {issued_fwd}, backwards issued {sorted(issued_bwd)})")
        st = SchedulerState(M, issued_fwd, set(ready) | issued_bwd, set(issued_bwd), 0)
        want = next_action(policy, st)
        got = (int(e["action"][0]), str(e["action"][1]))
        if want is None or tuple(want) != got:
            raise StaticModeViolation(f"decision {i} at t={e.get('t')}: log has {got}, the scheduler decides {want} "
                                      f"(ready_backwards {ready})")
        if got[1] == FWD:
            issued_fwd += 1
        else:
            issued_bwd.add(got[0])
        acts.append(got)
    return acts


def static_schedule(policy: SchedulePolicy, stages: int, fwd_cost: float = 1.0, bwd_cost: float = 2.0,
                    replay: list | None = None):
    """Record the scheduler's decisions on a P-stage chain and return per-stage op lists.

    Event model: a forward of microbatch m visits stages 0..P-1 (each busy fwd_cost),
    a backward visits P-1..0 (bwd_cost); stages execute their queue FIFO, one op at a
    time.  pp_rank 0 consults next_action whenever it is idle, exactly like the module
    server (pipeline.py:486-530).  Returns (decision_log, ops) with ops[stage] the ordered
    list of (microbatch, direction) that stage executes.

    replay: a decision log (checked with check_decision_log) whose action sequence rank 0
    issues verbatim instead of consulting next_action -- each action as soon as rank 0 is idle
    and, for a backward, its forward has completed in the model."""
    P, M = stages, policy.microbatches
    script = check_decision_log(policy, replay) if replay is not None else None
    st = SchedulerState(M)
    busy_until = [0.0] * P
    queues = [[] for _ in range(P)]  # (ready_time, seq, mb, dir)
    ops = [[] for _ in range(P)]
    log = []
    events = []  # (time, seq, stage, mb, dir) completions
    seq = 0
    t = 0.0
    done_bwd = 0
    while (done_bwd < M or (policy.forward_only and len(st.completed_fwd) < M)) and \
            (script is None or len(log) < len(script) or events or any(queues)):
        # rank 0 consults the scheduler when idle and nothing is queued for it
        if busy_until[0] <= t and not queues[0]:
            if script is None:
                act = next_action(policy, st)
            else:
                nxt = script[len(log)] if len(log) < len(script) else None
                act = nxt if nxt is not None and (nxt[1] == FWD or nxt[0] in st.completed_fwd) else None
            if act is not None:
                log.append({"t": t, "ready_backwards": ready_backwards(st), "action": list(act)})
                mb, d = act
                if d == FWD:
                    st.issued_fwd += 1
                    queues[0].append((t, seq, mb, d))
                else:
                    st.issued_bwd.add(mb)
                    queues[P - 1].append((t, seq, mb, d))
                seq += 1
        # start queued work on idle stages
        for s in range(P):
            if busy_until[s] <= t and queues[s]:
                queues[s].sort()
                rt, _, mb, d = queues[s].pop(0)
                cost = fwd_cost if d == FWD else bwd_cost
                busy_until[s] = max(t, rt) + cost
                ops[s].append((mb, d))
                heapq.heappush(events, (busy_until[s], seq, s, mb, d))
                seq += 1
        if not events:
            if policy.forward_only and len(st.completed_fwd) == M:
                break
            t += 1e-9
            continue
        t, _, s, mb, d = heapq.heappop(events)
        if d == FWD:
            if s + 1 < P:
                queues[s + 1].append((t, seq, mb, d))
                seq += 1
            else:
                st.completed_fwd.add(mb)
        else:
            if s > 0:
                queues[s - 1].append((t, seq, mb, d))
                seq += 1
            else:
                done_bwd += 1
                st.completed_bwd += 1
    if script is not None and len(log) < len(script):
        raise StaticModeViolation(f"replayed log: action {len(log)} {script[len(log)]} never became issuable")
    if done_bwd < M and not (policy.forward_only and len(st.completed_fwd) == M):
        raise StaticModeViolation(f"replayed log ends after {len(log)} actions with {M - done_bwd} microbatches "
                                  "unfinished")
    return log, ops


# ---------------------------------------------------------------------------
# routing + persistent buffer accounting (comm.py:157-225)
# ---------------------------------------------------------------------------

class D2DBuffers:
    def __init__(self, world_size: int, capacity_bytes: float):
        self.capacity = capacity_bytes
        self.send_used = [0.0] * world_size
        self.recv_used = [0.0] * world_size

    def reserve(self, rank: int, nbytes: float, kind: str) -> bool:
        if nbytes < 0:
            raise ValueError("cannot reserve negative bytes")
        used = self.send_used if kind == "send" else self.recv_used
        if used[rank] + nbytes > self.capacity:
            return False
        used[rank] += nbytes
        return True

    def release(self, rank: int, nbytes: float, kind: str) -> None:
        used = self.send_used if kind == "send" else self.recv_used
        if nbytes < 0 or used[rank] - nbytes < -1e-9:
            raise ValueError(f"release of {nbytes} bytes exceeds reservations on rank {rank}")
        used[rank] = max(used[rank] - nbytes, 0.0)

    def try_reserve_pair(self, src: int, dst: int, nbytes: float) -> bool:
        if not self.reserve(src, nbytes, "send"):
            return False
        if not self.reserve(dst, nbytes, "recv"):
            self.release(src, nbytes, "send")
            return False
        return True

    def release_pair(self, src: int, dst: int, nbytes: float) -> None:
        self.release(src, nbytes, "send")
        self.release(dst, nbytes, "recv")


def route(device: str, nbytes: float, src: int, dst: int, *, same_node: bool, nvlink: bool, rdma: bool,
          buffers: D2DBuffers) -> str:
    """MPI (host-staged fallback) vs D2D for one tensor transfer, reserving D2D space."""
    if src == dst:
        raise ValueError("route requires distinct src and dst ranks")
    if device == "cpu":
        return MPI
    if same_node:
        if not nvlink:
            return MPI
    elif not rdma:
        return MPI
    if not buffers.try_reserve_pair(src, dst, nbytes):
        return MPI
    return D2D


# ---------------------------------------------------------------------------
# D2D transport
# ---------------------------------------------------------------------------

FLAG_BYTES = 256  # ready word at +0 of the flag block; free word at +128


class _Ring:
    """Device allocation: [slots * slot_bytes payload][flag block]."""

    def __init__(self, slots: int, slot_bytes: int):
        self.slots, self.slot_bytes = slots, slot_bytes
        p = C.c_void_p()
        _lib.call("smpk_p2p_alloc", slots * slot_bytes + FLAG_BYTES, C.byref(p))
        self.base = p.value
        self.flags = self.base + slots * slot_bytes

    def handle(self) -> bytes:
        buf = C.create_string_buffer(64)
        _lib.call("smpk_p2p_export", self.base, buf)
        return buf.raw

    def free(self):
        if self.base:
            _lib.call("smpk_p2p_free", self.base)
            self.base = None


class StageChannel:
    """Directed D2D channel src_rank -> dst_rank with a ring of `slots` persistent buffers.

    Both ranks construct it (collectively over the PP group); the producer calls
    ``send(t)``, the consumer ``recv(out)``, each on its current stream, in the same
    order.  Flow control and completion are stream-ordered sequence words."""

    def __init__(self, src: int, dst: int, slot_bytes: int, slots: int = 4, group=None, *, connect: bool = True):
        self.src, self.dst, self.slots, self.slot_bytes = src, dst, slots, slot_bytes
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.seq = 0
        self.peer_base = None
        if self.rank not in (src, dst):
            raise ValueError("StageChannel must be built by its two endpoint ranks")
        self.is_dst = self.rank == dst
        # dst owns the receive ring (+ ready word); src owns only a flag block (free word)
        self.local = _Ring(slots if self.is_dst else 0, slot_bytes)
        if connect:
            gathered = [None] * dist.get_world_size(group)
            dist.all_gather_object(gathered, (self.rank, self.local.handle()), group=group)
            peer = [h for r, h in gathered if r == (src if self.is_dst else dst)]
            if not peer:
                raise RuntimeError("StageChannel: peer handle missing (both ranks must construct the channel)")
            self.connect(peer[0])

    def connect(self, peer_handle: bytes) -> None:
        """Map the peer endpoint's allocation (its IPC handle, exchanged by the caller)."""
        p = C.c_void_p()
        _lib.call("smpk_p2p_import", C.create_string_buffer(peer_handle, 64), C.byref(p))
        self.peer_base = p.value
        self.peer_flags = self.peer_base + (0 if self.is_dst else self.slots * self.slot_bytes)

    @staticmethod
    def _stream():
        return torch.cuda.current_stream().cuda_stream

    def send(self, t: torch.Tensor) -> None:
        assert self.rank == self.src
        t = t.contiguous()
        nbytes = t.numel() * t.element_size()
        if nbytes > self.slot_bytes:
            raise ValueError(f"StageChannel payload {nbytes} B exceeds slot size {self.slot_bytes} B")
        k = self.seq % self.slots
        wait_free = self.seq - self.slots + 1 if self.seq >= self.slots else 0
        _lib.call("smpk_p2p_send", self.peer_base + k * self.slot_bytes, t.data_ptr(), nbytes,
                  self.peer_flags, self.local.flags + 128, wait_free, self.seq, self._stream())
        self.seq += 1

    def recv(self, out: torch.Tensor) -> torch.Tensor:
        assert self.rank == self.dst
        nbytes = out.numel() * out.element_size()
        k = self.seq % self.slots
        _lib.call("smpk_p2p_recv", out.data_ptr(), self.local.base + k * self.slot_bytes, nbytes,
                  self.local.flags, self.peer_flags + 128, self.seq, self._stream())
        self.seq += 1
        return out

    def close(self):
        if getattr(self, "peer_base", None):
            _lib.call("smpk_p2p_close", self.peer_base)
            self.peer_base = None
        self.local.free()


# ---------------------------------------------------------------------------
# SPMD pipeline engine over a chain of stages
# ---------------------------------------------------------------------------

class PipelineEngine:
    """Runs one training step of a P-stage chain with M microbatches (one process per stage and
    TP rank: with tensor parallelism each TP rank drives its own chain of the same tp_rank,
    topology.py:49-50, and the stage module's TP collectives run inside the stage).

    stage_module: this rank's module (a callable on [mb, s, H] activations); the first
    stage receives its microbatch inputs, the last stage applies ``loss_fn``.  Activations
    go forward and gradients backward over D2D StageChannels; the per-stage op order is
    the recorded schedule of ``next_action`` (static_schedule), or -- with ``decision_log`` --
    the verbatim replay of a recorded log's actions (checked against next_action first).
    ``self.log`` is this engine's decision log in the reference format.

    Transport (PAPER.md:337-350 D2D backend): every send and receive runs on a dedicated
    send / receive stream, ordered against the compute stream by CUDA events -- a send starts
    as soon as its producer op finished and never blocks the next op's kernels, and the
    receive of the NEXT op is posted before the current op runs, so its payload lands while
    this stage computes.  Channels are built from one handle exchange over the PP group."""

    def __init__(self, stage_module, *, pp_rank: int, pp_size: int, ranks: list, act_shape, dtype=torch.bfloat16,
                 policy: SchedulePolicy, slots: int = 4, group=None, decision_log: list | None = None):
        self.mod, self.s, self.P, self.ranks = stage_module, pp_rank, pp_size, list(ranks)
        self.shape, self.dtype, self.policy = tuple(act_shape), dtype, policy
        nbytes = int(torch.Size(act_shape).numel()) * torch.tensor([], dtype=dtype).element_size()
        self.log, ops = static_schedule(policy, pp_size, replay=decision_log)
        self.ops = ops[pp_rank]
        self.fwd_in = self.fwd_out = self.bwd_in = self.bwd_out = None
        me = self.ranks[pp_rank]
        chans = {}
        if pp_rank > 0:  # from the previous stage: activations in, gradients out
            chans["fwd_in"] = StageChannel(self.ranks[pp_rank - 1], me, nbytes, slots, connect=False)
            chans["bwd_out"] = StageChannel(me, self.ranks[pp_rank - 1], nbytes, slots, connect=False)
        if pp_rank + 1 < pp_size:  # to the next stage
            chans["fwd_out"] = StageChannel(me, self.ranks[pp_rank + 1], nbytes, slots, connect=False)
            chans["bwd_in"] = StageChannel(self.ranks[pp_rank + 1], me, nbytes, slots, connect=False)
        mine = {k: c.local.handle() for k, c in chans.items()}
        if group is None and dist.is_initialized() and dist.get_world_size() == pp_size:
            group = dist.group.WORLD
        gathered = [None] * pp_size
        dist.all_gather_object(gathered, (pp_rank, mine), group=group)
        peer = {r: h for r, h in gathered}
        # the endpoint on the other side of each channel
        pairs = {"fwd_in": (pp_rank - 1, "fwd_out"), "bwd_out": (pp_rank - 1, "bwd_in"),
                 "fwd_out": (pp_rank + 1, "fwd_in"), "bwd_in": (pp_rank + 1, "bwd_out")}
        for k, c in chans.items():
            r, kk = pairs[k]
            c.connect(peer[r][kk])
            setattr(self, k, c)
        # separate FIFO streams for receives and sends: a receive posted ahead (waiting for its
        # ready word) must never hold back a send the peer is waiting for
        self.recv_stream, self.send_stream = torch.cuda.Stream(), torch.cuda.Stream()

    def _post_recv(self, op, dev):
        """Receive the payload of op (if it is a receiving op) on the comm stream; returns
        (tensor, ready event) or None."""
        mb, d = op
        ch = self.fwd_in if d == FWD else self.bwd_in
        if ch is None:
            return None
        buf = torch.empty(self.shape, dtype=self.dtype, device=dev)
        self.recv_stream.wait_stream(torch.cuda.current_stream())  # buf allocation
        with torch.cuda.stream(self.recv_stream):
            ch.recv(buf)
            ev = torch.cuda.Event()
            ev.record()
        buf.record_stream(self.recv_stream)
        return buf, ev

    def _send(self, ch, t):
        ev = torch.cuda.Event()
        ev.record()  # the producer op's kernels on the compute stream
        self.send_stream.wait_event(ev)
        with torch.cuda.stream(self.send_stream):
            ch.send(t)
        t.record_stream(self.send_stream)

    def step(self, inputs=None, loss_fn=None):
        """inputs: list of M microbatch tensors (stage 0); loss_fn(mb, y) -> scalar (last stage).
        Returns the list of per-microbatch losses on the last stage (None elsewhere)."""
        saved, losses = {}, {}
        dev = torch.device("cuda", torch.cuda.current_device())
        main = torch.cuda.current_stream()
        pending = self._post_recv(self.ops[0], dev) if self.ops else None
        for i, (mb, d) in enumerate(self.ops):
            cur, pending = pending, None
            if i + 1 < len(self.ops):  # the next op's payload streams in while this op computes
                pending = self._post_recv(self.ops[i + 1], dev)
            if cur is not None:
                main.wait_event(cur[1])
            if d == FWD:
                x = inputs[mb] if self.s == 0 else cur[0].requires_grad_(True)
                y = self.mod(x)
                saved[mb] = (x, y)
                if self.s == self.P - 1:
                    losses[mb] = loss_fn(mb, y)
                else:
                    self._send(self.fwd_out, y.detach())
            else:
                x, y = saved.pop(mb)
                if self.s == self.P - 1:
                    losses[mb].backward()
                else:
                    torch.autograd.backward(y, cur[0])
                if self.s > 0:
                    self._send(self.bwd_out, x.grad)
        main.wait_stream(self.send_stream)  # this step's sends are ordered before the next step's work
        main.wait_stream(self.recv_stream)
        if self.s == self.P - 1:
            return [losses[m] for m in range(self.policy.microbatches)]
        return None
