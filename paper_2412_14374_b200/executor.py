"""B200 pipeline runtime: the drop-in replacement for the reference hot path
``run_pipelined`` (pkg/src/pipecraft/executor.py:387-483).

Same boundary as the reference:

    run_pipelined(cp, tg, params, batch, lr=0.1, timeout_s=30.0, delay_fn=None,
                  strict_store=True) -> ExecutionResult(grads, losses, new_params, stats)

with identical ``RunStats`` semantics (driver messages = one dispatch + one
gather per actor, per-channel message counts, sent buffers, peak live / stash
counts, final live sets) and the same fault types (``ExecutorFault``,
``LivenessFault``, ``ChannelOrderFault``).  What changes is underneath:

* each actor's fused program is issued by one host thread onto that actor's
  CUDA compute stream, asynchronously (no host sync inside the step);
  ``RunTask`` launches libpp200 kernels (device.DeviceOps);
* a channel is either a zero-copy ``LocalChannel`` (actors sharing a GPU,
  events order the streams) or an ``NcclChannel`` (one 2-rank NCCL
  communicator and one send / one recv stream per directed pair; RecvStart
  posts the receive = real prefetch; RecvWait / SendWait are stream waits);
* gradient-merge chains accumulate in place (fp32 accumulator per param and
  stage) whenever the plan proves the running sum has no other reader;
* a watchdog turns host blocking and device hangs into ``LivenessFault``
  (device hangs abort the NCCL communicators first).

In a multi-process launch (torchrun, one process per GPU, world size == P)
each rank executes only its own actor's program; otherwise all actors run as
threads of this process (all on one GPU unless ``devices`` says otherwise).
"""
from __future__ import annotations

import itertools
import math
import os
import threading
import time
from collections import deque
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .comms import (
    CommPlan,
    Delete,
    FlushPendingDeletes,
    RecvStart,
    RecvWait,
    RunTask,
    SendStart,
    SendWait,
    _brief,
)
from .device import _PC as _PC_OF
from .device import MODES, Act, DeviceOps, Mode, Param, PeerBuf, Trans, strip, tensor_of, \
    to_device_input, to_device_param
from .ir import GPTConfig
from .taskgraph import GRAD_TOTAL, OPT_STATE, PARAM, STASH, TaskGraph


class ExecutorFault(RuntimeError):
    """Liveness or consistency failure inside the runtime."""


class ChannelOrderFault(ExecutorFault):
    pass


class LivenessFault(ExecutorFault):
    pass


# ---------------------------------------------------------------------------
# Results and statistics (executor.py:141-165)


@dataclass
class RunStats:
    driver_messages: int = 0
    channel_counts: dict = field(default_factory=dict)     # (src, dst) -> int
    sent_buffers: list = field(default_factory=list)       # (src, dst, buffer id)
    peak_live: dict = field(default_factory=dict)          # actor -> int
    peak_stash: dict = field(default_factory=dict)         # (actor, stage) -> int
    peak_stash_bytes: dict = field(default_factory=dict)   # actor -> device bytes held in stashes
    final_live: dict = field(default_factory=dict)         # actor -> sorted buffer ids
    timeline: list = field(default_factory=list)           # (actor, kind, uid, start_ms, end_ms)

    @property
    def channel_messages(self) -> int:
        return sum(self.channel_counts.values())

    def messages_for_param(self, tg: TaskGraph, param: str) -> int:
        return sum(1 for _, _, bid in self.sent_buffers
                   if tg.buffers[bid].meta.get("param") == param
                   and tg.buffers[bid].kind.startswith("param-grad"))

    def bubble_fraction(self, num_actors: int) -> float:
        """Idle share of the loop window (simulator.py:241-270 definition) from
        the measured per-task CUDA-event intervals."""
        loop = [e for e in self.timeline if e[1] in ("fwd", "bwd")]
        if not loop:
            return 0.0
        lo = min(e[3] for e in loop)
        hi = max(e[4] for e in loop)
        span = hi - lo
        if span <= 0:
            return 0.0
        busy = [0.0] * num_actors
        for a, _, _, s, e in self.timeline:
            busy[a] += max(0.0, min(e, hi) - max(s, lo))
        return sum(span - b for b in busy) / (num_actors * span)


@dataclass
class ExecutionResult:
    grads: dict
    losses: object
    new_params: dict
    stats: RunStats


def instrument(result: ExecutionResult) -> RunStats:
    return result.stats


# ---------------------------------------------------------------------------
# Control (executor.py:172-197)


class _Aborted(Exception):
    pass


class _Control:
    def __init__(self, timeout_s: float):
        self.deadline = time.monotonic() + timeout_s
        self.abort = threading.Event()
        self.heartbeat: dict[int, str] = {}
        self.faults: list[BaseException] = []
        self.lock = threading.Lock()

    def remaining(self) -> float:
        return self.deadline - time.monotonic()

    def fail(self, exc: BaseException):
        with self.lock:
            self.faults.append(exc)
        self.abort.set()

    def check(self, actor: int):
        if self.abort.is_set():
            raise _Aborted()
        if self.remaining() <= 0:
            raise LivenessFault(f"actor {actor} timed out")


# ---------------------------------------------------------------------------
# Channels


class LocalChannel:
    """Directed FIFO between two actors on the same GPU (reference Channel,
    executor.py:201-254, semantics kept exactly).  The payload is the device
    tensor itself (zero copy) plus the CUDA event after which it is valid on
    the sender's stream; the receiver orders its stream on that event."""

    def __init__(self, src: int, dst: int):
        self.src, self.dst = src, dst
        self.cond = threading.Condition()
        self.reset()

    def reset(self):
        self.q: deque = deque()
        self.mailbox: dict[int, tuple] = {}
        self.consumed: set[int] = set()

    def send(self, seq: int, bid: str, value, stream: torch.cuda.Stream):
        ev = torch.cuda.Event()
        ev.record(stream)
        with self.cond:
            if self.q and self.q[-1][0] >= seq:
                raise ChannelOrderFault(
                    f"channel {self.src}->{self.dst}: send seq {seq} out of order")
            self.q.append((seq, bid, strip(value), ev))
            self.cond.notify_all()

    def post_recv(self, seq: int, bid: str, stream=None):
        pass

    def recv(self, seq: int, ctl: _Control, actor: int, stream: torch.cuda.Stream):
        with self.cond:
            while True:
                if seq in self.mailbox:
                    bid, value, ev = self.mailbox.pop(seq)
                    break
                while not self.q:
                    ctl.check(actor)
                    self.cond.wait(timeout=min(0.05, max(ctl.remaining(), 0.001)))
                head, bid, value, ev = self.q.popleft()
                self.consumed.add(head)
                self.cond.notify_all()
                if head == seq:
                    break
                if head > seq:
                    raise ChannelOrderFault(
                        f"channel {self.src}->{self.dst}: receive expected seq {seq} "
                        f"but the channel already advanced to {head} ({bid})")
                self.mailbox[head] = (bid, value, ev)
        stream.wait_event(ev)
        if isinstance(value, torch.Tensor):
            value.record_stream(stream)
        return bid, value

    def wait_consumed(self, seq: int, ctl: _Control, actor: int, stream):
        with self.cond:
            while seq not in self.consumed:
                ctl.check(actor)
                self.cond.wait(timeout=min(0.05, max(ctl.remaining(), 0.001)))

    def is_consumed(self, seq: int) -> bool:
        with self.cond:
            return seq in self.consumed

    def drained(self) -> bool:
        with self.cond:
            return not self.q and not self.mailbox

    def abort(self):
        pass


class NcclChannel:
    """One side of a directed channel between two processes: a dedicated
    2-rank NCCL communicator (src = rank 0, dst = rank 1) and a dedicated
    stream on this side.  Sends and receives are posted in sequence order on
    that stream, which is the per-pair FIFO of the deadlock checker."""

    def __init__(self, src: int, dst: int, me: int, comm, device, wire_meta):
        self.src, self.dst, self.me = src, dst, me
        self.comm = comm
        self.stream = torch.cuda.Stream(device=device)
        self.wire_meta = wire_meta
        self.reset()

    def reset(self):
        self.sent: dict[int, torch.cuda.Event] = {}
        self.posted: dict[int, tuple] = {}
        self.last_seq = -1
        self.consumed: set[int] = set()

    def send(self, seq: int, bid: str, value, stream: torch.cuda.Stream):
        if seq <= self.last_seq:
            raise ChannelOrderFault(f"channel {self.src}->{self.dst}: send seq {seq} out of order")
        self.last_seq = seq
        t = strip(value)
        t = t if t.is_contiguous() else t.contiguous()
        ready = torch.cuda.Event()
        ready.record(stream)
        self.stream.wait_event(ready)
        _lib.call("pc_p2p_send", self.comm, t.data_ptr(), t.numel() * t.element_size(), 1,
                  self.stream.cuda_stream)
        t.record_stream(self.stream)
        done = torch.cuda.Event()
        done.record(self.stream)
        self.sent[seq] = done

    def post_recv(self, seq: int, bid: str, stream: torch.cuda.Stream | None = None):
        shape, dtype = self.wire_meta(bid)
        if stream is not None and torch.cuda.is_current_stream_capturing():
            # join the recv stream into the capture: the receive is posted in
            # program order, which is exactly the checker's model of RecvStart
            fork = torch.cuda.Event()
            fork.record(stream)
            self.stream.wait_event(fork)
        with torch.cuda.stream(self.stream):
            buf = torch.empty(shape, dtype=dtype, device=self.stream.device)
        _lib.call("pc_p2p_recv", self.comm, buf.data_ptr(), buf.numel() * buf.element_size(), 0,
                  self.stream.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(self.stream)
        self.posted[seq] = (bid, buf, ev)

    def recv(self, seq: int, ctl: _Control, actor: int, stream: torch.cuda.Stream):
        if seq not in self.posted:
            raise ChannelOrderFault(
                f"channel {self.src}->{self.dst}: wait on seq {seq} that was never posted")
        bid, buf, ev = self.posted.pop(seq)
        self.consumed.add(seq)
        stream.wait_event(ev)
        buf.record_stream(stream)
        return bid, buf

    def wait_consumed(self, seq: int, ctl: _Control, actor: int, stream):
        ev = self.sent.get(seq)
        if ev is not None:
            stream.wait_event(ev)

    def is_consumed(self, seq: int) -> bool:
        ev = self.sent.get(seq)
        if ev is None:
            return True
        if torch.cuda.is_current_stream_capturing():
            return False  # resolved by the flush after capture
        return ev.query()

    def drained(self) -> bool:
        return not self.posted

    def abort(self):
        if self.comm:
            try:
                _lib.call("pc_p2p_abort", self.comm)
            finally:
                self.comm = None


_TYPESTR = {torch.bfloat16: "<i2", torch.float32: "<f4", torch.float64: "<f8",
            torch.int32: "<i4"}


class _CAI:
    """__cuda_array_interface__ view of raw device memory (this GPU's own)."""

    def __init__(self, ptr: int, shape, dtype):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": _TYPESTR[dtype],
                                         "data": (ptr, False), "version": 3, "strides": None}


def _slot_layout(bids, wire_meta):
    """Receiver-slot layout of one channel: flag words first, then one
    256-byte-aligned slot per message in plan order."""
    n = len(bids)
    off = (4 * n + 255) // 256 * 256
    slots = []
    for bid in bids:
        shape, dtype = wire_meta(bid)
        nb = math.prod(shape) * torch.empty((), dtype=dtype).element_size()
        slots.append((off, tuple(shape), dtype, nb))
        off += (nb + 255) // 256 * 256
    return slots, off


class PeerChannel:
    """One side of a directed channel over NVLink peer memory (same node).

    The receiver owns one slot per message of the plan's channel list plus a
    flag word per message (``pc_peer_alloc``, CUDA IPC); the sender maps them.
    SendStart: the value is normally already in the slot (its producing
    kernel wrote it there, see ``_Actor._placement``), otherwise a copy engine
    moves it; then a stream memory write sets the flag, ordered after the
    producer.  RecvWait: the receiver's stream waits for the flag and re-arms
    it.  No transfer step and no communication kernel remain on the critical
    path.  A slot is rewritten only in the next step, after the receiver has
    finished the step that read it (the sender's next step needs this step's
    last gradient from the receiver).  Reference Channel: executor.py:201-254.
    """

    def __init__(self, src: int, dst: int, me: int, base: int, bids, slots, abort_word):
        self.src, self.dst, self.me = src, dst, me
        self.base, self.bids, self.slots = base, list(bids), slots
        self.abort_host, self.abort_dev = abort_word   # the engine's mapped host word
        self.reset()

    def reset(self):
        self.last_seq = -1
        self.in_place = 0   # messages whose producer wrote them into the slot
        self.copied = 0     # messages moved by a copy engine at SendStart

    def flag(self, seq: int) -> int:
        return self.base + 4 * seq

    def peer_slot(self, seq: int):
        off, shape, dtype, _ = self.slots[seq]
        return PeerBuf(self.base + off, shape, dtype)

    def send(self, seq: int, bid: str, value, stream: torch.cuda.Stream):
        if seq <= self.last_seq:
            raise ChannelOrderFault(f"channel {self.src}->{self.dst}: send seq {seq} out of order")
        self.last_seq = seq
        if self.bids[seq] != bid:
            raise ChannelOrderFault(f"channel {self.src}->{self.dst}: seq {seq} carries "
                                    f"{self.bids[seq]}, not {bid}")
        off, shape, dtype, nb = self.slots[seq]
        t = strip(value)
        if t.data_ptr() != self.base + off:
            if not isinstance(t, PeerBuf):
                t = t if t.is_contiguous() else t.contiguous()
            if t.numel() * t.element_size() != nb:
                raise ChannelOrderFault(f"channel {self.src}->{self.dst}: {bid} has "
                                        f"{t.numel() * t.element_size()} bytes, slot {nb}")
            _lib.call("pc_peer_copy", self.base + off, t.data_ptr(), nb, stream.cuda_stream)
            self.copied += 1
        else:
            self.in_place += 1
        _lib.call("pc_stream_write_u32", self.flag(seq), 1, stream.cuda_stream)

    def post_recv(self, seq: int, bid: str, stream=None):
        pass

    def recv(self, seq: int, ctl: _Control, actor: int, stream: torch.cuda.Stream):
        off, shape, dtype, _ = self.slots[seq]
        # spin kernel: waits for the flag, re-arms it, and gives up when the
        # engine's abort word is set (see abort)
        _lib.call("pc_peer_wait", self.flag(seq), self.abort_dev, stream.cuda_stream)
        t = torch.as_tensor(_CAI(self.base + off, shape, dtype), device=stream.device)
        return self.bids[seq], (t.view(torch.bfloat16) if dtype == torch.bfloat16 else t)

    def wait_consumed(self, seq: int, ctl: _Control, actor: int, stream):
        pass

    def is_consumed(self, seq: int) -> bool:
        return True

    def drained(self) -> bool:
        return True

    def abort(self):
        """Release this rank's parked receives: a plain CPU store to the engine's
        mapped abort word ends every pc_peer_wait spin, so the device drains (the
        data read is garbage; the step is failing).  No stream is involved: work
        queued to release a blocked stream could share its hardware queue."""
        import ctypes
        ctypes.c_uint32.from_address(self.abort_host).value = 1


# ---------------------------------------------------------------------------
# Per-actor store (executor.py:257-313)


class DeviceStore:
    """Buffer id -> device value, with the reference's pending-deletions queue
    for buffers whose sends are still in flight."""

    def __init__(self, actor: int, tg: TaskGraph, stats: RunStats):
        self.actor = actor
        self.tg = tg
        self.stats = stats
        self.data: dict[str, object] = {}
        self.pending: deque[str] = deque()
        self.outstanding: dict[str, list] = {}
        self.received: set[str] = set()
        self._stash_stage = {bid: b.meta["stage"] for bid, b in tg.buffers.items()
                             if b.kind == STASH}
        # running stash totals, updated on put / removal (not re-walked per put)
        self._stash_nbytes: dict[str, int] = {}
        self._stash_total = 0
        self._stash_count: dict[int, int] = {}

    def put(self, bid: str, value):
        if bid in self.data:
            self._forget(bid)
        self.data[bid] = value
        st = self._stash_stage.get(bid)
        if st is not None:
            nb = _stash_bytes(value)
            self._stash_nbytes[bid] = nb
            self._stash_total += nb
            self._stash_count[st] = self._stash_count.get(st, 0) + 1
        self._track(st)

    def _forget(self, bid: str):
        """Remove bid from the running stash totals (before it leaves data)."""
        nb = self._stash_nbytes.pop(bid, None)
        if nb is not None:
            self._stash_total -= nb
            self._stash_count[self._stash_stage[bid]] -= 1

    def _pop(self, bid: str):
        if bid in self.data:
            self._forget(bid)
            del self.data[bid]

    def get(self, bid: str, at: str):
        if bid not in self.data:
            raise LivenessFault(f"actor {self.actor} at {at}: missing buffer {bid}")
        return self.data[bid]

    def note_send(self, bid: str, ch, seq: int):
        self.outstanding.setdefault(bid, []).append((ch, seq))

    def sends_done(self, bid: str) -> bool:
        return all(ch.is_consumed(seq) for ch, seq in self.outstanding.get(bid, ()))

    def delete(self, bid: str, at: str):
        if bid not in self.data:
            raise LivenessFault(f"actor {self.actor} at {at}: delete of absent buffer {bid}")
        if self.sends_done(bid):
            self._pop(bid)
        else:
            self.pending.append(bid)

    def flush(self):
        keep = deque()
        while self.pending:
            bid = self.pending.popleft()
            if self.sends_done(bid):
                self._pop(bid)
            else:
                keep.append(bid)
        self.pending = keep

    def _track(self, stage):
        """Peak counters (executor.py:302-313): O(1) per put from the running totals
        (only the stage of the stash just put can reach a new peak)."""
        a = self.actor
        self.stats.peak_live[a] = max(self.stats.peak_live.get(a, 0), len(self.data))
        if stage is not None:
            key = (a, stage)
            self.stats.peak_stash[key] = max(self.stats.peak_stash.get(key, 0),
                                             self._stash_count[stage])
            self.stats.peak_stash_bytes[a] = max(self.stats.peak_stash_bytes.get(a, 0),
                                                 self._stash_total)


REMAT_NONE, REMAT_FULL = "none", "full-per-stage"   # simulator.py:48, :132-149


def _stash_bytes(stash) -> int:
    """Device bytes a stash holds (under remat: the retained forward inputs
    only; the parameter references it carries are not stash memory)."""
    if isinstance(stash, dict) and "__remat__" in stash:
        stash = stash["__remat__"][0]
    seen: dict[int, int] = {}

    def walk(v):
        if isinstance(v, torch.Tensor):
            seen[v.data_ptr()] = max(seen.get(v.data_ptr(), 0), v.numel() * v.element_size())
        elif isinstance(v, Act):
            walk(v.t)
            walk(v.saved)
        elif isinstance(v, Trans):
            walk(v.base)
        elif isinstance(v, dict):
            for x in v.values():
                walk(x)
        elif isinstance(v, (tuple, list)):
            for x in v:
                walk(x)

    walk(stash)
    return sum(seen.values())


def _retained(v):
    """A forward feed kept for the replay, by reference: nothing rewrites a feed
    before its backward in the same step (peer slots are per message and are
    rewritten only in the next step, NCCL receive buffers and local-channel
    values are fresh, stage forwards never write their inputs).  An Act's saved
    tensors are dropped: the replay recomputes them."""
    if isinstance(v, Act):
        return Act(v.t)
    return v


# ---------------------------------------------------------------------------
# Actor


class _Actor:
    def __init__(self, actor: int, tg: TaskGraph, ops: DeviceOps, stats: RunStats,
                 timeline: bool, inplace: bool = False, instrs=(), channels=None):
        self.actor = actor
        self.inplace = inplace       # resident training state: SGD overwrites the param
        self.tg = tg
        self.device = ops.device
        self.stream = ops.stream
        self.ops = ops
        self.store = DeviceStore(actor, tg, stats)
        self.timeline = timeline
        self.events: list = []       # (kind, uid, start slot, end slot)
        self.remat = REMAT_NONE      # PipelineEngine(remat=...) sets it
        self.ts = None               # int64 device buffer of %globaltimer stamps
        if timeline:
            n = 2 * sum(1 for t in tg.tasks.values() if t.actor == actor) + 1
            self.ts = torch.empty(n, dtype=torch.int64, device=self.device)
        self.end_event = None
        self.last_issued = -1
        # grad-merge adds of this actor by their partial (rhs) operand, and the
        # partials a producer already added onto the running sum
        self._add_by_rhs = {t.exec["rhs"]: (t.uid, t.exec["lhs"]) for t in tg.tasks.values()
                            if t.actor == actor and t.exec.get("type") == "add"}
        self.fused: set = set()
        # sent buffers with no reader on this actor whose one channel is a
        # peer-memory channel: produced straight into the receiver's slot
        sends: dict = {}
        for ins in instrs:
            if isinstance(ins, SendStart):
                sends.setdefault(ins.buffer, []).append((ins.dst, ins.seq))
        self._peer_out = {}
        for bid, dsts in sends.items():
            ch = (channels or {}).get((actor, dsts[0][0]))
            b = tg.buffers[bid]
            if (len(dsts) == 1 and isinstance(ch, PeerChannel) and not b.is_output
                    and all(tg.tasks[c].actor != actor for c in b.consumers)):
                self._peer_out[bid] = ch.peer_slot(dsts[0][1])

    def stamp(self, slot: int):
        _lib.call("pc_timestamp", self.ts.data_ptr() + 8 * slot, self.stream.cuda_stream)

    def read_timeline(self) -> list:
        """(actor, kind, uid, start_ms, end_ms) relative to this actor's program start."""
        if self.ts is None:
            return []
        t = self.ts.cpu().tolist()
        base = t[0]
        return [(self.actor, kind, uid, (t[s0] - base) / 1e6, (t[s1] - base) / 1e6)
                for kind, uid, s0, s1 in self.events]

    def run_task(self, task, at: str):
        ex = task.exec
        kind = ex["type"]
        st = self.store
        p = self.tg.partition
        if self.timeline:
            s0 = 1 + 2 * len(self.events)
            self.stamp(s0)
        if kind == "stage-fwd":
            prog = p.fwd_programs[ex["stage"]]
            env = {v: st.get(bid, at) for v, bid in ex["feeds"].items()}
            kept = None
            if ex["stash_out"] and self.remat == REMAT_FULL:
                # full per-stage rematerialisation: keep the forward's feeds only
                # (boundary activations and batch inputs copied before the
                # forward runs, since their channel slots are reused; parameters
                # by reference) and replay the forward inside the backward task
                # (simulator.py:144-149)
                params = set(prog.params_used)
                kept = ({v: _retained(t) for v, t in env.items() if v not in params},
                        {v: t for v, t in env.items() if v in params})
            self.ops.place = self._placement(ex)
            try:
                self.ops.run_ops(prog.ops, env)
            finally:
                self.ops.place = {}
            for v, bid in ex["outs"].items():
                st.put(bid, env[v])
            if kept is not None:
                st.put(ex["stash_out"], {"__remat__": kept})
            elif ex["stash_out"]:
                st.put(ex["stash_out"], {v: env[v] for v in prog.stash})
        elif kind == "stage-bwd":
            prog = p.bwd_programs[ex["stage"]]
            env = {v: st.get(bid, at) for v, bid in ex["feeds"].items()}
            if ex["stash_in"]:
                stash = st.get(ex["stash_in"], at)
                if "__remat__" in stash:
                    kept, params = stash["__remat__"]
                    fenv = {**kept, **params}
                    self.ops.run_ops(p.fwd_programs[ex["stage"]].ops, fenv)
                    stash = {v: fenv[v] for v in p.fwd_programs[ex["stage"]].stash}
                env.update(stash)
            acc = self._fusable_accumulators(ex) if self.ops.fuse_acc else {}
            self.ops.acc_into = acc
            self.ops.place = self._placement(ex)
            try:
                self.ops.run_ops(prog.ops, env)
            finally:
                self.ops.acc_into = {}
                self.ops.place = {}
            for v, bid in ex["outs"].items():
                st.put(bid, env[v])
                if v in acc and isinstance(env[v], torch.Tensor) and env[v] is acc[v]:
                    self.fused.add(bid)
        elif kind == "add":
            lhs = ex["lhs"]
            if ex["rhs"] in self.fused:   # its producer already added it onto lhs
                self.fused.discard(ex["rhs"])
                st.get(ex["rhs"], at)
                st.put(ex["out"], st.get(lhs, at))
            else:
                st.put(ex["out"], self.ops.add(st.get(lhs, at), st.get(ex["rhs"], at),
                                               inplace=self._may_overwrite(lhs, task.uid)))
        elif kind == "concat":
            st.put(ex["out"], self.ops.concat_losses([st.get(b, at) for b in ex["parts"]]))
        elif kind == "sgd-update":
            st.put(ex["out"], self.ops.sgd(st.get(ex["param"], at), st.get(ex["grad"], at),
                                           st.get(ex["lr"], at), inplace=self.inplace))
        else:
            raise ExecutorFault(f"unknown task payload {kind!r}")
        if self.timeline:
            self.stamp(s0 + 1)
            self.events.append((task.kind if task.is_loop else "aux", task.uid, s0, s0 + 1))

    def _placement(self, ex) -> dict:
        """{output value: peer slot} for this task's outputs that go to a
        peer-memory channel (DeviceOps.place)."""
        if not self._peer_out:
            return {}
        return {v: self._peer_out[bid] for v, bid in ex["outs"].items() if bid in self._peer_out}

    def _fusable_accumulators(self, ex) -> dict:
        """{bwd output value: running-sum tensor} for partial gradients whose
        only reader is the next grad-merge add on this actor, when that add may
        update its lhs in place and the lhs already exists: the producer then
        adds its partial onto the lhs itself (acc + p, the same fp32 add) and
        the add task only renames (taskgraph.py:369-433 order unchanged)."""
        out = {}
        for v, bid in ex["outs"].items():
            hit = self._add_by_rhs.get(bid)
            if hit is None:
                continue
            uid, lhs = hit
            b = self.tg.buffers[bid]
            if b.consumers != {uid} or b.is_output or lhs not in self.store.data:
                continue
            if not self._may_overwrite(lhs, uid):
                continue
            t = self.store.data[lhs]
            if isinstance(t, torch.Tensor) and t.dtype == torch.float32 and t.dim() == 1:
                out[v] = t
        return out

    def _may_overwrite(self, bid: str, uid: str) -> bool:
        """True when ``bid``'s only reader is this task, it is not a step output,
        not a received buffer, and has no send in flight: then the running sum
        can be updated in place (the fused accumulator)."""
        b = self.tg.buffers[bid]
        return (b.consumers == {uid} and not b.is_output and b.kind not in (PARAM, OPT_STATE)
                and bid not in self.store.received and not self.store.outstanding.get(bid))


def _wire_meta_fn(tg: TaskGraph, mode: Mode):
    g = tg.partition.graph

    def meta(bid: str):
        b = tg.buffers[bid]
        v = b.meta.get("value")
        if v is not None:
            spec = g.spec_of(v)
            op = g.producer(v)
            if op.kind == "input-read" and op.attr_or("token_ids", 0):
                return tuple(spec.dims), torch.int32
            if v in g.params:
                return tuple(spec.dims), mode.master
            return tuple(spec.dims), mode.act
        q = b.meta.get("param")
        if q is not None:
            return tuple(g.spec_of(q).dims), mode.master
        raise ExecutorFault(f"no wire layout for buffer {bid}")
    return meta


def _worker(act: _Actor, instrs, tg: TaskGraph, channels: dict, ctl: _Control, delay_fn,
            counting, epilogue=None):
    a = act.actor
    try:
        with torch.cuda.device(act.device), torch.cuda.stream(act.stream):
            if act.timeline:
                act.stamp(0)
            for idx, ins in enumerate(instrs):
                ctl.heartbeat[a] = f"[{idx}] {_brief(ins)}"
                if delay_fn is not None:
                    d = delay_fn(a, idx)
                    if d:
                        time.sleep(d)
                ctl.check(a)
                at = f"instruction {idx}"
                if isinstance(ins, RunTask):
                    act.run_task(tg.tasks[ins.task], at)
                elif isinstance(ins, SendStart):
                    ch = channels[(a, ins.dst)]
                    value = act.store.get(ins.buffer, at)
                    act.store.note_send(ins.buffer, ch, ins.seq)
                    counting(a, ins.dst, ins.buffer)
                    ch.send(ins.seq, ins.buffer, value, act.stream)
                elif isinstance(ins, SendWait):
                    channels[(a, ins.dst)].wait_consumed(ins.seq, ctl, a, act.stream)
                elif isinstance(ins, RecvStart):
                    channels[(ins.src, a)].post_recv(ins.seq, ins.buffer, act.stream)
                elif isinstance(ins, RecvWait):
                    bid, value = channels[(ins.src, a)].recv(ins.seq, ctl, a, act.stream)
                    act.store.received.add(bid)
                    act.store.put(bid, value)
                elif isinstance(ins, Delete):
                    act.store.delete(ins.buffer, at)
                elif isinstance(ins, FlushPendingDeletes):
                    act.store.flush()
                else:
                    raise ExecutorFault(f"actor {a}: unknown instruction {ins!r}")
                act.last_issued = idx
            if epilogue is not None:
                epilogue(act, ctl)
            act.end_event = torch.cuda.Event()
            act.end_event.record(act.stream)
        ctl.heartbeat[a] = "done"
    except _Aborted:
        pass
    except BaseException as e:  # noqa: BLE001 - forwarded to the driver
        ctl.fail(e)


# ---------------------------------------------------------------------------
# Engine


_ENGINE_IDS = itertools.count()


def exchange_channel_ids(store, tag: str, me: int, channels, new_id) -> dict:
    """Rendezvous for the per-directed-channel communicators.

    For every plan channel (src, dst) this rank belongs to, the sender creates
    the 128-byte NCCL unique id and publishes it under ``pp200/<tag>/src->dst``;
    the receiver reads it.  Channels are visited in one global sorted order on
    every rank, so the pairwise communicator inits that follow cannot wait on
    each other in a cycle.  Returns {(src, dst): id bytes} for this rank.
    """
    out = {}
    for src, dst in sorted(channels):
        if me not in (src, dst):
            continue
        key = f"pp200/{tag}/{src}->{dst}"
        if me == src:
            raw = new_id()
            store.set(key, raw)
        else:
            raw = store.get(key)
        out[(src, dst)] = bytes(raw)
    return out


def tied_holders(tg: TaskGraph) -> list:
    """[(param, low actor, {holder actor: param buffer id})] for parameters held
    by more than one actor (tied weights).  The reference updates such a
    parameter only on the actor owning its lowest stage (taskgraph.py:349-361);
    a multi-step run must carry the new value to the other holders before
    their next use -- the re-broadcast of SURVEY.md §8(f) item 4."""
    holders: dict = {}
    for bid, b in tg.buffers.items():
        if b.kind == PARAM and b.producer is None:   # seeded copies, not wnew outputs
            holders.setdefault(b.meta["param"], {})[b.home] = bid
    out = []
    for q in sorted(holders):
        if len(holders[q]) > 1:
            out.append((q, tg.tasks[f"opt:{q}"].actor, dict(sorted(holders[q].items()))))
    return out


def _clone_value(v):
    if isinstance(v, Param):
        return Param(v.master.clone(), None if v.shadow is None else v.shadow.clone())
    return tensor_of(v).clone()


def _dist_world():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        return dist.get_rank(), dist.get_world_size()
    return None


class PipelineEngine:
    """Reusable executor for one (CommPlan, TaskGraph): streams, channels and
    NCCL communicators are created once; ``step`` runs one training step."""

    def __init__(self, cp: CommPlan, tg: TaskGraph, mode: str | Mode = "fp64",
                 gpt: GPTConfig | None = None, devices=None, timeline: bool = False,
                 transport: str | None = None, remat: str = REMAT_NONE):
        if not cp.fused:
            raise ExecutorFault("plan must be fused before execution")
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2412_14374_b200 needs a CUDA device (no CPU fallback)")
        _lib.lib()  # fail loudly if the extension is missing
        self.cp, self.tg = cp, tg
        self.mode = MODES[mode] if isinstance(mode, str) else mode
        self.gpt = gpt
        if remat not in (REMAT_NONE, REMAT_FULL):
            raise ExecutorFault(f"unknown remat policy {remat!r}")
        self.remat = remat
        self.P = cp.num_actors
        self.timeline = timeline
        dw = _dist_world()
        self.distributed = dw is not None
        self.stats = RunStats()
        if self.distributed:
            rank, world = dw
            if world != self.P:
                raise ExecutorFault(f"world size {world} != plan actors {self.P}")
            self.local = [rank]
            dev = torch.device("cuda", torch.cuda.current_device())
            self.devices = {rank: dev}
        else:
            self.local = list(range(self.P))
            if devices is None:
                devices = [torch.cuda.current_device()]
            devs = [torch.device("cuda", d) if isinstance(d, int) else torch.device(d)
                    for d in devices]
            self.devices = {a: devs[a % len(devs)] for a in self.local}
            if len({self.devices[a] for a in self.local}) > 1 and cp.channels:
                raise ExecutorFault("single-process multi-GPU channels are not supported; "
                                    "launch one process per GPU (torchrun)")
        self._wire_meta = _wire_meta_fn(tg, self.mode)
        # inter-process channels: "peer" (NVLink peer memory, producers write
        # into the receiver's slots) or "nccl" (a communicator per channel)
        # (peer needs every rank on this node: CUDA IPC + NVLink)
        one_node = os.environ.get("LOCAL_WORLD_SIZE", os.environ.get("WORLD_SIZE", "1")) == \
            os.environ.get("WORLD_SIZE", "1")
        self.transport = transport or os.environ.get("PP200_TRANSPORT",
                                                     "peer" if one_node else "nccl")
        if self.transport not in ("peer", "nccl"):
            raise ExecutorFault(f"unknown transport {self.transport!r}")
        self._peer_allocs: list = []
        self._peer_opens: list = []
        self._peer_made = False
        self._abort_word = None  # (host, device) address of the peer waits' abort word
        self.peer_bytes = 0     # receive slots this rank allocated (outside torch's allocator)
        self._faulted = False   # a step raised: streams were released, state is garbage
        self._tag = next(_ENGINE_IDS)   # same sequence on every rank (engines built in order)
        self._resident: dict | None = None   # bid -> device value (load_params)
        self._tied = tied_holders(tg)
        self._tied_ch: dict = {}
        self._tied_ready = False
        self._captures: list = []
        self._ops = {a: DeviceOps(tg.partition, self.mode, self.devices[a],
                                  torch.cuda.Stream(device=self.devices[a]), gpt)
                     for a in self.local}
        self._channels = self._make_channels()

    def _make_channels(self, keys=None, wire_meta=None):
        plan = keys is None
        keys = self.cp.channels if keys is None else keys
        if not self.distributed:
            return {key: LocalChannel(*key) for key in keys}
        import ctypes

        import torch.distributed as dist
        store = dist.distributed_c10d._get_default_store()
        tag = next(_ENGINE_IDS)
        me = self.local[0]
        dev = self.devices[me]
        wire_meta = self._wire_meta if wire_meta is None else wire_meta
        if plan and self.transport == "peer":
            return self._make_peer_channels(store, tag, me, dev)

        def new_id() -> bytes:
            uid = (ctypes.c_char * 128)()
            _lib.call("pc_p2p_unique_id", uid)
            return bytes(uid)

        out = {}
        for (src, dst), raw in exchange_channel_ids(store, f"e{tag}", me, keys,
                                                    new_id).items():
            idbuf = (ctypes.c_char * 128).from_buffer_copy(raw)
            comm = ctypes.c_void_p()
            with torch.cuda.device(dev):
                _lib.call("pc_p2p_comm_init", ctypes.byref(comm), 2, idbuf, 0 if me == src else 1)
            out[(src, dst)] = NcclChannel(src, dst, me, comm, dev, wire_meta)
        return out

    def _make_peer_channels(self, store, tag, me, dev):
        """Receiver side allocates and publishes its slots first, then every
        sender maps its channels (so no rank waits on another's mapping)."""
        import ctypes
        self._peer_made = True
        hw, dw = ctypes.c_void_p(), ctypes.c_void_p()
        _lib.call("pc_host_word_alloc", ctypes.byref(hw), ctypes.byref(dw))
        self._abort_word = (hw.value, dw.value)
        out = {}
        layout = {key: _slot_layout(bids, self._wire_meta) for key, bids in self.cp.channels.items()}
        for (src, dst) in sorted(self.cp.channels):
            if dst != me:
                continue
            slots, total = layout[(src, dst)]
            ptr, h = ctypes.c_void_p(), (ctypes.c_char * 64)()
            with torch.cuda.device(dev):
                _lib.call("pc_peer_alloc", total, ctypes.byref(ptr), h)
            self._peer_allocs.append(ptr.value)
            self.peer_bytes += total
            store.set(f"pp200/e{tag}/peer/{src}->{dst}", bytes(h))
            out[(src, dst)] = PeerChannel(src, dst, me, ptr.value, self.cp.channels[(src, dst)],
                                          slots, self._abort_word)
        for (src, dst) in sorted(self.cp.channels):
            if src != me:
                continue
            slots, _ = layout[(src, dst)]
            h = (ctypes.c_char * 64).from_buffer_copy(store.get(f"pp200/e{tag}/peer/{src}->{dst}"))
            ptr = ctypes.c_void_p()
            with torch.cuda.device(dev):
                _lib.call("pc_peer_open", h, ctypes.byref(ptr))
            self._peer_opens.append(ptr.value)
            out[(src, dst)] = PeerChannel(src, dst, me, ptr.value, self.cp.channels[(src, dst)],
                                          slots, self._abort_word)
        return out

    # -- resident training state (multi-step) --
    def load_params(self, params):
        """Keep ``params`` resident on this process's actors for multi-step
        training: one private copy per holding actor (executor.py:409-410
        copies per actor too).  Afterwards ``step(None, batch)`` /
        ``capture(None, batch)`` train in place: the SGD task overwrites the
        resident value, and each tied parameter's new value is sent from the
        actor that updated it to its other holders at the end of the step
        (one extra message per holder, on its own channel), so step k+1 sees
        exactly what the reference would seed from step k's ``new_params``."""
        is_gpt = self.gpt is not None
        res = {}
        for bid, buf in self.tg.buffers.items():
            if buf.kind != PARAM or buf.producer is not None or buf.home not in self.local:
                continue
            dev = self.devices[buf.home]
            with torch.cuda.device(dev):
                res[bid] = _clone_value(to_device_param(params[buf.meta["param"]], self.mode,
                                                        dev, is_gpt))
        for d in {self.devices[a] for a in self.local}:
            torch.cuda.synchronize(d)
        self._resident = res
        if not self._tied_ready:   # every rank takes this branch once (same channel tags)
            self._tied_ready = True
            keys = sorted({(low, h) for _, low, hs in self._tied for h in hs if h != low})
            g = self.tg.partition.graph

            def meta(bid):
                return tuple(g.spec_of(bid.split(":", 1)[1]).dims), self.mode.master
            if keys:
                self._tied_ch = self._make_channels(keys, meta)

    def state_dict(self, to_host: bool = True) -> dict:
        """{param: current value} for the parameters this process updates
        (each taken from the actor owning its lowest stage)."""
        if self._resident is None:
            raise ExecutorFault("no resident parameters: call load_params first")
        out = {}
        for bid, v in self._resident.items():
            b = self.tg.buffers[bid]
            q = b.meta["param"]
            if self.tg.tasks[f"opt:{q}"].actor != b.home:
                continue
            t = v.master if isinstance(v, Param) else tensor_of(v)
            out[q] = t.detach().cpu().numpy() if to_host else t
        return out

    def _rebroadcast(self, act, ctl):
        """End-of-step epilogue in resident mode: low actor -> other holders."""
        a = act.actor
        for seq, (q, low, hs) in enumerate(self._tied):
            if a == low:
                src = self._resident[hs[low]]
                t = src.master if isinstance(src, Param) else tensor_of(src)
                for h in hs:
                    if h == low:
                        continue
                    ch = self._tied_ch[(low, h)]
                    ch.send(seq, f"wnew:{q}", t, act.stream)
                    if isinstance(ch, NcclChannel):
                        act.stream.wait_event(ch.sent[seq])   # joins the send stream
            elif a in hs:
                ch = self._tied_ch[(low, a)]
                ch.post_recv(seq, f"wnew:{q}", act.stream)
                _, buf = ch.recv(seq, ctl, a, act.stream)
                dst = self._resident[hs[a]]
                m = dst.master if isinstance(dst, Param) else tensor_of(dst)
                m.copy_(buf)
                if isinstance(dst, Param) and dst.shadow is not None:
                    _lib.call("pc_cast", _PC_OF[m.dtype], _lib.PC_BF16, m.numel(), m.data_ptr(),
                              dst.shadow.data_ptr(), act.stream.cuda_stream)

    def close(self):
        # graphs that captured NCCL work pin their communicators: release the
        # graphs first, then destroy
        for cs in self._captures:
            if cs.graph is not None:
                cs.graph.reset()
                cs.graph = None
        self._captures.clear()
        if self._faulted:
            # released streams drain within seconds; if one does not, leak the
            # transport state instead of hanging the process on it
            if not self._drain(30.0):
                self._peer_made = False
                return
        else:
            for d in {self.devices[a] for a in self.local}:
                torch.cuda.synchronize(d)
        for ch in list(self._channels.values()) + list(self._tied_ch.values()):
            if isinstance(ch, NcclChannel) and ch.comm:
                # the device is drained, so nothing is in flight on the pair: a local
                # abort frees the communicator (ncclCommDestroy can wait on the peer)
                _lib.call("pc_p2p_abort", ch.comm)
                ch.comm = None
        if self._peer_made:
            self._peer_made = False
            for ptr in self._peer_opens:
                _lib.call("pc_peer_close", ptr)
            self._peer_opens = []
            # free this rank's slots once every mapping of them is closed; a
            # peer that never gets here (it faulted and could not drain) makes
            # this rank leak its slots rather than block
            if self._close_barrier(60.0):
                for ptr in self._peer_allocs:
                    _lib.call("pc_peer_free", ptr)
            self._peer_allocs = []
            if self._abort_word is not None:
                _lib.call("pc_host_word_free", self._abort_word[0])
                self._abort_word = None

    # -- seeding (executor.py:405-414) --
    def _seed(self, actors: dict, params, batch, lr):
        tg = self.tg
        p = tg.partition
        M = tg.schedule.num_microbatches
        # one array for a single-input graph, else {input name: array}
        if isinstance(batch, dict):
            feeds = {name: split_batch(v, M) for name, v in batch.items()}
        else:
            (x_in,) = sorted(p.graph.inputs)
            feeds = {x_in: split_batch(batch, M)}
        is_tok = {name: p.graph.producer(name).attr_or("token_ids", 0) == 1 for name in feeds}
        is_gpt = self.gpt is not None
        if params is None and self._resident is None:
            raise ExecutorFault("params=None needs resident parameters (load_params)")
        for act in actors.values():  # per-step caches on parameters start over
            act.ops.step_epoch += 1
        for bid, buf in tg.buffers.items():
            if buf.producer is not None or buf.home not in actors:
                continue
            act = actors[buf.home]
            with torch.cuda.device(act.device), torch.cuda.stream(act.stream):
                if buf.kind == PARAM:
                    v = (self._resident[bid] if params is None else
                         to_device_param(params[buf.meta["param"]], self.mode, act.device, is_gpt))
                elif buf.kind == OPT_STATE:
                    v = float(lr)
                else:
                    name = buf.meta.get("value", buf.meta.get("input"))
                    if name not in feeds:
                        (name,) = feeds if len(feeds) == 1 else (None,)
                    v = to_device_input(feeds[name][buf.meta["microbatch"]], self.mode,
                                        act.device, is_tok[name])
                act.store.put(bid, v)

    def step(self, params, batch, lr: float = 0.1, timeout_s: float = 30.0, delay_fn=None,
             strict_store: bool = True, to_host: bool = True,
             timeline: bool | None = None) -> ExecutionResult:
        self._check_usable()
        stats = RunStats()
        tl = self.timeline if timeline is None else timeline
        ctl = _Control(timeout_s)
        resident = params is None
        for ch in list(self._channels.values()) + list(self._tied_ch.values()):
            ch.reset()
        actors = {a: _Actor(a, self.tg, self._ops[a], stats, tl, inplace=resident,
                            instrs=self.cp.programs[a].instrs, channels=self._channels)
                  for a in self.local}
        for act in actors.values():
            act.remat = self.remat
        for a, act in actors.items():
            # params / inputs are copied on the current stream; the actor stream waits
            with torch.cuda.device(act.device):
                act.stream.wait_stream(torch.cuda.current_stream(act.device))
        self._seed(actors, params, batch, lr)
        lock = threading.Lock()

        def counting(src, dst, bid):
            with lock:
                stats.channel_counts[(src, dst)] = stats.channel_counts.get((src, dst), 0) + 1
                stats.sent_buffers.append((src, dst, bid))

        if self.distributed:
            import torch.distributed as dist
            dist.barrier()
        workers = []
        for a in self.local:
            stats.driver_messages += 1  # program dispatch
            w = threading.Thread(target=_worker, name=f"actor-{a}",
                                 args=(actors[a], self.cp.programs[a].instrs, self.tg,
                                       self._channels, ctl, delay_fn, counting,
                                       self._rebroadcast if resident else None), daemon=True)
            workers.append(w)
            w.start()
        for w in workers:
            w.join(timeout=max(ctl.remaining(), 0.0) + 1.0)
        hung = [w for w in workers if w.is_alive()]
        if hung:
            ctl.abort.set()
            self._abort_channels()
            dump = ", ".join(f"actor {a}: {ctl.heartbeat.get(a, '?')}" for a in self.local)
            raise LivenessFault(f"watchdog timeout; blocked instructions: {dump}")
        if ctl.faults:
            # streams may already wait on messages the failed actor will never send
            self._abort_channels()
            raise ctl.faults[0]
        self._wait_devices(actors, ctl)
        if self.distributed and self._peer_faulted():
            # a released wait on the faulted rank lets its stream run on and send
            # garbage downstream: this rank finished on it and must not report it
            self._faulted = True
            raise LivenessFault("a peer rank faulted in this step (its watchdog fired); "
                                "results are invalid")
        for key, ch in list(self._channels.items()) + list(self._tied_ch.items()):
            if not ch.drained():
                raise ChannelOrderFault(f"channel {key} holds undelivered messages at step end")
        # after the device finished, in-flight sends are complete: final flush
        for act in actors.values():
            act.store.flush()
        return self._gather(actors, stats, strict_store, to_host)

    def capture(self, params, batch, lr: float = 0.1, timeout_s: float = 600.0,
                timeline: bool = False):
        """Capture this process's actor program as one CUDA graph.

        The host-side interpreter (store, deletions, channel bookkeeping) runs
        once while every launch -- libpp200 kernels, NCCL sends/receives on the
        channel streams, event waits -- is recorded; ``CapturedStep.replay``
        then re-issues the whole fused program with a single launch (the
        paper's one-dispatch-per-actor fusion, at zero host
        cost).  Needs one actor per process (P=1, or a torchrun launch) and a
        prior warm-up step (NCCL connects lazily).
        """
        if len(self.local) != 1:
            raise ExecutorFault("graph capture needs exactly one actor per process")
        self._check_usable()
        a = self.local[0]
        stats = RunStats()
        ctl = _Control(timeout_s)
        resident = params is None
        for ch in list(self._channels.values()) + list(self._tied_ch.values()):
            ch.reset()
        act = _Actor(a, self.tg, self._ops[a], stats, timeline, inplace=resident,
                     instrs=self.cp.programs[a].instrs, channels=self._channels)
        act.remat = self.remat
        actors = {a: act}
        with torch.cuda.device(act.device):
            act.stream.wait_stream(torch.cuda.current_stream(act.device))
        self._seed(actors, params, batch, lr)
        inputs = {bid: v for bid, v in act.store.data.items()
                  if self.tg.buffers[bid].kind not in (PARAM, OPT_STATE)}
        lock = threading.Lock()

        def counting(src, dst, bid):
            with lock:
                stats.channel_counts[(src, dst)] = stats.channel_counts.get((src, dst), 0) + 1
                stats.sent_buffers.append((src, dst, bid))

        if self.distributed:
            import torch.distributed as dist
            dist.barrier()
        stats.driver_messages += 1
        launches0 = _lib.launch_count
        graph = torch.cuda.CUDAGraph(keep_graph=True)
        with torch.cuda.device(act.device):
            torch.cuda.synchronize()
            try:
                with torch.cuda.graph(graph, stream=act.stream):
                    _worker(act, self.cp.programs[a].instrs, self.tg, self._channels, ctl, None,
                            counting, self._rebroadcast if resident else None)
            except Exception as e:
                # a fault inside the worker leaves the capture unjoined, and ending
                # the capture then fails too: report the fault, not that symptom
                if ctl.faults:
                    raise ctl.faults[0] from e
                raise
        if ctl.faults:
            raise ctl.faults[0]
        # send-completion events recorded into the graph cannot be queried; every
        # replay runs the sends to completion, so the captured buffers are free.
        for ch in list(self._channels.values()) + list(self._tied_ch.values()):
            if isinstance(ch, NcclChannel):
                ch.sent.clear()
        act.store.flush()
        tl_on, act.timeline = act.timeline, False   # timestamps are read after a replay
        result = self._gather(actors, stats, strict_store=False, to_host=False)
        act.timeline = tl_on
        import ctypes
        nk = ctypes.c_int64(0)
        _lib.call("pc_graph_kernel_nodes", ctypes.c_void_p(graph.raw_cuda_graph()), ctypes.byref(nk))
        graph.instantiate()
        cs = CapturedStep(self, graph, act, inputs, result)
        self._captures.append(cs)
        cs.launches = _lib.launch_count - launches0   # libpp200 calls recorded per replay
        cs.kernels = nk.value                         # kernel nodes = kernels per replay
        return cs

    def _close_barrier(self, timeout_s: float) -> bool:
        """All ranks reached close() (store counter; bounded, unlike dist.barrier)."""
        import torch.distributed as dist
        store = dist.distributed_c10d._get_default_store()
        key = f"pp200/close/{self._tag}"
        store.add(key, 1)
        world = dist.get_world_size()
        deadline = time.monotonic() + timeout_s
        while store.add(key, 0) < world:
            if time.monotonic() > deadline:
                return False
            time.sleep(0.002)
        return True

    def _fault_key(self) -> str:
        return f"pp200/fault/{self._tag}"

    def _peer_faulted(self) -> bool:
        import torch.distributed as dist
        return dist.distributed_c10d._get_default_store().check([self._fault_key()])

    def _abort_channels(self):
        """Fault path (executor.py:443-451): NCCL communicators are aborted, peer
        receivers release their own flag waits, so every stream drains; the
        engine refuses further steps.  Across processes the fault is posted to
        the rendezvous store first, so a rank whose step completes on the data
        the released streams sent afterwards raises too."""
        self._faulted = True
        if self.distributed:
            try:
                import torch.distributed as dist
                dist.distributed_c10d._get_default_store().set(self._fault_key(), "1")
            except Exception:  # noqa: BLE001 - best effort, the fault itself is reported
                pass
        for ch in list(self._channels.values()) + list(self._tied_ch.values()):
            try:
                ch.abort()
            except Exception:  # noqa: BLE001 - best effort, the fault itself is reported
                pass

    def _check_usable(self):
        if self._faulted:
            raise ExecutorFault("engine was aborted by an earlier fault; build a new PipelineEngine")

    def _drain(self, timeout_s: float) -> bool:
        """Bounded device synchronisation: True when every local device drained."""
        devs = sorted({self.devices[a] for a in self.local}, key=str)
        done = threading.Event()

        def sync():
            for d in devs:
                torch.cuda.synchronize(d)
            done.set()

        threading.Thread(target=sync, daemon=True, name="pp200-drain").start()
        return done.wait(timeout_s)

    def _wait_devices(self, actors, ctl: _Control):
        """Device-side watchdog: a stream that never drains (e.g. a receive
        whose send was dropped) aborts the communicators and raises."""
        pending = {a: act for a, act in actors.items() if act.end_event is not None}
        while pending:
            for a in list(pending):
                if pending[a].end_event.query():
                    del pending[a]
            if not pending:
                break
            if ctl.remaining() <= 0:
                self._abort_channels()
                dump = ", ".join(
                    f"actor {a}: device stream stalled after issuing [{act.last_issued}] "
                    f"{ctl.heartbeat.get(a, '?')}" for a, act in pending.items())
                raise LivenessFault(f"watchdog timeout; blocked instructions: {dump}")
            time.sleep(0.0005)

    def _gather(self, actors, stats: RunStats, strict_store: bool, to_host: bool):
        tg = self.tg
        grads, new_params, losses = {}, {}, None

        def out(v):
            t = v.master if isinstance(v, Param) else tensor_of(v)
            return t.detach().cpu().numpy() if to_host else t

        for a in sorted(actors):
            act = actors[a]
            store = act.store
            stats.driver_messages += 1  # result gather
            stats.final_live[a] = sorted(store.data)
            for bid in stats.final_live[a]:
                b = tg.buffers[bid]
                if b.kind == GRAD_TOTAL:
                    grads[b.meta["param"]] = out(store.data[bid])
                elif bid.startswith("wnew:"):
                    new_params[b.meta["param"]] = out(store.data[bid])
                elif bid == "loss:all":
                    losses = out(store.data[bid])
            if act.timeline:
                stats.timeline.extend(act.read_timeline())
        if strict_store:
            for a in sorted(actors):
                store = actors[a].store
                extra = [bid for bid in store.data
                         if tg.buffers[bid].kind not in (PARAM, OPT_STATE)
                         and not tg.buffers[bid].is_output]
                if extra or store.pending:
                    raise ExecutorFault(
                        f"actor {a} leaked buffers at step end: {sorted(extra)} "
                        f"pending={sorted(store.pending)}")
        if not self.distributed:
            missing = set(tg.partition.graph.params) - set(grads)
            if missing or losses is None:
                raise ExecutorFault(f"step outputs incomplete: grads missing {sorted(missing)}")
        self.stats = stats
        return ExecutionResult(grads=grads, losses=losses, new_params=new_params, stats=stats)


class CapturedStep:
    """A captured actor program: ``replay`` runs one full training step.

    ``result`` holds the step outputs (grads, losses, new params on this
    process's actor); their device memory belongs to the graph and is
    rewritten by every replay.  ``set_inputs`` copies a new batch into the
    graph's static input buffers (stream-ordered, before the replay)."""

    def __init__(self, engine, graph, act, inputs, result):
        self.engine, self.graph, self.act = engine, graph, act
        self.inputs = inputs
        self.result = result

    def set_inputs(self, batch):
        tg = self.engine.tg
        M = tg.schedule.num_microbatches
        # one array for a single-input graph, else {input name: array} (as _seed)
        if isinstance(batch, dict):
            split = {name: split_batch(v, M) for name, v in batch.items()}
        else:
            split = {None: split_batch(batch, M)}
        for bid, dst in self.inputs.items():
            meta = tg.buffers[bid].meta
            name = meta.get("value", meta.get("input"))
            mbs = split[name] if name in split else split[next(iter(split))]
            src = mbs[meta["microbatch"]]
            if isinstance(src, np.ndarray):
                src = torch.from_numpy(np.ascontiguousarray(src))
            dst = tensor_of(dst)
            dst.copy_(src.to(dst.dtype) if src.dtype != dst.dtype else src, non_blocking=True)

    def replay(self, batch=None, timeout_s: float | None = None):
        """Launch one captured step (asynchronous).  With ``timeout_s`` the call
        waits for the step and turns a device that does not drain in time into
        a LivenessFault, after releasing the channels (the graph's watchdog)."""
        if self.graph is None:
            raise ExecutorFault("captured step was released (engine closed)")
        self.engine._check_usable()
        if batch is not None:
            self.set_inputs(batch)
        self.graph.replay()
        if timeout_s is not None:
            ev = torch.cuda.Event()
            ev.record()
            deadline = time.monotonic() + timeout_s
            while not ev.query():
                if time.monotonic() > deadline:
                    self.engine._abort_channels()
                    raise LivenessFault(f"watchdog timeout: captured step of actor "
                                        f"{self.act.actor} did not finish in {timeout_s} s")
                time.sleep(0.0005)
        return self.result

    def release(self):
        """Free the graph (and its hold on the NCCL communicators) now."""
        if self.graph is not None:
            torch.cuda.synchronize(self.act.device)
            self.graph.reset()
            self.graph = None
        if self in self.engine._captures:
            self.engine._captures.remove(self)

    def timeline(self) -> list:
        """(actor, kind, uid, start_ms, end_ms) of the last replay, when the
        step was captured with ``timeline=True`` (timestamp kernels in the graph)."""
        torch.cuda.synchronize(self.act.device)
        return self.act.read_timeline()


def split_batch(batch, M: int):
    """executor.py:110-114 (rows split into M equal microbatches)."""
    n = batch.shape[0]
    if n % M != 0:
        raise ValueError(f"batch of {n} rows does not split into {M} microbatches")
    step = n // M
    return [batch[i * step:(i + 1) * step] for i in range(M)]


def run_pipelined(cp: CommPlan, tg: TaskGraph, params, batch, lr: float = 0.1,
                  timeout_s: float = 30.0, delay_fn=None, strict_store: bool = True,
                  mode: str | None = None, gpt: GPTConfig | None = None, devices=None,
                  timeline: bool = False, to_host: bool = True,
                  remat: str = REMAT_NONE) -> ExecutionResult:
    """Execute a fused plan on B200(s).  Drop-in for executor.py:387-483.

    ``mode`` defaults from the parameter dtype (float64 -> "fp64", float32 ->
    "fp32"); GPT graphs (``gpt`` given) default to "bf16".
    """
    if mode is None:
        if gpt is not None:
            mode = "bf16"
        else:
            any_p = next(iter(params.values()))
            mode = "fp32" if getattr(any_p, "dtype", None) in (np.float32, torch.float32) else "fp64"
    eng = PipelineEngine(cp, tg, mode=mode, gpt=gpt, devices=devices, timeline=timeline,
                         remat=remat)
    try:
        return eng.step(params, batch, lr=lr, timeout_s=timeout_s, delay_fn=delay_fn,
                        strict_store=strict_store, to_host=to_host)
    finally:
        eng.close()
