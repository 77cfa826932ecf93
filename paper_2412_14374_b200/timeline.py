"""Measured timelines -> schedule replay and Gantt chart.

``PipelineEngine.step(timeline=True)`` / ``CapturedStep.timeline()`` record one
(actor, kind, task uid, start ms, end ms) interval per task from device
``%globaltimer`` stamps.  This module

* ``replay``: re-times the fused ``CommPlan`` with those measured task
  durations under the same execution model as the reference's discrete-event
  simulator (pkg/src/pipecraft/simulator.py:1-8: every actor is one serial
  compute resource, every directed actor pair a link that moves one transfer at
  a time in send order while compute overlaps) -- the "achievable ideal" of a
  configuration given its real kernels: the bubble that is left once
  dispatch / transfer overheads are removed (link time 0) or modelled
  (``link_ms``);
* ``render_svg``: draws measured or replayed intervals per actor (forward /
  backward / other tasks coloured like the reference's gantt.py:14-54).

The bubble definition is the reference's (simulator.py:241-270): idle share of
P x span, span = first loop-task start .. last loop-task end over all actors,
busy = any task interval.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from .comms import CommPlan, RecvStart, RecvWait, RunTask, SendStart, SendWait


@dataclass
class Replay:
    intervals: list = field(default_factory=list)  # (actor, kind, uid, start_ms, end_ms)
    makespan_ms: float = 0.0

    def bubble_fraction(self, num_actors: int) -> float:
        return bubble_fraction(self.intervals, num_actors)


def bubble_fraction(intervals, num_actors: int) -> float:
    loop = [e for e in intervals if e[1] in ("fwd", "bwd")]
    if not loop:
        return 0.0
    lo = min(e[3] for e in loop)
    hi = max(e[4] for e in loop)
    span = hi - lo
    if span <= 0:
        return 0.0
    busy = [0.0] * num_actors
    for a, _, _, s, e in intervals:
        s, e = max(s, lo), min(e, hi)
        if e > s:
            busy[a] += e - s
    return sum(span - b for b in busy) / (num_actors * span)


def task_durations(timeline) -> dict:
    """{task uid: (kind, measured duration ms)} from a recorded timeline."""
    return {uid: (kind, e - s) for _, kind, uid, s, e in timeline}


def replay(cp: CommPlan, durations: dict, link_ms=0.0) -> Replay:
    """Longest-path sweep of the fused plan with measured task durations.

    ``durations``: {uid: (kind, ms)} (``task_durations``); tasks missing from
    it take 0.  ``link_ms``: constant per-transfer time or a callable
    ``(src, dst, buffer) -> ms``.  Each actor runs its instruction stream in
    order; a RecvWait blocks until the matching transfer has arrived; a
    transfer leaves at its SendStart once the previous transfer on the same
    directed link has arrived (one at a time, in send order).
    """
    link = link_ms if callable(link_ms) else (lambda s, d, b, c=float(link_ms): c)
    P = cp.num_actors
    pc = [0] * P            # next instruction per actor
    clock = [0.0] * P       # actor time
    link_free: dict = {}    # (src, dst) -> time the link is free
    arrive: dict = {}       # (src, dst, seq) -> arrival time
    out = Replay()
    progress = True
    while progress:
        progress = False
        for a in range(P):
            instrs = cp.programs[a].instrs
            while pc[a] < len(instrs):
                ins = instrs[pc[a]]
                if isinstance(ins, RunTask):
                    kind, ms = durations.get(ins.task, ("other", 0.0))
                    s = clock[a]
                    clock[a] = s + ms
                    out.intervals.append((a, kind, ins.task, s, clock[a]))
                elif isinstance(ins, SendStart):
                    key = (a, ins.dst)
                    start = max(clock[a], link_free.get(key, 0.0))
                    t = start + link(a, ins.dst, ins.buffer)
                    link_free[key] = t
                    arrive[(a, ins.dst, ins.seq)] = t
                elif isinstance(ins, RecvWait):
                    t = arrive.get((ins.src, a, ins.seq))
                    if t is None:  # the sender has not issued it yet: come back later
                        break
                    clock[a] = max(clock[a], t)
                # SendWait / RecvStart / Delete / FlushPendingDeletes take no time
                pc[a] += 1
                progress = True
    stuck = [a for a in range(P) if pc[a] < len(cp.programs[a].instrs)]
    if stuck:
        raise RuntimeError(f"replay deadlocked on actors {stuck}")
    out.makespan_ms = max(clock) if clock else 0.0
    return out


_COLOURS = {"fwd": "#4e79a7", "bwd": "#f28e2b", "add": "#59a14f", "sgd": "#b07aa1"}


def render_svg(intervals, num_actors: int, width_px: int = 960, title: str = "") -> str:
    """One row per actor, one rectangle per task (fwd blue, bwd orange, grad
    merge green, optimizer purple, other grey), time axis in ms."""
    if not intervals:
        return '<svg xmlns="http://www.w3.org/2000/svg" width="10" height="10"/>'
    t0 = min(e[3] for e in intervals)
    t1 = max(e[4] for e in intervals)
    span = max(t1 - t0, 1e-9)
    row, top, left = 28, 30, 60
    plot_w = width_px - left - 10
    h = top + row * num_actors + 30
    parts = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{width_px}" height="{h}" '
             f'font-family="monospace" font-size="11">',
             f'<text x="{left}" y="18">{title} span {span:.2f} ms, bubble '
             f'{bubble_fraction(intervals, num_actors):.3f}</text>']
    for a in range(num_actors):
        y = top + a * row
        parts.append(f'<text x="4" y="{y + 17}">GPU {a}</text>')
    for a, kind, uid, s, e in intervals:
        x = left + (s - t0) / span * plot_w
        w = max((e - s) / span * plot_w, 0.5)
        y = top + a * row + 3
        colour = _COLOURS.get(kind, "#9c9c9c")
        parts.append(f'<rect x="{x:.2f}" y="{y}" width="{w:.2f}" height="{row - 6}" '
                     f'fill="{colour}"><title>{uid} {e - s:.3f} ms</title></rect>')
    y = top + row * num_actors + 18
    parts.append(f'<text x="{left}" y="{y}">0 ms</text>')
    parts.append(f'<text x="{left + plot_w - 60}" y="{y}">{span:.2f} ms</text>')
    parts.append("</svg>")
    return "\n".join(parts)
