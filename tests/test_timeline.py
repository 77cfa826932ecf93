"""Schedule replay with task durations (timeline.py) on CPU: uniform task
costs reproduce the closed-form ideal bubble (simulator.py:346-348) for GPipe,
1F1B and interleaved 1F1B; link time only adds; the Gantt SVG is well formed."""
import xml.dom.minidom

import pytest

from paper_2412_14374_b200 import comms as C
from paper_2412_14374_b200 import ir as I
from paper_2412_14374_b200 import schedules as S
from paper_2412_14374_b200 import taskgraph as T
from paper_2412_14374_b200.timeline import render_svg, replay


def plan(P, M, V=1, fam="1f1b"):
    cfg = I.ModelConfig(layers=P * V * 2, width=8, microbatch_size=4, yield_every=2)
    p = I.derive_backward(I.partition_stages(I.build_model(cfg)))
    s = {"gpipe": lambda: S.gpipe(P, M), "1f1b": lambda: S.one_f_one_b(P, M),
         "int": lambda: S.interleaved_1f1b(P, M, V)}[fam]()
    tg = T.infer_outer_placement(T.commute_grad_accumulation(T.unroll(p, s)), p)
    return tg, C.plan_pipeline(tg)


def uniform(tg, bwd=2.0):
    d = {}
    for uid, t in tg.tasks.items():
        kind = t.exec.get("type", "")
        if kind == "stage-fwd":
            d[uid] = ("fwd", 1.0)
        elif kind == "stage-bwd":
            d[uid] = ("bwd", bwd)
    return d


@pytest.mark.parametrize("fam,P,M,V", [("gpipe", 2, 4, 1), ("1f1b", 4, 8, 1), ("1f1b", 8, 16, 1),
                                       ("int", 4, 8, 2)])
def test_uniform_replay_matches_ideal_bubble(fam, P, M, V):
    tg, cp = plan(P, M, V, fam)
    r = replay(cp, uniform(tg))
    ideal = (P - 1) / (V * M + P - 1)
    assert r.bubble_fraction(P) == pytest.approx(ideal, abs=1e-9)


def test_link_time_only_adds():
    tg, cp = plan(4, 8)
    base = replay(cp, uniform(tg)).makespan_ms
    slow = replay(cp, uniform(tg), link_ms=0.5).makespan_ms
    assert slow > base


def test_svg_well_formed():
    tg, cp = plan(2, 4, fam="gpipe")
    r = replay(cp, uniform(tg))
    doc = xml.dom.minidom.parseString(render_svg(r.intervals, 2, title="gpipe 2x4"))
    assert len(doc.getElementsByTagName("rect")) == sum(1 for e in r.intervals)
