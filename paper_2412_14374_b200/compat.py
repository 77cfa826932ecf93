"""Adapters for callers holding the reference package's objects.

A pipecraft user has ``(cp, tg)`` built by ``pipecraft`` (the reference,
pkg/src/pipecraft).  ``plan_from_reference`` rebuilds the same plan with this
package's planner from the reference objects' own JSON (forward graph,
schedule, commuting flag) and asserts that the resulting CommPlan JSON is
byte-identical to the reference's, so the B200 ``run_pipelined`` executes
exactly the program the reference planned.
"""
from __future__ import annotations

from . import comms as C
from . import ir as I
from . import schedules as S
from . import taskgraph as T


def graph_from_json(doc: dict, keep=None) -> I.StagedGraph:
    """StagedGraph from ``StagedGraph.to_json()`` output (optionally only op ids in ``keep``)."""
    ops = []
    for o in doc["ops"]:
        if keep is not None and o["id"] not in keep:
            continue
        spec = I.TensorSpec(tuple(o["result_spec"]["dims"]), o["result_spec"]["elem_bytes"])
        attrs = tuple(sorted(o.get("attrs", {}).items()))
        ops.append(I.OpNode(o["id"], o["kind"], tuple(o["operands"]), o["result"], spec,
                            flops=o["flops"], attrs=attrs))
    return I.StagedGraph(ops=ops, params=frozenset(doc["params"]), inputs=frozenset(doc["inputs"]),
                         outputs=tuple(doc["outputs"]))


def plan_from_reference(ref_cp, ref_tg, check: bool = True):
    """(CommPlan, TaskGraph) of this package equivalent to a reference plan."""
    part = ref_tg.partition
    fwd_ids = set(part.assignment)
    g = graph_from_json(part.graph.to_json(), keep=fwd_ids)
    p = I.derive_backward(I.partition_stages(g))
    s = S.schedule_from_json(ref_tg.schedule.to_json())
    tg = T.unroll(p, s)
    if ref_tg.commuted:
        tg = T.commute_grad_accumulation(tg)
    tg = T.infer_outer_placement(tg, p)
    cp = C.plan_pipeline(tg)
    if check and cp.to_json_str() != ref_cp.to_json_str():
        raise C.CommsError("re-planned program differs from the reference plan")
    return cp, tg
