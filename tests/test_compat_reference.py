"""Drop-in adapter: a plan built by the reference package (when it is
importable, i.e. in the build container) is re-planned here byte-identically."""
import pathlib
import sys

import pytest

REF = pathlib.Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference package not present")


@pytest.mark.parametrize("fam,P,M,V,tied,commute", [
    ("1f1b", 4, 8, 1, False, True), ("gpipe", 2, 4, 1, True, False),
    ("interleaved", 2, 4, 2, True, True)])
def test_plan_from_reference_objects(fam, P, M, V, tied, commute):
    sys.path.insert(0, str(REF))
    try:
        from pipecraft import comms as RC, ir as RI, schedules as RS, taskgraph as RT
    finally:
        sys.path.remove(str(REF))
    from paper_2412_14374_b200.compat import plan_from_reference
    L = max(P * V, 4 if tied else 2)
    p = RI.derive_backward(RI.partition_stages(RI.build_model(RI.ModelConfig(
        layers=L, width=4, microbatch_size=2, yield_every=L // (P * V), tied_weights=tied))))
    s = {"gpipe": lambda: RS.gpipe(P, M), "1f1b": lambda: RS.one_f_one_b(P, M),
         "interleaved": lambda: RS.interleaved_1f1b(P, M, V)}[fam]()
    tg = RT.unroll(p, s)
    if commute:
        tg = RT.commute_grad_accumulation(tg)
    tg = RT.infer_outer_placement(tg, p)
    cp = RC.plan_pipeline(tg)
    mine_cp, mine_tg = plan_from_reference(cp, tg)
    assert mine_cp.to_json_str() == cp.to_json_str()
    assert mine_tg.to_json_str() == tg.to_json_str()
