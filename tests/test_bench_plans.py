"""bench.py plans every workload it can be asked for -- the driver's scaling run
launches 1, 2, 4 and 8 GPUs -- without a GPU: stage boundaries from the cost
model, a deadlock-free comm plan with one program per GPU."""
import pytest

import bench


@pytest.mark.parametrize("wl", ["C2", "C3", "C4", "C5", "FFN-C2"])
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_plan_every_workload_and_gpu_count(wl, P):
    W = bench.WORKLOADS[wl]
    cfg, tg, cp = bench.build_plan(P, dict(W["kw"]), W["M"], mode="fp64" if W["family"] == "ffn" else "bf16",
                                   family=W["family"], schedule=W.get("schedule", "1f1b"), V=W.get("V", 1))
    assert len(cp.programs) == P
    inter = W.get("schedule") == "interleaved" and P > 1 and W.get("V", 1) > 1
    stages = P * W.get("V", 1) if inter else P
    assert len(tg.partition.fwd_programs) == stages
    if W["family"] != "ffn" and stages > 1:
        y = list(cfg.yields)
        assert len(y) == stages - 1 and y == sorted(set(y))


def test_cost_model_head_heavier_than_a_block():
    from paper_2412_14374_b200 import ir as I
    for wl, fn, Cfg in (("C2", bench.block_costs, I.GPTConfig), ("C5", bench.llama_block_costs, I.LlamaConfig)):
        kw = dict(bench.WORKLOADS[wl]["kw"])
        c = fn(Cfg(**kw, yield_every=kw["layers"] + 2))
        assert len(c) == kw["layers"] + 2
        assert c[-1] > 2 * c[1] > 0 and 0 < c[0] < c[1]
