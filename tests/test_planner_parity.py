"""Bit-exact plan parity with the reference planner (north_star: "the inferred
task order and communication plan must be bit-exact").

Golden hashes come from the reference package itself (tests/golden/make_golden.py):
schedule, partition, taskgraph and commplan JSON for a grid of FFN configs,
random schedules from the reference's helpers.random_schedule, the crossing
schedule's deadlock witness, and GPT stage layouts (canonicalised gradient
names) planned by the reference on a mirror graph with the same topology.
"""
import hashlib
import json
import pathlib
import re

import pytest

from paper_2412_14374_b200 import comms as C
from paper_2412_14374_b200 import ir as I
from paper_2412_14374_b200 import schedules as S
from paper_2412_14374_b200 import taskgraph as T

GOLD = json.loads((pathlib.Path(__file__).parent / "golden" / "plans.json").read_text())


def sha(s):
    return hashlib.sha256(s.encode()).hexdigest()


def make_sched(fam, P, M, V):
    return {"gpipe": lambda: S.gpipe(P, M), "1f1b": lambda: S.one_f_one_b(P, M),
            "interleaved": lambda: S.interleaved_1f1b(P, M, V)}[fam]()


def lower(p, s, commute=True):
    tg = T.unroll(p, s)
    if commute:
        tg = T.commute_grad_accumulation(tg)
    tg = T.infer_outer_placement(tg, p)
    cp = C.infer_comms(tg, s)
    assert C.check_deadlock_free(cp).ok
    return tg, C.fuse(C.insert_deletions(cp, tg), tg)


def canon_gv(text):
    names = {}
    return re.sub(r"\bgv\d+\b", lambda m: names.setdefault(m.group(0), f"G{len(names)}"), text)


@pytest.mark.parametrize("doc", GOLD["ffn"], ids=lambda d: "{fam}-P{P}-M{M}-V{V}-L{layers}-t{tied}-c{commute}".format(**d["config"]))
def test_ffn_plan_bit_exact(doc):
    c = doc["config"]
    p = I.derive_backward(I.partition_stages(I.build_model(I.ModelConfig(
        layers=c["layers"], width=c["width"], microbatch_size=c["mbs"],
        yield_every=c["yield_every"], tied_weights=c["tied"]))))
    s = make_sched(c["fam"], c["P"], c["M"], c["V"])
    tg, cp = lower(p, s, c["commute"])
    assert sha(json.dumps(s.to_json(), indent=2, sort_keys=True)) == doc["schedule"]
    assert sha(json.dumps(p.to_json(), indent=2, sort_keys=True)) == doc["partition"]
    assert sha(tg.to_json_str()) == doc["taskgraph"]
    assert sha(cp.to_json_str()) == doc["commplan"]


@pytest.mark.parametrize("k", range(len(GOLD["random"])))
def test_random_schedule_plans_bit_exact(k):
    doc = GOLD["random"][k]
    s = S.schedule_from_json(doc["schedule"])
    p = I.derive_backward(I.partition_stages(I.build_model(I.ModelConfig(
        layers=s.num_stages, width=4, microbatch_size=2, yield_every=1))))
    _, cp = lower(p, s)
    assert sha(cp.to_json_str()) == doc["commplan"]


def test_full_commplan_text_matches_reference():
    want = (pathlib.Path(__file__).parent / "golden" / "commplan_gpipe_2x4.json").read_text()
    p = I.derive_backward(I.partition_stages(I.build_model(I.ModelConfig(
        layers=4, width=8, microbatch_size=4, yield_every=2))))
    _, cp = lower(p, S.gpipe(2, 4))
    assert cp.to_json_str() + "\n" == want
    # and the JSON round-trips into an identical plan object
    assert C.CommPlan.from_json(json.loads(want)).to_json_str() == cp.to_json_str()


def test_crossing_schedule_naive_deadlocks_inferred_safe():
    doc = GOLD["crossing"]
    s = S.schedule_from_json(doc["schedule"])
    p = I.derive_backward(I.partition_stages(I.build_model(I.ModelConfig(
        layers=4, width=4, microbatch_size=2, yield_every=1))))
    tg = T.infer_outer_placement(T.unroll(p, s), p)
    naive = C.naive_lowering(tg, s)
    rep = C.check_deadlock_free(naive)
    assert not rep.ok
    assert str(rep) == doc["naive_report"]
    assert sha(naive.to_json_str()) == doc["naive_commplan"]
    inferred = C.infer_comms(tg, s)
    assert C.check_deadlock_free(inferred).ok == doc["inferred_ok"] is True
    assert sha(inferred.to_json_str()) == doc["inferred_commplan"]


@pytest.mark.parametrize("lay", GOLD["gpt_mirror"], ids=lambda d: d["name"])
def test_gpt_plan_isomorphic_to_reference(lay):
    """Plan of the real GPT graph == reference plan of the mirror graph, up to
    gradient-value renaming (tied embedding commuting + non-adjacent token skip)."""
    cfg = I.GPTConfig(layers=lay["layers"], d_model=64, n_heads=2, d_ff=128, vocab=128,
                      seq_len=16, microbatch_size=2, yields=tuple(lay["yields"]) or None,
                      yield_every=lay["layers"] + 2)
    p = I.derive_backward(I.partition_stages(I.build_gpt(cfg)))
    s = make_sched(lay["fam"], lay["P"], lay["M"], lay["V"])
    _, cp = lower(p, s)
    assert sha(canon_gv(cp.to_json_str())) == lay["commplan_canon"]
    assert sorted([list(k) for k in cp.channels]) == lay["channels"]
    assert sum(len(v) for v in cp.channels.values()) == lay["messages"]


def test_gpt_token_skip_is_non_adjacent():
    cfg = I.GPTConfig(layers=12, d_model=64, n_heads=2, d_ff=128, vocab=128, seq_len=16,
                      microbatch_size=2, yields=(5, 9, 13))
    p = I.derive_backward(I.partition_stages(I.build_gpt(cfg)))
    _, cp = lower(p, S.one_f_one_b(4, 8))
    assert cp.channels[(0, 3)] == [f"act:x:mb{i}" for i in range(8)]
    assert cp.channels[(3, 0)] == ["gsum:w0:s3:k7"]  # one commuted tied-weight send


def test_balanced_yields():
    assert I.balanced_yields([1, 1, 1, 1], 2) == (2,)
    assert I.balanced_yields([1, 4, 4, 4, 4, 9], 3) == (3, 5)
    ys = I.balanced_yields([0.1] + [1.0] * 12 + [4.5], 4)
    assert len(ys) == 3 and ys[-1] == 13


@pytest.mark.parametrize("k", range(len(GOLD["cli_plan"])))
def test_plan_artifacts_match_reference_cli(k, tmp_path):
    """schedule.json / taskgraph.json / commplan.json byte-identical to what
    ``pipecraft plan`` writes for the same config (cli.py:194-204)."""
    from paper_2412_14374_b200 import plan_io
    doc = GOLD["cli_plan"][k]
    cfg = plan_io.PlanConfig(dict(doc["config"], output={"dir": str(tmp_path)}), tmp_path)
    _, s, tg, cp = plan_io.compile_plan(cfg)
    files = plan_io.write_plan(cfg.out_dir, s, tg, cp)
    for name, want in doc["files"].items():
        assert sha(files[name].read_text()) == want, name
    # the written artifacts load back: schedule file drives an identical plan
    again = plan_io.PlanConfig(dict(doc["config"], parallel=dict(
        doc["config"]["parallel"], schedule_file="schedule.json")), tmp_path)
    _, _, _, cp2 = plan_io.compile_plan(again)
    assert cp2.to_json_str() == cp.to_json_str()
    assert plan_io.load_commplan(files["commplan.json"]).to_json_str() == cp.to_json_str()


def test_plan_config_errors_cite_fields(tmp_path):
    from paper_2412_14374_b200 import plan_io
    base = {"model": {"layers": 4, "width": 4, "microbatch_size": 2, "yield_every": 2},
            "parallel": {"num_actors": 2, "num_microbatches": 4}}
    with pytest.raises(plan_io.ConfigError, match="^model.layers"):
        plan_io.PlanConfig({"model": {"width": 4, "microbatch_size": 2},
                            "parallel": base["parallel"]})
    with pytest.raises(plan_io.ConfigError, match="^parallel.schedule:"):
        plan_io.PlanConfig(dict(base, parallel=dict(base["parallel"], schedule="zb")))
    with pytest.raises(plan_io.ConfigError, match="^model.yield_every"):
        plan_io.compile_plan(plan_io.PlanConfig(dict(base, parallel=dict(base["parallel"],
                                                                          num_actors=4))))
    with pytest.raises(plan_io.ConfigError, match="^config: invalid JSON"):
        (tmp_path / "bad.json").write_text("{")
        plan_io.PlanConfig.load(tmp_path / "bad.json")
