"""Generate the golden fixtures under tests/golden/ from the REFERENCE package.

Runs only in the build container (it imports ``pipecraft`` from
/root/reference/pkg/src, which does not exist on GPU boxes).  The fixtures it
writes are small JSON files committed to the repo; tests compare the B200
build's planner and the numpy oracle against them.

    python tests/golden/make_golden.py

Outputs
  plans.json      sha256 of schedule / partition / taskgraph / commplan JSON for
                  a grid of FFN configs (reference planner), random schedules
                  (the reference's helpers.random_schedule), the crossing-
                  schedule deadlock witness, and canonicalised plans for GPT
                  stage layouts planned on a reference "mirror" graph.
  commplan_gpipe_2x4.json   one full commplan, for readable diffs.
  numerics.json   run_reference losses / grads / new params (float64) for FFN
                  configs, including tied weights.
  golden_seed0.json         copy of pkg/tests/fixtures/golden_seed0.json.
"""
from __future__ import annotations

import hashlib
import json
import pathlib
import re
import shutil
import sys

import numpy as np

REF = pathlib.Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

from helpers import crossing_schedule, init_batch, init_params, random_schedule  # noqa: E402
from pipecraft import comms as C  # noqa: E402
from pipecraft import ir as I  # noqa: E402
from pipecraft import schedules as S  # noqa: E402
from pipecraft import taskgraph as T  # noqa: E402
from pipecraft.executor import run_reference  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent


def sha(s: str) -> str:
    return hashlib.sha256(s.encode()).hexdigest()


def make_sched(fam, P, M, V):
    if fam == "gpipe":
        return S.gpipe(P, M)
    if fam == "1f1b":
        return S.one_f_one_b(P, M)
    return S.interleaved_1f1b(P, M, V)


def lower(p, s, commute=True):
    tg = T.unroll(p, s)
    if commute:
        tg = T.commute_grad_accumulation(tg)
    tg = T.infer_outer_placement(tg, p)
    cp = C.infer_comms(tg, s)
    assert C.check_deadlock_free(cp).ok
    return tg, C.fuse(C.insert_deletions(cp, tg), tg)


def canon_gv(text: str) -> str:
    """Rename gradient value ids gv<n> by first appearance (isomorphism check)."""
    names: dict[str, str] = {}

    def sub(m):
        return names.setdefault(m.group(0), f"G{len(names)}")
    return re.sub(r"\bgv\d+\b", sub, text)


def ffn_grid():
    grid = []
    for fam, P, M, V in [("gpipe", 1, 3, 1), ("gpipe", 2, 2, 1), ("gpipe", 2, 4, 1),
                         ("gpipe", 4, 8, 1), ("1f1b", 2, 2, 1), ("1f1b", 2, 4, 1),
                         ("1f1b", 4, 8, 1), ("1f1b", 4, 2, 1), ("1f1b", 8, 16, 1),
                         ("1f1b", 8, 32, 1), ("interleaved", 2, 4, 2),
                         ("interleaved", 4, 8, 2), ("interleaved", 8, 32, 2),
                         ("interleaved", 2, 6, 3)]:
        for tied in (False, True):
            for commute in ((True, False) if tied else (True,)):
                for per_stage in (1, 2):
                    L = P * V * per_stage
                    if tied and L < 2:
                        L = 2 * P * V
                    grid.append(dict(layers=L, width=4, mbs=2, yield_every=L // (P * V),
                                     tied=tied, commute=commute, fam=fam, P=P, M=M, V=V))
    return grid


def plan_doc(cfg):
    p = I.derive_backward(I.partition_stages(I.build_model(I.ModelConfig(
        layers=cfg["layers"], width=cfg["width"], microbatch_size=cfg["mbs"],
        yield_every=cfg["yield_every"], tied_weights=cfg["tied"]))))
    s = make_sched(cfg["fam"], cfg["P"], cfg["M"], cfg["V"])
    tg, cp = lower(p, s, cfg["commute"])
    return {
        "config": cfg,
        "schedule": sha(json.dumps(s.to_json(), indent=2, sort_keys=True)),
        "partition": sha(json.dumps(p.to_json(), indent=2, sort_keys=True)),
        "taskgraph": sha(tg.to_json_str()),
        "commplan": sha(cp.to_json_str()),
        "instructions": sum(len(pg.instrs) for pg in cp.programs),
        "messages": sum(len(v) for v in cp.channels.values()),
    }


def gpt_mirror(layers, yields, mbs=2, w=4):
    """Reference graph with the GPT stage topology: embed ~ matmul(x, w0),
    block k ~ matmul(h, w_k), head ~ matmul(h, w0) + x (token ids consumed on
    the last stage) -> sub-sample-loss.  Same values, params and boundary
    structure as ir.build_gpt."""
    act = I.TensorSpec((mbs, w))
    wsp = I.TensorSpec((w, w))
    cut = set(yields)
    ops = [I.OpNode("read_x", "input-read", (), "x", act),
           I.OpNode("read_w0", "parameter-read", (), "w0", wsp),
           I.OpNode("embed", "matmul", ("x", "w0"), "h0", act)]
    params = ["w0"]
    cur, blk = "h0", 1
    if blk in cut:
        ops.append(I.OpNode(f"yield{blk}", "yield-marker", (cur,), f"y{blk}", act))
        cur = f"y{blk}"
    for k in range(1, layers + 1):
        ops.append(I.OpNode(f"read_w{k}", "parameter-read", (), f"w{k}", wsp))
        params.append(f"w{k}")
        ops.append(I.OpNode(f"block{k}", "matmul", (cur, f"w{k}"), f"h{k}", act))
        cur = f"h{k}"
        blk += 1
        if blk in cut:
            ops.append(I.OpNode(f"yield{blk}", "yield-marker", (cur,), f"y{blk}", act))
            cur = f"y{blk}"
    ops += [I.OpNode("head", "matmul", (cur, "w0"), "lg", act),
            I.OpNode("head_t", "add", ("lg", "x"), "lt", act),
            I.OpNode("head_loss", "sub-sample-loss", ("lt",), "loss", I.TensorSpec(()))]
    g = I.StagedGraph(ops=ops, params=frozenset(params), inputs=frozenset({"x"}),
                      outputs=("loss",))
    g.validate()
    return I.derive_backward(I.partition_stages(g))


# GPT stage layouts of the BASELINE configs (yields over [embed, L blocks, head]).
GPT_LAYOUTS = [
    dict(name="C1", layers=4, yields=[3], fam="gpipe", P=2, M=4, V=1),
    dict(name="C2", layers=12, yields=[5, 9, 13], fam="1f1b", P=4, M=8, V=1),
    dict(name="C2-P2", layers=12, yields=[8], fam="1f1b", P=2, M=8, V=1),
    dict(name="C2-P1", layers=12, yields=[], fam="1f1b", P=1, M=8, V=1),
    dict(name="C3", layers=24, yields=[4, 8, 12, 16, 20, 23, 25], fam="1f1b", P=8, M=16, V=1),
    dict(name="C4", layers=24, yields=[2, 4, 5, 7, 9, 10, 12, 14, 15, 17, 19, 20, 22, 24, 25],
         fam="interleaved", P=8, M=32, V=2),
    dict(name="tiny-P4-gpipe", layers=2, yields=[1, 2, 3], fam="gpipe", P=4, M=4, V=1),
]


def gpt_docs():
    out = []
    for lay in GPT_LAYOUTS:
        p = gpt_mirror(lay["layers"], lay["yields"])
        s = make_sched(lay["fam"], lay["P"], lay["M"], lay["V"])
        tg, cp = lower(p, s)
        text = canon_gv(cp.to_json_str())
        out.append({**lay, "commplan_canon": sha(text),
                    "messages": sum(len(v) for v in cp.channels.values()),
                    "channels": sorted([list(k) for k in cp.channels])})
    return out


def random_docs():
    out = []
    for seed, (P, M, V) in enumerate([(2, 2, 1), (2, 4, 1), (3, 3, 1), (4, 4, 1), (2, 4, 2),
                                      (3, 2, 2), (4, 8, 1), (2, 3, 3)] * 3):
        rng = np.random.default_rng(1000 + seed)
        s = random_schedule(rng, P, M, V)
        p = I.derive_backward(I.partition_stages(I.build_model(I.ModelConfig(
            layers=P * V, width=4, microbatch_size=2, yield_every=1))))
        tg, cp = lower(p, s)
        out.append({"schedule": s.to_json(), "commplan": sha(cp.to_json_str())})
    return out


def crossing_doc():
    s = crossing_schedule()
    p = I.derive_backward(I.partition_stages(I.build_model(I.ModelConfig(
        layers=4, width=4, microbatch_size=2, yield_every=1))))
    tg = T.infer_outer_placement(T.unroll(p, s), p)
    naive = C.naive_lowering(tg, s)
    rep = C.check_deadlock_free(naive)
    inferred = C.infer_comms(tg, s)
    return {"schedule": s.to_json(), "naive_report": str(rep),
            "naive_commplan": sha(naive.to_json_str()),
            "inferred_ok": C.check_deadlock_free(inferred).ok,
            "inferred_commplan": sha(inferred.to_json_str())}


def numerics_docs():
    out = []
    for (L, w, mbs, M, tied, ye, seed) in [(2, 8, 2, 2, False, 1, 0), (4, 6, 3, 4, False, 1, 1),
                                          (4, 6, 3, 4, True, 1, 2), (3, 5, 4, 3, False, 1, 3),
                                          (6, 16, 8, 4, True, 2, 4)]:
        p = I.derive_backward(I.partition_stages(I.build_model(I.ModelConfig(
            layers=L, width=w, microbatch_size=mbs, yield_every=ye, tied_weights=tied))))
        rng = np.random.default_rng(seed)
        params = init_params(p, rng)
        batch = init_batch(p, M, rng)
        g, losses, wn = run_reference(p, params, batch, M, 0.1)
        out.append({"layers": L, "width": w, "mbs": mbs, "M": M, "tied": tied, "yield_every": ye,
                    "seed": seed, "lr": 0.1,
                    "params": {q: v.tolist() for q, v in params.items()},
                    "batch": batch.tolist(),
                    "losses": losses.tolist(),
                    "grads": {q: v.tolist() for q, v in g.items()},
                    "new_params": {q: v.tolist() for q, v in wn.items()}})
    return out


CLI_CONFIGS = [
    {"version": 1, "model": {"layers": 4, "width": 8, "microbatch_size": 4, "yield_every": 2},
     "parallel": {"num_actors": 2, "num_microbatches": 4, "schedule": "gpipe"}},
    {"version": 1, "model": {"layers": 8, "width": 6, "microbatch_size": 2, "yield_every": 2,
                             "tied_weights": True},
     "parallel": {"num_actors": 4, "num_microbatches": 8, "schedule": "1f1b"}},
    {"version": 1, "model": {"layers": 8, "width": 4, "microbatch_size": 2, "yield_every": 1},
     "parallel": {"num_actors": 2, "num_microbatches": 4, "schedule": "interleaved",
                  "circular_repeat": 4, "commute_shared_grads": False}},
]


def cli_plan_docs():
    """sha256 of the three files ``pipecraft plan`` writes (cli.py:194-204)."""
    import contextlib
    import io
    import tempfile

    from pipecraft import cli
    out = []
    for doc in CLI_CONFIGS:
        with tempfile.TemporaryDirectory() as d:
            cfg_doc = dict(doc, output={"dir": d})
            with contextlib.redirect_stdout(io.StringIO()):
                rc = cli.cmd_plan(cli.RunConfig(cfg_doc, pathlib.Path(d)))
            assert rc == 0
            files = {n: sha((pathlib.Path(d) / n).read_text())
                     for n in ("schedule.json", "taskgraph.json", "commplan.json")}
        out.append({"config": doc, "files": files})
    return out


def main():
    plans = {"ffn": [plan_doc(c) for c in ffn_grid()], "gpt_mirror": gpt_docs(),
             "random": random_docs(), "crossing": crossing_doc(),
             "cli_plan": cli_plan_docs()}
    (OUT / "plans.json").write_text(json.dumps(plans, indent=1, sort_keys=True) + "\n")
    p = I.derive_backward(I.partition_stages(I.build_model(I.ModelConfig(
        layers=4, width=8, microbatch_size=4, yield_every=2))))
    _, cp = lower(p, S.gpipe(2, 4))
    (OUT / "commplan_gpipe_2x4.json").write_text(cp.to_json_str() + "\n")
    (OUT / "numerics.json").write_text(json.dumps(numerics_docs()) + "\n")
    shutil.copy(REF / "tests" / "fixtures" / "golden_seed0.json", OUT / "golden_seed0.json")
    print(f"wrote {len(plans['ffn'])} ffn plans, {len(plans['gpt_mirror'])} gpt layouts, "
          f"{len(plans['random'])} random schedules")


if __name__ == "__main__":
    main()
