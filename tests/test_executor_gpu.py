"""The reference's executor tests (pkg/tests/test_executor.py) re-run against the
B200 runtime, with the numpy oracle (oracle/ffn.py) as the serial reference.

fp64 mode must match to 1e-12 exactly like the reference's own gate
(test_executor.py:83-93, cli.py:59-60); fp32 mode to 1e-5 (north_star).
"""
import json
import pathlib

import numpy as np
import pytest

from oracle import ffn
from paper_2412_14374_b200 import comms as C
from paper_2412_14374_b200 import ir as I
from paper_2412_14374_b200 import schedules as S
from paper_2412_14374_b200 import taskgraph as T
from paper_2412_14374_b200.executor import (
    ExecutorFault,
    LivenessFault,
    instrument,
    run_pipelined,
)

pytestmark = pytest.mark.gpu
GOLD = pathlib.Path(__file__).parent / "golden"


def build(fam, P, M, V=1, layers=None, width=6, mbs=3, tied=False, commute=True, seed=0,
          dtype=np.float64):
    L = layers or max(P * V, 2 if not tied else 4)
    p = I.derive_backward(I.partition_stages(I.build_model(I.ModelConfig(
        layers=L, width=width, microbatch_size=mbs, yield_every=max(1, L // (P * V)),
        tied_weights=tied))))
    s = {"gpipe": lambda: S.gpipe(P, M), "1f1b": lambda: S.one_f_one_b(P, M),
         "interleaved": lambda: S.interleaved_1f1b(P, M, V)}[fam]()
    tg = T.unroll(p, s)
    if commute:
        tg = T.commute_grad_accumulation(tg)
    tg = T.infer_outer_placement(tg, p)
    cp = C.infer_comms(tg, s)
    assert C.check_deadlock_free(cp).ok
    cp = C.fuse(C.insert_deletions(cp, tg), tg)
    rng = np.random.default_rng(seed)
    dims = {q: p.graph.spec_of(q).dims for q in p.graph.params}
    params = {q: v.astype(dtype) for q, v in ffn.init_params(dims, rng).items()}
    batch = ffn.init_batch(M, mbs, width, rng).astype(dtype)
    return L, tied, tg, cp, params, batch


def reference(L, tied, params, batch, M):
    p64 = {q: v.astype(np.float64) for q, v in params.items()}
    return ffn.run_reference_ffn(p64, batch.astype(np.float64), M, L, tied)


@pytest.mark.parametrize("fam,P,M,V", [("gpipe", 2, 2, 1), ("1f1b", 2, 2, 1), ("1f1b", 4, 8, 1),
                                       ("interleaved", 2, 4, 2), ("gpipe", 1, 3, 1)])
def test_matches_reference_fp64(fam, P, M, V):
    L, tied, tg, cp, params, batch = build(fam, P, M, V)
    g, l, w = reference(L, tied, params, batch, M)
    res = run_pipelined(cp, tg, params, batch)
    assert max(ffn.rel(res.grads[q], g[q]) for q in g) < 1e-12
    assert ffn.rel(res.losses, l) < 1e-12
    assert max(ffn.rel(res.new_params[q], w[q]) for q in w) < 1e-12


@pytest.mark.parametrize("fam,P,M,V", [("gpipe", 2, 4, 1), ("1f1b", 4, 8, 1),
                                       ("interleaved", 2, 4, 2)])
def test_matches_reference_fp32(fam, P, M, V):
    L, tied, tg, cp, params, batch = build(fam, P, M, V, width=32, mbs=16, dtype=np.float32)
    g, l, w = reference(L, tied, params, batch, M)
    res = run_pipelined(cp, tg, params, batch)
    assert max(ffn.rel(res.grads[q], g[q]) for q in g) < 1e-5
    assert ffn.rel(res.losses, l) < 1e-5
    assert max(ffn.rel(res.new_params[q], w[q]) for q in w) < 1e-5


def test_golden_seed0_through_gpu_runtime():
    doc = json.loads((GOLD / "golden_seed0.json").read_text())
    P = 2
    p = I.derive_backward(I.partition_stages(I.build_model(I.ModelConfig(
        layers=doc["layers"], width=doc["width"], microbatch_size=doc["microbatch_size"],
        yield_every=doc["layers"] // P))))
    s = S.one_f_one_b(P, doc["M"])
    tg = T.infer_outer_placement(T.unroll(p, s), p)
    cp = C.fuse(C.insert_deletions(C.infer_comms(tg, s), tg), tg)
    rng = np.random.default_rng(doc["seed"])
    params = ffn.init_params({q: p.graph.spec_of(q).dims for q in p.graph.params}, rng)
    batch = ffn.init_batch(doc["M"], doc["microbatch_size"], doc["width"], rng)
    res = run_pipelined(cp, tg, params, batch, lr=doc["lr"])
    assert ffn.rel(res.losses, doc["losses"]) < 1e-12
    for q in doc["grads"]:
        assert ffn.rel(res.grads[q], doc["grads"][q]) < 1e-12
        assert ffn.rel(res.new_params[q], doc["new_params"][q]) < 1e-12


@pytest.mark.parametrize("commute", [True, False])
def test_tied_weights_and_commuting(commute):
    L, tied, tg, cp, params, batch = build("1f1b", 4, 4, tied=True, commute=commute)
    g, l, w = reference(L, tied, params, batch, 4)
    res = run_pipelined(cp, tg, params, batch)
    assert max(ffn.rel(res.grads[q], g[q]) for q in g) < 1e-12
    assert res.stats.messages_for_param(tg, "w0") == (1 if commute else 4)


def test_deterministic_under_injected_delays():
    L, tied, tg, cp, params, batch = build("1f1b", 2, 4)
    base = run_pipelined(cp, tg, params, batch)
    for seed in (1, 2):
        rng = np.random.default_rng(seed)
        delays = {(a, i): float(rng.uniform(0, 2e-4))
                  for a in range(2) for i in range(len(cp.programs[a].instrs))}
        res = run_pipelined(cp, tg, params, batch, delay_fn=lambda a, i: delays[(a, i)])
        for q in base.grads:
            assert ffn.rel(res.grads[q], base.grads[q]) == 0.0
        assert ffn.rel(res.losses, base.losses) == 0.0


def test_watchdog_reports_blocked_instruction():
    L, tied, tg, cp, params, batch = build("1f1b", 2, 2)
    prog = cp.programs[1]
    idx = next(i for i, ins in enumerate(prog.instrs) if isinstance(ins, C.RecvWait))
    prog.instrs.pop(idx)
    with pytest.raises((LivenessFault, ExecutorFault)) as err:
        run_pipelined(cp, tg, params, batch, timeout_s=1.0)
    assert "actor" in str(err.value)


def test_dropped_send_hangs_and_watchdog_fires():
    L, tied, tg, cp, params, batch = build("1f1b", 2, 2)
    prog = cp.programs[0]
    idx = max(i for i, ins in enumerate(prog.instrs) if isinstance(ins, C.SendStart))
    prog.instrs.pop(idx)
    with pytest.raises(LivenessFault, match="watchdog|timed out"):
        run_pipelined(cp, tg, params, batch, timeout_s=1.0)


def test_missing_buffer_fault_names_buffer():
    L, tied, tg, cp, params, batch = build("gpipe", 2, 2)
    prog = cp.programs[0]
    at = prog.instrs.index(C.RunTask("f:s0:mb0")) + 1
    prog.instrs.insert(at, C.Delete("input:x:mb1"))
    with pytest.raises((LivenessFault, ExecutorFault)) as err:
        run_pipelined(cp, tg, params, batch, timeout_s=2.0)
    assert "input:x:mb1" in str(err.value) or "leaked" in str(err.value)


def test_store_clean_at_step_end():
    L, tied, tg, cp, params, batch = build("interleaved", 2, 4, V=2)
    res = run_pipelined(cp, tg, params, batch)
    for a, live in res.stats.final_live.items():
        for bid in live:
            b = tg.buffers[bid]
            assert b.kind in ("param", "optimizer-state") or b.is_output, bid


def test_driver_messages_are_two_per_actor():
    for P in (1, 2, 4):
        L, tied, tg, cp, params, batch = build("1f1b", P, max(P, 2))
        res = run_pipelined(cp, tg, params, batch)
        assert instrument(res).driver_messages == 2 * P


def test_stash_peaks_match_memory_claim():
    peaks = {}
    for fam in ("gpipe", "1f1b"):
        L, tied, tg, cp, params, batch = build(fam, 4, 8)
        res = run_pipelined(cp, tg, params, batch)
        peaks[fam] = res.stats.peak_stash[(0, 0)]
    assert peaks == {"gpipe": 8, "1f1b": 4}


def test_channel_counts_match_plan():
    L, tied, tg, cp, params, batch = build("1f1b", 2, 4)
    res = run_pipelined(cp, tg, params, batch)
    assert res.stats.channel_counts == {k: len(v) for k, v in cp.channels.items()}


def test_timeline_bubble_measured():
    L, tied, tg, cp, params, batch = build("gpipe", 2, 4, width=64, mbs=64)
    res = run_pipelined(cp, tg, params, batch, timeline=True)
    tl = res.stats.timeline
    assert len([e for e in tl if e[1] in ("fwd", "bwd")]) == 2 * 2 * 4
    assert all(e[4] >= e[3] for e in tl)
    b = res.stats.bubble_fraction(2)
    assert 0.0 <= b < 1.0


@pytest.mark.parametrize("fam,P,M,V,tied", [("gpipe", 2, 4, 1, False), ("1f1b", 4, 8, 1, False),
                                            ("interleaved", 2, 4, 2, False),
                                            ("1f1b", 2, 4, 1, True)])
def test_full_remat_matches_reference_fp64(fam, P, M, V, tied):
    """FFN model under remat="full-per-stage" (forward replayed in each
    backward task): still the reference's run_reference to 1e-12, and bitwise
    equal to the stashing run, including interleaved chunks and tied weights."""
    L, tied, tg, cp, params, batch = build(fam, P, M, V, tied=tied)
    g, l, w = reference(L, tied, params, batch, M)
    a = run_pipelined(cp, tg, params, batch)
    b = run_pipelined(cp, tg, params, batch, remat="full-per-stage")
    assert max(ffn.rel(b.grads[q], g[q]) for q in g) < 1e-12
    assert ffn.rel(b.losses, l) < 1e-12
    assert max(ffn.rel(b.new_params[q], w[q]) for q in w) < 1e-12
    assert np.array_equal(a.losses, b.losses)
    for q in a.grads:
        assert np.array_equal(a.grads[q], b.grads[q]), q


@pytest.mark.parametrize("fam,P,M,V,tied", [("gpipe", 4, 4, 1, False), ("1f1b", 4, 8, 1, False),
                                            ("1f1b", 4, 8, 1, True), ("interleaved", 2, 4, 2, False)])
@pytest.mark.parametrize("remat", ["none", "full-per-stage"])
def test_differentiable_skips_match_oracle_fp64(fam, P, M, V, tied, remat):
    """activations joined to non-adjacent later blocks
    (ir.ModelConfig.skips) -- the activation is sent forward past a stage, its
    gradient comes back to the producer's stage and is summed there.  fp64
    results equal the oracle (pinned to torch autograd) to the reference's
    1e-12 gate, under stashing and full remat."""
    from test_skips_cpu import SKIPS, plan
    p, tg, cp = plan(fam, P, M, V, tied=tied)
    rng = np.random.default_rng(3)
    dims = {q: p.graph.spec_of(q).dims for q in p.graph.params}
    params = ffn.init_params(dims, rng)
    batch = ffn.init_batch(M, 4, 8, rng)
    g, l, w = ffn.run_reference_ffn(params, batch, M, 6, tied, skips=SKIPS)
    res = run_pipelined(cp, tg, params, batch, remat=remat)
    assert ffn.rel(res.losses, l) < 1e-12
    for q in g:
        assert ffn.rel(res.grads[q], g[q]) < 1e-12, q
        assert ffn.rel(res.new_params[q], w[q]) < 1e-12, q
