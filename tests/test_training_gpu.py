"""Multi-step training with resident parameters.

``PipelineEngine.load_params`` keeps one copy of every parameter per holding
actor; ``step(None, batch)`` / ``capture(None, batch)`` then update in place
and re-broadcast each tied parameter from the actor that updated it (the
lowest stage, taskgraph.py:349-361) to its other holders.  K resident steps
must equal K calls of the reference loop (executor.py:117-134) fed each
step's new parameters -- which is what a pipecraft user does by hand.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import ffn, gpt  # noqa: E402
from paper_2412_14374_b200 import comms as C  # noqa: E402
from paper_2412_14374_b200 import ir as I  # noqa: E402
from paper_2412_14374_b200 import schedules as S  # noqa: E402
from paper_2412_14374_b200 import taskgraph as T  # noqa: E402
from paper_2412_14374_b200.executor import PipelineEngine, tied_holders  # noqa: E402

pytestmark = pytest.mark.gpu

K = 3


def _plan(p, s):
    tg = T.infer_outer_placement(T.commute_grad_accumulation(T.unroll(p, s)), p)
    return tg, C.plan_pipeline(tg)


@pytest.mark.parametrize("fam,P,M,V", [("1f1b", 4, 4, 1), ("interleaved", 2, 4, 2),
                                       ("gpipe", 1, 2, 1)])
def test_ffn_fp64_resident_steps_match_oracle(fam, P, M, V):
    L = 4
    p = I.derive_backward(I.partition_stages(I.build_model(I.ModelConfig(
        layers=L, width=12, microbatch_size=6, yield_every=1 if P * V == 4 else L,
        tied_weights=True))))
    s = {"gpipe": lambda: S.gpipe(P, M), "1f1b": lambda: S.one_f_one_b(P, M),
         "interleaved": lambda: S.interleaved_1f1b(P, M, V)}[fam]()
    tg, cp = _plan(p, s)
    if P > 1:
        assert tied_holders(tg), "w0 must be held by two actors"
    rng = np.random.default_rng(7)
    params = ffn.init_params({q: p.graph.spec_of(q).dims for q in p.graph.params}, rng)
    batches = [ffn.init_batch(M, 6, 12, rng) for _ in range(K)]
    eng = PipelineEngine(cp, tg, mode="fp64")
    eng.load_params(params)
    ref = dict(params)
    for k in range(K):
        res = eng.step(None, batches[k], lr=0.1)
        g, losses, ref = ffn.run_reference_ffn(ref, batches[k], M, L, True)
        assert ffn.rel(res.losses, losses) < 1e-12, k
        for q in g:
            assert ffn.rel(res.grads[q], g[q]) < 1e-12, (k, q)
    state = eng.state_dict()
    for q in ref:
        assert ffn.rel(state[q], ref[q]) < 1e-12, q
    eng.close()


TINY = dict(layers=4, d_model=64, n_heads=4, d_ff=256, vocab=96, seq_len=32, microbatch_size=2)


def test_gpt_fp32_resident_steps_match_oracle():
    """Tied embedding on stage 0 and the LM head on stage 3: step 2 onward is
    only right if the head actor received the updated w0."""
    cfg = I.GPTConfig(**TINY, yields=(2, 3, 5), yield_every=TINY["layers"] + 2, elem_bytes=4)
    p = I.derive_backward(I.partition_stages(I.build_gpt(cfg)))
    tg, cp = _plan(p, S.one_f_one_b(4, 4))
    (q_tied, low, hs), = tied_holders(tg)
    assert q_tied == "w0" and low == 0 and sorted(hs) == [0, 3]
    oc = dict(layers=4, d=64, heads=4, ff=256, vocab=96, seq=32, mbs=2)
    rng = np.random.default_rng(1)
    params = gpt.init_params(oc, rng, std=0.1)
    toks = [gpt.init_tokens(oc, 4, rng) for _ in range(K)]
    eng = PipelineEngine(cp, tg, mode="fp32", gpt=cfg)
    eng.load_params({q: v.astype(np.float32) for q, v in params.items()})
    ref = dict(params)
    for k in range(K):
        res = eng.step(None, toks[k].reshape(8, 32), lr=0.1)
        _, losses, ref = gpt.run_reference_gpt(ref, toks[k], oc)
        assert ffn.rel(res.losses, losses) < 1e-5, k
    state = eng.state_dict()
    for q in ref:
        assert ffn.rel(state[q], ref[q]) < 1e-5, q
    eng.close()


def test_gpt_bf16_captured_replays_equal_resident_steps():
    """One CUDA-graph replay == one more training step, bit for bit."""
    cfg = I.GPTConfig(**TINY, yield_every=TINY["layers"] + 2, elem_bytes=2)
    p = I.derive_backward(I.partition_stages(I.build_gpt(cfg)))
    tg, cp = _plan(p, S.one_f_one_b(1, 4))
    oc = dict(layers=4, d=64, heads=4, ff=256, vocab=96, seq=32, mbs=2)
    rng = np.random.default_rng(2)
    params = {q: v.astype(np.float32) for q, v in gpt.init_params(oc, rng, std=0.05).items()}
    toks = [gpt.init_tokens(oc, 4, rng).reshape(8, 32) for _ in range(K + 1)]

    a = PipelineEngine(cp, tg, mode="bf16", gpt=cfg)
    a.load_params(params)
    la = [a.step(None, toks[k], lr=0.1).losses for k in range(K + 1)]
    sa = a.state_dict()

    b = PipelineEngine(cp, tg, mode="bf16", gpt=cfg)
    b.load_params(params)
    lb = [b.step(None, toks[0], lr=0.1).losses]            # warm-up = step 1
    cs = b.capture(None, toks[1], lr=0.1)
    for k in range(1, K + 1):
        r = cs.replay(torch.from_numpy(toks[k]))
        lb.append(r.losses.cpu().numpy())
    sb = b.state_dict()
    for k in range(K + 1):
        assert np.array_equal(la[k], lb[k]), k
    assert not np.array_equal(la[0], la[K])               # it did train
    for q in sa:
        assert np.array_equal(sa[q], sb[q]), q
