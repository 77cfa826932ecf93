"""Differentiable non-adjacent skip connections.

The reference planner rejects a gradient merge of an activation used on two
stages (pkg/src/pipecraft/ir.py:568-571, taskgraph.py:244-246).  Here the merge
is an ordinary op of the producer-side backward: the activation travels
forward to the non-adjacent stage, its gradient comes back, and the plan
stays deadlock-free.  There is no reference executor for this, so the numpy
oracle (oracle/ffn.py ffn_step_skips) is pinned to torch float64 autograd.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import ffn  # noqa: E402
from paper_2412_14374_b200 import comms as C  # noqa: E402
from paper_2412_14374_b200 import ir as I  # noqa: E402
from paper_2412_14374_b200 import schedules as S  # noqa: E402
from paper_2412_14374_b200 import taskgraph as T  # noqa: E402

SKIPS = ((0, 3), (1, 5), (2, 4))


def _autograd(params, x, layers, tied, skips):
    P = {q: torch.tensor(v, dtype=torch.float64, requires_grad=True) for q, v in params.items()}
    h = torch.tensor(x, dtype=torch.float64)
    acts = {}
    for k in range(layers):
        for src, dst in skips:
            if dst == k:
                h = h + acts[src]
        w = P["w0"] if (tied and k == layers - 1) else P[f"w{k}"]
        z = h @ w
        if k < layers - 1:
            h = torch.relu(z)
            acts[k] = h
        else:
            h = z
    loss = 0.5 * (h * h).sum()
    loss.backward()
    return loss.item(), {q: t.grad.numpy() for q, t in P.items()}


@pytest.mark.parametrize("tied", [False, True])
def test_oracle_with_skips_matches_autograd(tied):
    L, w, mbs = 6, 8, 5
    rng = np.random.default_rng(1)
    names = {f"w{k}": (w, w) for k in range(L - (1 if tied else 0))}
    params = ffn.init_params(names, rng)
    x = rng.standard_normal((mbs, w))
    loss, grads = ffn.ffn_step_skips(params, x, L, tied, SKIPS)
    l2, g2 = _autograd(params, x, L, tied, SKIPS)
    assert abs(loss - l2) <= 1e-12 * abs(l2)
    for q in g2:
        assert ffn.rel(grads[q], g2[q]) < 1e-12, q


def plan(fam, P, M, V=1, yields=(2, 3, 5), tied=False, skips=SKIPS):
    cfg = I.ModelConfig(layers=6, width=8, microbatch_size=4, yields=yields, tied_weights=tied,
                        skips=skips)
    p = I.derive_backward(I.partition_stages(I.build_model(cfg)))
    s = {"gpipe": lambda: S.gpipe(P, M), "1f1b": lambda: S.one_f_one_b(P, M),
         "interleaved": lambda: S.interleaved_1f1b(P, M, V)}[fam]()
    tg = T.infer_outer_placement(T.commute_grad_accumulation(T.unroll(p, s)), p)
    cp = C.infer_comms(tg, s)
    rep = C.check_deadlock_free(cp)
    assert rep.ok, str(rep)
    return p, tg, C.fuse(C.insert_deletions(cp, tg), tg)


@pytest.mark.parametrize("fam,P,M,V,yields", [("gpipe", 4, 4, 1, (2, 3, 5)),
                                              ("1f1b", 4, 8, 1, (2, 3, 5)),
                                              ("interleaved", 2, 4, 2, (2, 3, 5))])
def test_planner_accepts_skips_and_sends_gradients_back(fam, P, M, V, yields):
    p, tg, cp = plan(fam, P, M, V, yields)
    stage_of_block = lambda k: sum(1 for y in yields if y <= k)
    # every skip crossing a stage boundary: forward activation channel and a
    # gradient coming back to the producer's stage
    for src, dst in SKIPS:
        s0, s1 = stage_of_block(src), stage_of_block(dst)
        if s0 == s1:
            continue
        a0, a1 = s0 % P, s1 % P
        if a0 == a1:
            continue
        fwd = [b for b in cp.channels.get((a0, a1), []) if b.startswith(f"act:a{src}:")]
        assert len(fwd) == M, (src, dst, cp.channels.get((a0, a1)))
        assert any(b.startswith("gbuf:") for b in cp.channels.get((a1, a0), []))
    # the merge is a backward op of the producer's home stage, not a task-graph merge
    assert all(m.value in p.graph.params for m in p.cross_merges)


def test_skip_validation():
    with pytest.raises(I.GraphError):
        I.ModelConfig(layers=4, width=4, microbatch_size=2, skips=((3, 2),))
    with pytest.raises(I.GraphError):
        I.ModelConfig(layers=4, width=4, microbatch_size=2, skips=((3, 3),))
