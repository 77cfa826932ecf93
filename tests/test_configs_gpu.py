"""BASELINE.json configs through the GPU runtime vs the float64 oracle.

C1 runs at its exact size (the reference-runnable case).  C3 / C4 keep their
stage layouts (8-stage 1F1B with the stage0 -> stage7 token skip; 8x2
interleaved chunks) and head_dim (64 / 128) at reduced width so the oracle
finishes in seconds; all actors share one GPU through local channels.
"""
import numpy as np
import pytest

from oracle import ffn, gpt
from paper_2412_14374_b200 import comms as C
from paper_2412_14374_b200 import ir as I
from paper_2412_14374_b200 import schedules as S
from paper_2412_14374_b200 import taskgraph as T
from paper_2412_14374_b200.executor import run_pipelined

pytestmark = pytest.mark.gpu


def _costs(cfg):
    return [float(cfg.tokens * cfg.d_model)] + [cfg.block_fwd_flops()] * cfg.layers + \
        [cfg.head_fwd_flops()]


def run(kw, fam, P, M, V, mode, std=0.05, seed=0):
    base = I.GPTConfig(**kw, yield_every=kw["layers"] + 2)
    S_ = P * V
    yields = I.balanced_yields(_costs(base), S_) if S_ > 1 else None
    cfg = I.GPTConfig(**kw, yields=yields, yield_every=kw["layers"] + 2,
                      elem_bytes=2 if mode == "bf16" else 4)
    p = I.derive_backward(I.partition_stages(I.build_gpt(cfg)))
    s = {"gpipe": lambda: S.gpipe(P, M), "1f1b": lambda: S.one_f_one_b(P, M),
         "interleaved": lambda: S.interleaved_1f1b(P, M, V)}[fam]()
    tg = T.infer_outer_placement(T.commute_grad_accumulation(T.unroll(p, s)), p)
    cp = C.plan_pipeline(tg)
    oc = dict(layers=cfg.layers, d=cfg.d_model, heads=cfg.n_heads, ff=cfg.d_ff, vocab=cfg.vocab,
              seq=cfg.seq_len, mbs=cfg.microbatch_size)
    rng = np.random.default_rng(seed)
    params = gpt.init_params(oc, rng, std=std)
    tokens = gpt.init_tokens(oc, M, rng)
    g, l, w = gpt.run_reference_gpt(params, tokens, oc)
    res = run_pipelined(cp, tg, {q: v.astype(np.float32) for q, v in params.items()},
                        tokens.reshape(M * cfg.microbatch_size, cfg.seq_len), mode=mode, gpt=cfg)
    err = max([ffn.rel(res.losses, l)] + [ffn.rel(res.grads[q], g[q]) for q in g]
              + [ffn.rel(res.new_params[q], w[q]) for q in w])
    return err, cp, res


C1 = dict(layers=4, d_model=128, n_heads=4, d_ff=512, vocab=512, seq_len=64, microbatch_size=4)


def test_c1_exact_fp32():
    err, cp, res = run(C1, "gpipe", 2, 4, 1, "fp32", std=0.1)
    assert err < 1e-5
    assert res.stats.driver_messages == 4


def test_c1_bf16():
    err, _, _ = run(C1, "gpipe", 2, 4, 1, "bf16")
    assert err < 2e-2


def test_c3_layout_8_stage_1f1b():
    kw = dict(layers=24, d_model=128, n_heads=2, d_ff=256, vocab=128, seq_len=64,
              microbatch_size=2)
    err, cp, res = run(kw, "1f1b", 8, 16, 1, "bf16")
    assert err < 2e-2
    assert (0, 7) in cp.channels and (7, 0) in cp.channels  # token skip + tied grad
    assert res.stats.channel_counts == {k: len(v) for k, v in cp.channels.items()}


def test_c4_layout_interleaved_hd128():
    kw = dict(layers=8, d_model=256, n_heads=2, d_ff=512, vocab=128, seq_len=128,
              microbatch_size=2)
    err, cp, res = run(kw, "interleaved", 4, 8, 2, "bf16")
    assert err < 2e-2
