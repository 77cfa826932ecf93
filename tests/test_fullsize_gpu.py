"""Parity at BASELINE.json's full sizes through a size-independent property.

The float64 oracle cannot run GPT-2 small / medium at full size in test time,
but pipelining must not change the arithmetic: every kernel is deterministic
and every stage runs exactly the shapes of the unpipelined model, so a P-stage
1F1B step (all actors on one GPU, zero-copy local channels) reproduces the
single-stage step bit for bit -- losses, every block parameter's gradient and
new value.  The one exception is the tied embedding w0: its embedding and
LM-head partial gradients are merged in a different order once they live on
different stages (taskgraph.py commuting), so it is
compared at a tight float tolerance instead.
"""
import numpy as np
import pytest
import torch

import bench
from oracle import ffn
from paper_2412_14374_b200.executor import PipelineEngine

pytestmark = pytest.mark.gpu


def _step(cfg_kw, P, M, params_fn, tokens):
    cfg, tg, cp = bench.build_plan(P, cfg_kw, M)
    params = params_fn(cfg)
    eng = PipelineEngine(cp, tg, mode="bf16", gpt=cfg)
    res = eng.step(params, tokens, lr=1e-4, timeout_s=900, to_host=True)
    eng.close()
    return res


@pytest.mark.parametrize("name,cfg_kw,P,M", [
    ("C2 gpt2-small, 4-stage 1F1B", bench.C2, 4, 8),
    ("C3 layout: gpt2-medium width, 8-stage 1F1B",
     dict(bench.C2, layers=24, d_model=1024, n_heads=16, d_ff=4096), 8, 8),
])
def test_pipelined_equals_single_stage_bitwise(name, cfg_kw, P, M):
    dev = torch.device("cuda", 0)
    g = torch.Generator().manual_seed(0)
    tokens = torch.randint(0, cfg_kw["vocab"], (M * cfg_kw["microbatch_size"], cfg_kw["seq_len"]),
                           generator=g, dtype=torch.int32)
    params_fn = lambda cfg: bench.init_params_device(cfg, dev, seed=0)
    one = _step(cfg_kw, 1, M, params_fn, tokens)
    many = _step(cfg_kw, P, M, params_fn, tokens)
    assert np.isfinite(one.losses).all()
    assert np.array_equal(one.losses, many.losses), name
    assert set(one.grads) == set(many.grads) and len(one.grads) > 2
    assert set(one.new_params) == set(one.grads)
    for q in one.grads:
        a, b = one.grads[q], many.grads[q]
        if q == "w0":  # tied: embedding + head partials merged in another order
            assert ffn.rel(a, b) < 1e-6, (name, q)
        else:
            assert np.array_equal(a, b), (name, q, ffn.rel(a, b))
    for q in one.new_params:
        a, b = one.new_params[q], many.new_params[q]
        if q == "w0":
            assert ffn.rel(a, b) < 1e-6, (name, q)
        else:
            assert np.array_equal(a, b), (name, q)


def test_c5_llama_width_pipelined_equals_single_stage_bitwise():
    """BASELINE C5 at full width and sequence (Llama-3-8B block: d 4096, 32 heads,
    8 KV heads, head_dim 128, SwiGLU 14336, vocab 128256, seq 4096), reduced to
    2 blocks so one GPU holds it: a 2-stage 1F1B step with the position ids
    sent 0 -> 1 equals the single-stage step bit for bit (untied head, so every
    parameter is compared exactly)."""
    dev = torch.device("cuda", 0)
    kw = dict(layers=2, d_model=4096, n_heads=32, n_kv_heads=8, d_ff=14336, vocab=128256,
              seq_len=4096, microbatch_size=1)
    M = 2
    g = torch.Generator(device=dev).manual_seed(0)
    tokens = torch.randint(0, kw["vocab"], (M, kw["seq_len"]), generator=g, device=dev,
                           dtype=torch.int32)
    pos = torch.arange(kw["seq_len"], device=dev, dtype=torch.int32).repeat(M, 1)
    out = []
    for P, yields in ((1, None), (2, (2,))):
        from paper_2412_14374_b200 import comms as C, ir as I, schedules as S, taskgraph as T
        cfg = I.LlamaConfig(**kw, yields=yields, yield_every=kw["layers"] + 2)
        p = I.derive_backward(I.partition_stages(I.build_llama(cfg)))
        s = S.one_f_one_b(P, M)
        tg = T.infer_outer_placement(T.commute_grad_accumulation(T.unroll(p, s)), p)
        cp = C.plan_pipeline(tg)
        pg = torch.Generator(device=dev).manual_seed(1)
        params = {q: torch.randn(p.graph.spec_of(q).num_elems, generator=pg, device=dev) * 0.02
                  for q in sorted(p.graph.params)}
        eng = PipelineEngine(cp, tg, mode="bf16", gpt=cfg)
        res = eng.step(params, {"x": tokens, "pos": pos}, lr=1e-4, timeout_s=900, to_host=True)
        eng.close()
        out.append(res)
        del params, eng
        torch.cuda.empty_cache()
    one, two = out
    assert np.isfinite(one.losses).all()
    assert np.array_equal(one.losses, two.losses)
    assert set(one.grads) == set(two.grads)
    for q in one.grads:
        assert np.array_equal(one.grads[q], two.grads[q]), (q, ffn.rel(one.grads[q], two.grads[q]))
