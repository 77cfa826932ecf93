"""Pin the CPU oracle before trusting it.

FFN half: bit-exact against the reference's own golden fixture
(pkg/tests/fixtures/golden_seed0.json, checked with rel == 0 exactly as
pkg/tests/test_executor.py:63-75) and against run_reference outputs generated
from the reference (tests/golden/numerics.json).

GPT half (no reference counterpart): central finite differences like
pkg/tests/test_ir.py:32-49, plus torch float64 autograd on identical inputs.
"""
import json
import math
import pathlib

import numpy as np
import pytest

from oracle import ffn, gpt

GOLD = pathlib.Path(__file__).parent / "golden"


def ffn_param_dims(layers, width, tied):
    return {f"w{k}": (width, width) for k in range(layers - (1 if tied else 0))}


def test_golden_seed0_bit_exact():
    doc = json.loads((GOLD / "golden_seed0.json").read_text())
    rng = np.random.default_rng(doc["seed"])
    params = ffn.init_params(ffn_param_dims(doc["layers"], doc["width"], False), rng)
    batch = ffn.init_batch(doc["M"], doc["microbatch_size"], doc["width"], rng)
    grads, losses, new = ffn.run_reference_ffn(params, batch, doc["M"], doc["layers"], False,
                                               doc["lr"])
    assert losses.tolist() == doc["losses"]
    for q, want in doc["grads"].items():
        assert ffn.rel(grads[q], want) == 0.0
    for q, want in doc["new_params"].items():
        assert ffn.rel(new[q], want) == 0.0


@pytest.mark.parametrize("k", range(5))
def test_reference_numerics_bit_exact(k):
    doc = json.loads((GOLD / "numerics.json").read_text())[k]
    params = {q: np.array(v) for q, v in doc["params"].items()}
    batch = np.array(doc["batch"])
    grads, losses, new = ffn.run_reference_ffn(params, batch, doc["M"], doc["layers"],
                                               doc["tied"], doc["lr"])
    assert ffn.rel(losses, doc["losses"]) == 0.0
    for q in params:
        assert ffn.rel(grads[q], doc["grads"][q]) == 0.0
        assert ffn.rel(new[q], doc["new_params"][q]) == 0.0


def test_eval_op_vocabulary():
    a = np.arange(6.0).reshape(2, 3) - 2
    assert np.array_equal(ffn.eval_op("relu", [a]), np.maximum(a, 0))
    assert np.array_equal(ffn.eval_op("relu-grad", [np.ones_like(a), a]), (a > 0) * 1.0)
    assert ffn.eval_op("sub-sample-loss", [a]) == 0.5 * np.sum(a * a)
    assert ffn.eval_op("sum-to", [np.ones((4, 2, 3))], result_dims=(1, 3)).tolist() == [[8.0] * 3]
    assert ffn.eval_op("slice", [a], {"offset": 1, "length": 1}).tolist() == [a[1].tolist()]
    assert ffn.eval_op("broadcast", [np.ones(3)], result_dims=(2, 3)).shape == (2, 3)


TINY = dict(layers=2, d=8, heads=2, ff=16, vocab=11, seq=5, mbs=2)


def _loss(params, tokens):
    return gpt.gpt_step(params, tokens, TINY)[0]


def test_gpt_oracle_finite_differences():
    rng = np.random.default_rng(0)
    params = gpt.init_params(TINY, rng, std=0.3)
    tokens = gpt.init_tokens(TINY, 1, rng)[0]
    _, grads = gpt.gpt_step(params, tokens, TINY)
    eps = 1e-6
    for q, flat in params.items():
        idx = rng.choice(flat.size, size=min(25, flat.size), replace=False)
        for j in idx:
            saved = flat[j]
            flat[j] = saved + eps
            up = _loss(params, tokens)
            flat[j] = saved - eps
            dn = _loss(params, tokens)
            flat[j] = saved
            fd = (up - dn) / (2 * eps)
            assert abs(fd - grads[q][j]) <= 1e-6 * max(1.0, abs(fd)), (q, j, fd, grads[q][j])


def test_gpt_oracle_matches_torch_autograd():
    torch = pytest.importorskip("torch")
    F = torch.nn.functional
    cfg = dict(layers=2, d=16, heads=4, ff=32, vocab=23, seq=7, mbs=3)
    rng = np.random.default_rng(1)
    params = gpt.init_params(cfg, rng, std=0.2)
    tokens = gpt.init_tokens(cfg, 1, rng)[0]
    loss, grads = gpt.gpt_step(params, tokens, cfg)

    tp = {q: torch.tensor(v, dtype=torch.float64, requires_grad=True) for q, v in params.items()}
    B, S, d, H = cfg["mbs"], cfg["seq"], cfg["d"], cfg["heads"]

    def view(flat, layout):
        return {k: flat[o:o + math.prod(dims)].reshape(dims) for k, (o, dims) in layout.items()}

    E = view(tp["w0"], gpt.embed_layout(cfg)[0])
    tok = torch.tensor(tokens, dtype=torch.long)
    h = E["wte"][tok.reshape(-1)] + E["wpe"][torch.arange(S).repeat(B)]
    for k in range(1, cfg["layers"] + 1):
        final = k == cfg["layers"]
        P = view(tp[f"w{k}"], gpt.block_layout(cfg, final)[0])
        a = F.layer_norm(h, (d,), P["ln1_g"], P["ln1_b"], eps=gpt.LN_EPS)
        qkv = a @ P["w_qkv"].T + P["b_qkv"]
        q, kk, v = (qkv[:, i * d:(i + 1) * d].reshape(B, S, H, -1).transpose(1, 2) for i in range(3))
        o = F.scaled_dot_product_attention(q, kk, v, is_causal=True)
        o = o.transpose(1, 2).reshape(B * S, d)
        h = h + o @ P["w_o"].T + P["b_o"]
        a2 = F.layer_norm(h, (d,), P["ln2_g"], P["ln2_b"], eps=gpt.LN_EPS)
        h = h + F.gelu(a2 @ P["w_fc1"].T + P["b_fc1"], approximate="tanh") @ P["w_fc2"].T + P["b_fc2"]
        if final:
            h = F.layer_norm(h, (d,), P["lnf_g"], P["lnf_b"], eps=gpt.LN_EPS)
    logits = (h @ E["wte"].T).reshape(B, S, -1)
    tl = F.cross_entropy(logits[:, :-1].reshape(-1, logits.shape[-1]), tok[:, 1:].reshape(-1),
                         reduction="sum")
    tl.backward()
    assert abs(tl.item() - loss) < 1e-10 * abs(loss)
    for q in params:
        assert ffn.rel(tp[q].grad.numpy(), grads[q]) < 1e-10


def test_gpt_accumulation_linear_in_microbatches():
    """Summed loss => accumulating M microbatches equals one big batch."""
    cfg1 = dict(TINY, mbs=4)
    cfg2 = dict(TINY, mbs=2)
    rng = np.random.default_rng(2)
    params = gpt.init_params(cfg1, rng, std=0.3)
    tokens = gpt.init_tokens(cfg1, 1, rng)
    g1, l1, _ = gpt.run_reference_gpt(params, tokens, cfg1)
    g2, l2, _ = gpt.run_reference_gpt(params, tokens.reshape(2, 2, -1), cfg2)
    assert abs(l1.sum() - l2.sum()) < 1e-10 * abs(l1.sum())
    for q in params:
        assert ffn.rel(g1[q], g2[q]) < 1e-12


# ---------------------------------------------------------------------------
# Llama-style oracle (BASELINE C5: RMSNorm, RoPE, GQA, SwiGLU, untied head)

from oracle import llama  # noqa: E402

LTINY = dict(layers=2, d=16, heads=4, kv_heads=2, ff=24, vocab=13, seq=6, mbs=2, theta=10000.0)


def _lpos(cfg, rng):
    # non-trivial position ids (e.g. packed documents) exercise RoPE fully
    return rng.integers(0, 50, size=(cfg["mbs"], cfg["seq"])).astype(np.int32)


def test_llama_oracle_finite_differences():
    rng = np.random.default_rng(3)
    params = llama.init_params(LTINY, rng, std=0.3)
    tokens = llama.init_tokens(LTINY, 1, rng)[0]
    pos = _lpos(LTINY, rng)
    _, grads = llama.llama_step(params, tokens, pos, LTINY)
    eps = 1e-6
    for q, flat in params.items():
        idx = rng.choice(flat.size, size=min(25, flat.size), replace=False)
        for j in idx:
            saved = flat[j]
            flat[j] = saved + eps
            up = llama.llama_step(params, tokens, pos, LTINY)[0]
            flat[j] = saved - eps
            dn = llama.llama_step(params, tokens, pos, LTINY)[0]
            flat[j] = saved
            fd = (up - dn) / (2 * eps)
            assert abs(fd - grads[q][j]) <= 1e-6 * max(1.0, abs(fd)), (q, j, fd, grads[q][j])


def test_llama_oracle_matches_torch_autograd():
    torch = pytest.importorskip("torch")
    F = torch.nn.functional
    cfg = dict(layers=2, d=32, heads=4, kv_heads=2, ff=40, vocab=29, seq=9, mbs=3, theta=500.0)
    rng = np.random.default_rng(4)
    params = llama.init_params(cfg, rng, std=0.2)
    tokens = llama.init_tokens(cfg, 1, rng)[0]
    pos = _lpos(cfg, rng)
    loss, grads = llama.llama_step(params, tokens, pos, cfg)

    tp = {q: torch.tensor(v, dtype=torch.float64, requires_grad=True) for q, v in params.items()}
    B, S, d, H, Hkv, f = cfg["mbs"], cfg["seq"], cfg["d"], cfg["heads"], cfg["kv_heads"], cfg["ff"]
    hd = d // H

    def view(flat, layout):
        return {k: flat[o:o + math.prod(dims)].reshape(dims) for k, (o, dims) in layout.items()}

    def rms(x, g):
        return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + llama.RMS_EPS) * g

    ang = torch.tensor(pos.reshape(-1), dtype=torch.float64)[:, None] * \
        cfg["theta"] ** (-torch.arange(0, hd // 2, dtype=torch.float64) * 2.0 / hd)
    cos, sin = torch.cos(ang)[:, None, :], torch.sin(ang)[:, None, :]

    def rope(t):  # [T, nh, hd], rotate-half
        t1, t2 = t[..., :hd // 2], t[..., hd // 2:]
        return torch.cat([t1 * cos - t2 * sin, t2 * cos + t1 * sin], -1)

    tok = torch.tensor(tokens, dtype=torch.long)
    h = view(tp["w0"], llama.embed_layout(cfg)[0])["wte"][tok.reshape(-1)]
    for k in range(1, cfg["layers"] + 1):
        final = k == cfg["layers"]
        P = view(tp[f"w{k}"], llama.block_layout(cfg, final)[0])
        qkv = rms(h, P["rms1_g"]) @ P["w_qkv"].T
        q = rope(qkv[:, :H * hd].reshape(-1, H, hd))
        kk = rope(qkv[:, H * hd:(H + Hkv) * hd].reshape(-1, Hkv, hd))
        v = qkv[:, (H + Hkv) * hd:].reshape(-1, Hkv, hd)
        q4 = q.reshape(B, S, H, hd).transpose(1, 2)
        k4 = kk.reshape(B, S, Hkv, hd).transpose(1, 2).repeat_interleave(H // Hkv, dim=1)
        v4 = v.reshape(B, S, Hkv, hd).transpose(1, 2).repeat_interleave(H // Hkv, dim=1)
        o = F.scaled_dot_product_attention(q4, k4, v4, is_causal=True)
        h = h + o.transpose(1, 2).reshape(B * S, H * hd) @ P["w_o"].T
        gu = rms(h, P["rms2_g"]) @ P["w_gu"].T
        h = h + (F.silu(gu[:, :f]) * gu[:, f:]) @ P["w_down"].T
        if final:
            h = rms(h, P["rmsf_g"])
    logits = (h @ view(tp["wout"], llama.head_layout(cfg)[0])["w_head"].T).reshape(B, S, -1)
    tl = F.cross_entropy(logits[:, :-1].reshape(-1, logits.shape[-1]), tok[:, 1:].reshape(-1),
                         reduction="sum")
    tl.backward()
    assert abs(tl.item() - loss) < 1e-10 * abs(loss)
    for q in params:
        assert ffn.rel(tp[q].grad.numpy(), grads[q]) < 1e-10, q
