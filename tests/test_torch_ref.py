"""Pin the float64 torch restatements (tests/torch_ref.py) to the numpy oracle
(oracle/gpt.py, oracle/llama.py) on small inputs, on the CPU, rel < 1e-12.  The
full-size GPU tests (tests/test_fullsize_kernels_gpu.py) use these restatements
as their reference, so this is the link from them back to the oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import torch_ref as R  # noqa: E402
from oracle import gpt, llama  # noqa: E402


def _t(x):
    return torch.tensor(x, dtype=torch.float64)


@pytest.mark.parametrize("H,Hkv,S", [(3, 3, 40), (4, 2, 33), (8, 1, 16)])
def test_attention_matches_oracle(H, Hkv, S):
    B, hd = 2, 16
    rng = np.random.default_rng(H * 10 + Hkv)
    q = rng.standard_normal((B, H, S, hd))
    k = rng.standard_normal((B, Hkv, S, hd))
    v = rng.standard_normal((B, Hkv, S, hd))
    do = rng.standard_normal((B, H, S, hd))
    if H == Hkv:
        o, p = gpt.attention(q, k, v)
        dq, dk, dv = gpt.attention_bwd(do, q, k, v, p)
    else:
        o, p = llama.gqa_attention(q, k, v)
        dq, dk, dv = llama.gqa_attention_bwd(do, q, k, v, p)
    to, lse = R.attention_fwd(_t(q), _t(k), _t(v))
    tq, tk, tv = R.attention_bwd(_t(do), _t(q), _t(k), _t(v), lse)
    for a, b in ((to, o), (tq, dq), (tk, dk), (tv, dv)):
        assert R.rel(a, _t(b)) < 1e-12


def test_xent_matches_oracle_head_loss():
    B, S, V, d = 3, 7, 29, 5
    rng = np.random.default_rng(1)
    h = rng.standard_normal((B * S, V))
    tokens = rng.integers(0, V, (B, S))
    loss, dh, _ = gpt.head_loss(h, np.eye(V), tokens)  # identity head: logits = h
    rl, dl = R.xent_rows(_t(h), torch.tensor(tokens))
    assert abs(rl.sum().item() - loss) < 1e-12 * abs(loss)
    assert R.rel(dl, _t(dh)) < 1e-12


def test_embedding_bwd_matches_add_at():
    T, d, V, seq = 48, 6, 11, 8
    rng = np.random.default_rng(2)
    tokens = rng.integers(0, V, T)
    dh = rng.standard_normal((T, d))
    want_te = np.zeros((V, d))
    np.add.at(want_te, tokens, dh)
    want_pe = np.zeros((seq, d))
    np.add.at(want_pe, np.arange(T) % seq, dh)
    te, pe = R.embedding_bwd(torch.tensor(tokens), _t(dh), V, seq)
    assert R.rel(te, _t(want_te)) < 1e-12
    assert R.rel(pe, _t(want_pe)) < 1e-12
