"""Parity at the sizes the bench runs, on the kernels the bench runs.

The small-shape kernel tests (tests/test_gpt_gpu.py) launch fewer work items
than the GPU has SMs, so every persistent CTA does one tile.  These tests run
the BASELINE shapes themselves against float64 references:

* causal attention at C2 geometry (B 8, H 12, S 1024, head_dim 64: 768 forward
  tiles, 768 dQ and 384 dK/dV items over 148 SMs, so the persistent tcgen05
  backward walks several tiles per CTA with next-tile prefetch and ring phases
  carried across tiles) and at C3 geometry (H 16);
* the fused next-token cross-entropy on [8192, 50304] bf16 logits (C2's LM head);
* the deterministic embedding backward at T 8192, V 50304, d 768;
* one training step of a GPT-2-small-width model (d 768, seq 1024, vocab 50304,
  2 layers, 2-stage 1F1B) against the numpy float64 oracle itself.

References: tests/torch_ref.py (float64 torch, pinned to oracle/gpt.py by
tests/test_torch_ref.py) on the device, or oracle/gpt.py directly.  Tolerance:
the reference's max-normalised rel (cli.py:257-259), bf16 2e-2 (north_star).
"""
import ctypes

import numpy as np
import pytest
import torch

import torch_ref as R
from oracle import ffn, gpt
from paper_2412_14374_b200 import _lib

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _heads(t, B, S, H):
    return t.reshape(B, S, H, -1).permute(0, 2, 1, 3)


def _merge(t):
    B, H, S, hd = t.shape
    return t.permute(0, 2, 1, 3).reshape(B * S, H * hd)


def _attention_case(B, H, S, hd, std, seed, Hkv=None):
    """Run pc_attention_gqa_fwd/bwd on seeded bf16 inputs and return the max rel
    error of o, lse, dq, dk, dv against the float64 reference (tests/torch_ref.py),
    computed one (batch, kv-head group) at a time to bound the float64 memory."""
    Hkv = Hkv or H
    G = H // Hkv
    dq_, dkv = H * hd, Hkv * hd
    ld = dq_ + 2 * dkv
    g = torch.Generator(device="cuda").manual_seed(seed)
    qkv = (torch.randn(B * S, ld, device="cuda", generator=g) * std).to(torch.bfloat16)
    do = torch.randn(B * S, dq_, device="cuda", generator=g).to(torch.bfloat16)
    o = torch.empty(B * S, dq_, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * H * S, device="cuda")
    st = _stream()
    _lib.call("pc_attention_gqa_fwd", _lib.PC_BF16, B, H, Hkv, S, hd, qkv.data_ptr(), ld,
              o.data_ptr(), dq_, lse.data_ptr(), st)
    dqkv = torch.empty(B * S, ld, device="cuda", dtype=torch.bfloat16)
    delta = torch.empty(B * H * S, device="cuda")
    _lib.call("pc_attention_gqa_bwd", _lib.PC_BF16, B, H, Hkv, S, hd, qkv.data_ptr(), ld,
              o.data_ptr(), do.data_ptr(), dq_, lse.data_ptr(), delta.data_ptr(),
              dqkv.data_ptr(), ld, st)
    # a second backward must reproduce the first bit for bit (no atomics)
    dqkv2 = torch.empty_like(dqkv)
    _lib.call("pc_attention_gqa_bwd", _lib.PC_BF16, B, H, Hkv, S, hd, qkv.data_ptr(), ld,
              o.data_ptr(), do.data_ptr(), dq_, lse.data_ptr(), delta.data_ptr(),
              dqkv2.data_ptr(), ld, st)
    torch.cuda.synchronize()
    assert torch.equal(dqkv, dqkv2)
    q = _heads(qkv[:, :dq_].double(), B, S, H)
    k = _heads(qkv[:, dq_:dq_ + dkv].double(), B, S, Hkv)
    v = _heads(qkv[:, dq_ + dkv:].double(), B, S, Hkv)
    gd = _heads(do.double(), B, S, H)
    got = {"o": _heads(o.double(), B, S, H), "dq": _heads(dqkv[:, :dq_].double(), B, S, H),
           "dk": _heads(dqkv[:, dq_:dq_ + dkv].double(), B, S, Hkv),
           "dv": _heads(dqkv[:, dq_ + dkv:].double(), B, S, Hkv), "lse": lse.view(B, H, S)}
    want = {key: torch.empty_like(t, dtype=torch.float64) for key, t in got.items()}
    for b in range(B):
        for hk in range(Hkv):
            qs = slice(hk * G, (hk + 1) * G)
            ks = slice(hk, hk + 1)
            ro, rlse = R.attention_fwd(q[b:b + 1, qs], k[b:b + 1, ks], v[b:b + 1, ks])
            rq, rk, rv = R.attention_bwd(gd[b:b + 1, qs], q[b:b + 1, qs], k[b:b + 1, ks],
                                         v[b:b + 1, ks], rlse)
            want["o"][b, qs], want["lse"][b, qs] = ro[0], rlse[0]
            want["dq"][b, qs], want["dk"][b, ks], want["dv"][b, ks] = rq[0], rk[0], rv[0]
    return {key: R.rel(got[key], want[key]) for key in got}


@pytest.mark.parametrize("name,B,H,S,std", [
    ("C2 geometry", 8, 12, 1024, 1.0),
    ("C3 geometry", 8, 16, 1024, 1.0),
    ("C2 geometry, peaked scores", 8, 12, 1024, 3.0),
    ("ragged S, persistent", 5, 12, 1000, 1.0),
])
def test_attention_hd64_bench_shapes(name, B, H, S, std):
    errs = _attention_case(B, H, S, 64, std, seed=B * 1000 + H)
    assert errs["lse"] < 1e-3, (name, errs)
    for key in ("o", "dq", "dk", "dv"):
        assert errs[key] < TOL, (name, key, errs)


@pytest.mark.parametrize("name,B,H,Hkv,S,hd,std", [
    ("hd128 small, one tile", 1, 2, 2, 128, 128, 1.0),
    ("hd128 ragged", 2, 3, 3, 200, 128, 1.0),
    ("C4 geometry (GPT-3 1.3B: 16 heads x 128, seq 2048, mbs 4)", 4, 16, 16, 2048, 128, 1.0),
    ("GQA hd64 small", 2, 4, 2, 256, 64, 1.0),
    ("GQA hd128 ragged, group 4", 1, 8, 2, 520, 128, 2.0),
    ("C5 geometry (Llama-8B: 32 q / 8 kv heads x 128, seq 4096)", 1, 32, 8, 4096, 128, 1.0),
])
def test_attention_hd128_and_gqa(name, B, H, Hkv, S, hd, std):
    """tcgen05 kernels for head_dim 128 and grouped-query heads (native: kv heads
    addressed in the TMA coordinates, the group's dK / dV summed in TMEM)."""
    errs = _attention_case(B, H, S, hd, std, seed=H * 100 + S, Hkv=Hkv)
    assert errs["lse"] < 1e-3, (name, errs)
    for key in ("o", "dq", "dk", "dv"):
        assert errs[key] < TOL, (name, key, errs)


def test_xent_c2_lm_head_shape():
    """pc_xent_fwd_bwd at C2's LM head: 8 sequences x 1024 tokens x vocab 50304, bf16
    logits overwritten with dlogits, fp32 row losses."""
    B, S, V = 8, 1024, 50304
    g = torch.Generator(device="cuda").manual_seed(0)
    logits = (torch.randn(B * S, V, device="cuda", generator=g) * 2.0).to(torch.bfloat16)
    tokens = torch.randint(0, V, (B, S), device="cuda", generator=g, dtype=torch.int32)
    ref_in = logits.double()
    row_loss = torch.empty(B * S, device="cuda")
    _lib.call("pc_xent_fwd_bwd", _lib.PC_BF16, B * S, V, S, logits.data_ptr(), V, tokens.data_ptr(),
              row_loss.data_ptr(), _stream())
    torch.cuda.synchronize()
    rl, dl = R.xent_rows(ref_in, tokens)
    assert R.rel(row_loss, rl) < 1e-5
    assert abs(row_loss.double().sum().item() - rl.sum().item()) < 1e-5 * rl.sum().abs().item()
    assert R.rel(logits, dl) < TOL
    # the no-target rows (last position of each sequence) are exactly zero
    assert torch.count_nonzero(logits.view(B, S, V)[:, -1]).item() == 0
    assert torch.count_nonzero(row_loss.view(B, S)[:, -1]).item() == 0


@pytest.mark.parametrize("accumulate", [0, 1])
def test_embedding_bwd_c2_shape(accumulate):
    T, d, seq, V = 8192, 768, 1024, 50304
    g = torch.Generator(device="cuda").manual_seed(1)
    # a skewed token distribution: long runs of repeated ids stress the segment sums
    tokens = torch.where(torch.rand(T, device="cuda", generator=g) < 0.3,
                         torch.full((T,), 17, device="cuda", dtype=torch.int32),
                         torch.randint(0, V, (T,), device="cuda", generator=g, dtype=torch.int32))
    dh = torch.randn(T, d, device="cuda", generator=g).to(torch.bfloat16)
    nb = ctypes.c_int64()
    _lib.call("pc_embedding_bwd_workspace_bytes", T, ctypes.byref(nb))
    outs = []
    for _ in range(2):
        ws = torch.zeros(nb.value, dtype=torch.uint8, device="cuda")
        dwte = torch.full((V, d), 0.25, device="cuda")
        dwpe = torch.full((seq, d), -0.5, device="cuda")
        _lib.call("pc_embedding_bwd_acc", _lib.PC_BF16, T, d, seq, V, tokens.data_ptr(),
                  dh.data_ptr(), dwte.data_ptr(), dwpe.data_ptr(), accumulate, ws.data_ptr(),
                  nb.value, _stream())
        outs.append((dwte, dwpe))
    torch.cuda.synchronize()
    te, pe = R.embedding_bwd(tokens, dh.double(), V, seq)
    if accumulate:
        te, pe = te + 0.25, pe - 0.5
    assert R.rel(outs[0][0], te) < 1e-5
    assert R.rel(outs[0][1], pe) < 1e-5
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


def test_gpt2_small_width_step_matches_oracle():
    """One 2-stage 1F1B bf16 training step at GPT-2-small width and sequence (d 768,
    12 heads, ffn 3072, vocab 50304, seq 1024, 2 sequences per microbatch, 2 blocks)
    against the float64 numpy oracle: losses, every gradient and every new parameter."""
    from test_gpt_gpu import run_case
    from paper_2412_14374_b200 import ir as I
    cfg = I.GPTConfig(layers=2, d_model=768, n_heads=12, d_ff=3072, vocab=50304, seq_len=1024,
                      microbatch_size=2, yields=(2,), yield_every=4, elem_bytes=2)
    res, g, l, w = run_case(cfg, "1f1b", 2, 2, 1, "bf16", seed=3, std=0.02)
    assert ffn.rel(res.losses, l) < TOL
    for q in g:
        assert ffn.rel(res.grads[q], g[q]) < TOL, (q, ffn.rel(res.grads[q], g[q]))
        assert ffn.rel(res.new_params[q], w[q]) < TOL, q


@pytest.mark.parametrize("name,B,S,V,d", [
    ("C2 LM head (8 x 1024 tokens, vocab 50304, d 768)", 8, 1024, 50304, 768),
    ("ragged vocab tile, short sequences", 3, 40, 1000, 256),
    ("C5 LM head slice (1 x 1024 tokens, vocab 128256, d 4096)", 1, 1024, 128256, 4096),
])
def test_lmhead_xent_fused(name, B, S, V, d):
    """pc_lmhead_xent_fwd (softmax statistics from the logits GEMM's epilogue + one
    streaming pass) and pc_lmhead_xent_bwd against float64: row losses, dlogits
    (overwriting the logits), dh and dW (onto an existing accumulator)."""
    T = B * S
    g = torch.Generator(device="cuda").manual_seed(V + d)
    h = (torch.randn(T, d, device="cuda", generator=g)).to(torch.bfloat16)
    w = (torch.randn(V, d, device="cuda", generator=g) * (2.0 / d ** 0.5)).to(torch.bfloat16)
    tokens = torch.randint(0, V, (B, S), device="cuda", generator=g, dtype=torch.int32)
    lds, nb = ctypes.c_int64(), ctypes.c_int64()
    _lib.call("pc_lmhead_xent_workspace", T, V, d, ctypes.byref(lds), ctypes.byref(nb))
    ws = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
    logits = torch.empty(T, V, device="cuda", dtype=torch.bfloat16)
    rows = torch.empty(T, device="cuda")
    st = _stream()
    _lib.call("pc_lmhead_xent_fwd", T, V, d, S, h.data_ptr(), d, w.data_ptr(), d, tokens.data_ptr(),
              logits.data_ptr(), V, ws.data_ptr(), ws.numel(), rows.data_ptr(), st)
    wt = w.t().contiguous()
    dh = torch.empty(T, d, device="cuda", dtype=torch.bfloat16)
    dw = torch.full((V, d), 0.5, device="cuda")
    _lib.call("pc_lmhead_xent_bwd", T, V, d, logits.data_ptr(), V, h.data_ptr(), d, wt.data_ptr(), V,
              dh.data_ptr(), d, dw.data_ptr(), d, 1, st)
    torch.cuda.synchronize()
    ref_logits = h.double() @ w.double().t()
    rl, dl = R.xent_rows(ref_logits, tokens)
    assert R.rel(rows, rl) < 1e-2, name
    assert abs(rows.double().sum().item() - rl.sum().item()) < 1e-3 * rl.abs().sum().item(), name
    assert R.rel(logits, dl) < TOL, name
    assert torch.count_nonzero(logits.view(B, S, V)[:, -1]).item() == 0
    rdh = dl @ w.double()
    rdw = dl.t() @ h.double() + 0.5
    assert R.rel(dh, rdh) < TOL, name
    assert R.rel(dw, rdw) < TOL, name
