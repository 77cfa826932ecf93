"""The tcgen05 attention kernels' alternative schedules (pc_attention_tune, the
A/B hooks behind tools/attn_ab.py) against the defaults the product runs.

One or two MMA-issuing warps only reorder when MMAs are issued, never what
they compute, so those pairs must agree bitwise; the head_dim-64 forward's
FMA-pipe exp2 share (EMU) changes P within bf16 rounding.  Persistent shapes
(more tiles than CTAs) and a ragged sequence length are included.
"""
import pytest
import torch

from paper_2412_14374_b200 import _lib

pytestmark = pytest.mark.gpu

# pc_attention_tune keys: 0 head_dim-64 forward design, 1 its EMU, 2 head_dim-128
# forward issuers, 3 dQ kernel issuers (defaults 3, 6, 1, 1)
DEFAULTS = {0: 3, 1: 6, 2: 1, 3: 1}


@pytest.fixture(autouse=True)
def _restore_defaults():
    yield
    for k, v in DEFAULTS.items():
        _lib.call("pc_attention_tune", k, v)


def _run(B, H, Hkv, S, hd, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    ld = (H + 2 * Hkv) * hd
    qkv = (torch.randn(B * S, ld, device="cuda", generator=g) * 0.5).bfloat16()
    do = torch.randn(B * S, H * hd, device="cuda", generator=g).bfloat16()
    o = torch.empty(B * S, H * hd, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * H * S, device="cuda")
    delta = torch.empty_like(lse)
    dqkv = torch.zeros_like(qkv)
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("pc_attention_gqa_fwd", 2, B, H, Hkv, S, hd, qkv.data_ptr(), ld, o.data_ptr(), H * hd,
              lse.data_ptr(), st)
    _lib.call("pc_attention_gqa_bwd", 2, B, H, Hkv, S, hd, qkv.data_ptr(), ld, o.data_ptr(),
              do.data_ptr(), H * hd, lse.data_ptr(), delta.data_ptr(), dqkv.data_ptr(), ld, st)
    torch.cuda.synchronize()
    return o, lse, dqkv


SHAPES64 = [(4, 12, 12, 1024), (3, 6, 6, 1000)]
SHAPES128 = [(2, 16, 16, 2048), (1, 16, 4, 1500)]


@pytest.mark.parametrize("B,H,Hkv,S", SHAPES64)
def test_hd64_forward_issuers_bitwise(B, H, Hkv, S):
    ref = _run(B, H, Hkv, S, 64)
    _lib.call("pc_attention_tune", 0, 2)   # one issuing warp
    alt = _run(B, H, Hkv, S, 64)
    for a, b in zip(ref, alt):
        assert torch.equal(a, b)


@pytest.mark.parametrize("B,H,Hkv,S", SHAPES64)
@pytest.mark.parametrize("design", [1, 3])
def test_hd64_forward_exp2_share(B, H, Hkv, S, design):
    _lib.call("pc_attention_tune", 0, design)
    _lib.call("pc_attention_tune", 1, 0)   # every exponential on MUFU
    o0, l0, _ = _run(B, H, Hkv, S, 64)
    _lib.call("pc_attention_tune", 0, 3)
    _lib.call("pc_attention_tune", 1, 6)
    o6, l6, _ = _run(B, H, Hkv, S, 64)
    assert float((o0.float() - o6.float()).abs().max()) <= 8e-3
    assert float((l0 - l6).abs().max()) <= 1e-3


@pytest.mark.parametrize("B,H,Hkv,S", SHAPES128)
def test_hd128_forward_issuers_bitwise(B, H, Hkv, S):
    ref = _run(B, H, Hkv, S, 128)
    _lib.call("pc_attention_tune", 2, 0)
    alt = _run(B, H, Hkv, S, 128)
    for a, b in zip(ref, alt):
        assert torch.equal(a, b)


@pytest.mark.parametrize("B,H,Hkv,S,hd", [s + (64,) for s in SHAPES64] + [s + (128,) for s in SHAPES128])
def test_dq_issuers_bitwise(B, H, Hkv, S, hd):
    ref = _run(B, H, Hkv, S, hd)
    _lib.call("pc_attention_tune", 3, 0)
    alt = _run(B, H, Hkv, S, hd)
    for a, b in zip(ref, alt):
        assert torch.equal(a, b)


def test_tune_rejects_unknown_values():
    with pytest.raises(_lib.PCError):
        _lib.call("pc_attention_tune", 2, 7)
    with pytest.raises(_lib.PCError):
        _lib.call("pc_attention_tune", 9, 0)
