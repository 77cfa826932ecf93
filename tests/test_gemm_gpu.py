"""GEMM numerics through the C-ABI (pc_gemm) against a torch fp32/fp64 reference.

Covers every operand-major combination of the tcgen05 bf16 kernel (the
reference's explicit transposes, ir.py:519-529, become majors), ragged
shapes that exercise TMA out-of-bounds fill and epilogue guards, every tile
width, and each fused epilogue.
"""
import pytest

torch = pytest.importorskip("torch")

from paper_2412_14374_b200 import _lib  # noqa: E402

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = a.double()
    b = b.double()
    scale = max(a.abs().max().item(), b.abs().max().item(), 1e-30)
    return (a - b).abs().max().item() / scale


def _ptr(t):
    return t.data_ptr() if t is not None else None


def run_gemm(A, B, ta, tb, M, N, K, out_dtype, epi=0, bias=None, aux=None, aux_out=None, C=None):
    dev = A.device
    dt_in = {torch.bfloat16: _lib.PC_BF16, torch.float32: _lib.PC_F32,
             torch.float64: _lib.PC_F64}[A.dtype]
    dt_out = {torch.bfloat16: _lib.PC_BF16, torch.float32: _lib.PC_F32,
              torch.float64: _lib.PC_F64}[out_dtype]
    if C is None:
        C = torch.empty(M, N, dtype=out_dtype, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("pc_gemm", dt_in, dt_out, ta, tb, M, N, K, _ptr(A), A.stride(0), _ptr(B),
              B.stride(0), _ptr(C), C.stride(0), epi, _ptr(bias), _ptr(aux),
              (aux.stride(0) if aux.dim() > 1 else aux.numel()) if aux is not None else 0,
              _ptr(aux_out),
              aux_out.stride(0) if aux_out is not None else 0, st)
    return C


def make_operands(M, N, K, ta, tb, dtype, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    A = torch.randn((K, M) if ta else (M, K), device="cuda", generator=g).to(dtype)
    B = torch.randn((N, K) if tb else (K, N), device="cuda", generator=g).to(dtype)
    opA = A.double().t() if ta else A.double()
    opB = B.double().t() if tb else B.double()
    return A, B, opA @ opB


class forced:
    """Pin the GEMM tile width / CTA-pair mode / store path for one block."""

    def __init__(self, bn=0, pair=0, tma=1):
        self.v = (bn, pair, tma)

    def __enter__(self):
        bn, pair, tma = self.v
        _lib.call("pc_gemm_set_tile_n", bn)
        _lib.call("pc_gemm_set_cta_pair", pair)
        _lib.call("pc_gemm_set_tma_store", tma)

    def __exit__(self, *a):
        _lib.call("pc_gemm_set_tile_n", 0)
        _lib.call("pc_gemm_set_cta_pair", 0)
        _lib.call("pc_gemm_set_tma_store", 1)


@pytest.mark.parametrize("tma", [1, 0])
@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("bn,pair", [(64, 1), (128, 1), (192, 1), (256, 1), (128, 2), (192, 2),
                                     (256, 2)])
@pytest.mark.parametrize("shape", [(128, 256, 64), (256, 512, 256), (200, 136, 72), (1024, 768, 768),
                                   (392, 200, 136)])
def test_bf16_tcgen05_majors(ta, tb, bn, pair, shape, tma):
    M, N, K = shape
    A, B, ref = make_operands(M, N, K, ta, tb, torch.bfloat16)
    with forced(bn, pair, tma):
        C32 = run_gemm(A, B, ta, tb, M, N, K, torch.float32)
        C16 = run_gemm(A, B, ta, tb, M, N, K, torch.bfloat16)
    torch.cuda.synchronize()
    assert rel(C32, ref) < 1e-5
    assert rel(C16, ref) < 1e-2


def test_bf16_large_persistent():
    M, N, K = 8192, 2304, 768
    A, B, ref = make_operands(M, N, K, 0, 1, torch.bfloat16, seed=3)
    C = run_gemm(A, B, 0, 1, M, N, K, torch.float32)
    torch.cuda.synchronize()
    assert rel(C, ref) < 1e-5


@pytest.mark.parametrize("ta,tb", [(0, 1), (1, 0), (0, 0)])
@pytest.mark.parametrize("shape", [(8192, 768, 5000), (5000, 768, 8192), (8200, 200, 4104)])
def test_bf16_n_raster_large_a(shape, ta, tb):
    """A operand larger than L2 (the LM-head gradient GEMMs): tiles walk N so
    the A rows stream from DRAM once; results as with the M raster."""
    M, N, K = shape
    A, B, ref = make_operands(M, N, K, ta, tb, torch.bfloat16, seed=6)
    C = run_gemm(A, B, ta, tb, M, N, K, torch.float32)
    torch.cuda.synchronize()
    assert rel(C, ref) < 3e-5   # fp32 accumulation over K = 8192 unit-normal products


@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-5), (torch.float64, 1e-13)])
@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_simt_gemm(dtype, tol, ta, tb):
    M, N, K = 70, 45, 33
    A, B, ref = make_operands(M, N, K, ta, tb, dtype, seed=1)
    C = run_gemm(A, B, ta, tb, M, N, K, dtype)
    torch.cuda.synchronize()
    assert rel(C, ref) < tol


@pytest.mark.parametrize("pair", [0, 2])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_epilogues(dtype, pair):
    with forced(0, pair):
        _epilogues(dtype)


def _epilogues(dtype):
    M, N, K = 512, 192, 128
    A, B, ref = make_operands(M, N, K, 0, 1, dtype, seed=2)
    out = torch.bfloat16 if dtype == torch.bfloat16 else torch.float32
    tol = 2e-2 if dtype == torch.bfloat16 else 1e-5
    bias = torch.randn(N, device="cuda", dtype=torch.float32)
    pre = torch.empty(M, N, device="cuda", dtype=out)
    C = run_gemm(A, B, 0, 1, M, N, K, out, epi=_lib.EPI_BIAS | _lib.EPI_GELU, bias=bias,
                 aux_out=pre)
    z = ref + bias.double()
    assert rel(pre, z) < tol
    assert rel(C, torch.nn.functional.gelu(z, approximate="tanh")) < tol
    aux = torch.randn(M, N, device="cuda").to(out)
    C = run_gemm(A, B, 0, 1, M, N, K, out, epi=_lib.EPI_RESIDUAL, aux=aux)
    assert rel(C, ref + aux.double()) < tol
    u = aux.double().requires_grad_(True)
    gelu_u = torch.nn.functional.gelu(u, approximate="tanh")
    (dgelu,) = torch.autograd.grad(gelu_u.sum(), u)
    C = run_gemm(A, B, 0, 1, M, N, K, out, epi=_lib.EPI_GELU_GRAD, aux=aux)
    assert rel(C, ref * dgelu) < tol
    C = run_gemm(A, B, 0, 1, M, N, K, out, epi=_lib.EPI_RELU, aux_out=pre)
    assert rel(C, ref.clamp_min(0)) < tol
    C = run_gemm(A, B, 0, 1, M, N, K, out, epi=_lib.EPI_RELU_GRAD, aux=aux)
    assert rel(C, ref * (aux.double() > 0)) < tol
    acc = torch.randn(M, N, device="cuda", dtype=torch.float32)
    want = acc.double() + ref
    run_gemm(A, B, 0, 1, M, N, K, torch.float32, epi=_lib.EPI_ACCUM, C=acc)
    torch.cuda.synchronize()
    assert rel(acc, want) < (1e-5 if dtype != torch.bfloat16 else 1e-5)


@pytest.mark.parametrize("pair", [1, 2])
@pytest.mark.parametrize("shape", [(768, 768, 8192), (256, 192, 4096), (200, 72, 2000)])
def test_splitk_zero_c_deterministic(shape, pair):
    """The split-K hint (two K halves reduce-added onto a zero C) is exact to the
    reference and bitwise reproducible run to run."""
    M, N, K = shape
    A, B, ref = make_operands(M, N, K, 1, 0, torch.bfloat16, seed=5)
    outs = []
    with forced(0, pair):
        for _ in range(3):
            C = torch.zeros(M, N, device="cuda", dtype=torch.float32)
            run_gemm(A, B, 1, 0, M, N, K, torch.float32, epi=_lib.EPI_SPLITK_ZERO_C, C=C)
            outs.append(C)
    torch.cuda.synchronize()
    assert rel(outs[0], ref) < 1e-5
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])


@pytest.mark.parametrize("tma", [1, 0])
@pytest.mark.parametrize("pair", [1, 2])
@pytest.mark.parametrize("shape", [(768, 3072, 8192), (200, 136, 1100), (256, 512, 256)])
def test_accumulate_equals_store_then_add(shape, pair, tma):
    """fp32 C += op(A) op(B) (TMA reduce-add, or the direct read-modify-write)
    is bitwise the unsplit product stored, then added onto C."""
    M, N, K = shape
    A, B, ref = make_operands(M, N, K, 1, 0, torch.bfloat16, seed=9)
    g = torch.Generator(device="cuda").manual_seed(3)
    acc0 = torch.randn(M, N, device="cuda", generator=g)
    with forced(0, pair, tma):
        fused = run_gemm(A, B, 1, 0, M, N, K, torch.float32, epi=_lib.EPI_ACCUM, C=acc0.clone())
        part = run_gemm(A, B, 1, 0, M, N, K, torch.float32)
    want = acc0.clone()
    _lib.call("pc_accumulate", _lib.PC_F32, _lib.PC_F32, want.numel(), want.data_ptr(),
              part.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(fused, want)
    assert rel(fused - acc0, ref) < 1e-4


def test_tile_choice_reports_split():
    import ctypes
    bn, cg, ks = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _lib.call("pc_gemm_tile_choice", 0, 768, 768, 8192, 1, ctypes.byref(bn), ctypes.byref(cg),
              ctypes.byref(ks))
    assert ks.value == 2 and bn.value in (64, 128, 192, 256)
    _lib.call("pc_gemm_tile_choice", 0, 768, 768, 8192, 0, ctypes.byref(bn), ctypes.byref(cg),
              ctypes.byref(ks))
    assert ks.value == 1


def _ordered_bounds(nk, ks):
    """Split boundaries of the ordered split-K (gemm_tc.cu k_split_at)."""
    if ks == 1:
        return [0, nk]
    dl = (nk + 4 * ks - 1) // (4 * ks)
    l0 = (nk - dl * ks * (ks - 1) // 2) // ks
    return [s * l0 + dl * s * (s - 1) // 2 for s in range(ks)] + [nk]


@pytest.mark.parametrize("shape", [(768, 768, 8192), (2304, 768, 8192), (768, 3072, 8192),
                                   (256, 256, 4096)])
def test_ordered_splitk_accumulate(shape):
    """C += op(A) op(B) split in K and added in a fixed order, ((C + h0) + h1)
    + ..., sequenced per tile by flags: equal to the unsplit part-products
    added one after the other, run-to-run identical, flags left zeroed."""
    import ctypes
    M, N, K = shape
    # 256-wide CTA-pair tiles leave most SMs idle without a K split on these
    # shapes, so the chooser splits (the production choice may be an unsplit
    # narrower tile; this test is about the split protocol)
    _lib.call("pc_gemm_set_tile_n", 256)
    _lib.call("pc_gemm_set_cta_pair", 2)
    try:
        _ordered_splitk_case(M, N, K)
    finally:
        _lib.call("pc_gemm_set_tile_n", 0)
        _lib.call("pc_gemm_set_cta_pair", 0)


def _ordered_splitk_case(M, N, K):
    import ctypes
    bn, cg, ks = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _lib.call("pc_gemm_tile_choice", 0, M, N, K, 2, ctypes.byref(bn), ctypes.byref(cg),
              ctypes.byref(ks))
    assert ks.value in (2, 4)
    A, B, ref = make_operands(M, N, K, 1, 0, torch.bfloat16, seed=4)
    g = torch.Generator(device="cuda").manual_seed(8)
    acc0 = torch.randn(M, N, device="cuda", generator=g)
    flags = torch.zeros(1 << 16, dtype=torch.int32, device="cuda")
    outs = []
    for _ in range(3):
        C = acc0.clone()
        run_gemm(A, B, 1, 0, M, N, K, torch.float32,
                 epi=_lib.EPI_ACCUM | _lib.EPI_SPLITK_ORDERED, aux=flags, C=C)
        outs.append(C)
    bounds = [64 * b for b in _ordered_bounds((K + 63) // 64, ks.value)]
    bounds[-1] = K
    want = acc0.clone()
    st = torch.cuda.current_stream().cuda_stream
    with forced(bn.value, cg.value):
        for lo, hi in zip(bounds[:-1], bounds[1:]):
            h = run_gemm(A[lo:hi], B[lo:hi], 1, 0, M, N, hi - lo, torch.float32)
            _lib.call("pc_accumulate", _lib.PC_F32, _lib.PC_F32, want.numel(), want.data_ptr(),
                      h.data_ptr(), st)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])
    assert torch.equal(outs[0], want)
    assert int(flags.abs().sum()) == 0
    assert rel(outs[0] - acc0, ref) < 1e-4


@pytest.mark.parametrize("M1,M2,N,K", [(2304, 768, 768, 8192), (256, 200, 192, 1024),
                                       (1024, 4096, 1024, 8192)])
@pytest.mark.parametrize("ordered", [False, True])
def test_wgrad_pair_matches_two_products(M1, M2, N, K, ordered):
    """pc_gemm_wgrad_pair: C1 (+)= A1^T B1 and C2 (+)= A2^T B2 in one launch (the
    attention-output + qkv weight gradients of a block), both within fp32
    rounding of the float64 products, run-to-run identical, flags left zeroed."""
    g = torch.Generator(device="cuda").manual_seed(M1 + M2 + N)
    A1 = torch.randn(K, M1, device="cuda", generator=g).to(torch.bfloat16)
    B1 = torch.randn(K, N, device="cuda", generator=g).to(torch.bfloat16)
    A2 = torch.randn(K, M2, device="cuda", generator=g).to(torch.bfloat16)
    B2 = torch.randn(K, N, device="cuda", generator=g).to(torch.bfloat16)
    acc1 = torch.randn(M1, N, device="cuda", generator=g)
    acc2 = torch.randn(M2, N, device="cuda", generator=g)
    flags = torch.zeros(1 << 16, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    outs = []
    for _ in range(2):
        if ordered:
            C1, C2 = acc1.clone(), acc2.clone()
            epi, aux = _lib.EPI_ACCUM | _lib.EPI_SPLITK_ORDERED, flags.data_ptr()
        else:
            C1, C2 = torch.zeros_like(acc1), torch.zeros_like(acc2)
            epi, aux = _lib.EPI_SPLITK_ZERO_C, None
        _lib.call("pc_gemm_wgrad_pair", M1, M2, N, K, A1.data_ptr(), M1, B1.data_ptr(), N,
                  C1.data_ptr(), N, A2.data_ptr(), M2, B2.data_ptr(), N, C2.data_ptr(), N, epi, aux,
                  flags.numel(), st)
        outs.append((C1, C2))
    torch.cuda.synchronize()
    ref1 = A1.double().t() @ B1.double()
    ref2 = A2.double().t() @ B2.double()
    base1, base2 = (acc1.double(), acc2.double()) if ordered else (0.0, 0.0)
    assert rel(outs[0][0].double() - base1, ref1) < 1e-4
    assert rel(outs[0][1].double() - base2, ref2) < 1e-4
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    assert int(flags.abs().sum()) == 0


@pytest.mark.parametrize("bn,pair", [(256, 2), (256, 1)])
def test_wgrad_pair_forced_split(bn, pair):
    """The grouped pair under a forced tile that makes the chooser split K: the
    ordered split-K flags are indexed by the pair's global tile, so both
    problems' chains stay sequenced; equal to the fp64 products, deterministic."""
    import ctypes
    M1, M2, N, K = 2304, 768, 768, 8192
    _lib.call("pc_gemm_set_tile_n", bn)
    _lib.call("pc_gemm_set_cta_pair", pair)
    try:
        b_, c_, ks = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _lib.call("pc_gemm_tile_choice", 0, M1 + M2, N, K, 2, ctypes.byref(b_), ctypes.byref(c_),
                  ctypes.byref(ks))
        assert ks.value > 1
        g = torch.Generator(device="cuda").manual_seed(11)
        A1 = torch.randn(K, M1, device="cuda", generator=g).to(torch.bfloat16)
        B1 = torch.randn(K, N, device="cuda", generator=g).to(torch.bfloat16)
        A2 = torch.randn(K, M2, device="cuda", generator=g).to(torch.bfloat16)
        B2 = torch.randn(K, N, device="cuda", generator=g).to(torch.bfloat16)
        acc1 = torch.randn(M1, N, device="cuda", generator=g)
        acc2 = torch.randn(M2, N, device="cuda", generator=g)
        flags = torch.zeros(1 << 16, dtype=torch.int32, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        outs = []
        for _ in range(2):
            C1, C2 = acc1.clone(), acc2.clone()
            _lib.call("pc_gemm_wgrad_pair", M1, M2, N, K, A1.data_ptr(), M1, B1.data_ptr(), N,
                      C1.data_ptr(), N, A2.data_ptr(), M2, B2.data_ptr(), N, C2.data_ptr(), N,
                      _lib.EPI_ACCUM | _lib.EPI_SPLITK_ORDERED, flags.data_ptr(), flags.numel(), st)
            outs.append((C1, C2))
        torch.cuda.synchronize()
    finally:
        _lib.call("pc_gemm_set_tile_n", 0)
        _lib.call("pc_gemm_set_cta_pair", 0)
    assert rel(outs[0][0].double() - acc1.double(), A1.double().t() @ B1.double()) < 1e-4
    assert rel(outs[0][1].double() - acc2.double(), A2.double().t() @ B2.double()) < 1e-4
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    assert int(flags.abs().sum()) == 0
