"""GPT path on the GPU vs the float64 numpy oracle (oracle/gpt.py).

fp32 mode: rel < 1e-5 (north_star).  bf16 mode: rel < 2e-2 (north_star).
The pipeline runs the tied-embedding GPT graph (ir.build_gpt) through the
same planner and runtime as the FFN tests: GPipe / 1F1B / interleaved on one
GPU with local channels, including the non-adjacent token skip to the last
stage and the commuted tied-weight gradient.
"""
import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import ffn, gpt  # noqa: E402
from paper_2412_14374_b200 import _lib  # noqa: E402
from paper_2412_14374_b200 import comms as C  # noqa: E402
from paper_2412_14374_b200 import ir as I  # noqa: E402
from paper_2412_14374_b200 import schedules as S  # noqa: E402
from paper_2412_14374_b200 import taskgraph as T  # noqa: E402
from paper_2412_14374_b200.executor import run_pipelined  # noqa: E402

pytestmark = pytest.mark.gpu


def plan(cfg: I.GPTConfig, fam, P, M, V=1):
    p = I.derive_backward(I.partition_stages(I.build_gpt(cfg)))
    s = {"gpipe": lambda: S.gpipe(P, M), "1f1b": lambda: S.one_f_one_b(P, M),
         "interleaved": lambda: S.interleaved_1f1b(P, M, V)}[fam]()
    tg = T.infer_outer_placement(T.commute_grad_accumulation(T.unroll(p, s)), p)
    cp = C.infer_comms(tg, s)
    assert C.check_deadlock_free(cp).ok
    return p, tg, C.fuse(C.insert_deletions(cp, tg), tg)


def oracle_cfg(cfg: I.GPTConfig):
    return dict(layers=cfg.layers, d=cfg.d_model, heads=cfg.n_heads, ff=cfg.d_ff,
                vocab=cfg.vocab, seq=cfg.seq_len, mbs=cfg.microbatch_size)


def run_case(cfg, fam, P, M, V, mode, seed=0, std=0.02):
    p, tg, cp = plan(cfg, fam, P, M, V)
    oc = oracle_cfg(cfg)
    rng = np.random.default_rng(seed)
    params = gpt.init_params(oc, rng, std=std)
    tokens = gpt.init_tokens(oc, M, rng)
    g, l, w = gpt.run_reference_gpt(params, tokens, oc)
    res = run_pipelined(cp, tg, {q: v.astype(np.float32) for q, v in params.items()},
                        tokens.reshape(M * cfg.microbatch_size, cfg.seq_len), mode=mode, gpt=cfg)
    return res, g, l, w


TINY = dict(layers=4, d_model=64, n_heads=4, d_ff=256, vocab=96, seq_len=32, microbatch_size=2)


@pytest.mark.parametrize("fam,P,M,V,yields", [
    ("gpipe", 1, 2, 1, None), ("gpipe", 2, 4, 1, (3,)), ("1f1b", 4, 4, 1, (2, 3, 5)),
    ("interleaved", 2, 4, 2, (1, 3, 4))])
def test_gpt_fp32_matches_oracle(fam, P, M, V, yields):
    cfg = I.GPTConfig(**TINY, yields=yields, yield_every=TINY["layers"] + 2, elem_bytes=4)
    res, g, l, w = run_case(cfg, fam, P, M, V, "fp32", std=0.1)
    assert ffn.rel(res.losses, l) < 1e-5
    for q in g:
        assert ffn.rel(res.grads[q], g[q]) < 1e-5, q
        assert ffn.rel(res.new_params[q], w[q]) < 1e-5, q


@pytest.mark.parametrize("fam,P,M,yields", [("gpipe", 2, 4, (3,)), ("1f1b", 4, 8, (2, 3, 5))])
def test_gpt_bf16_matches_oracle(fam, P, M, yields):
    cfg = I.GPTConfig(**dict(TINY, d_model=128, n_heads=2, d_ff=512, vocab=256, seq_len=64),
                      yields=yields, yield_every=TINY["layers"] + 2, elem_bytes=2)
    res, g, l, w = run_case(cfg, fam, P, M, 1, "bf16", std=0.05)
    assert ffn.rel(res.losses, l) < 2e-2
    for q in g:
        assert ffn.rel(res.grads[q], g[q]) < 2e-2, q
        assert ffn.rel(res.new_params[q], w[q]) < 2e-2, q


def test_gpt_bf16_deterministic_rerun():
    cfg = I.GPTConfig(**TINY, yields=(3,), yield_every=TINY["layers"] + 2)
    a, *_ = run_case(cfg, "1f1b", 2, 4, 1, "bf16")
    b, *_ = run_case(cfg, "1f1b", 2, 4, 1, "bf16")
    for q in a.grads:
        assert np.array_equal(a.grads[q], b.grads[q])
    assert np.array_equal(a.losses, b.losses)


# ---------------------------------------------------------------- kernels


def _t(x, dt=torch.float32):
    return torch.tensor(x, device="cuda", dtype=dt)


@pytest.mark.parametrize("dt,tol", [(torch.float32, 1e-5), (torch.bfloat16, 2e-2)])
@pytest.mark.parametrize("impl", [0, 1, 2])
@pytest.mark.parametrize("S", [80, 256])
def test_attention_kernels(dt, tol, impl, S):
    B, H, hd = 2, 3, 64
    rng = np.random.default_rng(3)
    qkv = rng.standard_normal((B * S, 3 * H * hd)) * 0.5
    do = rng.standard_normal((B * S, H * hd))
    d = H * hd
    q, k, v = (qkv[:, i * d:(i + 1) * d].reshape(B, S, H, hd).transpose(0, 2, 1, 3) for i in range(3))
    o4, p = gpt.attention(q, k, v)
    dq, dk, dv = gpt.attention_bwd(do.reshape(B, S, H, hd).transpose(0, 2, 1, 3), q, k, v, p)
    merge = lambda t: t.transpose(0, 2, 1, 3).reshape(B * S, d)
    tq = _t(qkv, dt)
    o = torch.empty(B * S, d, device="cuda", dtype=dt)
    lse = torch.empty(B * H * S, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("pc_attention_set_impl", impl)
    try:
        _lib.call("pc_attention_fwd", _lib.PC_F32 if dt == torch.float32 else _lib.PC_BF16, B, H,
                  S, hd, tq.data_ptr(), 3 * d, o.data_ptr(), d, lse.data_ptr(), st)
        tdo = _t(do, dt)
        dqkv = torch.empty(B * S, 3 * d, device="cuda", dtype=dt)
        delta = torch.empty(B * H * S, device="cuda")
        _lib.call("pc_attention_bwd", _lib.PC_F32 if dt == torch.float32 else _lib.PC_BF16, B, H,
                  S, hd, tq.data_ptr(), 3 * d, o.data_ptr(), tdo.data_ptr(), d, lse.data_ptr(),
                  delta.data_ptr(), dqkv.data_ptr(), 3 * d, st)
    finally:
        _lib.call("pc_attention_set_impl", 0)
    torch.cuda.synchronize()
    assert ffn.rel(o.double().cpu().numpy(), merge(o4)) < tol
    got = dqkv.double().cpu().numpy()
    assert ffn.rel(got[:, :d], merge(dq)) < tol
    assert ffn.rel(got[:, d:2 * d], merge(dk)) < tol
    assert ffn.rel(got[:, 2 * d:], merge(dv)) < tol


def test_layernorm_and_xent_kernels():
    rows, d, V, seq = 64, 96, 50, 16
    rng = np.random.default_rng(4)
    x = rng.standard_normal((rows, d))
    g, b = rng.standard_normal(d), rng.standard_normal(d)
    dy = rng.standard_normal((rows, d))
    y, cache = gpt.layer_norm(x, g, b)
    dx, dg, db = gpt.layer_norm_bwd(dy, g, cache)
    tx, tg_, tb, tdy = _t(x), _t(g), _t(b), _t(dy)
    ty = torch.empty_like(tx)
    mean = torch.empty(rows, device="cuda")
    rstd = torch.empty(rows, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("pc_layernorm_fwd", _lib.PC_F32, rows, d, tx.data_ptr(), tg_.data_ptr(),
              tb.data_ptr(), ty.data_ptr(), mean.data_ptr(), rstd.data_ptr(), 1e-5, st)
    tdx = torch.empty_like(tx)
    tdg = torch.empty(d, device="cuda")
    tdb = torch.empty(d, device="cuda")
    _lib.call("pc_layernorm_bwd", _lib.PC_F32, rows, d, tdy.data_ptr(), tx.data_ptr(),
              tg_.data_ptr(), mean.data_ptr(), rstd.data_ptr(), None, tdx.data_ptr(),
              tdg.data_ptr(), tdb.data_ptr(), None, 0, st)
    # the many-CTA two-stage reduction (with workspace) gives the same parameter grads
    import ctypes
    nb = ctypes.c_int64()
    _lib.call("pc_reduce_workspace_bytes", rows, d, ctypes.byref(nb))
    ws = torch.zeros(nb.value, dtype=torch.uint8, device="cuda")  # arrival counters start at 0
    tdg2, tdb2 = torch.empty(d, device="cuda"), torch.empty(d, device="cuda")
    _lib.call("pc_layernorm_bwd", _lib.PC_F32, rows, d, tdy.data_ptr(), tx.data_ptr(),
              tg_.data_ptr(), mean.data_ptr(), rstd.data_ptr(), None, tdx.data_ptr(),
              tdg2.data_ptr(), tdb2.data_ptr(), ws.data_ptr(), nb.value, st)
    torch.cuda.synchronize()
    assert ffn.rel(ty.cpu().numpy(), y) < 1e-5
    assert ffn.rel(tdx.cpu().numpy(), dx) < 1e-5
    assert ffn.rel(tdg.cpu().numpy(), dg) < 1e-5
    assert ffn.rel(tdb.cpu().numpy(), db) < 1e-5
    assert ffn.rel(tdg2.cpu().numpy(), dg) < 1e-5
    assert ffn.rel(tdb2.cpu().numpy(), db) < 1e-5
    # column sums (bias gradients), single- and two-stage
    cs1, cs2 = torch.empty(d, device="cuda"), torch.empty(d, device="cuda")
    _lib.call("pc_col_sum", _lib.PC_F32, _lib.PC_F32, rows, d, tdy.data_ptr(), d, cs1.data_ptr(),
              0, None, 0, st)
    _lib.call("pc_col_sum", _lib.PC_F32, _lib.PC_F32, rows, d, tdy.data_ptr(), d, cs2.data_ptr(),
              0, ws.data_ptr(), nb.value, st)
    torch.cuda.synchronize()
    assert ffn.rel(cs1.cpu().numpy(), dy.sum(0)) < 1e-5
    assert ffn.rel(cs2.cpu().numpy(), dy.sum(0)) < 1e-5
    # cross-entropy against the oracle head (identity "wte" so logits = h)
    h = rng.standard_normal((rows, V))
    tokens = rng.integers(0, V, size=(rows // seq, seq)).astype(np.int32)
    loss, dh, _ = gpt.head_loss(h, np.eye(V), tokens)
    tl = _t(h)
    tt = torch.tensor(tokens, device="cuda")
    row_loss = torch.empty(rows, device="cuda")
    _lib.call("pc_xent_fwd_bwd", _lib.PC_F32, rows, V, seq, tl.data_ptr(), V, tt.data_ptr(),
              row_loss.data_ptr(), st)
    torch.cuda.synchronize()
    assert abs(row_loss.sum().item() - loss) < 1e-4 * abs(loss)
    assert ffn.rel(tl.cpu().numpy(), dh) < 1e-5


def test_embedding_kernels_deterministic():
    T_, d, seq, V = 256, 64, 32, 40
    rng = np.random.default_rng(5)
    wte = rng.standard_normal((V, d))
    wpe = rng.standard_normal((seq, d))
    tokens = rng.integers(0, V, size=T_).astype(np.int32)
    dh = rng.standard_normal((T_, d))
    st = torch.cuda.current_stream().cuda_stream
    tt = torch.tensor(tokens, device="cuda")
    out = torch.empty(T_, d, device="cuda")
    twte, twpe, tdh = _t(wte), _t(wpe), _t(dh)   # keep alive across the async launches
    _lib.call("pc_embedding_fwd", _lib.PC_F32, T_, d, seq, tt.data_ptr(), twte.data_ptr(),
              twpe.data_ptr(), out.data_ptr(), st)
    torch.cuda.synchronize()
    ref = wte[tokens] + wpe[np.arange(T_) % seq]
    assert ffn.rel(out.cpu().numpy(), ref) < 1e-6
    import ctypes
    nb = ctypes.c_int64()
    _lib.call("pc_embedding_bwd_workspace_bytes", T_, ctypes.byref(nb))
    ws = torch.zeros(nb.value, dtype=torch.uint8, device="cuda")  # arrival counters start at 0
    outs = []
    for _ in range(2):
        dwte = torch.empty(V, d, device="cuda")
        dwpe = torch.empty(seq, d, device="cuda")
        _lib.call("pc_embedding_bwd", _lib.PC_F32, T_, d, seq, V, tt.data_ptr(), tdh.data_ptr(),
                  dwte.data_ptr(), dwpe.data_ptr(), ws.data_ptr(), nb.value, st)
        torch.cuda.synchronize()
        outs.append((dwte.cpu().numpy(), dwpe.cpu().numpy()))
    want_te = np.zeros((V, d))
    np.add.at(want_te, tokens, dh)
    want_pe = np.zeros((seq, d))
    np.add.at(want_pe, np.arange(T_) % seq, dh)
    assert ffn.rel(outs[0][0], want_te) < 1e-5
    assert ffn.rel(outs[0][1], want_pe) < 1e-5
    assert np.array_equal(outs[0][0], outs[1][0])


def test_xent_bf16_vectorised_path():
    rows, V, seq = 96, 136, 24
    rng = np.random.default_rng(6)
    h = rng.standard_normal((rows, V)) * 2
    tokens = rng.integers(0, V, size=(rows // seq, seq)).astype(np.int32)
    tl = _t(h, torch.bfloat16)
    hb = tl.double().cpu().numpy()
    loss, dh, _ = gpt.head_loss(hb, np.eye(V), tokens)
    tt = torch.tensor(tokens, device="cuda")
    row_loss = torch.empty(rows, device="cuda")
    _lib.call("pc_xent_fwd_bwd", _lib.PC_BF16, rows, V, seq, tl.data_ptr(), V, tt.data_ptr(),
              row_loss.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert abs(row_loss.sum().item() - loss) < 1e-4 * abs(loss)
    assert ffn.rel(tl.double().cpu().numpy(), dh) < 1e-2


def test_cuda_graph_replay_matches_eager():
    """One actor per process: the captured program replays to the same results
    as the eager step (bitwise), including after new inputs are copied in."""
    from paper_2412_14374_b200.executor import PipelineEngine
    cfg = I.GPTConfig(**TINY, yield_every=TINY["layers"] + 2, elem_bytes=2)
    p, tg, cp = plan(cfg, "1f1b", 1, 4)
    oc = oracle_cfg(cfg)
    rng = np.random.default_rng(7)
    params = {q: v.astype(np.float32) for q, v in gpt.init_params(oc, rng, std=0.05).items()}
    t1 = gpt.init_tokens(oc, 4, rng).reshape(8, -1)
    t2 = gpt.init_tokens(oc, 4, rng).reshape(8, -1)
    eng = PipelineEngine(cp, tg, mode="bf16", gpt=cfg)
    e1 = eng.step(params, t1)
    e2 = eng.step(params, t2)
    cap = eng.capture(params, t1)
    r = cap.replay()
    torch.cuda.synchronize()
    assert np.array_equal(r.losses.cpu().numpy(), e1.losses)
    for q in e1.grads:
        assert np.array_equal(r.grads[q].cpu().numpy(), e1.grads[q]), q
    r = cap.replay(t2)
    torch.cuda.synchronize()
    assert np.array_equal(r.losses.cpu().numpy(), e2.losses)
    for q in e2.grads:
        assert np.array_equal(r.grads[q].cpu().numpy(), e2.grads[q]), q


@pytest.mark.parametrize("d", [96, 256, 768, 1024])
@pytest.mark.parametrize("dt,tol", [(torch.float32, 1e-5), (torch.bfloat16, 2e-2)])
def test_layernorm_vectorised_paths(d, dt, tol):
    import ctypes
    rows = 200
    rng = np.random.default_rng(8)
    x = rng.standard_normal((rows, d))
    g, b = rng.standard_normal(d), rng.standard_normal(d)
    dy = rng.standard_normal((rows, d))
    res = rng.standard_normal((rows, d))
    tx, tdy, tres = _t(x, dt), _t(dy, dt), _t(res, dt)
    xq, dyq, resq = (t.double().cpu().numpy() for t in (tx, tdy, tres))
    y, cache = gpt.layer_norm(xq, g, b)
    dx, dg, db = gpt.layer_norm_bwd(dyq, g, cache)
    tg_, tb = _t(g), _t(b)
    ty = torch.empty_like(tx)
    mean = torch.empty(rows, device="cuda")
    rstd = torch.empty(rows, device="cuda")
    pc = _lib.PC_F32 if dt == torch.float32 else _lib.PC_BF16
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("pc_layernorm_fwd", pc, rows, d, tx.data_ptr(), tg_.data_ptr(), tb.data_ptr(),
              ty.data_ptr(), mean.data_ptr(), rstd.data_ptr(), 1e-5, st)
    nb = ctypes.c_int64()
    _lib.call("pc_reduce_workspace_bytes", rows, d, ctypes.byref(nb))
    ws = torch.zeros(nb.value, dtype=torch.uint8, device="cuda")
    tdx = torch.empty_like(tx)
    tdg, tdb = torch.empty(d, device="cuda"), torch.empty(d, device="cuda")
    _lib.call("pc_layernorm_bwd", pc, rows, d, tdy.data_ptr(), tx.data_ptr(), tg_.data_ptr(),
              mean.data_ptr(), rstd.data_ptr(), tres.data_ptr(), tdx.data_ptr(), tdg.data_ptr(),
              tdb.data_ptr(), ws.data_ptr(), nb.value, st)
    cs = torch.empty(d, device="cuda")
    _lib.call("pc_col_sum", pc, _lib.PC_F32, rows, d, tdy.data_ptr(), d, cs.data_ptr(), 0,
              ws.data_ptr(), nb.value, st)
    torch.cuda.synchronize()
    assert ffn.rel(ty.double().cpu().numpy(), y) < tol
    assert ffn.rel(tdx.double().cpu().numpy(), dx + resq) < tol
    assert ffn.rel(tdg.cpu().numpy(), dg) < tol
    assert ffn.rel(tdb.cpu().numpy(), db) < tol
    assert ffn.rel(cs.cpu().numpy(), dyq.sum(0)) < 1e-5


@pytest.mark.parametrize("rows,cols", [(8192, 768), (8192, 2304), (1000, 768), (37, 768),
                                       (8191, 1024), (8192, 770), (1, 256)])
def test_col_sum_bf16_shapes_and_determinism(rows, cols):
    """Bias-gradient column sums (the `sum-to` of executor.py:50-56) at the C2
    shapes and ragged ones: short row chunks (all of a warp's rows loaded at
    once), long chunks, column tails; equal to the float64 sum within fp32
    rounding, bitwise identical run to run, and accumulate = out + sum."""
    g = torch.Generator(device="cuda").manual_seed(rows * 7 + cols)
    a = torch.randn(rows, cols, device="cuda", generator=g).to(torch.bfloat16)
    nb = ctypes.c_int64()
    _lib.call("pc_reduce_workspace_bytes", rows, cols, ctypes.byref(nb))
    ws = torch.zeros(nb.value, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    outs = []
    for _ in range(2):
        o = torch.empty(cols, device="cuda")
        _lib.call("pc_col_sum", _lib.PC_BF16, _lib.PC_F32, rows, cols, a.data_ptr(), cols,
                  o.data_ptr(), 0, ws.data_ptr(), nb.value, st)
        outs.append(o)
    acc = torch.full((cols,), 0.5, device="cuda")
    _lib.call("pc_col_sum", _lib.PC_BF16, _lib.PC_F32, rows, cols, a.data_ptr(), cols,
              acc.data_ptr(), 1, ws.data_ptr(), nb.value, st)
    torch.cuda.synchronize()
    ref = a.double().sum(0)
    err = ((outs[0].double() - ref).abs().max() / ref.abs().max()).item()
    assert err < 1e-5, err
    assert torch.equal(outs[0], outs[1])
    assert torch.allclose(acc, outs[0] + 0.5, rtol=1e-6, atol=1e-5)


@pytest.mark.parametrize("rows,d", [(8192, 768), (8192, 1024), (1000, 768), (37, 256), (8191, 2048)])
@pytest.mark.parametrize("accumulate", [0, 1])
def test_layernorm_param_bias_grads_equal_the_separate_sums(rows, d, accumulate):
    """pc_layernorm_param_bias_grads (LN2's dgamma / dbeta plus the fc2 and
    attention-output bias gradients in one pass) is bitwise equal to
    pc_layernorm_param_grads + two pc_col_sum calls, with and without
    accumulation onto a running sum, and within fp32 rounding of fp64."""
    g = torch.Generator(device="cuda").manual_seed(rows + d)
    dy, x, y3, y4 = (torch.randn(rows, d, device="cuda", generator=g).to(torch.bfloat16)
                     for _ in range(4))
    mean = torch.randn(rows, device="cuda", generator=g) * 0.1
    rstd = torch.rand(rows, device="cuda", generator=g) + 0.5
    nb = ctypes.c_int64()
    _lib.call("pc_reduce_workspace_bytes", rows, d, ctypes.byref(nb))
    ws = torch.zeros(nb.value, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    init = torch.randn(4, d, device="cuda", generator=g)
    sep, one = init.clone(), init.clone()
    _lib.call("pc_layernorm_param_grads", _lib.PC_BF16, rows, d, dy.data_ptr(), x.data_ptr(),
              mean.data_ptr(), rstd.data_ptr(), sep[0].data_ptr(), sep[1].data_ptr(), accumulate,
              ws.data_ptr(), nb.value, st)
    for i, y in ((2, y3), (3, y4)):
        _lib.call("pc_col_sum", _lib.PC_BF16, _lib.PC_F32, rows, d, y.data_ptr(), d,
                  sep[i].data_ptr(), accumulate, ws.data_ptr(), nb.value, st)
    _lib.call("pc_layernorm_param_bias_grads", rows, d, dy.data_ptr(), x.data_ptr(),
              mean.data_ptr(), rstd.data_ptr(), one[0].data_ptr(), one[1].data_ptr(),
              y3.data_ptr(), one[2].data_ptr(), y4.data_ptr(), one[3].data_ptr(), accumulate, st)
    torch.cuda.synchronize()
    assert torch.equal(sep, one)
    xhat = (x.double() - mean.double()[:, None]) * rstd.double()[:, None]
    ref = torch.stack([(dy.double() * xhat).sum(0), dy.double().sum(0), y3.double().sum(0),
                       y4.double().sum(0)])
    if accumulate:
        ref = ref + init.double()
    err = ((one.double() - ref).abs().max() / ref.abs().max()).item()
    assert err < 1e-5, err


def test_fused_grad_accumulation_matches_the_add_chain():
    """Block weight / bias / LN gradients added onto the running sum by their
    producers (GEMM TMA reduce-add, reductions with accumulate) reproduce the
    grad-merge chain (taskgraph.py:369-433): bitwise where the producer adds
    one partial (bias, LN, unsplit GEMMs), (acc + h0) + h1 instead of
    acc + (h0 + h1) for split-K GEMMs; deterministic either way.  T = 1024
    tokens per microbatch so both kinds of weight GEMM occur."""
    from paper_2412_14374_b200.executor import PipelineEngine
    cfg = I.GPTConfig(layers=4, d_model=128, n_heads=2, d_ff=512, vocab=256, seq_len=256,
                      microbatch_size=4, yields=(3,), yield_every=6, elem_bytes=2)
    p, tg, cp = plan(cfg, "1f1b", 2, 4)
    oc = oracle_cfg(cfg)
    rng = np.random.default_rng(11)
    params = {q: v.astype(np.float32) for q, v in gpt.init_params(oc, rng, std=0.05).items()}
    tokens = gpt.init_tokens(oc, 4, rng).reshape(16, 256)
    out = []
    for fuse in (True, False, True):
        eng = PipelineEngine(cp, tg, mode="bf16", gpt=cfg)
        for ops in eng._ops.values():
            ops.fuse_acc = fuse
        out.append(eng.step(params, tokens))
        eng.close()
    a, b, c = out
    assert np.array_equal(a.losses, b.losses)
    for q in a.grads:
        assert ffn.rel(a.grads[q], b.grads[q]) < 1e-6, (q, ffn.rel(a.grads[q], b.grads[q]))
        assert np.array_equal(a.grads[q], c.grads[q]), q


@pytest.mark.parametrize("mode,fam,P,M,yields", [("bf16", "1f1b", 2, 4, (3,)),
                                                 ("fp32", "gpipe", 2, 4, (3,)),
                                                 ("bf16", "1f1b", 4, 8, (2, 3, 5))])
def test_full_remat_replays_the_forward_bitwise(mode, fam, P, M, yields):
    """remat="full-per-stage" (the reference simulator's policy,
    simulator.py:132-149, made real): each stage keeps only its forward feeds
    and replays the forward inside the backward task.  Deterministic kernels
    make every gradient, loss and updated parameter bitwise equal to the
    stashing run, with less stash memory per actor."""
    from paper_2412_14374_b200.executor import ExecutorFault, PipelineEngine
    cfg = I.GPTConfig(**TINY, yields=yields, yield_every=TINY["layers"] + 2,
                      elem_bytes=2 if mode == "bf16" else 4)
    _, tg, cp = plan(cfg, fam, P, M)
    oc = oracle_cfg(cfg)
    rng = np.random.default_rng(5)
    params = {q: v.astype(np.float32) for q, v in gpt.init_params(oc, rng, std=0.05).items()}
    tokens = gpt.init_tokens(oc, M, rng).reshape(M * cfg.microbatch_size, cfg.seq_len)
    a = run_pipelined(cp, tg, params, tokens, mode=mode, gpt=cfg)
    b = run_pipelined(cp, tg, params, tokens, mode=mode, gpt=cfg, remat="full-per-stage")
    assert np.array_equal(a.losses, b.losses)
    for q in a.grads:
        assert np.array_equal(a.grads[q], b.grads[q]), q
        assert np.array_equal(a.new_params[q], b.new_params[q]), q
    for actor in range(P):
        assert b.stats.peak_stash_bytes[actor] < a.stats.peak_stash_bytes[actor], actor
    with pytest.raises(ExecutorFault):
        PipelineEngine(cp, tg, mode=mode, gpt=cfg, remat="selective")


@pytest.mark.parametrize("d", [256, 768, 1024])
@pytest.mark.parametrize("dt,tol", [(torch.float32, 1e-5), (torch.bfloat16, 2e-2)])
def test_layernorm_bwd_partials_then_col_sum(d, dt, tol):
    """pc_layernorm_bwd_partials (dx plus per-CTA partial rows of dgamma / dbeta in
    one read of dy and x) followed by pc_col_sum over the partial rows equals the
    oracle's LayerNorm backward; deterministic across runs."""
    rows = 8192 if d == 768 else 300
    rng = np.random.default_rng(9)
    x = rng.standard_normal((rows, d))
    g, b = rng.standard_normal(d), rng.standard_normal(d)
    dy = rng.standard_normal((rows, d))
    res = rng.standard_normal((rows, d))
    tx, tdy, tres = _t(x, dt), _t(dy, dt), _t(res, dt)
    xq, dyq, resq = (t.double().cpu().numpy() for t in (tx, tdy, tres))
    y, cache = gpt.layer_norm(xq, g, b)
    dx, dg, db = gpt.layer_norm_bwd(dyq, g, cache)
    tg_, tb = _t(g), _t(b)
    ty = torch.empty_like(tx)
    mean, rstd = torch.empty(rows, device="cuda"), torch.empty(rows, device="cuda")
    pc = _lib.PC_F32 if dt == torch.float32 else _lib.PC_BF16
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("pc_layernorm_fwd", pc, rows, d, tx.data_ptr(), tg_.data_ptr(), tb.data_ptr(),
              ty.data_ptr(), mean.data_ptr(), rstd.data_ptr(), 1e-5, st)
    n = ctypes.c_int64()
    _lib.call("pc_layernorm_partial_rows", rows, d, ctypes.byref(n))
    nb = ctypes.c_int64()
    _lib.call("pc_reduce_workspace_bytes", n.value, d, ctypes.byref(nb))
    ws = torch.zeros(nb.value, dtype=torch.uint8, device="cuda")
    outs = []
    for _ in range(2):
        parts = torch.empty(2 * n.value * d, device="cuda")
        tdx = torch.empty_like(tx)
        _lib.call("pc_layernorm_bwd_partials", pc, rows, d, tdy.data_ptr(), tx.data_ptr(),
                  tg_.data_ptr(), mean.data_ptr(), rstd.data_ptr(), tres.data_ptr(),
                  tdx.data_ptr(), parts.data_ptr(), n.value, st)
        tdg = torch.full((d,), 0.25, device="cuda")
        tdb = torch.empty(d, device="cuda")
        _lib.call("pc_col_sum", _lib.PC_F32, _lib.PC_F32, n.value, d, parts.data_ptr(), d,
                  tdg.data_ptr(), 1, ws.data_ptr(), nb.value, st)
        _lib.call("pc_col_sum", _lib.PC_F32, _lib.PC_F32, n.value, d,
                  parts[n.value * d:].data_ptr(), d, tdb.data_ptr(), 0, ws.data_ptr(), nb.value, st)
        outs.append((tdx, tdg, tdb))
    torch.cuda.synchronize()
    tdx, tdg, tdb = outs[0]
    assert ffn.rel(tdx.double().cpu().numpy(), dx + resq) < tol
    assert ffn.rel(tdg.cpu().numpy(), dg + 0.25) < 1e-5
    assert ffn.rel(tdb.cpu().numpy(), db) < 1e-5
    for a, c in zip(outs[0], outs[1]):
        assert torch.equal(a, c)


@pytest.mark.parametrize("dt,pc", [(torch.float64, "PC_F64"), (torch.float32, "PC_F32"),
                                   (torch.bfloat16, "PC_BF16")])
def test_copy2d_zero_source_stride_broadcasts(dt, pc):
    """pc_copy2d with lds = 0 repeats a row (the generic vocabulary's `broadcast`
    of a [n] value to [m, n], executor.py:78-95) and a scalar (cols = 1), one launch."""
    st = torch.cuda.current_stream().cuda_stream
    row = torch.randn(37, device="cuda").to(dt)
    out = torch.empty(5, 37, device="cuda", dtype=dt)
    _lib.call("pc_copy2d", getattr(_lib, pc), 5, 37, row.data_ptr(), 0, 0, out.data_ptr(), 37, st)
    one = torch.randn(1, device="cuda").to(dt)
    out2 = torch.empty(3, 4, device="cuda", dtype=dt)
    _lib.call("pc_copy2d", getattr(_lib, pc), 12, 1, one.data_ptr(), 0, 0, out2.data_ptr(), 1, st)
    torch.cuda.synchronize()
    assert torch.equal(out, row.expand(5, 37))
    assert torch.equal(out2, one.expand(3, 4))
