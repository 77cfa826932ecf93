"""Device time (CUDA-graph replay, warm) of the HBM-bound C2 kernels at their
step shapes, against the bytes they must move: LayerNorm fwd / bwd, bias
column sums, cross-entropy.  usage: python tools/hbm_kernels_perf.py"""
import ctypes
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from paper_2412_14374_b200 import _lib  # noqa: E402

T, d, f, V, S = 8192, 768, 3072, 50304, 1024
st = torch.cuda.Stream()
peak = json.loads((pathlib.Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())


def timed(fn, reps=10):
    with torch.cuda.stream(st):
        for _ in range(2):
            fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                fn()
        g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.replay()
        e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


bf = torch.bfloat16
dev = "cuda"
x = torch.randn(T, d, device=dev).to(bf)
y = torch.empty_like(x)
dy = torch.randn(T, d, device=dev).to(bf)
dx = torch.empty_like(x)
g_ = torch.ones(d, device=dev)
b_ = torch.zeros(d, device=dev)
mean = torch.empty(T, device=dev)
rstd = torch.empty(T, device=dev)
dg = torch.zeros(d, device=dev)
db = torch.zeros(d, device=dev)
nb = ctypes.c_int64()
_lib.call("pc_reduce_workspace_bytes", T, f, ctypes.byref(nb))
ws = torch.zeros(nb.value, dtype=torch.uint8, device=dev)
s = st.cuda_stream
rows = []
us = timed(lambda: _lib.call("pc_layernorm_fwd", _lib.PC_BF16, T, d, x.data_ptr(), g_.data_ptr(),
                             b_.data_ptr(), y.data_ptr(), mean.data_ptr(), rstd.data_ptr(), 1e-5, s))
rows.append(("layernorm_fwd [8192,768]", us, 2 * T * d * 2 + 8 * T))
for cl in (0, 1):  # pc_colsum_set_cluster A/B: two-stage workspace vs one-pass cluster
    _lib.call("pc_colsum_set_cluster", cl)
    tag = "cluster" if cl else "2-stage"
    dg.zero_(); db.zero_()
    us = timed(lambda: _lib.call("pc_layernorm_bwd_acc", _lib.PC_BF16, T, d, dy.data_ptr(), x.data_ptr(),
                                 g_.data_ptr(), mean.data_ptr(), rstd.data_ptr(), dy.data_ptr(),
                                 dx.data_ptr(), dg.data_ptr(), db.data_ptr(), 1, ws.data_ptr(),
                                 ws.numel(), s))
    rows.append((f"layernorm_bwd(+params) [8192,768] {tag}", us, 4 * T * d * 2 + 8 * T))
    for n in (768, 2304, 3072):
        torch.manual_seed(n)
        a = torch.randn(T, n, device=dev).to(bf)
        out = torch.zeros(n, device=dev)
        us = timed(lambda: _lib.call("pc_col_sum", _lib.PC_BF16, _lib.PC_F32, T, n, a.data_ptr(), n,
                                     out.data_ptr(), 1, ws.data_ptr(), ws.numel(), s))
        out.zero_()
        _lib.call("pc_col_sum", _lib.PC_BF16, _lib.PC_F32, T, n, a.data_ptr(), n, out.data_ptr(), 0,
                  ws.data_ptr(), ws.numel(), s)
        torch.cuda.synchronize()
        ref = a.double().sum(0)
        err = float((out.double() - ref).abs().max() / ref.abs().max())
        rows.append((f"bias col_sum [8192,{n}] {tag} (rel err {err:.1e})", us, T * n * 2))
_lib.call("pc_colsum_set_cluster", 1)
# a GPT block's LN2 side-stream sums: dgamma / dbeta + the fc2 / attention-output bias sums,
# three launches (param grads + two column sums) vs one four-sum pass
y3 = torch.randn(T, d, device=dev).to(bf)
y4 = torch.randn(T, d, device=dev).to(bf)
s3, s4 = torch.zeros(d, device=dev), torch.zeros(d, device=dev)
mean.normal_(0, 0.1)
rstd.uniform_(0.5, 1.5)


def three():
    _lib.call("pc_layernorm_param_grads", _lib.PC_BF16, T, d, dy.data_ptr(), x.data_ptr(),
              mean.data_ptr(), rstd.data_ptr(), dg.data_ptr(), db.data_ptr(), 1, ws.data_ptr(),
              ws.numel(), s)
    for yy, ss in ((y3, s3), (y4, s4)):
        _lib.call("pc_col_sum", _lib.PC_BF16, _lib.PC_F32, T, d, yy.data_ptr(), d, ss.data_ptr(), 1,
                  ws.data_ptr(), ws.numel(), s)


us = timed(three)
rows.append(("LN2 params + 2 bias col_sums [8192,768], 3 launches", us, 4 * T * d * 2 + 8 * T))
us = timed(lambda: _lib.call("pc_layernorm_param_bias_grads", T, d, dy.data_ptr(), x.data_ptr(),
                             mean.data_ptr(), rstd.data_ptr(), dg.data_ptr(), db.data_ptr(),
                             y3.data_ptr(), s3.data_ptr(), y4.data_ptr(), s4.data_ptr(), 1, s))
rows.append(("LN2 params + 2 bias col_sums [8192,768], one pass", us, 4 * T * d * 2 + 8 * T))
logits = torch.randn(T, V, device=dev).to(bf)
tok = torch.randint(0, V, (T,), device=dev, dtype=torch.int32)
rl = torch.empty(T, device=dev)
us = timed(lambda: _lib.call("pc_xent_fwd_bwd", _lib.PC_BF16, T, V, S, logits.data_ptr(), V,
                             tok.data_ptr(), rl.data_ptr(), s), reps=3)
rows.append(("xent fwd+bwd [8192,50304]", us, 2 * T * V * 2))
hbm = peak.get("hbm_gbs", 6546.2)
for name, us, by in rows:
    print(f"{name:56s} {us:8.1f} us  {by / us / 1e3:7.0f} GB/s  ({by / us / 1e3 / hbm:.2f} of {hbm:.0f})")
