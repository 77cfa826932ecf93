"""pc_col_sum (bias-gradient column sums) on the C2 shapes: time and GB/s."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import ctypes
import torch
from paper_2412_14374_b200 import _lib

T = 8192
for N in (768, 2304, 3072):
    x = torch.randn(T, N, device="cuda").bfloat16()
    out = torch.empty(N, device="cuda")
    nb = ctypes.c_int64()
    _lib.call("pc_reduce_workspace_bytes", T, N, ctypes.byref(nb))
    ws = torch.zeros(nb.value, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    f = lambda: _lib.call("pc_col_sum", _lib.PC_BF16, _lib.PC_F32, T, N, x.data_ptr(), N,
                          out.data_ptr(), 0, ws.data_ptr(), nb.value, st)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    ref = x.float().sum(0)
    err = (out - ref).abs().max().item()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(50):
        f()
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / 50 * 1e3
    print(f"col_sum [{T} x {N}] bf16: {us:.1f} us  {T * N * 2 / us / 1e3:.0f} GB/s  maxerr {err:.2e}")
