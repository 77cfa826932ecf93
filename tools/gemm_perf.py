"""Time pc_gemm (tcgen05 bf16) on the GPT-2-small stage shapes vs torch.matmul (cuBLAS)."""
import sys
import pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2412_14374_b200 import _lib

SHAPES = [  # (name, M, N, K, transA, transB)
    ("fwd qkv", 8192, 2304, 768, 0, 1),
    ("fwd fc1", 8192, 3072, 768, 0, 1),
    ("fwd fc2", 8192, 768, 3072, 0, 1),
    ("dgrad fc1", 8192, 768, 3072, 0, 0),
    ("wgrad qkv", 2304, 768, 8192, 1, 0),
    ("wgrad fc2", 768, 3072, 8192, 1, 0),
    ("head fwd", 8192, 50304, 768, 0, 1),
    ("sq 8192", 8192, 8192, 8192, 0, 1),
    ("dgrad qkv", 8192, 768, 2304, 0, 0),
    ("wgrad fc1", 3072, 768, 8192, 1, 0),
]
VARIANTS = [("auto", 0, 0), ("192", 192, 1), ("256", 256, 1), ("128", 128, 1),
            ("p128", 128, 2), ("p192", 192, 2), ("p256", 256, 2)]


def bench(fn, iters=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


for name, M, N, K, ta, tb in SHAPES:
    A = torch.randn((K, M) if ta else (M, K), device="cuda").bfloat16()
    B = torch.randn((N, K) if tb else (K, N), device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream
    f = lambda: _lib.call("pc_gemm", 2, 2, ta, tb, M, N, K, A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0), C.data_ptr(), C.stride(0), 0, None, None, 0, None, 0, st)
    opA = A.t() if ta else A
    opB = B.t() if tb else B
    g = lambda: torch.matmul(opA, opB, out=C)
    res = {}
    for tag, bn, pair in VARIANTS:
        _lib.call("pc_gemm_set_tile_n", bn)
        _lib.call("pc_gemm_set_cta_pair", pair)
        ms = bench(f)
        res[tag] = 2 * M * N * K / ms / 1e9
    _lib.call("pc_gemm_set_tile_n", 0)
    _lib.call("pc_gemm_set_cta_pair", 0)
    if ta:  # weight gradients run with fp32 output and the split-K hint in the step
        C32 = torch.zeros(M, N, device="cuda", dtype=torch.float32)
        h = lambda: _lib.call("pc_gemm", 2, 0, ta, tb, M, N, K, A.data_ptr(), A.stride(0),
                              B.data_ptr(), B.stride(0), C32.data_ptr(), C32.stride(0),
                              _lib.EPI_SPLITK_ZERO_C, None, None, 0, None, 0, st)
        res["prod-f32-splitk"] = 2 * M * N * K / bench(h) / 1e9
    ref = 2 * M * N * K / bench(g) / 1e9
    print(f"{name:12s} M={M} N={N} K={K} ta={ta} tb={tb}: pp200 TFLOP/s " +
          " ".join(f"{k}={v:.0f}" for k, v in res.items()) + f" | cuBLAS {ref:.0f}", flush=True)
