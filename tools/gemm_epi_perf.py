"""The fused-epilogue GEMMs of one GPT block as the step issues them (bias+GELU
with the pre-activation stored, bias+residual, GELU-derivative from the stored
pre-activation), vs the same GEMM with a plain epilogue."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2412_14374_b200 import _lib

T, d, f = 8192, 768, 3072


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
    return s.elapsed_time(e) / iters * 1e3


st = torch.cuda.current_stream().cuda_stream
cases = [  # name, M, N, K, ta, tb, epi, (aux?), (aux_out?)
    ("fc1 fwd bias+gelu+U", T, f, d, 0, 1, _lib.EPI_BIAS | _lib.EPI_GELU, False, True),
    ("fc2 fwd bias+resid", T, d, f, 0, 1, _lib.EPI_BIAS | _lib.EPI_RESIDUAL, True, False),
    ("out fwd bias+resid", T, d, d, 0, 1, _lib.EPI_BIAS | _lib.EPI_RESIDUAL, True, False),
    ("fc1 dgrad gelu'", T, f, d, 0, 0, _lib.EPI_GELU_GRAD, True, False),
]
for name, M, N, K, ta, tb, epi, has_aux, has_u in cases:
    A = torch.randn((K, M) if ta else (M, K), device="cuda").bfloat16()
    B = torch.randn((N, K) if tb else (K, N), device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    aux = torch.randn(M, N, device="cuda").bfloat16() if has_aux else None
    U = torch.empty(M, N, device="cuda", dtype=torch.bfloat16) if has_u else None
    bias = torch.randn(N, device="cuda")
    def run(e):
        _lib.call("pc_gemm", 2, 2, ta, tb, M, N, K, A.data_ptr(), A.stride(0), B.data_ptr(),
                  B.stride(0), C.data_ptr(), N, e, bias.data_ptr(),
                  aux.data_ptr() if aux is not None else None, N,
                  U.data_ptr() if U is not None else None, N, st)
    out = []
    for ab in (0, 1, 4):
        _lib.call("pc_gemm_set_ablation", ab)
        out.append((bench(lambda: run(epi)), bench(lambda: run(0))))
    _lib.call("pc_gemm_set_ablation", 0)
    fl = 2.0 * M * N * K
    (fe, fp), (ne, np_), (xe, _) = out
    print(f"{name:22s} fused {fe:6.1f} us ({fl / fe / 1e6:5.0f} TF/s)  plain {fp:6.1f} us  "
          f"| no-epi: fused {ne:6.1f}  plain {np_:6.1f} | no aux loads: fused {xe:6.1f}", flush=True)
