"""One launch each of pc_gemm (BN=256 single-CTA, BN=256 CTA pair) and cuBLAS
on one C2 GEMM shape, for a side-by-side `ncu --set full` capture.
usage: python tools/ncu_gemm_cmp.py M N K transA transB"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2412_14374_b200 import _lib

M, N, K, ta, tb = (int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (8192, 2304, 768, 0, 1)))
A = torch.randn((K, M) if ta else (M, K), device="cuda").bfloat16()
B = torch.randn((N, K) if tb else (K, N), device="cuda").bfloat16()
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream
opA = A.t() if ta else A
opB = B.t() if tb else B
for bn, pair in ((256, 1), (256, 2), (192, 1)):
    _lib.call("pc_gemm_set_tile_n", bn)
    _lib.call("pc_gemm_set_cta_pair", pair)
    for _ in range(2):
        _lib.call("pc_gemm", 2, 2, ta, tb, M, N, K, A.data_ptr(), A.stride(0), B.data_ptr(),
                  B.stride(0), C.data_ptr(), C.stride(0), 0, None, None, 0, None, 0, st)
for _ in range(2):
    torch.matmul(opA, opB, out=C)
torch.cuda.synchronize()
print("ok")
