"""The dominant kernel (tcgen05 GEMM) on the C2 fc1 forward shape with its
bias+GELU epilogue, for one ncu --set full capture."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2412_14374_b200 import _lib
M, N, K = 8192, 3072, 768
A = torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(N, K, device="cuda").bfloat16()
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
U = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
bias = torch.zeros(N, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    _lib.call("pc_gemm", 2, 2, 0, 1, M, N, K, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N,
              _lib.EPI_BIAS | _lib.EPI_GELU, bias.data_ptr(), None, 0, U.data_ptr(), N, st)
torch.cuda.synchronize()
print("ok")
