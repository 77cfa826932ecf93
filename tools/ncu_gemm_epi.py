"""One fc1-forward GEMM with the bias+GELU epilogue and stored pre-activation
(C2 shape 8192x3072x768), then the same GEMM plain, for an ncu --set full capture."""
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
for epi, u in ((_lib.EPI_BIAS | _lib.EPI_GELU, U), (_lib.EPI_BIAS, None)):
    for _ in range(2):
        _lib.call("pc_gemm", 2, 2, 0, 1, M, N, K, A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N,
                  epi, bias.data_ptr(), None, 0, u.data_ptr() if u is not None else None, N, st)
torch.cuda.synchronize()
print("ok")
