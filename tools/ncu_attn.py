"""C2 attention shapes (B=8, H=12, S=1024, hd=64): fwd + bwd, for ncu captures."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2412_14374_b200 import _lib
B, H, S, hd = 8, 12, 1024, 64
d = H * hd
qkv = (torch.randn(B * S, 3 * d, device="cuda") * 0.5).bfloat16()
o = torch.empty(B * S, d, device="cuda", dtype=torch.bfloat16)
do = torch.randn(B * S, d, device="cuda").bfloat16()
dqkv = torch.empty_like(qkv)
lse = torch.empty(B * H * S, device="cuda"); delta = torch.empty_like(lse)
st = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    _lib.call("pc_attention_fwd", 2, B, H, S, hd, qkv.data_ptr(), 3 * d, o.data_ptr(), d, lse.data_ptr(), st)
    _lib.call("pc_attention_bwd", 2, B, H, S, hd, qkv.data_ptr(), 3 * d, o.data_ptr(), do.data_ptr(), d, lse.data_ptr(), delta.data_ptr(), dqkv.data_ptr(), 3 * d, st)
torch.cuda.synchronize()
print("ok")
