"""One fwd + bwd of the tcgen05 attention at a BASELINE shape, for ncu captures:
    python tools/ncu_attn.py [C2|C5]"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2412_14374_b200 import _lib
SH = {"C2": (8, 12, 12, 1024, 64), "C4": (4, 16, 16, 2048, 128), "C5": (1, 32, 8, 4096, 128)}
B, H, Hkv, S, hd = SH[sys.argv[1] if len(sys.argv) > 1 else "C2"]
dq_, dkv = H * hd, Hkv * hd
ld = dq_ + 2 * dkv
qkv = (torch.randn(B * S, ld, device="cuda") * 0.5).bfloat16()
o = torch.empty(B * S, dq_, device="cuda", dtype=torch.bfloat16)
do = torch.randn(B * S, dq_, device="cuda").bfloat16()
dqkv = torch.empty_like(qkv)
lse = torch.empty(B * H * S, device="cuda"); delta = torch.empty_like(lse)
st = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    _lib.call("pc_attention_gqa_fwd", 2, B, H, Hkv, S, hd, qkv.data_ptr(), ld, o.data_ptr(), dq_, lse.data_ptr(), st)
    _lib.call("pc_attention_gqa_bwd", 2, B, H, Hkv, S, hd, qkv.data_ptr(), ld, o.data_ptr(), do.data_ptr(), dq_,
              lse.data_ptr(), delta.data_ptr(), dqkv.data_ptr(), ld, st)
torch.cuda.synchronize()
print("ok")
