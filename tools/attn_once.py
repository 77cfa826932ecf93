"""One forward + backward of the tcgen05 attention at a BASELINE shape (for an
`ncu --set full` capture of exactly those kernels).
usage: python tools/attn_once.py C2|C3|C4|C5"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2412_14374_b200 import _lib

SHAPES = {"C2": (8, 12, 12, 1024, 64), "C3": (8, 16, 16, 1024, 64), "C4": (4, 16, 16, 2048, 128),
          "C5": (1, 32, 8, 4096, 128)}
B, H, Hkv, S, hd = SHAPES[sys.argv[1] if len(sys.argv) > 1 else "C5"]
ld = (H + 2 * Hkv) * hd
qkv = (torch.randn(B * S, ld, device="cuda") * 0.5).bfloat16()
do = torch.randn(B * S, H * hd, device="cuda").bfloat16()
o = torch.empty(B * S, H * hd, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B * H * S, device="cuda")
delta = torch.empty_like(lse)
dqkv = torch.empty_like(qkv)
st = torch.cuda.current_stream().cuda_stream
_lib.call("pc_attention_gqa_fwd", 2, B, H, Hkv, S, hd, qkv.data_ptr(), ld, o.data_ptr(), H * hd, lse.data_ptr(), st)
_lib.call("pc_attention_gqa_bwd", 2, B, H, Hkv, S, hd, qkv.data_ptr(), ld, o.data_ptr(), do.data_ptr(), H * hd,
          lse.data_ptr(), delta.data_ptr(), dqkv.data_ptr(), ld, st)
torch.cuda.synchronize()
print("ok", sys.argv[1:] or ["C5"])
