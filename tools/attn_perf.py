"""Time pc_attention_fwd/bwd (tensor-core vs SIMT) on GPT-2-small shapes."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2412_14374_b200 import _lib

def bench(fn, iters=10):
    for _ in range(2): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters

for (B, H, S, hd) in [(8, 12, 1024, 64), (4, 16, 2048, 128), (8, 16, 1024, 64)]:
    d = H * hd
    qkv = (torch.randn(B * S, 3 * d, device="cuda") * 0.5).bfloat16()
    o = torch.empty(B * S, d, device="cuda", dtype=torch.bfloat16)
    do = torch.randn(B * S, d, device="cuda").bfloat16()
    dqkv = torch.empty_like(qkv)
    lse = torch.empty(B * H * S, device="cuda"); delta = torch.empty_like(lse)
    st = torch.cuda.current_stream().cuda_stream
    f = lambda: _lib.call("pc_attention_fwd", 2, B, H, S, hd, qkv.data_ptr(), 3 * d, o.data_ptr(), d, lse.data_ptr(), st)
    b = lambda: _lib.call("pc_attention_bwd", 2, B, H, S, hd, qkv.data_ptr(), 3 * d, o.data_ptr(), do.data_ptr(), d, lse.data_ptr(), delta.data_ptr(), dqkv.data_ptr(), 3 * d, st)
    flops_f = 4 * B * H * S * S * hd / 2  # causal
    for impl in (0, 2):
        _lib.call("pc_attention_set_impl", impl)
        tf = bench(f, 20); tb = bench(b, 20)
        print(f"B{B} H{H} S{S} hd{hd} {['tcgen05', 'simt', 'mma.sync'][impl]}: fwd {tf:.3f} ms ({flops_f/tf/1e9:.0f} TF/s) bwd {tb:.3f} ms ({2.5*flops_f/tb/1e9:.0f} TF/s eq)", flush=True)
    _lib.call("pc_attention_set_impl", 0)
    # flash (sdpa) reference timing
    q = qkv[:, :d].view(B, S, H, hd).transpose(1, 2); k = qkv[:, d:2*d].view(B, S, H, hd).transpose(1, 2); v = qkv[:, 2*d:].view(B, S, H, hd).transpose(1, 2)
    g = lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
    print(f"   torch sdpa fwd {bench(g):.3f} ms", flush=True)
