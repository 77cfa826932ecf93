"""Time the attention kernels (pc_attention_gqa_fwd/bwd) at the BASELINE shapes.

For each shape: the tcgen05 kernels, and for comparison the mma.sync kernels
(head_dim 64/128 multi-head; grouped-query heads through the old expand ->
multi-head -> group-sum path, pc_gqa_kv).  FLOPs: causal forward 2 GEMMs of
B*H*S^2/2*hd each (4 B H S^2 hd / 2), backward 2.5x forward (FA convention:
dV, dP, dQ, dK plus half a recompute of S).  CUDA events on the launch
stream, 20 back-to-back launches after warm-up.
"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import json
import torch
from paper_2412_14374_b200 import _lib


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


SHAPES = [("C2", 8, 12, 12, 1024, 64), ("C3", 8, 16, 16, 1024, 64),
          ("C4", 4, 16, 16, 2048, 128), ("C5", 1, 32, 8, 4096, 128)]
rows = []
st = torch.cuda.current_stream().cuda_stream
for (name, B, H, Hkv, S, hd) in SHAPES:
    dq_, dkv = H * hd, Hkv * hd
    ld = dq_ + 2 * dkv
    qkv = (torch.randn(B * S, ld, device="cuda") * 0.5).bfloat16()
    o = torch.empty(B * S, dq_, device="cuda", dtype=torch.bfloat16)
    do = torch.randn(B * S, dq_, device="cuda").bfloat16()
    dqkv = torch.empty_like(qkv)
    lse = torch.empty(B * H * S, device="cuda")
    delta = torch.empty_like(lse)
    flops_f = 4.0 * B * H * S * S * hd / 2
    f = lambda: _lib.call("pc_attention_gqa_fwd", 2, B, H, Hkv, S, hd, qkv.data_ptr(), ld,
                          o.data_ptr(), dq_, lse.data_ptr(), st)
    b = lambda: _lib.call("pc_attention_gqa_bwd", 2, B, H, Hkv, S, hd, qkv.data_ptr(), ld,
                          o.data_ptr(), do.data_ptr(), dq_, lse.data_ptr(), delta.data_ptr(),
                          dqkv.data_ptr(), ld, st)
    tf, tb = bench(f), bench(b)
    row = dict(shape=name, B=B, H=H, Hkv=Hkv, S=S, hd=hd, impl="tcgen05",
               fwd_ms=round(tf, 4), fwd_tflops=round(flops_f / tf / 1e9, 1),
               bwd_ms=round(tb, 4), bwd_tflops=round(2.5 * flops_f / tb / 1e9, 1))
    rows.append(row)
    print(json.dumps(row), flush=True)
    # legacy mma.sync kernels (expanded heads for GQA)
    _lib.call("pc_attention_set_impl", 2)
    try:
        if Hkv != H:
            T = B * S
            ex = torch.empty(T, 3 * dq_, device="cuda", dtype=torch.bfloat16)
            dex = torch.empty_like(ex)

            def f2():
                _lib.call("pc_gqa_kv", 2, T, H, Hkv, hd, qkv.data_ptr(), ld, ex.data_ptr(), 3 * dq_, 0, st)
                _lib.call("pc_attention_fwd", 2, B, H, S, hd, ex.data_ptr(), 3 * dq_, o.data_ptr(), dq_,
                          lse.data_ptr(), st)

            def b2():
                _lib.call("pc_attention_bwd", 2, B, H, S, hd, ex.data_ptr(), 3 * dq_, o.data_ptr(),
                          do.data_ptr(), dq_, lse.data_ptr(), delta.data_ptr(), dex.data_ptr(), 3 * dq_, st)
                _lib.call("pc_gqa_kv", 2, T, H, Hkv, hd, dex.data_ptr(), 3 * dq_, dqkv.data_ptr(), ld, 1, st)
        else:
            f2 = lambda: _lib.call("pc_attention_fwd", 2, B, H, S, hd, qkv.data_ptr(), ld, o.data_ptr(),
                                   dq_, lse.data_ptr(), st)
            b2 = lambda: _lib.call("pc_attention_bwd", 2, B, H, S, hd, qkv.data_ptr(), ld, o.data_ptr(),
                                   do.data_ptr(), dq_, lse.data_ptr(), delta.data_ptr(), dqkv.data_ptr(),
                                   ld, st)
        tf2, tb2 = bench(f2), bench(b2)
    finally:
        _lib.call("pc_attention_set_impl", 0)
    row2 = dict(shape=name, impl="mma.sync" + (" + gqa expand/reduce" if Hkv != H else ""),
                fwd_ms=round(tf2, 4), fwd_tflops=round(flops_f / tf2 / 1e9, 1),
                bwd_ms=round(tb2, 4), bwd_tflops=round(2.5 * flops_f / tb2 / 1e9, 1),
                speedup_fwd=round(tf2 / tf, 2), speedup_bwd=round(tb2 / tb, 2))
    rows.append(row2)
    print(json.dumps(row2), flush=True)
    del qkv, o, do, dqkv
    torch.cuda.empty_cache()
