"""A/B the head_dim-64 attention kernel variants (pc_attention_tune) at the
C2 / C3 shapes: time (CUDA events, 20 back-to-back launches) and agreement
with the legacy design (max |o - o_ref|, max |lse - lse_ref|).
usage: python tools/attn_ab.py [fwd|bwd|all] [design,emu ...]  (default: all variants)
       python tools/attn_ab.py fwd128   (head_dim 128 forward, C4 / C5: one vs two issuing warps)
       python tools/attn_ab.py dqsplit  (backward, C2-C5: dQ kernel with one vs two issuing warps)"""
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


def fwd128():
    st = torch.cuda.current_stream().cuda_stream
    torch.manual_seed(0)
    for (name, B, H, Hkv, S) in [("C4", 4, 16, 16, 2048), ("C5", 1, 32, 8, 4096)]:
        hd = 128
        ld = (H + 2 * Hkv) * hd
        qkv = (torch.randn(B * S, ld, device="cuda") * 0.5).bfloat16()
        flops = 4.0 * B * H * S * S * hd / 2
        ref = None
        for split in (0, 1, 0, 1, 0, 1):
            _lib.call("pc_attention_tune", 2, split)
            o = torch.empty(B * S, H * hd, device="cuda", dtype=torch.bfloat16)
            lse = torch.empty(B * H * S, device="cuda")

            def run():
                _lib.call("pc_attention_gqa_fwd", 2, B, H, Hkv, S, hd, qkv.data_ptr(), ld, o.data_ptr(), H * hd,
                          lse.data_ptr(), st)
            run()
            torch.cuda.synchronize()
            t = bench(run)
            row = dict(shape=name, split=split, fwd_us=round(t * 1e3, 2), fwd_tflops=round(flops / t / 1e9, 1))
            if ref is None:
                ref = (o.clone(), lse.clone())
            else:
                row.update(o_maxdiff=float((o.float() - ref[0].float()).abs().max()),
                           lse_maxdiff=float((lse - ref[1]).abs().max()))
            print(json.dumps(row), flush=True)
    _lib.call("pc_attention_tune", 2, 1)


def dqsplit():
    st = torch.cuda.current_stream().cuda_stream
    torch.manual_seed(0)
    for (name, B, H, Hkv, S, hd) in [("C2", 8, 12, 12, 1024, 64), ("C3", 8, 16, 16, 1024, 64),
                                     ("C4", 4, 16, 16, 2048, 128), ("C5", 1, 32, 8, 4096, 128)]:
        ld = (H + 2 * Hkv) * hd
        qkv = (torch.randn(B * S, ld, device="cuda") * 0.5).bfloat16()
        do = torch.randn(B * S, H * hd, device="cuda").bfloat16()
        o = torch.empty(B * S, H * hd, device="cuda", dtype=torch.bfloat16)
        lse = torch.empty(B * H * S, device="cuda")
        _lib.call("pc_attention_gqa_fwd", 2, B, H, Hkv, S, hd, qkv.data_ptr(), ld, o.data_ptr(), H * hd,
                  lse.data_ptr(), st)
        flops = 2.5 * 4.0 * B * H * S * S * hd / 2
        ref = None
        for split in (0, 1, 0, 1, 0, 1):
            _lib.call("pc_attention_tune", 3, split)
            delta = torch.empty_like(lse)
            dqkv = torch.zeros_like(qkv)

            def run():
                _lib.call("pc_attention_gqa_bwd", 2, B, H, Hkv, S, hd, qkv.data_ptr(), ld, o.data_ptr(),
                          do.data_ptr(), H * hd, lse.data_ptr(), delta.data_ptr(), dqkv.data_ptr(), ld, st)
            run()
            torch.cuda.synchronize()
            t = bench(run)
            row = dict(shape=name, dq_split=split, bwd_us=round(t * 1e3, 2), bwd_tflops=round(flops / t / 1e9, 1))
            if ref is None:
                ref = dqkv.clone()
            else:
                row.update(bitwise=bool(torch.equal(dqkv, ref)))
            print(json.dumps(row), flush=True)
    _lib.call("pc_attention_tune", 3, 1)


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what == "fwd128":
        return fwd128()
    if what == "dqsplit":
        return dqsplit()
    st = torch.cuda.current_stream().cuda_stream
    torch.manual_seed(0)
    for (name, B, H, S) in [("C2", 8, 12, 1024), ("C3", 8, 16, 1024), ("C2-S1000", 8, 12, 1000)]:
        hd = 64
        ld = 3 * H * hd
        qkv = (torch.randn(B * S, ld, device="cuda") * 0.5).bfloat16()
        do = torch.randn(B * S, H * hd, device="cuda").bfloat16()
        flops_f = 4.0 * B * H * S * S * hd / 2

        def run_fwd(o, lse):
            _lib.call("pc_attention_gqa_fwd", 2, B, H, H, S, hd, qkv.data_ptr(), ld, o.data_ptr(), H * hd,
                      lse.data_ptr(), st)

        def run_bwd(o, lse, delta, dqkv):
            _lib.call("pc_attention_gqa_bwd", 2, B, H, H, S, hd, qkv.data_ptr(), ld, o.data_ptr(),
                      do.data_ptr(), H * hd, lse.data_ptr(), delta.data_ptr(), dqkv.data_ptr(), ld, st)

        variants = [(1, 0), (2, 6), (3, 6), (2, 101), (3, 101)]
        if len(sys.argv) > 2:
            variants = [tuple(int(x) for x in a.split(",")) for a in sys.argv[2:]]
        ref = None
        for (design, emu) in variants:
            _lib.call("pc_attention_tune", 0, design)
            _lib.call("pc_attention_tune", 1, emu)
            o = torch.empty(B * S, H * hd, device="cuda", dtype=torch.bfloat16)
            lse = torch.empty(B * H * S, device="cuda")
            run_fwd(o, lse)
            torch.cuda.synchronize()
            row = dict(shape=name, design=design, emu=emu)
            if what in ("fwd", "all"):
                t = bench(lambda: run_fwd(o, lse))
                row.update(fwd_us=round(t * 1e3, 2), fwd_tflops=round(flops_f / t / 1e9, 1))
            if ref is None:
                ref = (o.clone(), lse.clone())
            else:
                row.update(o_nan=int(torch.isnan(o.float()).sum()), lse_nan=int(torch.isnan(lse).sum()),
                           o_maxdiff=float((o.float() - ref[0].float()).abs().max()),
                           lse_maxdiff=float((lse - ref[1]).abs().max()))
            if what in ("bwd", "all"):
                delta = torch.empty_like(lse)
                dqkv = torch.empty_like(qkv)
                t = bench(lambda: run_bwd(o, lse, delta, dqkv))
                row.update(bwd_us=round(t * 1e3, 2), bwd_tflops=round(2.5 * flops_f / t / 1e9, 1))
            if name == "small" and emu:
                bad = torch.isnan(o.float()).any(dim=1).nonzero().flatten().tolist()
                row.update(nan_rows=bad[:8] + ["..."] + bad[-4:], n_bad=len(bad))
            print(json.dumps(row), flush=True)
        _lib.call("pc_attention_tune", 0, 3)
        _lib.call("pc_attention_tune", 1, 6)


if __name__ == "__main__":
    main()
