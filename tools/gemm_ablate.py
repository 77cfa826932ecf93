"""Where does the tcgen05 GEMM lose time?  Times each tile variant with the full
kernel, without epilogue work, without operand loads, and with neither (pure
MMA issue), on the C2 shapes.  usage: python tools/gemm_ablate.py"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2412_14374_b200 import _lib

SHAPES = [("fwd qkv", 8192, 2304, 768, 0, 1), ("fwd fc2", 8192, 768, 3072, 0, 1),
          ("sq 8192", 8192, 8192, 8192, 0, 1)]
if len(sys.argv) > 1 and sys.argv[1] == "wgrad":  # MN-major operands vs a K-major control
    SHAPES = [("wg fc2", 768, 3072, 8192, 1, 0), ("wg fc2 K", 768, 3072, 8192, 0, 1),
              ("wg fc1", 3072, 768, 8192, 1, 0), ("wg fc1 K", 3072, 768, 8192, 0, 1),
              ("wg fc1 AK", 3072, 768, 8192, 0, 0), ("wg fc1 BK", 3072, 768, 8192, 1, 1)]
TILES = ((256, 2), (128, 2), (256, 1), (128, 1))
if len(sys.argv) > 1 and sys.argv[1] == "proj":  # short-K, N = 768 GEMMs (attention out / its dX)
    SHAPES = [("proj", 8192, 768, 768, 0, 1), ("fc1dX", 8192, 768, 3072, 0, 1)]
    TILES = ((192, 2), (128, 2), (256, 2), (192, 1), (128, 1), (256, 1))


ST = torch.cuda.Stream()


def bench(fn, iters=20):
    """Device time per launch: iters launches captured in a CUDA graph."""
    with torch.cuda.stream(ST):
        for _ in range(3):
            fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=ST):
            for _ in range(iters):
                fn()
        g.replay()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(ST)
        g.replay()
        e.record(ST)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


for name, M, N, K, ta, tb in SHAPES:
    A = torch.randn((K, M) if ta else (M, K), device="cuda").bfloat16()
    B = torch.randn((N, K) if tb else (K, N), device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    st = ST.cuda_stream
    f = lambda: _lib.call("pc_gemm", 2, 2, ta, tb, M, N, K, A.data_ptr(), A.stride(0), B.data_ptr(),
                          B.stride(0), C.data_ptr(), C.stride(0), 0, None, None, 0, None, 0, st)
    for bn, pair in TILES:
        _lib.call("pc_gemm_set_tile_n", bn)
        _lib.call("pc_gemm_set_cta_pair", pair)
        out = []
        for ab in (0, 1, 2, 3):
            _lib.call("pc_gemm_set_ablation", ab)
            out.append(bench(f))
        _lib.call("pc_gemm_set_ablation", 0)
        fl = 2 * M * N * K / 1e9
        print(f"{name:8s} bn={bn} pair={pair}: full {out[0]*1e3:.1f} us ({fl/out[0]:.0f})  "
              f"no-epi {out[1]*1e3:.1f}  no-load {out[2]*1e3:.1f}  mma-only {out[3]*1e3:.1f} us",
              flush=True)
_lib.call("pc_gemm_set_tile_n", 0)
_lib.call("pc_gemm_set_cta_pair", 0)
