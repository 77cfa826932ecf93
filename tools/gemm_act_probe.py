"""Where does the activation epilogue (bias + GELU / ReLU, pre-activation U and
C both stored) cost time on the C2 fc1 GEMM [8192 x 3072 x 768]?  Times the
shape with: no epilogue, bias, bias+ReLU (U + C), bias+GELU (U + C), and the
latter with the epilogue work ablated (pc_gemm_set_ablation 1), for each
tile choice.  usage: python tools/gemm_act_probe.py [M N K [ablate-plain]]"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
import bench
from paper_2412_14374_b200 import _lib

M, N, K = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (8192, 3072, 768)
ST = torch.cuda.Stream()


def timed(args, iters=20):
    with torch.cuda.stream(ST):
        for _ in range(3):
            _lib.call("pc_gemm", *args)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=ST):
            for _ in range(iters):
                _lib.call("pc_gemm", *args)
        g.replay()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(ST)
        g.replay()
        e.record(ST)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


B_, G_, R_ = _lib.EPI_BIAS, _lib.EPI_GELU, _lib.EPI_RELU
cases = [("plain", 0, 0), ("bias", B_, 0), ("bias+relu U,C", B_ | R_, 1), ("bias+gelu U,C", B_ | G_, 1)]
if len(sys.argv) > 4:   # plain-store ablations too
    cases = [("plain", 0, 0), ("bias+gelu U,C", B_ | G_, 1)]
for bn, pair in ((0, 0), (192, 2), (256, 2), (128, 2)):
    _lib.call("pc_gemm_set_tile_n", bn)
    _lib.call("pc_gemm_set_cta_pair", pair)
    row = []
    for name, epi, has_u in cases:
        args, keep = bench.gemm_args((M, N, K, 0, 1, epi, 0, has_u, 0), ST)
        row.append(f"{name} {timed(args):.1f}")
        if name.startswith("bias+gelu") or (len(sys.argv) > 4 and name == "plain"):
            _lib.call("pc_gemm_set_ablation", 1)
            row.append(f"(no-epi {timed(args):.1f})")
            _lib.call("pc_gemm_set_ablation", 2)
            row.append(f"(no-load {timed(args):.1f})")
            _lib.call("pc_gemm_set_ablation", 3)
            row.append(f"(mma-only {timed(args):.1f})")
            _lib.call("pc_gemm_set_ablation", 0)
    print(f"tile {'auto' if bn == 0 else f'{bn}x{pair}'}: " + " | ".join(row) + " us", flush=True)
_lib.call("pc_gemm_set_tile_n", 0)
_lib.call("pc_gemm_set_cta_pair", 0)
