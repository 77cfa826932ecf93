"""Device time (CUDA-graph replay) of one GEMM shape under every forced tile
width / CTA-pair choice, with the production epilogue.
usage: python tools/gemm_tile_sweep.py M N K transA transB epi"""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
import bench
from paper_2412_14374_b200 import _lib

M, N, K, ta, tb, epi = (int(x) for x in sys.argv[1:7])
f32 = 1 if epi & (_lib.EPI_ACCUM | _lib.EPI_SPLITK_ZERO_C) else 0
st = torch.cuda.Stream()
args, keep = bench.gemm_args((M, N, K, ta, tb, epi, 0, 0, f32), st)


def t():
    with torch.cuda.stream(st):
        for _ in range(3):
            _lib.call("pc_gemm", *args)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(10):
                _lib.call("pc_gemm", *args)
        g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.replay()
        e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 10 * 1e3


splits = [int(x) for x in sys.argv[7].split(",")] if len(sys.argv) > 7 else [2]
for ks in splits:
    _lib.call("pc_gemm_set_max_split", ks)
    print(f"max_split={ks} auto: {t():.1f} us", flush=True)
    for bn in (64, 128, 192, 256):
        for pair in (1, 2):
            _lib.call("pc_gemm_set_tile_n", bn)
            _lib.call("pc_gemm_set_cta_pair", pair)
            try:
                print(f"  max_split={ks} bn={bn} pair={pair}: {t():.1f} us", flush=True)
            except Exception as e:  # noqa: BLE001
                print(f"  max_split={ks} bn={bn} pair={pair}: {e}", flush=True)
    _lib.call("pc_gemm_set_tile_n", 0)
    _lib.call("pc_gemm_set_cta_pair", 0)
_lib.call("pc_gemm_set_max_split", 4)
