"""Every C2 GEMM shape (as bench.gemm_shapes issues it: epilogue, aux / pre-activation
inputs, fp32 accumulate) under every forced tile width x CTA-pair choice and the
automatic choice, device time per launch from CUDA-graph replays.  Calibrates the
per-tile efficiency table of gemm_tc.cu choose_tiles.
usage: python tools/gemm_sweep_mix.py [C2|C3|C4|C5]"""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2412_14374_b200 import _lib  # noqa: E402
from paper_2412_14374_b200 import ir as I  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
kw = dict(bench.WORKLOADS[wl]["kw"])
fam = bench.WORKLOADS[wl]["family"]
if fam == "gpt":
    cfg = I.GPTConfig(**kw, yield_every=kw["layers"] + 2)
else:
    cfg, _, _ = bench.build_plan(1, kw, bench.WORKLOADS[wl]["M"], family=fam)
block, head = bench.gemm_shapes(cfg, 1)
st = torch.cuda.Stream()


def timed(args):
    with torch.cuda.stream(st):
        for _ in range(2):
            _lib.call("pc_gemm", *args)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(5):
                _lib.call("pc_gemm", *args)
        g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.replay()
        e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 5 * 1e3


for sh in block + head:
    M, N, K = sh[:3]
    args, keep = bench.gemm_args(sh, st)
    row = {"shape": list(sh[:6]), "auto": round(timed(args), 1)}
    for bn in (64, 128, 192, 256):
        for pair in (1, 2):
            _lib.call("pc_gemm_set_tile_n", bn)
            _lib.call("pc_gemm_set_cta_pair", pair)
            try:
                row[f"{bn}x{pair}"] = round(timed(args), 1)
            except Exception:  # noqa: BLE001 - combination not realisable for this shape
                row[f"{bn}x{pair}"] = None
    _lib.call("pc_gemm_set_tile_n", 0)
    _lib.call("pc_gemm_set_cta_pair", 0)
    best = min((v, k) for k, v in row.items() if k not in ("shape",) and v)
    row["best"] = best[1]
    row["tflops_auto"] = round(2.0 * M * N * K / row["auto"] / 1e6, 1)
    print(json.dumps(row), flush=True)
    del keep
