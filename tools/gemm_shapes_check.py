"""Launch every GEMM shape of a bench workload once (as bench.gemm_roofline
issues it) and report which ones finish: python tools/gemm_shapes_check.py C4 [index]"""
import subprocess, sys, pathlib, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import bench

wl = bench.WORKLOADS[sys.argv[1]]
cfg, tg, cp = bench.build_plan(1, wl["kw"], wl["M"], family=wl["family"])
block, head = bench.gemm_shapes(cfg, 1)
shapes = block + head
if len(sys.argv) > 2:
    import torch
    from paper_2412_14374_b200 import _lib
    st = torch.cuda.Stream()
    args, keep = bench.gemm_args(shapes[int(sys.argv[2])], st)
    with torch.cuda.stream(st):
        for _ in range(3):
            _lib.call("pc_gemm", *args)
    torch.cuda.synchronize()
    sys.exit(0)
for i, sh in enumerate(shapes):
    t0 = time.time()
    try:
        r = subprocess.run([sys.executable, __file__, sys.argv[1], str(i)], timeout=60,
                           capture_output=True, text=True)
        status = "ok" if r.returncode == 0 else f"rc={r.returncode} {r.stderr[-300:]}"
    except subprocess.TimeoutExpired:
        status = "TIMEOUT"
    print(i, sh, status, f"{time.time() - t0:.1f}s", flush=True)
