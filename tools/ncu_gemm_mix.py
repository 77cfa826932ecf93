"""Issue every C2 GEMM of one stage step once, exactly as bench.gemm_roofline
(and device.py) issue them, for an `ncu --set full -k regex:tc_gemm` capture;
then (here, no GPU) `python tools/ncu_gemm_mix.py --parse rep.csv` writes
profiles/r02_ncu_gemm_mix.json: DRAM bytes read + written per launch, keyed
like bench.gemm_traffic().

  GPU:  ncu --set full --clock-control none -k regex:tc_gemm -c 15 --csv --page raw \\
            --log-file gpurun_out/gemm_mix_raw.csv python tools/ncu_gemm_mix.py
"""
import csv
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def shapes():
    from paper_2412_14374_b200 import ir as I
    cfg = I.GPTConfig(**bench.C2, yield_every=bench.C2["layers"] + 2)
    block, head = bench.gemm_shapes(cfg, 1)
    return block + head


def run():
    import torch
    from paper_2412_14374_b200 import _lib
    st = torch.cuda.current_stream()
    for s in shapes():
        args, keep = bench.gemm_args(s, st)
        _lib.call("pc_gemm", *args)
        torch.cuda.synchronize()
        del keep


def parse(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    units = rows[0] if rows and rows[0].get("ID") == "" else None
    data = [r for r in rows if r.get("ID", "").isdigit()]
    out = {}
    for s, r in zip(shapes(), data):
        M, N, K, _, _, epi = s[:6]
        rd = float(r["dram__bytes_read.sum"].replace(",", ""))
        wr = float(r["dram__bytes_write.sum"].replace(",", ""))
        scale = 1.0
        if units:
            u = units.get("dram__bytes_read.sum", "byte")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        t = float(r["gpu__time_duration.sum"].replace(",", ""))
        out[f"{M}x{N}x{K}:{epi}"] = {"dram_bytes": int((rd + wr) * scale),
                                    "read_bytes": int(rd * scale), "write_bytes": int(wr * scale),
                                    "kernel": r.get("Kernel Name", "")[:60],
                                    "ncu_time": t}
    doc = {"source": "ncu --set full --clock-control none -k regex:tc_gemm, one launch per "
                     "shape (tools/ncu_gemm_mix.py); cold L2, replayed: compare bytes, not time",
           "shapes": out}
    dst = pathlib.Path(__file__).resolve().parents[1] / "profiles" / "r02_ncu_gemm_mix.json"
    dst.write_text(json.dumps(doc, indent=1) + "\n")
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--parse":
        parse(sys.argv[2])
    else:
        run()
