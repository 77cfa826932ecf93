"""One warm eager C2 step (P=1) for ncu launch lists: warm-up step first, then
the profiled step (skip the warm-up's launches with ncu -s)."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
import bench
from paper_2412_14374_b200 import _lib
from paper_2412_14374_b200.executor import PipelineEngine
cfg, tg, cp = bench.build_plan(1, bench.C2, bench.M_MICRO)
dev = torch.device("cuda", 0)
params = bench.init_params_device(cfg, dev)
tok = torch.randint(0, cfg.vocab, (bench.M_MICRO * cfg.microbatch_size, cfg.seq_len), dtype=torch.int32, device=dev)
eng = PipelineEngine(cp, tg, mode="bf16", gpt=cfg)
eng.step(params, tok, lr=1e-4, timeout_s=600, to_host=False)
torch.cuda.synchronize()
n0 = _lib.launch_count
torch.cuda.profiler.start()   # ncu --profile-from-start off: only this step
eng.step(params, tok, lr=1e-4, timeout_s=600, to_host=False)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("libpp200 calls per step:", _lib.launch_count - n0)
