"""Per-kernel GPU time breakdown of one C2 pipeline step (P=1) + host issue time.

CUPTI (torch.profiler) records every kernel in the process, including the
libpp200 ones; this is a development aid, not a bench number.
"""
import sys, pathlib, time, collections, json
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch
import bench
from paper_2412_14374_b200.executor import PipelineEngine

cfg, tg, cp = bench.build_plan(1, bench.C2, bench.M_MICRO)
dev = torch.device("cuda", 0)
params = bench.init_params_device(cfg, dev)
tok = torch.randint(0, cfg.vocab, (bench.M_MICRO * cfg.microbatch_size, cfg.seq_len), dtype=torch.int32, device=dev)
eng = PipelineEngine(cp, tg, mode="bf16", gpt=cfg)
for _ in range(2):
    eng.step(params, tok, lr=1e-4, timeout_s=600, to_host=False)
torch.cuda.synchronize()
# host issue time vs device time
import paper_2412_14374_b200.executor as E
orig = E.PipelineEngine._wait_devices
stamps = {}
def timed_wait(self, actors, ctl):
    stamps["issued"] = time.perf_counter()
    return orig(self, actors, ctl)
E.PipelineEngine._wait_devices = timed_wait
t0 = time.perf_counter()
eng.step(params, tok, lr=1e-4, timeout_s=600, to_host=False)
t1 = time.perf_counter()
print(f"host issue {1000*(stamps['issued']-t0):.1f} ms, step wall {1000*(t1-t0):.1f} ms")
E.PipelineEngine._wait_devices = orig
from torch.profiler import profile, ProfilerActivity
cap = eng.capture(params, tok, lr=1e-4)
for _ in range(2):
    cap.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); cap.replay(); e1.record(); torch.cuda.synchronize()
print(f"graph replay step {e0.elapsed_time(e1):.2f} ms")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    cap.replay()
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        name = ev.name.replace("(anonymous namespace)::", "").replace("pp200::", "")
        name = name.replace("void ", "")
        name = name.split("(")[0][:90]
        agg[name][0] += 1
        agg[name][1] += ev.device_time_total / 1000.0 if hasattr(ev, "device_time_total") else ev.cuda_time_total / 1000.0
tot = sum(v[1] for v in agg.values())
print(f"total kernel time {tot:.1f} ms")
for name, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{ms:9.2f} ms {100*ms/tot:5.1f}%  x{n:5d}  {name}")
