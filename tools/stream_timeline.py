"""Where one graph-replayed C2 step (P=1) spends its time per CUDA stream:
CUPTI kernel records (torch.profiler) of one CapturedStep.replay, grouped by
stream -- busy time (union of kernel intervals), the step span, how much of
the span each stream and both together cover, and the top kernels on the
compute stream.  A development aid, not a bench number.
usage: python tools/stream_timeline.py"""
import collections
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2412_14374_b200.executor import PipelineEngine  # noqa: E402

cfg, tg, cp = bench.build_plan(1, bench.C2, bench.M_MICRO)
dev = torch.device("cuda", 0)
params = bench.init_params_device(cfg, dev)
tok = torch.randint(0, cfg.vocab, (bench.M_MICRO * cfg.microbatch_size, cfg.seq_len),
                    dtype=torch.int32, device=dev)
eng = PipelineEngine(cp, tg, mode="bf16", gpt=cfg)
eng.load_params(params)
for _ in range(2):
    eng.step(None, tok, lr=1e-4, timeout_s=600, to_host=False)
cap = eng.capture(None, tok, lr=1e-4)
for _ in range(3):
    cap.replay()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    cap.replay()
    torch.cuda.synchronize()
out = pathlib.Path("gpurun_out/stream_trace.json")
out.parent.mkdir(exist_ok=True)
prof.export_chrome_trace(str(out))
ev = [e for e in json.loads(out.read_text())["traceEvents"]
      if e.get("cat") == "kernel" and "dur" in e]
by = collections.defaultdict(list)
for e in ev:
    by[e["args"].get("stream", e.get("tid"))].append((e["ts"], e["ts"] + e["dur"], e["name"]))
t0 = min(s for v in by.values() for s, _, _ in v)
t1 = max(t for v in by.values() for _, t, _ in v)


def union(iv):
    iv = sorted(iv)
    tot, cs, ce = 0.0, None, None
    for s, t in iv:
        if cs is None or s > ce:
            if cs is not None:
                tot += ce - cs
            cs, ce = s, t
        else:
            ce = max(ce, t)
    return tot + (ce - cs if cs is not None else 0.0)


print(f"step span {(t1 - t0) / 1e3:.2f} ms, {len(ev)} kernels")
allv = []
for st, v in sorted(by.items(), key=lambda kv: -len(kv[1])):
    iv = [(s, t) for s, t, _ in v]
    allv += iv
    print(f"  stream {st}: {len(v)} kernels, busy {union(iv) / 1e3:.2f} ms "
          f"({union(iv) / (t1 - t0):.1%} of the span), kernel time {sum(t - s for s, t in iv) / 1e3:.2f} ms")
print(f"  any stream busy: {union(allv) / 1e3:.2f} ms ({union(allv) / (t1 - t0):.1%}); "
      f"idle {(t1 - t0 - union(allv)) / 1e3:.2f} ms")
main = max(by.items(), key=lambda kv: len(kv[1]))[1]
agg = collections.defaultdict(lambda: [0, 0.0])
for s, t, n in main:
    k = n.split("(")[0][:60]
    agg[k][0] += 1
    agg[k][1] += t - s
print("compute stream, top kernels:")
for k, (c, d) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:14]:
    print(f"  {d / 1e3:7.2f} ms x{c:4d}  {k}")
