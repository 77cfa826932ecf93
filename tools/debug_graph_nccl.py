"""2-rank capture/replay smoke with phase logging (debugging aid)."""
import os, sys, time, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch, torch.distributed as dist
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"]); local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
def log(*a):
    print(f"[r{rank} {time.strftime('%H:%M:%S')}]", *a, flush=True)
from paper_2412_14374_b200 import comms as C, ir as I, schedules as S, taskgraph as T
from paper_2412_14374_b200.executor import PipelineEngine
from oracle import gpt
cfg = I.GPTConfig(layers=4, d_model=128, n_heads=2, d_ff=512, vocab=256, seq_len=64, microbatch_size=2, yields=(3,), yield_every=6)
p = I.derive_backward(I.partition_stages(I.build_gpt(cfg)))
s = S.one_f_one_b(world, 4)
tg = T.infer_outer_placement(T.commute_grad_accumulation(T.unroll(p, s)), p)
cp = C.plan_pipeline(tg)
oc = dict(layers=4, d=128, heads=2, ff=512, vocab=256, seq=64, mbs=2)
rng = np.random.default_rng(0)
params = {q: v.astype(np.float32) for q, v in gpt.init_params(oc, rng, std=0.05).items()}
tokens = gpt.init_tokens(oc, 4, rng).reshape(8, -1)
eng = PipelineEngine(cp, tg, mode="bf16", gpt=cfg)
log("eager 1"); r1 = eng.step(params, tokens, timeout_s=60); log("eager 2"); eng.step(params, tokens, timeout_s=60)
torch.cuda.synchronize(); log("capture")
cap = eng.capture(params, tokens, timeout_s=60); torch.cuda.synchronize(); log("captured")
dist.barrier(); log("replay")
r = cap.replay(); torch.cuda.synchronize(); log("replayed")
for q in r1.grads:
    same = np.array_equal(r.grads[q].cpu().numpy(), r1.grads[q])
    log(q, "bitwise equal" if same else "DIFFERENT")
if r1.losses is not None:
    log("loss equal", np.array_equal(r.losses.cpu().numpy(), r1.losses))
dist.barrier(); dist.destroy_process_group(); log("done")
