"""Point-to-point transfer time of one C2 stage-boundary message (12.6 MB bf16)
between two GPUs: NCCL send/recv (the runtime's NcclChannel path, torchrun
2 ranks) and, in rank 0 alone, a copy-engine peer copy.  usage: torchrun
--nproc-per-node 2 tools/p2p_bw.py"""
import os
import torch
import torch.distributed as dist

rank = int(os.environ["RANK"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
n = 8 * 1024 * 768  # tokens x d_model, bf16 = 12.6 MB
for nbytes_mult in (1, 4):
    t = torch.empty(n * nbytes_mult, dtype=torch.bfloat16, device="cuda")
    for _ in range(5):
        (dist.send if rank == 0 else dist.recv)(t, 1 - rank)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        (dist.send if rank == 0 else dist.recv)(t, 1 - rank)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    if rank == 1:
        print(f"nccl send/recv {t.numel()*2/1e6:.1f} MB: {ms*1e3:.1f} us, {t.numel()*2/ms/1e6:.0f} GB/s", flush=True)
dist.barrier()
if rank == 0:
    src = torch.empty(n, dtype=torch.bfloat16, device="cuda:0")
    dst = torch.empty(n, dtype=torch.bfloat16, device="cuda:1")
    for _ in range(5):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        dst.copy_(src, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"peer copy (copy engine) 12.6 MB: {ms*1e3:.1f} us, {n*2/ms/1e6:.0f} GB/s", flush=True)
dist.barrier()
dist.destroy_process_group()
