"""Host-side logic of the N>1 path on CPU with a world_size-2 gloo group.

What is tested here without GPUs: every rank derives the byte-identical plan
(the runtime relies on each process planning independently), the
communicator-id rendezvous pairs each directed channel's sender and receiver
with the same id, the per-rank program split covers all instructions exactly
once, and both ends of every channel agree on the wire shape/dtype of every
message (the receiver preallocates at RecvStart).  The NCCL data path itself is
covered by the 2-GPU test under gpurun (tests/test_nccl_gpu.py).
"""
import hashlib
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_14374_b200 import comms as C
from paper_2412_14374_b200 import ir as I
from paper_2412_14374_b200 import schedules as S
from paper_2412_14374_b200 import taskgraph as T


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _plan(P):
    cfg = I.GPTConfig(layers=4, d_model=64, n_heads=2, d_ff=128, vocab=64, seq_len=16,
                      microbatch_size=2, yields=(3,) if P == 2 else None, yield_every=6)
    p = I.derive_backward(I.partition_stages(I.build_gpt(cfg)))
    s = S.one_f_one_b(P, 4)
    tg = T.infer_outer_placement(T.commute_grad_accumulation(T.unroll(p, s)), p)
    cp = C.fuse(C.insert_deletions(C.infer_comms(tg, s), tg), tg)
    return cfg, tg, cp


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2412_14374_b200.device import MODES
        from paper_2412_14374_b200.executor import _wire_meta_fn, exchange_channel_ids
        cfg, tg, cp = _plan(world)
        digest = hashlib.sha256(cp.to_json_str().encode()).hexdigest()
        digests = [None] * world
        dist.all_gather_object(digests, digest)
        store = dist.distributed_c10d._get_default_store()
        ids = exchange_channel_ids(store, "test", rank, cp.channels,
                                   lambda: hashlib.sha256(f"{rank}-{os.getpid()}".encode()).digest() * 4)
        all_ids = [None] * world
        dist.all_gather_object(all_ids, ids)
        meta = _wire_meta_fn(tg, MODES["bf16"])
        mine = {}
        for ins in cp.programs[rank].instrs:
            if isinstance(ins, (C.SendStart, C.RecvStart)):
                shape, dt = meta(ins.buffer)
                mine[ins.buffer] = (shape, str(dt))
        metas = [None] * world
        dist.all_gather_object(metas, mine)
        q.put((rank, digests, all_ids, metas))
    finally:
        dist.destroy_process_group()


@pytest.mark.slow
def test_two_rank_rendezvous_and_wire_agreement():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    _, digests, all_ids, metas = results[0]
    assert len(set(digests)) == 1, "ranks planned different programs"
    _, _, cp = _plan(world)
    assert set(cp.channels) == {(0, 1), (1, 0)}
    for (src, dst) in cp.channels:
        assert all_ids[src][(src, dst)] == all_ids[dst][(src, dst)]
        assert len(all_ids[src][(src, dst)]) == 128
    # the two ends agree on every message's layout; tokens travel as int32
    common = set(metas[0]) & set(metas[1])
    assert common == {b for bufs in cp.channels.values() for b in bufs}
    for b in common:
        assert metas[0][b] == metas[1][b]
    assert metas[0]["act:x:mb0"][1] == str(torch.int32)


def test_programs_partition_instructions_by_rank():
    _, tg, cp = _plan(2)
    runs = [ins.task for pg in cp.programs for ins in pg.instrs if isinstance(ins, C.RunTask)]
    assert sorted(runs) == sorted(tg.tasks)
    for pg in cp.programs:
        for ins in pg.instrs:
            if isinstance(ins, C.RunTask):
                assert tg.tasks[ins.task].actor == pg.actor
