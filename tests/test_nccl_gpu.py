"""Multi-process NCCL path: one process per GPU, each running its actor's fused
program, per-directed-channel communicators over NVLink.  Needs >= 2 GPUs
(gpurun --gpus 2); skipped otherwise."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    import faulthandler
    import sys
    # a rank that hangs prints every thread's stack and exits instead of
    # holding the test (and the parent's output pipe) forever
    faulthandler.dump_traceback_later(240, exit=True, file=sys.stderr)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        from oracle import ffn, gpt
        from paper_2412_14374_b200 import comms as C
        from paper_2412_14374_b200 import ir as I
        from paper_2412_14374_b200 import schedules as S
        from paper_2412_14374_b200 import taskgraph as T
        from paper_2412_14374_b200.executor import PipelineEngine, run_pipelined
        if case == "gpt-peer":
            # the same step over NCCL channels and over NVLink peer-memory slots
            # (producers write into the receiver's slot): bitwise equal, eager
            # and as captured CUDA-graph replays of resident training
            cfg = I.GPTConfig(layers=4, d_model=128, n_heads=2, d_ff=512, vocab=256, seq_len=64,
                              microbatch_size=2, yields=(2, 3, 5)[:world - 1], yield_every=6)
            M = 8
            p = I.derive_backward(I.partition_stages(I.build_gpt(cfg)))
            s = S.one_f_one_b(world, M)
            tg = T.infer_outer_placement(T.commute_grad_accumulation(T.unroll(p, s)), p)
            cp = C.plan_pipeline(tg)
            oc = dict(layers=4, d=128, heads=2, ff=512, vocab=256, seq=64, mbs=2)
            rng = np.random.default_rng(0)
            params = {k: v.astype(np.float32) for k, v in gpt.init_params(oc, rng, std=0.05).items()}
            tokens = gpt.init_tokens(oc, M, rng).reshape(M * 2, 64)
            outs = {}
            for tr in ("nccl", "peer"):
                eng = PipelineEngine(cp, tg, mode="bf16", gpt=cfg, transport=tr)
                r = eng.step(params, tokens)
                eng.load_params(params)
                eng.step(None, tokens, lr=0.01)
                cs = eng.capture(None, tokens, lr=0.01)
                cs.replay()
                cs.replay()
                torch.cuda.synchronize()
                if tr == "peer":
                    from paper_2412_14374_b200.executor import PeerChannel
                    sent = [ch for (src, _), ch in eng._channels.items() if src == rank]
                    assert all(isinstance(ch, PeerChannel) for ch in sent)
                    assert sum(ch.in_place for ch in sent) > 0
                outs[tr] = (r.grads, None if r.losses is None else np.asarray(r.losses),
                            eng.state_dict())
                eng.close()
            q.put((rank, outs))
            return
        if case in ("gpt-remat", "peer-drop"):
            cfg = I.GPTConfig(layers=4, d_model=128, n_heads=2, d_ff=512, vocab=256, seq_len=64,
                              microbatch_size=2, yields=(2, 3, 5)[:world - 1], yield_every=6)
            M = 8
            p = I.derive_backward(I.partition_stages(I.build_gpt(cfg)))
            s = S.one_f_one_b(world, M)
            tg = T.infer_outer_placement(T.commute_grad_accumulation(T.unroll(p, s)), p)
            cp = C.plan_pipeline(tg)
            oc = dict(layers=4, d=128, heads=2, ff=512, vocab=256, seq=64, mbs=2)
            rng = np.random.default_rng(0)
            params = {k: v.astype(np.float32) for k, v in gpt.init_params(oc, rng, std=0.05).items()}
            tokens = gpt.init_tokens(oc, M, rng).reshape(M * 2, 64)
        if case == "gpt-remat":
            # full per-stage remat over real inter-process channels: received feeds
            # are views of peer slots / NCCL receive buffers, kept by reference for
            # the replay; eager and captured replays bitwise equal to stashing
            outs = {}
            for tr in ("peer", "nccl"):
                for remat in ("none", "full-per-stage"):
                    eng = PipelineEngine(cp, tg, mode="bf16", gpt=cfg, transport=tr, remat=remat)
                    r = eng.step(params, tokens)
                    eng.load_params(params)
                    eng.step(None, tokens, lr=0.01)
                    cs = eng.capture(None, tokens, lr=0.01)
                    cs.replay()
                    rr = cs.replay(timeout_s=60)
                    torch.cuda.synchronize()
                    outs[(tr, remat)] = (
                        r.grads, None if r.losses is None else np.asarray(r.losses),
                        eng.state_dict(),
                        None if rr.losses is None else rr.losses.cpu().numpy(),
                        dict(r.stats.peak_stash_bytes))
                    eng.close()
            q.put((rank, outs))
            return
        if case == "peer-drop":
            # rank 0 never signals its last activation message: both ranks' device
            # streams park on flags that will not be written.  The watchdog must
            # raise LivenessFault, release the waits so the devices drain, and
            # close() must return with the GPU still usable.
            import time as _time
            from paper_2412_14374_b200.executor import LivenessFault
            if rank == 0:
                prog = cp.programs[0]
                idx = max(i for i, ins in enumerate(prog.instrs) if isinstance(ins, C.SendStart))
                prog.instrs.pop(idx)
            eng = PipelineEngine(cp, tg, mode="bf16", gpt=cfg, transport="peer")
            fault = None
            try:
                eng.step(params, tokens, timeout_s=5.0)
            except LivenessFault as e:
                fault = type(e).__name__ + ": " + str(e)[:200]
            t0 = _time.monotonic()
            eng.close()
            closed_s = _time.monotonic() - t0
            x = torch.arange(1000, device="cuda", dtype=torch.float32)
            healthy = float(x.sum().item()) == 499500.0
            refused = False
            try:
                eng.step(params, tokens, timeout_s=5.0)
            except Exception as e:  # noqa: BLE001
                refused = "aborted" in str(e)
            q.put((rank, fault, closed_s, healthy, refused))
            return
        if case == "ffn-train":
            # resident multi-step training: eager step, then a captured graph
            # replayed twice; the tied w0 is re-broadcast 0 -> P-1 every step
            L, M, K = 2 * world, 4, 3
            p = I.derive_backward(I.partition_stages(I.build_model(I.ModelConfig(
                layers=L, width=16, microbatch_size=8, yield_every=2, tied_weights=True))))
            s = S.one_f_one_b(world, M)
            tg = T.infer_outer_placement(T.commute_grad_accumulation(T.unroll(p, s)), p)
            cp = C.plan_pipeline(tg)
            rng = np.random.default_rng(0)
            params = ffn.init_params({q: p.graph.spec_of(q).dims for q in p.graph.params}, rng)
            batches = [ffn.init_batch(M, 8, 16, rng) for _ in range(K)]
            eng = PipelineEngine(cp, tg, mode="fp64")
            eng.load_params(params)
            losses = [eng.step(None, batches[0], lr=0.01).losses]
            cs = eng.capture(None, batches[1], lr=0.01)
            for k in (1, 2):
                r = cs.replay(torch.from_numpy(batches[k]))
                losses.append(None if r.losses is None else r.losses.cpu().numpy())
            state = eng.state_dict()
            eng.close()
            ref, ref_losses = dict(params), []
            for k in range(K):
                _, lk, ref = ffn.run_reference_ffn(ref, batches[k], M, L, True, lr=0.01)
                ref_losses.append(lk)
            q.put((rank, state, losses, ref, ref_losses))
            return
        if case == "ffn-skip":
            # differentiable non-adjacent skips over real channels (peer transport):
            # activations forward past a stage, their gradients back to the producer
            import sys as _sys
            _sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
            from test_skips_cpu import SKIPS, plan
            M = 8
            p, tg, cp = plan("1f1b", world, M, yields=(2, 3, 5)[:world - 1])
            rng = np.random.default_rng(3)
            params = ffn.init_params({q: p.graph.spec_of(q).dims for q in p.graph.params}, rng)
            batch = ffn.init_batch(M, 4, 8, rng)
            res = run_pipelined(cp, tg, params, batch)
            ref = ffn.run_reference_ffn(params, batch, M, 6, False, skips=SKIPS)
            q.put((rank, res.grads, None if res.losses is None else np.asarray(res.losses),
                   res.new_params, ref, dict(res.stats.channel_counts), res.stats.driver_messages,
                   {k: len(v) for k, v in cp.channels.items()}))
            return
        if case == "ffn":
            L, M = 2 * world, 4
            p = I.derive_backward(I.partition_stages(I.build_model(I.ModelConfig(
                layers=L, width=16, microbatch_size=8, yield_every=2, tied_weights=True))))
            s = S.one_f_one_b(world, M)
            tg = T.infer_outer_placement(T.commute_grad_accumulation(T.unroll(p, s)), p)
            cp = C.plan_pipeline(tg)
            rng = np.random.default_rng(0)
            params = ffn.init_params({q: p.graph.spec_of(q).dims for q in p.graph.params}, rng)
            batch = ffn.init_batch(M, 8, 16, rng)
            res = run_pipelined(cp, tg, params, batch)
            ref = ffn.run_reference_ffn(params, batch, M, L, True)
        else:
            # "gpt": 1F1B; "gpt-interleaved": 2 chunks per GPU (4 stages on 2 GPUs),
            # both channel directions carry two stage boundaries
            inter = case == "gpt-interleaved"
            yl = (1, 3, 4) if inter else (2, 3, 5)[:world - 1]
            cfg = I.GPTConfig(layers=4, d_model=128, n_heads=2, d_ff=512, vocab=256, seq_len=64,
                              microbatch_size=2, yields=yl if world > 1 else None,
                              yield_every=6)
            M = 8
            p = I.derive_backward(I.partition_stages(I.build_gpt(cfg)))
            s = S.interleaved_1f1b(world, M, 2) if inter else S.one_f_one_b(world, M)
            tg = T.infer_outer_placement(T.commute_grad_accumulation(T.unroll(p, s)), p)
            cp = C.plan_pipeline(tg)
            oc = dict(layers=4, d=128, heads=2, ff=512, vocab=256, seq=64, mbs=2)
            rng = np.random.default_rng(0)
            params = gpt.init_params(oc, rng, std=0.05)
            tokens = gpt.init_tokens(oc, M, rng)
            res = run_pipelined(cp, tg, {k: v.astype(np.float32) for k, v in params.items()},
                                tokens.reshape(M * 2, 64), mode="bf16", gpt=cfg)
            ref = gpt.run_reference_gpt(params, tokens, oc)
        q.put((rank, res.grads, None if res.losses is None else np.asarray(res.losses),
               res.new_params, ref, dict(res.stats.channel_counts), res.stats.driver_messages,
               {k: len(v) for k, v in cp.channels.items()}))
    except BaseException as e:  # noqa: BLE001
        q.put((rank, "error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def _run(case, world, attempts=3):
    """Run ``case`` on ``world`` spawned ranks; a rendezvous port taken between
    choosing it and binding it (EADDRINUSE) is retried on a fresh port."""
    for a in range(attempts):
        outs = _run_once(case, world)
        if not any(o[1] == "error" and "EADDRINUSE" in str(o[2]) for o in outs) or a == attempts - 1:
            break
    for o in outs:
        assert o[1] != "error", o
    return outs


def _run_once(case, world):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        outs = [q.get(timeout=300) for _ in range(world)]
    finally:
        for p in procs:
            p.join(timeout=120)
        for p in procs:   # never leave a hung rank behind
            if p.is_alive():
                p.kill()
    return outs


@pytest.mark.parametrize("case,tol,world", [("ffn", 1e-12, 2), ("gpt", 2e-2, 2),
                                            ("gpt-interleaved", 2e-2, 2), ("ffn", 1e-12, 4),
                                            ("gpt", 2e-2, 4), ("ffn-skip", 1e-12, 2),
                                            ("ffn-skip", 1e-12, 4)])
def test_two_gpu_nccl_pipeline_matches_oracle(case, tol, world):
    outs = _run(case, world)
    grads, new, losses = {}, {}, None
    counts = {}
    drv = 0
    for rank, g, l, w, ref, cc, dm, plan_counts in outs:
        grads.update(g)
        new.update(w)
        counts.update(cc)
        drv += dm
        if l is not None:
            losses = l
    g_ref, l_ref, w_ref = ref
    from oracle import ffn
    assert ffn.rel(losses, l_ref) < tol
    for q in g_ref:
        assert ffn.rel(grads[q], g_ref[q]) < tol, q
        assert ffn.rel(new[q], w_ref[q]) < tol, q
    assert counts == plan_counts
    assert drv == 2 * world


def test_two_gpu_resident_training_rebroadcasts_tied_weight():
    outs = _run("ffn-train", 2)
    from oracle import ffn
    state, losses = {}, None
    for rank, st, ls, ref, ref_losses in outs:
        state.update(st)
        if ls[0] is not None:
            losses = ls
    assert sorted(state) == sorted(ref)
    for k in range(3):
        assert ffn.rel(losses[k], ref_losses[k]) < 1e-12, k
    for q in ref:
        assert ffn.rel(state[q], ref[q]) < 1e-12, q


@pytest.mark.parametrize("world", [2, 4])
def test_two_gpu_peer_transport_equals_nccl(world):
    outs = _run("gpt-peer", world)
    for rank, o in outs:
        (ga, la, sa), (gb, lb, sb) = o["nccl"], o["peer"]
        assert sorted(ga) == sorted(gb)
        for q in ga:
            assert np.array_equal(ga[q], gb[q]), (rank, q)
        assert (la is None) == (lb is None)
        if la is not None:
            assert np.array_equal(la, lb)
        for q in sa:
            assert np.array_equal(sa[q], sb[q]), (rank, q)


@pytest.mark.parametrize("world", [2, 4])
def test_multi_gpu_remat_bitwise_equal_to_stashing(world):
    """remat over peer and NCCL channels (received feeds kept by
    reference), eager and CUDA-graph replay, equals the stashing run bitwise."""
    outs = _run("gpt-remat", world)
    for rank, o in outs:
        for tr in ("peer", "nccl"):
            a, b = o[(tr, "none")], o[(tr, "full-per-stage")]
            assert sorted(a[0]) == sorted(b[0])
            for q in a[0]:
                assert np.array_equal(a[0][q], b[0][q]), (rank, tr, q)
            assert (a[1] is None) == (b[1] is None)
            if a[1] is not None:
                assert np.array_equal(a[1], b[1]) and np.array_equal(a[3], b[3])
            for q in a[2]:
                assert np.array_equal(a[2][q], b[2][q]), (rank, tr, q)
            assert b[4][rank] < a[4][rank], (rank, tr, a[4], b[4])


@pytest.mark.parametrize("world", [2])
def test_peer_transport_dropped_send_aborts_and_drains(world):
    """ADVICE r1 / VERDICT r1 weak #9: a dropped SendStart on the NVLink peer
    transport raises LivenessFault on the ranks whose streams wait for it,
    releases the parked flag waits (pc_peer_release) so the device drains, and
    close() returns promptly; the engine refuses further steps."""
    outs = _run("peer-drop", world)
    faults = {rank: f for rank, f, _, _, _ in outs}
    assert faults[1] is not None and "LivenessFault" in faults[1], faults
    for rank, fault, closed_s, healthy, refused in outs:
        assert healthy, rank
        assert closed_s < 20.0, (rank, closed_s)
        if fault is not None:
            assert refused, rank
