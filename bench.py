"""Benchmark: one pipelined GPT training step on N B200s (one process per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (BASELINE.json configs[1], "C2"): GPT-2 small (12 layers, d=768, 12
heads, d_ff=3072, vocab 50304, seq 1024), 1F1B over 8 microbatches of 8x1024
tokens, bf16 compute / fp32 master + accumulators, SGD update inside the step,
random-init weights and synthetic uniform tokens.  N GPUs = N pipeline stages
(stage boundaries balanced by FLOPs); total work per step is fixed as N grows
("scaling": "strong").  Inputs exceed L2 (activations of one stage ~1.5 GB per
microbatch), so no explicit flush is needed between steps.

Prints one JSON line (rank 0): value = tokens/s for the whole job, plus
model TFLOPS/GPU, measured vs ideal bubble, roofline of the dominant kernel
(the tcgen05 GEMM), the numpy CPU baseline, the e2e number through the public
API with host<->device copies, clocks, and libpp200 launch count.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

C2 = dict(layers=12, d_model=768, n_heads=12, d_ff=3072, vocab=50304, seq_len=1024,
          microbatch_size=8)
M_MICRO = 8
# BASELINE configs[2] (C3, GPT-2 medium; quoted there on 8 stages x 16 microbatches):
# `--workload C3` runs it on the GPUs given (the default bench line stays C2)
C3 = dict(C2, layers=24, d_model=1024, n_heads=16, d_ff=4096)
# BASELINE configs[3] (C4, GPT-3 1.3B shape: head_dim 128, quoted on 8 GPUs with interleaved
# 1F1B, 2 virtual stages per GPU, 32 microbatches) and configs[4] (C5, Llama-3-8B shape:
# RMSNorm / RoPE / GQA 32:8 / SwiGLU, untied head, position ids as skip tensors from stage 0
# to every later stage, 8-stage 1F1B, 16 microbatches).  `--workload C4|C5` runs them on the
# GPUs given (one pipeline stage -- or V virtual stages -- per GPU).
C4 = dict(layers=24, d_model=2048, n_heads=16, d_ff=8192, vocab=50304, seq_len=2048,
          microbatch_size=4)
C5 = dict(layers=32, d_model=4096, n_heads=32, n_kv_heads=8, d_ff=14336, vocab=128256,
          seq_len=4096, microbatch_size=1)
WORKLOADS = {
    "C2": dict(family="gpt", kw=C2, M=8, schedule="1f1b", V=1,
               name="C2 gpt2-small 12L d768 h12 ff3072 V50304 seq1024"),
    "C3": dict(family="gpt", kw=C3, M=16, schedule="1f1b", V=1,
               name="C3 gpt2-medium 24L d1024 h16 ff4096 V50304 seq1024"),
    "C4": dict(family="gpt", kw=C4, M=32, schedule="interleaved", V=2,
               name="C4 gpt3-1.3B 24L d2048 h16x128 ff8192 V50304 seq2048"),
    "C5": dict(family="llama", kw=C5, M=16, schedule="1f1b", V=1,
               name="C5 llama-8B 32L d4096 h32/kv8x128 swiglu14336 V128256 seq4096"),
    # The reference's own model (pipecraft ModelConfig: H = relu(H W), summed-square
    # loss) as the FFN surrogate of C2: 12 blocks of width 768,
    # 8 microbatches x 8192 rows, float64 -- the reference's arithmetic -- so the
    # reference's run_reference (oracle/ffn.py, bit-identical to it) is timed on
    # exactly this configuration by --impl reference --workload FFN-C2.
    "FFN-C2": dict(family="ffn", kw=dict(layers=12, width=768, microbatch_size=8192), M=8,
                   schedule="1f1b", V=1,
                   name="FFN-C2 pipecraft FFN surrogate of C2: 12L w768 rows8192 fp64"),
}


def ffn_flops_per_row(kw) -> float:
    """Algorithmic FLOPs of one row through the FFN stack, fwd + bwd: 3 GEMMs of
    2 w^2 per block (the reference's dead first-block dX, ir.py:510-511, not counted)."""
    return 6.0 * kw["layers"] * kw["width"] ** 2


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d["bf16_tflops"], d.get("bf16_tflops_sustained"), d["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


# In-situ rates calibrated from tools/profile_step.py (C2, P=1, round-1 kernels):
# block GEMMs ~1.05 PFLOP/s, the large-N LM-head GEMMs ~1.2, attention ~0.35
# (fwd+bwd equivalent), norms / reductions ~3 TB/s, the streaming loss ~6 TB/s.
_GEMM_RATE, _HEAD_RATE, _ATTN_RATE, _HBM_RATE, _STREAM_RATE = 1.05e15, 1.2e15, 0.35e15, 3e12, 6e12


def block_costs(cfg):
    """Per-block fwd+bwd time estimates (s) for stage balancing: FLOPs alone
    over-weight the LM head, whose GEMMs run much faster than attention."""
    T, d, f, V, S = cfg.tokens, cfg.d_model, cfg.d_ff, cfg.vocab, cfg.seq_len
    gemm = 3 * 2.0 * T * (4 * d * d + 2 * d * f)
    attn = 3.5 * 2.0 * T * S * d            # causal fwd + recomputing bwd
    elem = 2 * 20.0 * T * d + 2 * 6.0 * T * f  # LN, residuals, GELU, bias grads (bytes)
    blk = gemm / _GEMM_RATE + attn / _ATTN_RATE + elem / _HBM_RATE
    head = 3 * 2.0 * T * d * V / _HEAD_RATE + 3 * 2.0 * T * V / _STREAM_RATE
    emb = 4.0 * T * d * 4 / _HBM_RATE
    return [emb] + [blk] * cfg.layers + [head]


def llama_block_costs(cfg):
    """Per-block time estimates (s) for the Llama stack (C5), same rates."""
    T, d, V, S = cfg.tokens, cfg.d_model, cfg.vocab, cfg.seq_len
    H, hd, f = cfg.n_heads, cfg.head_dim, cfg.d_ff
    gemm = 3 * 2.0 * T * d * (cfg.qkv_width + H * hd + 3 * f)
    attn = 3.5 * 2.0 * T * S * H * hd
    elem = 2 * 16.0 * T * d + 2 * 8.0 * T * f
    blk = gemm / _GEMM_RATE + attn / _ATTN_RATE + elem / _HBM_RATE
    # untied head + loss: measured at 2.9 blocks' time on the C5 4-GPU timeline
    # (bubble.busy_ms_per_gpu), 1.8x what its FLOPs at _HEAD_RATE give
    scale = float(os.environ.get("PP200_LLAMA_HEAD_SCALE", "1.8"))   # A/B hook
    head = scale * (3 * 2.0 * T * d * V / _HEAD_RATE + 3 * 2.0 * T * V / _STREAM_RATE)
    emb = 4.0 * T * d * 4 / _HBM_RATE
    return [emb] + [blk] * cfg.layers + [head]


METRIC = "tokens/s (model TFLOPS/GPU and bubble alongside)"
WORKLOAD = "C2 gpt2-small 12L d768 h12 ff3072 V50304 seq1024"


def build_plan(P, cfg_kw, M, mode="bf16", family="gpt", schedule="1f1b", V=1):
    """Plan one workload on P GPUs: P stages (1F1B) or P x V virtual stages
    (interleaved 1F1B), stage boundaries balanced by the cost model."""
    from paper_2412_14374_b200 import comms as C
    from paper_2412_14374_b200 import ir as I
    from paper_2412_14374_b200 import schedules as S
    from paper_2412_14374_b200 import taskgraph as T
    inter = schedule == "interleaved" and P > 1 and V > 1
    stages = P * V if inter else P
    if family == "ffn":
        L = cfg_kw["layers"]
        base = dict(cfg_kw, elem_bytes=8 if mode == "fp64" else (4 if mode == "fp32" else 2))
        yields = I.balanced_yields([1.0] * L, stages) if stages > 1 else None
        cfg = I.ModelConfig(**base, yields=yields, yield_every=L)
        p = I.derive_backward(I.partition_stages(I.build_model(cfg)))
        s = S.interleaved_1f1b(P, M, V) if inter else S.one_f_one_b(P, M)
        tg = T.infer_outer_placement(T.commute_grad_accumulation(T.unroll(p, s)), p)
        cp = C.infer_comms(tg, s)
        rep = C.check_deadlock_free(cp)
        assert rep.ok, str(rep)
        return cfg, tg, C.fuse(C.insert_deletions(cp, tg), tg)
    Cfg, build = (I.GPTConfig, I.build_gpt) if family == "gpt" else (I.LlamaConfig, I.build_llama)
    costs_fn = block_costs if family == "gpt" else llama_block_costs
    base = Cfg(**cfg_kw, yield_every=cfg_kw["layers"] + 2)
    yields = I.balanced_yields(costs_fn(base), stages) if stages > 1 else None
    cfg = Cfg(**cfg_kw, yields=yields, yield_every=cfg_kw["layers"] + 2,
              elem_bytes=2 if mode == "bf16" else 4)
    p = I.derive_backward(I.partition_stages(build(cfg)))
    s = S.interleaved_1f1b(P, M, V) if inter else S.one_f_one_b(P, M)
    tg = T.infer_outer_placement(T.commute_grad_accumulation(T.unroll(p, s)), p)
    cp = C.infer_comms(tg, s)
    rep = C.check_deadlock_free(cp)
    assert rep.ok, str(rep)
    return cfg, tg, C.fuse(C.insert_deletions(cp, tg), tg)


def init_params_device(cfg, device, seed=0):
    """N(0, 0.02) weights (GPT: out projections / sqrt(2L)), norm gains 1, on device."""
    import torch
    from paper_2412_14374_b200 import _lib
    from paper_2412_14374_b200.device import Param
    from paper_2412_14374_b200.ir import layout_size
    g = torch.Generator(device=device).manual_seed(seed)
    out = {}
    st = torch.cuda.current_stream(device).cuda_stream

    def make(layout, name_filter):
        n = layout_size(layout)
        m = torch.zeros(n, device=device)
        for name, (off, dims) in layout.items():
            if name == "__size__":
                continue
            sz = int(np.prod(dims))
            if name.endswith("_g"):
                m[off:off + sz] = 1.0
            elif name.startswith("w"):
                std = 0.02 / np.sqrt(2 * cfg.layers) if name in ("w_o", "w_fc2", "w_down") else 0.02
                m[off:off + sz] = torch.randn(sz, device=device, generator=g) * std
        sh = torch.empty(n, device=device, dtype=torch.bfloat16)
        _lib.call("pc_cast", _lib.PC_F32, _lib.PC_BF16, n, m.data_ptr(), sh.data_ptr(), st)
        return Param(m, sh)

    out["w0"] = make(cfg.embed_layout(), None)
    for k in range(1, cfg.layers + 1):
        out[f"w{k}"] = make(cfg.block_layout(k == cfg.layers), None)
    if hasattr(cfg, "head_layout"):   # Llama: untied LM head
        out["wout"] = make(cfg.head_layout(), None)
    return out


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list = []  # (arrival time, csv line)
        self.window = None     # (t0, t1) of the timed region, perf_counter clock

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def wait_first(self, timeout_s: float = 5.0):
        """nvidia-smi needs up to ~1 s before its first sample: wait for it so a
        short timed region is still covered."""
        t_end = time.perf_counter() + timeout_s
        while self.proc is not None and not self.lines and time.perf_counter() < t_end:
            time.sleep(0.05)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        if self.window is not None and lines:
            t0, t1 = self.window
            inside = [x for x in lines if t0 - 0.1 <= x[0] <= t1 + 0.3]
            # a region shorter than the 200 ms period: the samples nearest to it
            lines = inside or sorted(lines, key=lambda x: abs(x[0] - 0.5 * (t0 + t1)))[:2]
        for _, ln in lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def gemm_shapes(cfg, P):
    """(M, N, K, transA, transB, epilogue, has_aux, has_u, fp32 out) of every
    tcgen05 GEMM of one stage step, with launches per microbatch: per GPT
    block and, on the last stage, the LM head.  Weight gradients accumulate
    into the running sum (device.py _wgrad_into: TMA reduce-add, ordered
    split-K) as in every microbatch after the first."""
    from paper_2412_14374_b200 import _lib as E
    T, d, f, V = cfg.tokens, cfg.d_model, cfg.d_ff, cfg.vocab
    WG = E.EPI_ACCUM | E.EPI_SPLITK_ORDERED
    if hasattr(cfg, "n_kv_heads"):   # Llama block (device.py _llama_block_fwd / _bwd)
        qw, ho = cfg.qkv_width, cfg.n_heads * cfg.head_dim
        block = [(T, qw, d, 0, 1, 0, 0, 0, 0),                                 # qkv
                 (T, d, ho, 0, 1, E.EPI_RESIDUAL, 1, 0, 0),                    # o (+h)
                 (T, 2 * f, d, 0, 1, 0, 0, 0, 0),                              # gate | up
                 (T, d, f, 0, 1, E.EPI_RESIDUAL, 1, 0, 0),                     # down (+h1)
                 (d, f, T, 1, 0, WG, 0, 0, 1),                                 # dW down
                 (T, f, d, 0, 1, 0, 0, 0, 0),                                  # dX down
                 (2 * f, d, T, 1, 0, WG, 0, 0, 1),                             # dW gate|up
                 (T, d, 2 * f, 0, 1, 0, 0, 0, 0),                              # dX gate|up
                 (d, ho, T, 1, 0, WG, 0, 0, 1),                                # dW o
                 (T, ho, d, 0, 1, 0, 0, 0, 0),                                 # dX o
                 (qw, d, T, 1, 0, WG, 0, 0, 1),                                # dW qkv
                 (T, d, qw, 0, 1, 0, 0, 0, 0)]                                 # dX qkv
        head = [(T, V, d, 0, 1, 0, 0, 0, 0), (T, d, V, 0, 1, 0, 0, 0, 0),
                (V, d, T, 1, 0, WG, 0, 0, 1)]
        return block, head
    block = [(T, 3 * d, d, 0, 1, E.EPI_BIAS, 0, 0, 0),                        # qkv
             (T, d, d, 0, 1, E.EPI_BIAS | E.EPI_RESIDUAL, 1, 0, 0),            # attn out
             (T, f, d, 0, 1, E.EPI_BIAS | E.EPI_GELU, 0, 1, 0),                # fc1
             (T, d, f, 0, 1, E.EPI_BIAS | E.EPI_RESIDUAL, 1, 0, 0),            # fc2
             (d, f, T, 1, 0, WG, 0, 0, 1),                                     # dW fc2
             (T, f, d, 0, 1, E.EPI_GELU_GRAD, 1, 0, 0),                        # dX fc2 (gelu')
             (f, d, T, 1, 0, WG, 0, 0, 1),                                     # dW fc1
             (T, d, f, 0, 1, 0, 0, 0, 0),                                      # dX fc1
             (d, d, T, 1, 0, WG, 0, 0, 1),                                     # dW out
             (T, d, d, 0, 1, 0, 0, 0, 0),                                      # dX out
             (3 * d, d, T, 1, 0, WG, 0, 0, 1),                                 # dW qkv
             (T, d, 3 * d, 0, 1, 0, 0, 0, 0)]                                  # dX qkv
    head = [(T, V, d, 0, 1, 0, 0, 0, 0), (T, d, V, 0, 1, 0, 0, 0, 0),
            (V, d, T, 1, 0, E.EPI_SPLITK_ZERO_C, 0, 0, 1)]
    return block, head


def gemm_args(shape, st):
    """Operands and pc_gemm arguments for one entry of gemm_shapes."""
    import torch
    from paper_2412_14374_b200 import _lib
    Mm, N, K, ta, tb, epi, has_aux, has_u, f32 = shape
    A = torch.randn((K, Mm) if ta else (Mm, K), device="cuda").bfloat16()
    B = torch.randn((N, K) if tb else (K, N), device="cuda").bfloat16()
    C = torch.zeros(Mm, N, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
    bias = torch.zeros(N, device="cuda")
    if epi & _lib.EPI_SPLITK_ORDERED:
        aux, ldaux = torch.zeros(1 << 16, dtype=torch.int32, device="cuda"), 1 << 16
    else:
        aux = torch.randn(Mm, N, device="cuda").bfloat16() if has_aux else None
        ldaux = N
    U = torch.empty(Mm, N, device="cuda", dtype=torch.bfloat16) if has_u else None
    args = (_lib.PC_BF16, _lib.PC_F32 if f32 else _lib.PC_BF16, ta, tb, Mm, N, K,
            A.data_ptr(), A.shape[1], B.data_ptr(), B.shape[1], C.data_ptr(), N, epi,
            bias.data_ptr(), aux.data_ptr() if aux is not None else None, ldaux,
            U.data_ptr() if U is not None else None, N, st.cuda_stream)
    return args, (A, B, C, bias, aux, U)


def gemm_roofline(cfg, P, stage_blocks, step_ms, peak, M=M_MICRO):
    """Average achieved TFLOP/s of the tcgen05 GEMM over the shape mix of one
    stage step, each GEMM issued exactly as device.py issues it (operand
    majors, fused epilogue, split-K hint) and timed with CUDA events on its
    launch stream (warm, back to back, replayed from a CUDA graph); share of
    the step it accounts for."""
    import torch
    from paper_2412_14374_b200 import _lib
    block, head = gemm_shapes(cfg, P)
    st = torch.cuda.Stream()
    tot_flops = tot_ms = 0.0
    per = []
    traffic = gemm_traffic()
    # GPT blocks issue the attention-output and qkv weight gradients as one
    # grouped launch (device.py _wgrad_pair_into): time them that way
    WG = _lib.EPI_ACCUM | _lib.EPI_SPLITK_ORDERED
    d = cfg.d_model
    pair = None
    if not hasattr(cfg, "n_kv_heads") and (3 * d) % 256 == 0 and \
            os.environ.get("PP200_WGRAD_PAIR", "1") != "0":
        wo, wq = (d, d, cfg.tokens, 1, 0, WG, 0, 0, 1), (3 * d, d, cfg.tokens, 1, 0, WG, 0, 0, 1)
        if wo in block and wq in block:
            block = [s for s in block if s not in (wo, wq)] + [("pair", 3 * d, d, d, cfg.tokens)]
    for shape, count in [(s, stage_blocks) for s in block] + [(s, 1 if P == 1 else 0) for s in head]:
        if count == 0:
            continue
        if os.environ.get("PP200_BENCH_VERBOSE") == "1":
            print(f"[bench] roofline shape {shape}", file=sys.stderr, flush=True)
        if shape[0] == "pair":
            _, M1, M2, N, K = shape
            A1 = torch.randn(K, M1, device="cuda").bfloat16()
            A2 = torch.randn(K, M2, device="cuda").bfloat16()
            B1 = torch.randn(K, N, device="cuda").bfloat16()
            B2 = torch.randn(K, N, device="cuda").bfloat16()
            C1 = torch.zeros(M1, N, device="cuda")
            C2 = torch.zeros(M2, N, device="cuda")
            flags = torch.zeros(1 << 16, dtype=torch.int32, device="cuda")
            fn = "pc_gemm_wgrad_pair"
            args = (M1, M2, N, K, A1.data_ptr(), M1, B1.data_ptr(), N, C1.data_ptr(), N,
                    A2.data_ptr(), M2, B2.data_ptr(), N, C2.data_ptr(), N, WG, flags.data_ptr(),
                    flags.numel(), st.cuda_stream)
            keep = (A1, A2, B1, B2, C1, C2, flags)
            Mm, ta, tb, epi = M1 + M2, 1, 0, WG
        else:
            Mm, N, K, ta, tb, epi = shape[:6]
            fn = "pc_gemm"
            args, keep = gemm_args(shape, st)
        # device time of back-to-back launches, issued from a CUDA graph as in
        # the step (host launch cost would otherwise pace the short GEMMs)
        with torch.cuda.stream(st):
            for _ in range(3):
                _lib.call(fn, *args)
            reps = 10
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for _ in range(reps):
                    _lib.call(fn, *args)
            g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            g.replay()
            e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        del g
        fl = 2.0 * Mm * N * K
        row = {"shape": [Mm, N, K, ta, tb], "epilogue": epi, "ms": round(ms, 4),
               "tflops": round(fl / ms / 1e9, 1), "launches_per_mb": count}
        if shape[0] == "pair":
            row["pair"] = [shape[1], shape[2]]
            k1, k2 = f"{shape[1]}x{N}x{K}:{epi}", f"{shape[2]}x{N}x{K}:{epi}"
            if k1 in traffic and k2 in traffic:
                row["dram_bytes"] = traffic[k1] + traffic[k2]
        else:
            key = f"{Mm}x{N}x{K}:{epi}"
            if key in traffic:
                row["dram_bytes"] = traffic[key]
        per.append(row)
        tot_flops += fl * count * M
        tot_ms += ms * count * M
        del keep
    achieved = tot_flops / tot_ms / 1e9 if tot_ms else 0.0
    # DRAM bytes per launch over the same mix, from the committed ncu --set full capture
    have = [r for r in per if "dram_bytes" in r]
    tr = (sum(r["dram_bytes"] * r["launches_per_mb"] for r in have) /
          sum(r["launches_per_mb"] for r in have)) if have and len(have) == len(per) else None
    return {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak, "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4),
            "traffic": None if tr is None else round(tr),
            "traffic_source": f"profiles/{_gemm_mix_file().name} (ncu --set full, per launch)"
            if tr is not None else None,
            "kernel": "tc_gemm_kernel (tcgen05.mma kind::f16, TMA, TMEM)",
            "share_of_step": round(tot_ms / step_ms, 3) if step_ms else None,
            "shapes": per}


def _gemm_mix_file() -> Path:
    """The newest committed ncu --set full capture of the GEMM mix."""
    d = Path(__file__).resolve().parent / "profiles"
    for name in ("r02_ncu_gemm_mix.json", "r01_ncu_gemm_mix.json"):
        if (d / name).exists():
            return d / name
    return d / "r02_ncu_gemm_mix.json"


def gemm_traffic() -> dict:
    """{"MxNxK:epilogue": dram bytes read + written per launch} from the
    committed ncu --set full capture of the GEMM mix (tools/ncu_gemm_mix.py)."""
    p = _gemm_mix_file()
    try:
        return {k: v["dram_bytes"] for k, v in json.loads(p.read_text())["shapes"].items()}
    except (OSError, ValueError, KeyError):
        return {}


def _oracle_sample(wl):
    """Time the float64 numpy oracle (oracle/gpt.py or oracle/llama.py: the
    reference's run_reference loop, executor.py:117-134, over this model's
    vocabulary) on a bounded sample of workload ``wl`` on the host cores.
    C2: the full 12-layer model on one 1024-token sequence.  Larger configs
    (a full-size sequence alone is minutes to hours of fp64 CPU work): a slice
    of the same width -- 1 block + embedding + LM head on one shorter
    sequence -- whose time per token is scaled to the full model by the FLOP
    ratio (both counted with ir.*Config.flops_per_token).  Returns
    (tokens/s of the full model, seconds timed, description)."""
    from threadpoolctl import threadpool_limits
    from paper_2412_14374_b200 import ir as I
    kw = wl["kw"]
    if wl["family"] == "ffn":
        # one whole microbatch of the same configuration through run_reference
        from oracle import ffn as of
        rng = np.random.default_rng(0)
        L, w, rows = kw["layers"], kw["width"], kw["microbatch_size"]
        params = of.init_params({f"w{k}": (w, w) for k in range(L)}, rng)
        batch = of.init_batch(1, rows, w, rng)
        with threadpool_limits(limits=os.cpu_count()):
            t0 = time.perf_counter()
            of.run_reference_ffn(params, batch, 1, L, False)
            dt = time.perf_counter() - t0
        return rows / dt, dt, (f"oracle/ffn.py run_reference (bit-identical restatement of "
                               f"executor.py:117-134, numpy float64), 1 microbatch x {rows} rows "
                               f"of the same config ({dt:.1f} s)")
    llama = wl["family"] == "llama"
    full = (I.LlamaConfig if llama else I.GPTConfig)(**kw)
    small = kw is C2
    layers = kw["layers"] if small else 1
    seq = kw["seq_len"] if small else 256
    sample = dict(kw, layers=layers, seq_len=seq, microbatch_size=1)
    samp = (I.LlamaConfig if llama else I.GPTConfig)(**sample)
    rng = np.random.default_rng(0)
    if llama:
        from oracle import llama as om
        oc = dict(layers=layers, d=kw["d_model"], heads=kw["n_heads"], kv_heads=kw["n_kv_heads"],
                  ff=kw["d_ff"], vocab=kw["vocab"], seq=seq, mbs=1, theta=10000.0)
        params = om.init_params(oc, rng)
        tokens = om.init_tokens(oc, 1, rng)
        pos = om.positions(oc, 1)
        run = lambda: om.run_reference_llama(params, tokens, pos, oc)
        what = "oracle/llama.py"
    else:
        from oracle import gpt as og
        oc = dict(layers=layers, d=kw["d_model"], heads=kw["n_heads"], ff=kw["d_ff"],
                  vocab=kw["vocab"], seq=seq, mbs=1)
        params = og.init_params(oc, rng)
        tokens = og.init_tokens(oc, 1, rng)
        run = lambda: og.run_reference_gpt(params, tokens, oc)
        what = "oracle/gpt.py"
    with threadpool_limits(limits=os.cpu_count()):
        t0 = time.perf_counter()
        run()
        dt = time.perf_counter() - t0
    tok_s = seq / dt * (samp.flops_per_token() / full.flops_per_token())
    desc = (f"{what} float64 numpy fwd+bwd+SGD, {layers} block(s) at full width, 1 sequence x "
            f"{seq} tokens ({dt:.1f} s)")
    if not small:
        desc += "; tokens/s scaled to the full model by the FLOP-per-token ratio"
    return tok_s, dt, desc


def cpu_baseline(wl):
    tok_s, dt, desc = _oracle_sample(wl)
    return {"value": round(tok_s, 3), "unit": "tokens/s", "cores": os.cpu_count(),
            "kind": "port", "sample": desc}


def run_reference_impl(args, rank, world):
    """--impl reference: the reference's CPU implementation of the path (the
    numpy oracle port; the Python reference cannot travel to the GPU box),
    on the host cores, one bounded sample of the workload per step."""
    if rank != 0:
        return 0
    wl = WORKLOADS[args.workload]
    for _ in range(min(args.warmup, 1)):
        _oracle_sample(wl)
    rates, times, desc = [], [], ""
    for _ in range(args.steps):
        tok_s, dt, desc = _oracle_sample(wl)
        rates.append(tok_s)
        times.append(dt)
    tok_s = float(np.mean(rates))
    from paper_2412_14374_b200 import ir as I
    if wl["family"] == "ffn":
        fpt = ffn_flops_per_row(wl["kw"])
    else:
        fpt = (I.LlamaConfig if wl["family"] == "llama" else I.GPTConfig)(**wl["kw"]).flops_per_token()
    line = {
        "impl": "reference", "metric": METRIC,
        "value": round(tok_s, 3), "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1000 * float(np.mean(times)), 2),
        "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl["name"], "schedule": wl["schedule"],
                   "microbatches": wl["M"],
                   "sample": desc + " per step (bounded CPU sample)"},
        "model_tflops_per_gpu": round(fpt * tok_s / 1e12, 5),
        "cpu_baseline": {"value": round(tok_s, 3), "unit": "tokens/s", "cores": os.cpu_count(),
                         "kind": "port", "sample": desc},
        "e2e": {"value": round(tok_s, 3), "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _isolate_stdout():
    """Native writes to fd 1 (NCCL's "NCCL version" banner, printed with printf under
    NCCL_DEBUG=WARN / VERSION) go to stderr; Python's sys.stdout keeps the original
    stdout, so rank 0's stdout carries only the one JSON line."""
    sys.stdout.flush()
    keep = os.dup(1)
    os.dup2(2, 1)
    sys.stdout = os.fdopen(keep, "w", buffering=1)


def main():
    _isolate_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--microbatches", type=int, default=None,
                    help="default: the workload's (C2: 8, C3: 16)")
    ap.add_argument("--workload", default="C2", choices=sorted(WORKLOADS))
    ap.add_argument("--schedule", default=None, choices=["1f1b", "interleaved"],
                    help="default: the workload's (C4: interleaved)")
    ap.add_argument("--vstages", type=int, default=None,
                    help="virtual stages per GPU for interleaved 1F1B (default: the workload's)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--gantt", default=None, help="write the measured timeline as an SVG Gantt chart")
    ap.add_argument("--remat", default="none", choices=["none", "full-per-stage"],
                    help="full-per-stage: stages keep their forward feeds and replay the "
                         "forward in the backward (model FLOPs unchanged in the metric)")
    ap.add_argument("--no-graph", action="store_true",
                    help="issue every step from Python instead of replaying the captured graph")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference_impl(args, rank, world)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2412_14374_b200 import _lib
    from paper_2412_14374_b200.executor import PipelineEngine

    P = world
    wl = WORKLOADS[args.workload]
    wl_kw, wl_name = wl["kw"], wl["name"]
    M = args.microbatches or wl["M"]
    Vv = args.vstages if args.vstages is not None else wl["V"]
    sched = args.schedule or wl["schedule"]
    ffn_wl = wl["family"] == "ffn"
    mode = "fp64" if ffn_wl else "bf16"
    cfg, tg, cp = build_plan(P, wl_kw, M, mode=mode, family=wl["family"], schedule=sched, V=Vv)
    sched_used = "interleaved" if (sched == "interleaved" and P > 1 and Vv > 1) else "1f1b"
    dev = torch.device("cuda", local)
    rng = np.random.default_rng(1234)
    if ffn_wl:
        g = torch.Generator(device=dev).manual_seed(0)
        w_ = wl_kw["width"]
        params = {q: torch.randn(w_, w_, device=dev, generator=g, dtype=torch.float64) * 0.4
                  / np.sqrt(w_) for q in sorted(tg.partition.graph.params)}
        tokens_host = rng.standard_normal((M * wl_kw["microbatch_size"], w_))
    else:
        params = init_params_device(cfg, dev)
        tokens_host = rng.integers(0, cfg.vocab, size=(M * cfg.microbatch_size, cfg.seq_len),
                                   dtype=np.int32)
    if wl["family"] == "llama":
        # token ids + position ids (the skip tensors every later stage reads)
        pos_host = np.tile(np.arange(cfg.seq_len, dtype=np.int32), (M * cfg.microbatch_size, 1))
        tokens_dev = {"x": torch.from_numpy(tokens_host).to(dev),
                      "pos": torch.from_numpy(pos_host).to(dev)}
        tokens_pinned = {"x": torch.from_numpy(tokens_host).pin_memory(),
                         "pos": torch.from_numpy(pos_host).pin_memory()}
        h2d_bytes = int(tokens_host.nbytes + pos_host.nbytes)
    else:
        tokens_dev = torch.from_numpy(tokens_host).to(dev)
        tokens_pinned = torch.from_numpy(tokens_host).pin_memory()
        h2d_bytes = int(tokens_host.nbytes)
    t_start = time.perf_counter()

    def progress(msg):
        if rank == 0:
            print(f"[bench {time.perf_counter() - t_start:7.1f}s] {msg}", file=sys.stderr, flush=True)

    progress(f"{args.workload}: plan built, {len(tg.partition.fwd_programs)} stages, M={M}")
    eng = PipelineEngine(cp, tg, mode=mode, gpt=None if ffn_wl else cfg, remat=args.remat)
    # resident training state: every step (eager or replayed) is a real SGD
    # step on the previous step's weights, tied w0 re-broadcast included
    eng.load_params(params)
    del params
    use_graph = not args.no_graph
    for _ in range(2):   # eager warm-up: NCCL connections, kernel attributes, allocator
        eng.step(None, tokens_dev, lr=1e-4, timeout_s=600, to_host=False)
    torch.cuda.synchronize()
    progress("eager warm-up steps done")
    if use_graph:
        cap = eng.capture(None, tokens_dev, lr=1e-4)
        run = lambda b: cap.replay(None if b is tokens_dev else b)
    else:
        run = lambda b: eng.step(None, b, lr=1e-4, timeout_s=600, to_host=False)
    for _ in range(max(args.warmup, 3)):
        run(tokens_dev)
    torch.cuda.synchronize()
    if os.environ.get("PP200_NCU_ONE_STEP") == "1":
        # `ncu --profile-from-start off`: the launch list of exactly one timed
        # step (graph replay); numbers printed by such a run are not bench values
        torch.cuda.profiler.start()
        run(tokens_dev)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    progress("captured, warm")
    # ---- device-resident timed region ----
    torch.cuda.reset_peak_memory_stats(dev)
    clocks = ClockSampler(local)
    clocks.start()
    clocks.wait_first()
    barrier()
    launches0 = _lib.launch_count
    t0 = time.perf_counter()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        run(tokens_dev)
    ev1.record()
    barrier()
    wall = time.perf_counter() - t0
    clocks.window = (t0, t0 + wall)
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    # peak HBM of the timed steps: torch allocations (the graph pool, params,
    # activations) plus this rank's peer receive slots (cudaMalloc'd outside torch)
    peak_hbm = torch.cuda.max_memory_allocated(dev) + eng.peer_bytes
    # kernels per step: the captured graph's kernel nodes (libpp200 calls when eager)
    launches = cap.kernels if use_graph else int((_lib.launch_count - launches0) / args.steps)
    clk = clocks.stop()

    progress(f"timed: {ms:.1f} ms/step")
    # ---- e2e through the public API: pinned host tokens -> device, losses -> host ----
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        res = run(tokens_pinned)
        if res.losses is not None:
            res.losses.cpu()
    e1.record()
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)

    progress(f"e2e: {e2e_ms:.1f} ms/step")
    # ---- one instrumented step (same warmed engine) for the bubble ----
    barrier()
    if use_graph:
        cap.release()   # its graph memory pool: the instrumented capture needs its own
        cap_tl = eng.capture(None, tokens_dev, lr=1e-4, timeline=True)
        barrier()
        cap_tl.replay()
        barrier()
        timeline = cap_tl.timeline()
        cap_tl.release()
    else:
        timeline = eng.step(None, tokens_dev, lr=1e-4, timeout_s=600, to_host=False,
                            timeline=True).stats.timeline
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, timeline)
        timeline = [e for part in gathered for e in part]
    progress("timeline step done")
    from paper_2412_14374_b200.executor import RunStats
    from paper_2412_14374_b200 import timeline as TL
    bubble = RunStats(timeline=timeline).bubble_fraction(P)
    # achievable ideal: the plan replayed with the measured task durations and
    # free transfers / dispatch
    achievable = TL.replay(cp, TL.task_durations(timeline)).bubble_fraction(P)
    # per-GPU busy time of the loop tasks: the balance the stage boundaries reached
    busy = [0.0] * P
    for a, kind, _, t0_, t1_ in timeline:
        if kind in ("fwd", "bwd") and a < P:
            busy[a] += t1_ - t0_
    if args.gantt and rank == 0:
        with open(args.gantt, "w") as f:
            f.write(TL.render_svg(timeline, P, title=f"{args.workload} 1F1B P={P} M={M} measured,"))

    tokens_per_step = M * (wl_kw["microbatch_size"] if ffn_wl else cfg.tokens)
    value = tokens_per_step / (ms / 1000)
    e2e = tokens_per_step / (e2e_ms / 1000)
    flops_step = (ffn_flops_per_row(wl_kw) if ffn_wl else cfg.flops_per_token()) * tokens_per_step
    tflops_gpu = flops_step / (ms / 1000) / P / 1e12
    burst, sustained, hbm, peak_kind = peaks()
    Vi = Vv if sched_used == "interleaved" else 1
    ideal = (P - 1) / (Vi * M + P - 1)   # simulator.py:346-348

    if rank == 0:
        # blocks on rank 0: its stages are s = 0, P, 2P, ... (schedules.py:60-61)
        fp = tg.partition.fwd_programs
        stage_blocks = sum(1 for st in range(0, len(fp), P) for op in fp[st].ops
                           if op.kind in ("gpt-block", "llama-block"))
        progress("bubble / achievable computed")
        if ffn_wl:
            # fp64 DFMA GEMMs: no bf16 tensor-core roofline applies (the FFN workload
            # exists for the same-config comparison with the reference's CPU path)
            roof = None
        else:
            roof = gemm_roofline(cfg, P, stage_blocks, ms, burst, M)
            roof["peak_kind"] = peak_kind
        progress("roofline measured")
        cpu = None if args.no_cpu_baseline else cpu_baseline(wl)
        progress("cpu baseline measured")
        mbs_ = wl_kw["microbatch_size"]
        seq_ = 1 if ffn_wl else cfg.seq_len
        line = {
            "metric": METRIC,
            "value": round(value, 1), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64" if ffn_wl else "bf16",
            "data": ("synthetic N(0,1) rows (tokens = rows), random-init weights" if ffn_wl
                     else "synthetic tokens, random-init weights"),
            "config": {"workload": wl_name,
                       "global_batch": M * mbs_, "seq_len": seq_,
                       "microbatches": M, "microbatch_size": mbs_,
                       "schedule": sched_used, "virtual_stages_per_gpu": Vv if sched_used ==
                       "interleaved" else 1, "stages": len(tg.partition.fwd_programs),
                       "yields": list(cfg.yields or []),
                       "parallelism": f"pp{P}", "l2": "inputs > L2 (no flush needed)",
                       "issue": "cuda-graph replay per actor" if use_graph else "python per op",
                       "transport": eng.transport if world > 1 else None,
                       "remat": args.remat,
                       "training": "resident params, in-place SGD each step"
                                   + (", tied w0 re-broadcast to the head stage"
                                      if P > 1 and not ffn_wl else "")},
            "model_tflops_per_gpu": round(tflops_gpu, 1),
            "peak_hbm_gb_rank0": round(peak_hbm / 1e9, 2),
            "peak_hbm_covers": "timed steps: torch allocator peak (reset before the timed region) "
                               "+ peer receive slots; excludes NCCL-internal buffers",
            "frac_of_bf16_peak": None if ffn_wl else round(tflops_gpu / burst, 4),
            "bubble": {"measured": round(bubble, 4), "ideal": round(ideal, 4),
                       "achievable": round(achievable, 4),
                       "busy_ms_per_gpu": [round(b, 3) for b in busy]},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e, 1), "unit": "tokens/s",
                    "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": 4 * M},
            "gpu_launches": launches,
            "clocks": clk,
            "wall_s": round(wall, 3),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        # Captured graphs hold references to the per-channel NCCL communicators;
        # tearing those down blocks, so ranks leave right after a final barrier
        # (process exit releases every GPU resource).
        dist.barrier()
        sys.stdout.flush()
        sys.stderr.flush()
        os._exit(0)
    if use_graph:
        del cap
    eng.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
