"""Stage compute on one B200: the GPU counterpart of the reference's op
interpreter (``eval_op``/``evaluate_ops``, pkg/src/pipecraft/executor.py:59-103)
and task payloads (``_run_task``, executor.py:316-346).

Every op is a libpp200 launch on the actor's compute stream (no host sync, no
torch compute kernels; torch only allocates memory).  Values are device
tensors; a transposed value is a zero-copy view that becomes a GEMM operand
major; ``Act`` carries the saved-for-backward tensors an op attaches to its
first operand (the stash keeps that value alive, exactly the reference's stash
dict, executor.py:326-327).

Compute modes
  fp64  float64 everywhere (FFN oracle mode: the reference's own 1e-12 tests)
  fp32  float32, FFMA GEMMs (no TF32), fp32 parity mode (rtol 1e-5)
  bf16  bf16 activations, tcgen05 GEMMs with fp32 accumulation, fp32 master
        params + bf16 shadow, fp32 gradients and accumulators (rtol 2e-2)
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import call
from .ir import GPTConfig, OpNode, StagePartition, layout_size

RMS_EPS = 1e-5  # oracle/llama.py RMS_EPS
LN_EPS = 1e-5

_PC = {torch.float32: _lib.PC_F32, torch.float64: _lib.PC_F64, torch.bfloat16: _lib.PC_BF16,
       torch.int32: _lib.PC_I32}


@dataclass(frozen=True)
class Mode:
    name: str
    act: torch.dtype       # activations / activation gradients
    master: torch.dtype    # parameters and parameter gradients

    @property
    def pc_act(self) -> int:
        return _PC[self.act]

    @property
    def pc_master(self) -> int:
        return _PC[self.master]


MODES = {
    "fp64": Mode("fp64", torch.float64, torch.float64),
    "fp32": Mode("fp32", torch.float32, torch.float32),
    "bf16": Mode("bf16", torch.bfloat16, torch.float32),
}


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


class Trans:
    """Lazy transpose of a 2-D value (reference `transpose`, executor.py:78-79)."""

    __slots__ = ("base",)

    def __init__(self, base):
        self.base = base


class Act:
    """A device activation plus tensors saved for backward, keyed by op id."""

    __slots__ = ("t", "saved")

    def __init__(self, t: torch.Tensor):
        self.t = t
        self.saved: dict = {}


_ABLATE_BIAS = os.environ.get("PP200_ABLATE_BIAS_GRAD") == "1"
# Profiling ablations (results are garbage while set): comma-separated subset of
# attn_fwd, attn_bwd, wgrad, lnp (LayerNorm / RMSNorm parameter gradients) --
# the step time without that work bounds what optimising it can save.
_ABLATE = set(filter(None, os.environ.get("PP200_ABLATE", "").split(",")))
_LN_PARAMS_MAIN = os.environ.get("PP200_LN_PARAMS_MAIN") == "1"   # A/B switch for profiling
# A/B switch, off by default: LayerNorm dx + parameter-gradient partial rows in one pass
# (pc_layernorm_bwd_partials) with the column sums on the side stream.  Measured on C2
# N=1 it is slower (75.0-75.6 vs 71.3-72.2 ms): the compute-stream kernel loses more to
# its row-chunked grid than the side-stream reduction it replaces costs.
_LN_FUSED = os.environ.get("PP200_LN_FUSED", "0") == "1"
# A/B switch, on by default: a GPT block's LN2 parameter gradients and its fc2 /
# attention-output bias gradients in one side-stream pass (pc_layernorm_param_bias_grads)
# instead of three column-sum launches; bitwise equal either way.
_LN_BIAS_FUSED = os.environ.get("PP200_LN_BIAS_FUSED", "1") != "0"
# A/B switch: 0 = logits GEMM then the stand-alone cross-entropy kernel (pc_xent_fwd_bwd)
_XENT_FUSED = os.environ.get("PP200_XENT_FUSED", "1") != "0"
# A/B switch: 0 = bf16 column sums through the two-stage workspace kernel instead of
# the one-pass cluster reduction (pc_colsum_set_cluster)
_COLSUM_CLUSTER = os.environ.get("PP200_COLSUM_CLUSTER", "1") != "0"
# A/B switch: 0 = the attention-output and qkv weight gradients as two GEMMs
_WGRAD_PAIR = os.environ.get("PP200_WGRAD_PAIR", "1") != "0"
# A/B switch: 0 = the compute stream waits for each GPT block's side-stream work
# (weight / bias / LayerNorm-parameter gradients) before the next block
_DEFER_JOIN = os.environ.get("PP200_DEFER_JOIN", "1") != "0"
# deferred side-stream pieces (one per block backward / head weight gradient) in
# flight before the compute stream waits for the oldest: bounds the tensors kept
# alive for them (a one-stage C5 program would otherwise keep every block's);
# C2 N=1 same box: depth 3 70.35 ms, unbounded 70.36 / 70.14 ms
_DEFER_DEPTH = int(os.environ.get("PP200_DEFER_DEPTH", "3"))


class PeerBuf:
    """A message slot in another GPU's memory (NVLink peer mapping): the
    producing kernel of a sent value writes here directly.  Only its address
    is used (kernels take raw pointers); it is never read on this GPU."""

    __slots__ = ("ptr", "shape", "dtype")

    def __init__(self, ptr: int, shape, dtype):
        self.ptr, self.shape, self.dtype = ptr, tuple(shape), dtype

    def data_ptr(self) -> int:
        return self.ptr

    def numel(self) -> int:
        return math.prod(self.shape)

    def element_size(self) -> int:
        return torch.empty((), dtype=self.dtype).element_size()

    def is_contiguous(self) -> bool:
        return True


@dataclass
class Param:
    """A parameter as stored on an actor: fp32 master (+ bf16 shadow in bf16 mode)."""

    master: torch.Tensor
    shadow: torch.Tensor | None = None
    # bf16 shadow with each GPT block matrix stored transposed (same flat
    # offsets), built lazily once per step (DeviceOps.step_epoch) for the
    # data-gradient GEMMs
    shadow_t: torch.Tensor | None = None
    shadow_t_epoch: int = -1

    def compute(self) -> torch.Tensor:
        return self.shadow if self.shadow is not None else self.master


def tensor_of(v) -> torch.Tensor:
    if isinstance(v, Act):
        return v.t
    if isinstance(v, Param):
        return v.compute()
    if isinstance(v, Trans):
        raise TypeError("transposed view used where a tensor is required")
    return v


def strip(v):
    """The wire form of a value: what crosses a channel (no saved state)."""
    if isinstance(v, Act):
        return v.t
    return v


@dataclass
class _StagePlan:
    fused_into_prev: set = field(default_factory=set)     # op indices skipped
    epilogue: dict = field(default_factory=dict)          # op index -> (kind, partner idx)


class DeviceOps:
    """Executes stage programs and task payloads for one actor on one device."""

    def __init__(self, p: StagePartition, mode: Mode, device: torch.device,
                 stream: torch.cuda.Stream, gpt: GPTConfig | None = None):
        self.p = p
        self.mode = mode
        self.device = device
        self.stream = stream
        self.gpt = gpt
        self._side_pending = False   # side-stream work not yet joined (run_ops joins it)
        # (event, tensors) per deferred piece of side-stream work: the tensors it
        # reads stay alive until the compute stream has waited for its event
        # (not record_stream: under CUDA-graph capture that defers every such free
        # to the end of the capture, which ran C4 / C3-M64 out of memory)
        self._side_ring: list = []
        if not _COLSUM_CLUSTER:
            call("pc_colsum_set_cluster", 0)
        self._plans: dict[int, _StagePlan] = {}
        # {param-grad value: fp32 accumulator} for the stage-bwd task being run:
        # the producer adds its partial straight onto the running sum (the
        # grad-merge `add` that follows becomes a rename, see _Actor.run_task)
        self.acc_into: dict = {}
        # {value: PeerBuf} for the task being run: outputs that are sent to a
        # peer-memory channel are produced straight into the receiver's slot
        self.place: dict = {}
        self._split_flags = None
        self.fuse_acc = os.environ.get("PP200_FUSE_ACC", "1") != "0"
        self._consumers = {}
        for op in p.graph.ops:
            for v in op.operands:
                self._consumers.setdefault(v, []).append(op)
        self._stage_outputs = set()
        for bp in p.bwd_programs:
            self._stage_outputs.update(bp.grads_out)
        for fp in p.fwd_programs:
            self._stage_outputs.update(fp.boundary_out)
            self._stage_outputs.update(fp.stash)
        if gpt is not None:
            self._elay = gpt.embed_layout()
            self._blay = {False: gpt.block_layout(False), True: gpt.block_layout(True)}
            if hasattr(gpt, "head_layout"):  # Llama-style: untied LM head
                self._hlay = gpt.head_layout()
        self._emb_ws = None
        self._red = None
        self._red_side = None
        self._side_stream = None
        self._xent_ws = None     # LM-head softmax statistics (pc_lmhead_xent_fwd)
        self._ln_parts: dict = {}  # LayerNorm parameter-gradient partial rows per LayerNorm
        self.step_epoch = 0  # bumped by the executor at every step

    # ------------------------------------------------------------------ alloc
    def red_ws(self, rows: int, cols: int, side: bool = False) -> tuple[int, int]:
        """Scratch for the two-stage column reductions, one per stream of the
        actor (reuse is ordered within each stream)."""
        nb = ctypes.c_int64(0)
        call("pc_reduce_workspace_bytes", rows, cols, ctypes.byref(nb))
        key = "_red_side" if side else "_red"
        buf = getattr(self, key)
        if buf is None or buf.numel() < nb.value:
            n = (nb.value + 3) // 4 * 4
            buf = self.empty((n,), torch.uint8)
            call("pc_fill", _lib.PC_F32, n // 4, 0.0, buf.data_ptr(), self.st)  # counters
            if side:  # the side stream must see the zeroed counters
                self._fork()
            setattr(self, key, buf)
        return buf.data_ptr(), buf.numel()

    def _side(self) -> torch.cuda.Stream:
        """Second stream of the actor: weight gradients run here, beside the
        data-gradient chain, and fill the wave tails of its GEMMs."""
        if self._side_stream is None:
            if os.environ.get("PP200_SINGLE_STREAM") == "1":  # A/B switch for profiling
                self._side_stream = self.stream
            else:
                self._side_stream = torch.cuda.Stream(device=self.device)
        return self._side_stream

    def _fork(self):
        """Side stream waits for everything issued so far on the compute stream."""
        ev = torch.cuda.Event()
        ev.record(self.stream)
        self._side().wait_event(ev)

    def _join(self):
        ev = torch.cuda.Event()
        ev.record(self._side())
        self.stream.wait_event(ev)

    def empty(self, shape, dtype) -> torch.Tensor:
        return torch.empty(shape, dtype=dtype, device=self.device)

    def _out(self, value: str, shape, dtype):
        """Output buffer of ``value``: its peer slot when placed (directly or
        through the yield-marker that makes it the stage output), else new."""
        pb = self.place.get(value)
        if pb is None and self.place:
            for u in self._consumers.get(value, ()):
                if u.kind == "yield-marker" and u.result in self.place:
                    pb = self.place[u.result]
        if pb is not None and pb.shape == tuple(shape) and pb.dtype == dtype:
            return pb
        return self.empty(shape, dtype)

    def _placed_elem(self, op, index: int, shape, dtype):
        """As _out for the ``index``-th element of a tuple-valued op."""
        if self.place:
            for u in self._consumers.get(op.result, ()):
                if u.kind == "tuple-get" and u.attr("index") == index and u.result in self.place:
                    return self._out(u.result, shape, dtype)
        return self.empty(shape, dtype)

    def zeros(self, shape, dtype) -> torch.Tensor:
        t = self.empty(shape, dtype)
        call("pc_fill", _PC[dtype], t.numel(), 0.0, t.data_ptr(), self.st)
        return t

    @property
    def st(self) -> int:
        return self.stream.cuda_stream

    # ---------------------------------------------------------- stage programs
    def run_ops(self, ops: list[OpNode], env: dict) -> dict:
        plan = self._plan(ops)
        for k, op in enumerate(ops):
            if k in plan.fused_into_prev:
                continue
            self._eval(op, env, k, ops, plan)
        # the blocks' side-stream gradient work joins at the end of the stage
        # program (every reader of those gradients comes after it)
        self._join_side()
        return env

    def _defer_side(self, tensors):
        """Side-stream work just enqueued reads ``tensors``; the compute stream
        goes on without waiting for it.  Once more than _DEFER_DEPTH pieces are
        in flight the compute stream waits for the oldest, whose tensors may
        then go back to the allocator."""
        ev = torch.cuda.Event()
        ev.record(self._side())
        self._side_ring.append((ev, tensors))
        self._side_pending = True
        while len(self._side_ring) > _DEFER_DEPTH:
            self.stream.wait_event(self._side_ring.pop(0)[0])

    def _join_side(self):
        if self._side_pending:
            self._join()
            self._side_pending = False
            self._side_ring.clear()

    def _plan(self, ops: list[OpNode]) -> _StagePlan:
        """Peephole fusion over one stage program: matmul -> relu becomes one
        GEMM with a ReLU epilogue; a dX matmul whose only consumer is a
        relu-grad becomes one GEMM with a relu-grad epilogue."""
        key = id(ops)
        plan = self._plans.get(key)
        if plan is not None:
            return plan
        plan = _StagePlan()
        idx = {op.result: k for k, op in enumerate(ops)}
        for k, op in enumerate(ops):
            if op.kind != "matmul":
                continue
            users = self._consumers.get(op.result, [])
            local = [u for u in users if u.result in idx and idx[u.result] > k]
            relu = [u for u in local if u.kind == "relu"]
            if relu:
                # z stays materialised (aux_out), so other readers are fine.
                j = idx[relu[0].result]
                plan.epilogue[k] = ("relu", j)
                plan.fused_into_prev.add(j)
                continue
            if len(users) != 1 or not local or op.result in self._stage_outputs:
                continue
            u = local[0]
            if u.kind == "relu-grad" and u.operands[0] == op.result and u.operands[1] != op.result:
                aux_src = u.operands[1]
                # the mask operand must already exist when the matmul runs
                if aux_src not in idx or idx[aux_src] < k:
                    plan.epilogue[k] = ("relu-grad", idx[u.result])
                    plan.fused_into_prev.add(idx[u.result])
        self._plans[key] = plan
        return plan

    def _eval(self, op: OpNode, env: dict, k: int, ops, plan: _StagePlan):
        kind = op.kind
        if kind in ("parameter-read", "input-read"):
            if op.result not in env:
                raise KeyError(f"{kind} {op.id}: value {op.result} was not fed")
            return
        a = env[op.operands[0]] if op.operands else None
        if kind == "yield-marker":
            env[op.result] = a
        elif kind == "transpose":
            env[op.result] = a.base if isinstance(a, Trans) else Trans(a)
        elif kind == "matmul":
            self._matmul(op, env, plan.epilogue.get(k), ops)
        elif kind == "relu":
            x = tensor_of(a)
            out = self.empty(x.shape, x.dtype)
            call("pc_ewise", _lib.EW_RELU, _PC[x.dtype], x.numel(), x.data_ptr(), None, 0,
                 out.data_ptr(), self.st)
            env[op.result] = out
        elif kind == "relu-grad":
            x, z = tensor_of(a), tensor_of(env[op.operands[1]])
            out = self.empty(x.shape, x.dtype)
            call("pc_ewise", _lib.EW_RELU_GRAD, _PC[x.dtype], x.numel(), x.data_ptr(),
                 z.data_ptr(), z.numel(), out.data_ptr(), self.st)
            env[op.result] = out
        elif kind == "add" and self._fused_add(op, env):
            pass
        elif kind in ("add", "scale", "mul"):
            x, y = tensor_of(a), tensor_of(env[op.operands[1]])
            out = self.empty(x.shape, x.dtype)
            opc = _lib.EW_ADD if kind == "add" else _lib.EW_MUL
            call("pc_ewise", opc, _PC[x.dtype], x.numel(), x.data_ptr(), y.data_ptr(), y.numel(),
                 out.data_ptr(), self.st)
            env[op.result] = out
        elif kind == "sub-sample-loss":
            x = tensor_of(a)
            out = self.empty((), x.dtype)
            call("pc_sumsq_half", _PC[x.dtype], x.numel(), x.data_ptr(), out.data_ptr(), self.st)
            env[op.result] = out
        elif kind == "sum-to":
            env[op.result] = self._sum_to(tensor_of(a), op.result_spec.dims)
        elif kind == "broadcast":
            env[op.result] = self._broadcast(tensor_of(a), op.result_spec.dims)
        elif kind == "slice":
            x = tensor_of(a)
            off, ln = op.attr("offset"), op.attr("length")
            env[op.result] = x.reshape(-1)[off:off + ln] if x.dim() == 1 else x[off:off + ln]
        elif kind == "concat":
            env[op.result] = self._concat([tensor_of(env[v]) for v in op.operands])
        elif kind == "tuple-get":
            env[op.result] = a[op.attr("index")]
        elif kind == "embed":
            env[op.result] = Act(self._embed(env))
        elif kind == "gpt-block":
            self._block_fwd(op, env)
        elif kind == "gpt-block-grad":
            env[op.result] = self._block_bwd(op, env, acc=self._acc_target(op, 1))
        elif kind == "lmhead-xent":
            env[op.result] = self._head_fwd(op, env)
        elif kind == "lmhead-xent-grad":
            env[op.result] = self._head_bwd(op, env, acc=self._acc_for_tuple(op, 1))
        elif kind == "embed-grad":
            env[op.result] = self._embed_bwd(op, env, acc=self._acc_for_value(op.result))
        elif kind == "llama-embed":
            env[op.result] = Act(self._llama_embed(op, env))
        elif kind == "llama-embed-grad":
            env[op.result] = self._llama_embed_bwd(op, env, acc=self._acc_for_value(op.result))
        elif kind == "llama-block":
            self._llama_block_fwd(op, env)
        elif kind == "llama-block-grad":
            env[op.result] = self._llama_block_bwd(op, env, acc=self._acc_target(op, 1))
        elif kind == "llama-head":
            env[op.result] = self._llama_head_fwd(op, env)
        elif kind == "llama-head-grad":
            env[op.result] = self._llama_head_bwd(op, env, acc=self._acc_for_tuple(op, 1))
        else:
            raise ValueError(f"no device rule for op kind {kind!r}")

    # ------------------------------------------------------------- FFN pieces
    @staticmethod
    def _operand(v):
        if isinstance(v, Trans):
            t = tensor_of(v.base)
            return t, 1, t.shape[1], t.shape[0]  # op(A) = A^T: rows = cols of base
        t = tensor_of(v)
        return t, 0, t.shape[0], t.shape[1]

    def _matmul(self, op: OpNode, env: dict, fuse, ops):
        A, ta, m, ka = self._operand(env[op.operands[0]])
        B, tb, kb, n = self._operand(env[op.operands[1]])
        if ka != kb:
            raise ValueError(f"matmul {op.id}: inner dims {ka} != {kb}")
        if not A.is_contiguous() or not B.is_contiguous():
            A, B = A.contiguous(), B.contiguous()
        dt = A.dtype
        out = self.empty((m, n), dt)
        epi, aux, aux_out = 0, None, None
        if fuse is not None:
            tag, j = fuse
            partner = ops[j]
            if tag == "relu":
                epi, aux_out = _lib.EPI_RELU, self.empty((m, n), dt)
            else:
                epi, aux = _lib.EPI_RELU_GRAD, tensor_of(env[partner.operands[1]])
        call("pc_gemm", _PC[dt], _PC[dt], ta, tb, m, n, ka, A.data_ptr(), A.shape[1],
             B.data_ptr(), B.shape[1], out.data_ptr(), n, epi, None, ptr(aux), n if aux is not None else 0,
             ptr(aux_out), n if aux_out is not None else 0, self.st)
        if fuse is None:
            env[op.result] = out
        elif fuse[0] == "relu":
            env[op.result] = aux_out           # z (pre-activation)
            env[ops[fuse[1]].result] = out     # relu(z)
        else:
            env[ops[fuse[1]].result] = out     # relu-grad(dX, z); dX never materialised

    def _sum_to(self, x: torch.Tensor, dims) -> torch.Tensor:
        dims = tuple(dims)
        if tuple(x.shape) == dims:
            return x
        if x.dim() == 2 and (dims == (x.shape[1],) or dims == (1, x.shape[1])):
            out = self.empty(dims, x.dtype)
            call("pc_col_sum", _PC[x.dtype], _PC[x.dtype], x.shape[0], x.shape[1], x.data_ptr(),
                 x.shape[1], out.data_ptr(), 0, None, 0, self.st)
            return out
        if len(dims) == 0 or math.prod(dims) == 1:
            out = self.empty(dims, x.dtype)
            flat = x.reshape(1, -1) if x.is_contiguous() else x.contiguous().reshape(1, -1)
            tmp = self.empty((flat.shape[1],), x.dtype)
            call("pc_copy2d", _PC[x.dtype], 1, flat.shape[1], flat.data_ptr(), flat.shape[1], 0,
                 tmp.data_ptr(), flat.shape[1], self.st)
            col = tmp.reshape(-1, 1)
            call("pc_col_sum", _PC[x.dtype], _PC[x.dtype], col.shape[0], 1, col.data_ptr(), 1,
                 out.data_ptr(), 0, None, 0, self.st)
            return out
        raise ValueError(f"sum-to {tuple(x.shape)} -> {dims} unsupported on device")

    def _broadcast(self, x: torch.Tensor, dims) -> torch.Tensor:
        dims = tuple(dims)
        out = self.empty(dims, x.dtype)
        # one launch each: a zero source row stride repeats the row (or the scalar)
        if len(dims) == 2 and x.numel() == dims[1]:
            call("pc_copy2d", _PC[x.dtype], dims[0], dims[1], x.data_ptr(), 0, 0,
                 out.data_ptr(), dims[1], self.st)
            return out
        if x.numel() == 1:
            call("pc_copy2d", _PC[x.dtype], out.numel(), 1, x.data_ptr(), 0, 0, out.data_ptr(), 1,
                 self.st)
            return out
        raise ValueError(f"broadcast {tuple(x.shape)} -> {dims} unsupported on device")

    def _concat(self, parts: list[torch.Tensor]) -> torch.Tensor:
        rows = [p.reshape(1) if p.dim() == 0 else p for p in parts]
        tail = rows[0].shape[1:]
        out = self.empty((sum(r.shape[0] for r in rows), *tail), rows[0].dtype)
        width = int(math.prod(tail)) if tail else 1
        off = 0
        for r in rows:
            call("pc_copy2d", _PC[r.dtype], r.shape[0], width, r.data_ptr(), width, 0,
                 out.data_ptr() + off * width * r.element_size(), width, self.st)
            off += r.shape[0]
        return out

    # ------------------------------------------------------------ task payloads
    def add(self, lhs, rhs, inplace: bool):
        """Grad-merge `add` (executor.py:335-336).  In place into ``lhs`` when
        the planner's chain guarantees it has no other reader."""
        x, y = tensor_of(lhs), tensor_of(rhs)
        if inplace and x.dtype in (torch.float32, torch.float64) and y.dtype == x.dtype:
            call("pc_accumulate", _PC[x.dtype], _PC[y.dtype], x.numel(), x.data_ptr(),
                 y.data_ptr(), self.st)
            return lhs
        out = self.empty(x.shape, x.dtype)
        call("pc_ewise", _lib.EW_ADD, _PC[x.dtype], x.numel(), x.data_ptr(), y.data_ptr(),
             y.numel(), out.data_ptr(), self.st)
        return out

    def concat_losses(self, parts) -> torch.Tensor:
        return self._concat([tensor_of(p) for p in parts])

    def sgd(self, w, g, lr: float, inplace: bool = False):
        """executor.py:340-344: w - lr*g (fp32/fp64 master; bf16 shadow refreshed).

        ``inplace``: the update overwrites ``w`` (resident training state,
        every reader of w is ordered before the update by the task graph)."""
        if isinstance(w, Param):
            master = w.master
            if inplace:
                newm, shadow = master, w.shadow
            else:
                newm = self.empty(master.shape, master.dtype)
                shadow = self.empty(master.shape, torch.bfloat16) if w.shadow is not None else None
            call("pc_sgd_update", _PC[master.dtype], master.numel(), master.data_ptr(),
                 tensor_of(g).data_ptr(), float(lr), newm.data_ptr(), ptr(shadow), self.st)
            return w if inplace else Param(newm, shadow)
        wt = tensor_of(w)
        out = wt if inplace else self.empty(wt.shape, wt.dtype)
        call("pc_sgd_update", _PC[wt.dtype], wt.numel(), wt.data_ptr(), tensor_of(g).data_ptr(),
             float(lr), out.data_ptr(), None, self.st)
        return out

    # ------------------------------------------------------------- GPT pieces
    def _slice(self, flat: torch.Tensor, layout, name):
        off, dims = layout[name]
        return flat[off:off + math.prod(dims)].view(*dims)

    _BLOCK_MATS = ("w_qkv", "w_o", "w_fc1", "w_fc2")

    def _shadow_t(self, w: "Param", lay, names=_BLOCK_MATS) -> torch.Tensor:
        """Transposed bf16 copies of the block matrices (W^T at W's offset), so
        the dX GEMMs read B K-major and can use the CTA-pair tiles.  Cached on
        the Param: one set of transposes per block per step."""
        if w.shadow_t is None or w.shadow_t_epoch != self.step_epoch:
            wt = self.empty(w.shadow.shape, torch.bfloat16)
            for name in names:
                off, (r, c) = lay[name]
                call("pc_copy2d", _lib.PC_BF16, c, r, w.shadow[off:].data_ptr(), c, 1,
                     wt[off:].data_ptr(), r, self.st)
            w.shadow_t, w.shadow_t_epoch = wt, self.step_epoch
        return w.shadow_t

    def _slice_t(self, flat: torch.Tensor, layout, name):
        off, (r, c) = layout[name]
        return flat[off:off + r * c].view(c, r)

    def _gemm(self, out_dtype, ta, tb, M, N, K, A, lda, B, ldb, C, ldc, epi=0, bias=None,
              aux=None, ldaux=0, aux_out=None, ldaux_out=0, st=None):
        call("pc_gemm", self.mode.pc_act, _PC[out_dtype], ta, tb, M, N, K, A.data_ptr(), lda,
             B.data_ptr(), ldb, C.data_ptr(), ldc, epi, ptr(bias), ptr(aux), ldaux, ptr(aux_out),
             ldaux_out, self.st if st is None else st)

    def _embed(self, env):
        cfg = self.gpt
        x = tensor_of(env["x"])
        w0: Param = env["w0"]
        T, d = cfg.tokens, cfg.d_model
        out = self.empty((T, d), self.mode.act)
        wte = self._slice(w0.master, self._elay, "wte")
        wpe = self._slice(w0.master, self._elay, "wpe")
        call("pc_embedding_fwd", self.mode.pc_act, T, d, cfg.seq_len, x.data_ptr(),
             wte.data_ptr(), wpe.data_ptr(), out.data_ptr(), self.st)
        return out

    def _embed_bwd(self, op, env, acc=None):
        self._join_side()   # the head weight gradient adds into the same tied sum
        cfg = self.gpt
        g = tensor_of(env[op.operands[0]])
        x = tensor_of(env[op.operands[1]])
        n = layout_size(self._elay)
        dw = acc if acc is not None else self.zeros((n,), torch.float32)
        T, d = cfg.tokens, cfg.d_model
        if self._emb_ws is None:
            nb = ctypes.c_int64(0)
            call("pc_embedding_bwd_workspace_bytes", T, ctypes.byref(nb))
            self._emb_ws = self.empty((nb.value,), torch.uint8)
        ws = self._emb_ws
        # accumulate: onto the running sum when fused, else onto the zeros above
        # (one zero-fill instead of two)
        call("pc_embedding_bwd_acc", self.mode.pc_act, T, d, cfg.seq_len, cfg.vocab,
             x.data_ptr(), g.data_ptr(), self._slice(dw, self._elay, "wte").data_ptr(),
             self._slice(dw, self._elay, "wpe").data_ptr(), 1, ws.data_ptr(), ws.numel(),
             self.st)
        ws.record_stream(self.stream)
        return dw

    def _block_fwd(self, op, env):
        cfg = self.gpt
        final = bool(op.attr("final_ln"))
        lay = self._blay[final]
        hv = env[op.operands[0]]
        if not isinstance(hv, Act):
            hv = env[op.operands[0]] = Act(tensor_of(hv))
        h = hv.t
        w: Param = env[op.operands[1]]
        W, Mst = w.compute(), w.master
        T, d, f, H = cfg.tokens, cfg.d_model, cfg.d_ff, cfg.n_heads
        act = self.mode.act
        sl = lambda name: self._slice(W, lay, name)
        ms = lambda name: self._slice(Mst, lay, name)
        a = self.empty((T, d), act)
        mean1 = self.empty((T,), torch.float32)
        rstd1 = self.empty((T,), torch.float32)
        call("pc_layernorm_fwd", self.mode.pc_act, T, d, h.data_ptr(), ms("ln1_g").data_ptr(),
             ms("ln1_b").data_ptr(), a.data_ptr(), mean1.data_ptr(), rstd1.data_ptr(), LN_EPS,
             self.st)
        qkv = self.empty((T, 3 * d), act)
        self._gemm(act, 0, 1, T, 3 * d, d, a, d, sl("w_qkv"), d, qkv, 3 * d, _lib.EPI_BIAS,
                   bias=ms("b_qkv"))
        o = self.empty((T, d), act)
        lse = self.empty((cfg.microbatch_size * H * cfg.seq_len,), torch.float32)
        if "attn_fwd" not in _ABLATE:
            call("pc_attention_fwd", self.mode.pc_act, cfg.microbatch_size, H, cfg.seq_len,
                 cfg.head_dim, qkv.data_ptr(), 3 * d, o.data_ptr(), d, lse.data_ptr(), self.st)
        h1 = self.empty((T, d), act)
        self._gemm(act, 0, 1, T, d, d, o, d, sl("w_o"), d, h1, d,
                   _lib.EPI_BIAS | _lib.EPI_RESIDUAL, bias=ms("b_o"), aux=h, ldaux=d)
        a2 = self.empty((T, d), act)
        mean2 = self.empty((T,), torch.float32)
        rstd2 = self.empty((T,), torch.float32)
        call("pc_layernorm_fwd", self.mode.pc_act, T, d, h1.data_ptr(), ms("ln2_g").data_ptr(),
             ms("ln2_b").data_ptr(), a2.data_ptr(), mean2.data_ptr(), rstd2.data_ptr(), LN_EPS,
             self.st)
        u = self.empty((T, f), act)
        gu = self.empty((T, f), act)
        self._gemm(act, 0, 1, T, f, d, a2, d, sl("w_fc1"), d, gu, f,
                   _lib.EPI_BIAS | _lib.EPI_GELU, bias=ms("b_fc1"), aux_out=u, ldaux_out=f)
        # a block output that leaves the stage is written straight into the
        # next stage's receive slot (NVLink peer memory) by this GEMM
        out = self.empty((T, d), act) if final else self._out(op.result, (T, d), act)
        self._gemm(act, 0, 1, T, d, f, gu, f, sl("w_fc2"), f, out, d,
                   _lib.EPI_BIAS | _lib.EPI_RESIDUAL, bias=ms("b_fc2"), aux=h1, ldaux=d)
        saved = dict(a=a, mean1=mean1, rstd1=rstd1, qkv=qkv, o=o, lse=lse, h1=h1, a2=a2,
                     mean2=mean2, rstd2=rstd2, u=u, gu=gu)
        if final:
            z = self.empty((T, d), act)
            meanf = self.empty((T,), torch.float32)
            rstdf = self.empty((T,), torch.float32)
            call("pc_layernorm_fwd", self.mode.pc_act, T, d, out.data_ptr(),
                 ms("lnf_g").data_ptr(), ms("lnf_b").data_ptr(), z.data_ptr(), meanf.data_ptr(),
                 rstdf.data_ptr(), LN_EPS, self.st)
            saved.update(out=out, meanf=meanf, rstdf=rstdf)
            out = z
        hv.saved[op.id] = saved
        env[op.result] = Act(out)

    def _ln_partials(self, key: str, rows: int, d: int):
        """Partial-row buffer [2, n, d] fp32 of one LayerNorm of the block (one per
        LayerNorm: the side stream may still sum the previous one's rows)."""
        n = ctypes.c_int64(0)
        call("pc_layernorm_partial_rows", rows, d, ctypes.byref(n))
        buf = self._ln_parts.get(key)
        if buf is None or buf.numel() < 2 * n.value * d:
            buf = self.empty((2 * n.value * d,), torch.float32)
            self._ln_parts[key] = buf
        return buf, n.value

    def _acc_for_value(self, v: str):
        """Running sum a parameter partial ``v`` may be added onto: v is a task
        output in acc_into, or v's only reader is the in-stage ``add`` that
        merges the tied embedding's partials into such an output (then both
        partials go onto the sum and the add is a rename, see _fused_add)."""
        if not self.acc_into:
            return None
        if v in self.acc_into:
            return self.acc_into[v]
        users = self._consumers.get(v, ())
        if len(users) == 1 and users[0].kind == "add" and users[0].result in self.acc_into:
            return self.acc_into[users[0].result]
        return None

    def _acc_for_tuple(self, op, index: int):
        if not self.acc_into:
            return None
        for u in self._consumers.get(op.result, ()):
            if u.kind == "tuple-get" and u.attr("index") == index:
                return self._acc_for_value(u.result)
        return None

    def _fused_add(self, op, env) -> bool:
        """The in-stage add of partials already added onto the running sum
        (or one of them): finish in place and alias the result."""
        acc = self.acc_into.get(op.result) if self.acc_into else None
        if acc is None:
            return False
        x, y = env[op.operands[0]], env[op.operands[1]]
        xs, ys = x is acc, y is acc
        if not (xs or ys):
            return False
        if not (xs and ys):
            other = tensor_of(y if xs else x)
            call("pc_accumulate", _PC[acc.dtype], _PC[other.dtype], acc.numel(), acc.data_ptr(),
                 other.data_ptr(), self.st)
        env[op.result] = acc
        return True

    def _acc_target(self, op, index: int):
        """The accumulator the ``index``-th tuple element of ``op`` may add
        onto (its only reader is a tuple-get whose value is in acc_into)."""
        if not self.acc_into:
            return None
        for u in self._consumers.get(op.result, ()):
            if u.kind == "tuple-get" and u.attr("index") == index and u.result in self.acc_into:
                return self.acc_into[u.result]
        return None

    def _wgrad_into(self, M_, N_, K_, A, lda, Bm, ldb, C, acc: bool, side: torch.cuda.Stream):
        """C (fp32 [M_, N_]) = the weight-gradient product, or C += it when
        ``acc``: the GEMM adds through its TMA reduce-add store -- unsplit,
        C + p (one fp32 add, bitwise the stored partial added after); split
        in two K halves, (C + h0) + h1 in that order (flag-sequenced per tile,
        deterministic)."""
        f32 = torch.float32
        st = side.cuda_stream
        if not acc:
            self._gemm(f32, 1, 0, M_, N_, K_, A, lda, Bm, ldb, C, N_, _lib.EPI_SPLITK_ZERO_C, st=st)
            return
        if self._split_flags is None:   # zero once; every ordered GEMM leaves them zero
            with torch.cuda.stream(side):
                self._split_flags = torch.zeros(1 << 16, dtype=torch.int32, device=self.device)
        self._gemm(f32, 1, 0, M_, N_, K_, A, lda, Bm, ldb, C, N_,
                   _lib.EPI_ACCUM | _lib.EPI_SPLITK_ORDERED, aux=self._split_flags,
                   ldaux=self._split_flags.numel(), st=st)

    def _wgrad_pair_into(self, M1, M2, N_, K_, A1, lda1, B1, ldb1, C1, A2, lda2, B2, ldb2, C2,
                         acc: bool, side: torch.cuda.Stream):
        """Two weight gradients with the same N and K in one launch
        (pc_gemm_wgrad_pair): the same per-gradient sums as two _wgrad_into
        calls, the second problem's tiles filling the first's partial wave."""
        st = side.cuda_stream
        if acc:
            if self._split_flags is None:
                with torch.cuda.stream(side):
                    self._split_flags = torch.zeros(1 << 16, dtype=torch.int32, device=self.device)
            epi, aux, ldaux = (_lib.EPI_ACCUM | _lib.EPI_SPLITK_ORDERED, self._split_flags.data_ptr(),
                               self._split_flags.numel())
        else:
            epi, aux, ldaux = _lib.EPI_SPLITK_ZERO_C, None, 0
        call("pc_gemm_wgrad_pair", M1, M2, N_, K_, A1.data_ptr(), lda1, B1.data_ptr(), ldb1,
             C1.data_ptr(), N_, A2.data_ptr(), lda2, B2.data_ptr(), ldb2, C2.data_ptr(), N_, epi, aux,
             ldaux, st)

    def _block_bwd(self, op, env, acc=None):
        cfg = self.gpt
        final = bool(op.attr("final_ln"))
        lay = self._blay[final]
        fwd_id = f"block{op.attr('layer')}"
        dz = tensor_of(env[op.operands[0]])
        hv = env[op.operands[1]]
        h = tensor_of(hv)
        sv = hv.saved[fwd_id]
        w: Param = env[op.operands[2]]
        W, Mst = w.compute(), w.master
        T, d, f, H = cfg.tokens, cfg.d_model, cfg.d_ff, cfg.n_heads
        act = self.mode.act
        f32 = torch.float32
        sl = lambda name: self._slice(W, lay, name)
        ms = lambda name: self._slice(Mst, lay, name)
        # dX GEMMs: B = W^T read K-major from the transposed shadow (bf16 mode),
        # else W read MN-major
        if w.shadow is not None:
            Wt = self._shadow_t(w, lay)
            wB = lambda name: (1, self._slice_t(Wt, lay, name), lay[name][1][0])
        else:
            wB = lambda name: (0, sl(name), lay[name][1][1])
        fused = acc is not None
        dW = acc if fused else self.zeros((layout_size(lay),), f32)
        gs = lambda name: self._slice(dW, lay, name)
        # the side stream's reduction workspace, sized once for the widest sum
        # (never reallocated while side work may still read it)
        self.red_ws(T, max(f, 3 * d), side=True)

        def ln_bwd(dy, x, gname, bname, mean, rstd, dres, dx, biases=None):
            """LayerNorm backward: dx on the compute stream; gamma / beta gradients
            (a reduction nothing downstream waits for) beside it on the side
            stream.  PP200_LN_FUSED=1: one pass for dx and partial rows of the
            parameter gradients, their column sums on the side stream.  biases =
            (y3, name3, y4, name4): two bias gradients (column sums of y3 and of
            y4, which may be dx itself) in the same side-stream pass, after dx."""
            if biases is not None:
                y3, n3, y4, n4 = biases
                call("pc_layernorm_bwd_acc", self.mode.pc_act, T, d, dy.data_ptr(), x.data_ptr(),
                     ms(gname).data_ptr(), mean.data_ptr(), rstd.data_ptr(),
                     None if dres is None else dres.data_ptr(), dx.data_ptr(), None, None, 0,
                     *self.red_ws(T, d), self.st)
                self._fork()
                call("pc_layernorm_param_bias_grads", T, d, dy.data_ptr(), x.data_ptr(),
                     mean.data_ptr(), rstd.data_ptr(), gs(gname).data_ptr(), gs(bname).data_ptr(),
                     y3.data_ptr(), gs(n3).data_ptr(), y4.data_ptr(), gs(n4).data_ptr(), int(fused),
                     sst)
                return
            if _LN_FUSED and "lnp" not in _ABLATE and d % 256 == 0 and d <= 1024:
                # dx and the parameter-gradient partial rows in one pass on the
                # compute stream; their fixed-order column sums on the side stream
                parts, npart = self._ln_partials(gname, T, d)
                call("pc_layernorm_bwd_partials", self.mode.pc_act, T, d, dy.data_ptr(),
                     x.data_ptr(), ms(gname).data_ptr(), mean.data_ptr(), rstd.data_ptr(),
                     None if dres is None else dres.data_ptr(), dx.data_ptr(), parts.data_ptr(),
                     npart, self.st)
                self._fork()
                ws = self.red_ws(npart, d, side=True)
                call("pc_col_sum", _lib.PC_F32, _lib.PC_F32, npart, d, parts.data_ptr(), d,
                     gs(gname).data_ptr(), int(fused), *ws, sst)
                call("pc_col_sum", _lib.PC_F32, _lib.PC_F32, npart, d,
                     parts[npart * d:].data_ptr(), d, gs(bname).data_ptr(), int(fused), *ws, sst)
                return
            on_side = not _LN_PARAMS_MAIN
            if on_side:
                self._fork()
            if "lnp" not in _ABLATE:
                call("pc_layernorm_param_grads", self.mode.pc_act, T, d, dy.data_ptr(), x.data_ptr(),
                     mean.data_ptr(), rstd.data_ptr(), gs(gname).data_ptr(), gs(bname).data_ptr(),
                     int(fused), *self.red_ws(T, d, side=on_side),
                     self._side().cuda_stream if on_side else self.st)
            call("pc_layernorm_bwd_acc", self.mode.pc_act, T, d, dy.data_ptr(), x.data_ptr(),
                 ms(gname).data_ptr(), mean.data_ptr(), rstd.data_ptr(),
                 None if dres is None else dres.data_ptr(), dx.data_ptr(), None, None, 0,
                 *self.red_ws(T, d), self.st)

        sst = self._side().cuda_stream
        if final:
            dout = self.empty((T, d), act)
            ln_bwd(dz, sv["out"], "lnf_g", "lnf_b", sv["meanf"], sv["rstdf"], None, dout)
        else:
            dout = dz
        # Weight gradients and their bias sums run on the side stream (they do
        # not feed the dX chain); each fork orders them after their inputs.

        def wgrad(M_, N_, A, lda, Bm, ldb, wname, bname, weight=True, bias=True):
            self._fork()
            if weight and "wgrad" not in _ABLATE:
                self._wgrad_into(M_, N_, T, A, lda, Bm, ldb, gs(wname), fused, self._side())
            if _ABLATE_BIAS or not bias:   # _ABLATE_BIAS: profiling only, left unset
                return
            call("pc_col_sum", self.mode.pc_act, _lib.PC_F32, T, M_, A.data_ptr(), lda,
                 gs(bname).data_ptr(), int(fused), *self.red_ws(T, M_, side=True), sst)

        # the attention-output and qkv weight gradients share N = d and K = T: one
        # grouped launch once both inputs exist (dW_o alone left most SMs idle)
        pair = self.mode.act == torch.bfloat16 and (3 * d) % 256 == 0 and _WGRAD_PAIR

        # the fc2 and attention-output bias gradients ride on LN2's parameter pass
        lnb = (_LN_BIAS_FUSED and act == torch.bfloat16 and not _LN_FUSED and not _LN_PARAMS_MAIN
               and not _ABLATE_BIAS and "lnp" not in _ABLATE and d % 8 == 0
               and dout.data_ptr() % 16 == 0 and sv["h1"].data_ptr() % 16 == 0)

        # MLP
        wgrad(d, f, dout, d, sv["gu"], f, "w_fc2", "b_fc2", bias=not lnb)
        du = self.empty((T, f), act)
        tb, B, ldb = wB("w_fc2")
        self._gemm(act, 0, tb, T, f, d, dout, d, B, ldb, du, f, _lib.EPI_GELU_GRAD,
                   aux=sv["u"], ldaux=f)
        wgrad(f, d, du, f, sv["a2"], d, "w_fc1", "b_fc1")
        da2 = self.empty((T, d), act)
        tb, B, ldb = wB("w_fc1")
        self._gemm(act, 0, tb, T, d, f, du, f, B, ldb, da2, d)
        dh1 = self.empty((T, d), act)
        ln_bwd(da2, sv["h1"], "ln2_g", "ln2_b", sv["mean2"], sv["rstd2"], dout, dh1,
               biases=(dout, "b_fc2", dh1, "b_o") if lnb else None)
        # attention
        wgrad(d, d, dh1, d, sv["o"], d, "w_o", "b_o", weight=not pair, bias=not lnb)
        do = self.empty((T, d), act)
        tb, B, ldb = wB("w_o")
        self._gemm(act, 0, tb, T, d, d, dh1, d, B, ldb, do, d)
        dqkv = self.empty((T, 3 * d), act)
        delta = self.empty((cfg.microbatch_size * H * cfg.seq_len,), f32)
        if "attn_bwd" not in _ABLATE:
            call("pc_attention_bwd", self.mode.pc_act, cfg.microbatch_size, H, cfg.seq_len,
                 cfg.head_dim, sv["qkv"].data_ptr(), 3 * d, sv["o"].data_ptr(), do.data_ptr(), d,
                 sv["lse"].data_ptr(), delta.data_ptr(), dqkv.data_ptr(), 3 * d, self.st)
        wgrad(3 * d, d, dqkv, 3 * d, sv["a"], d, "w_qkv", "b_qkv", weight=not pair)
        if pair and "wgrad" not in _ABLATE:   # after the fork above: dqkv and dh1 exist
            self._wgrad_pair_into(3 * d, d, d, T, dqkv, 3 * d, sv["a"], d, gs("w_qkv"), dh1, d,
                                  sv["o"], d, gs("w_o"), fused, self._side())
        da = self.empty((T, d), act)
        tb, B, ldb = wB("w_qkv")
        self._gemm(act, 0, tb, T, d, 3 * d, dqkv, 3 * d, B, ldb, da, d)
        dh = self._placed_elem(op, 0, (T, d), act)   # into the previous stage's slot when sent
        ln_bwd(da, h, "ln1_g", "ln1_b", sv["mean1"], sv["rstd1"], dh1, dh)
        if _DEFER_JOIN:
            # the next block's data-gradient chain does not wait for this block's
            # side-stream work; every tensor that work reads stays alive until
            # the compute stream has waited for it (_defer_side)
            self._defer_side((dz, dout, du, da2, dh1, dqkv, da, h, sv))
        else:
            self._join()
        return (dh, dW)

    def _head_fwd(self, op, env):
        cfg = self.gpt
        hv = env[op.operands[0]]
        if not isinstance(hv, Act):
            hv = env[op.operands[0]] = Act(tensor_of(hv))
        h = hv.t
        w0: Param = env[op.operands[1]]
        x = tensor_of(env[op.operands[2]])
        T, d, V = cfg.tokens, cfg.d_model, cfg.vocab
        logits, rows = self._lmhead_xent(h, self._slice(w0.compute(), self._elay, "wte"), x)
        loss = self.empty((), torch.float32)
        call("pc_sum_f32", T, rows.data_ptr(), loss.data_ptr(), self.st)
        hv.saved[op.id] = dict(dlogits=logits)
        return loss

    def _lmhead_xent(self, h, w, x):
        """logits = h W^T with the cross-entropy folded in: (dlogits in place of
        the logits, per-row losses).  bf16: pc_lmhead_xent_fwd (softmax statistics
        from the GEMM epilogue, one streaming pass); fp32 parity mode: GEMM then
        pc_xent_fwd_bwd."""
        cfg = self.gpt
        T, d, V = cfg.tokens, cfg.d_model, cfg.vocab
        logits = self.empty((T, V), self.mode.act)
        rows = self.empty((T,), torch.float32)
        if self.mode.act == torch.bfloat16 and V % 8 == 0 and _XENT_FUSED:
            if self._xent_ws is None:
                lds, nb = ctypes.c_int64(), ctypes.c_int64()
                call("pc_lmhead_xent_workspace", T, V, d, ctypes.byref(lds), ctypes.byref(nb))
                self._xent_ws = self.empty((nb.value,), torch.uint8)
            call("pc_lmhead_xent_fwd", T, V, d, cfg.seq_len, h.data_ptr(), d, w.data_ptr(), d,
                 x.data_ptr(), logits.data_ptr(), V, self._xent_ws.data_ptr(),
                 self._xent_ws.numel(), rows.data_ptr(), self.st)
            return logits, rows
        self._gemm(self.mode.act, 0, 1, T, V, d, h, d, w, d, logits, V)
        call("pc_xent_fwd_bwd", self.mode.pc_act, T, V, cfg.seq_len, logits.data_ptr(), V,
             x.data_ptr(), rows.data_ptr(), self.st)
        return logits, rows

    def _head_bwd(self, op, env, acc=None):
        cfg = self.gpt
        hv = env[op.operands[0]]
        h = tensor_of(hv)
        dlogits = hv.saved["head"]["dlogits"]
        w0: Param = env[op.operands[1]]
        T, d, V = cfg.tokens, cfg.d_model, cfg.vocab
        # the stage input gradient: into the previous stage's slot when sent
        dh = self._placed_elem(op, 0, (T, d), self.mode.act)
        if w0.shadow is not None:  # B = wte^T, K-major, from the transposed shadow
            wt = self._shadow_t(w0, self._elay, ("wte",))
            self._gemm(self.mode.act, 0, 1, T, d, V, dlogits, V,
                       self._slice_t(wt, self._elay, "wte"), V, dh, d)
        else:
            wte = self._slice(w0.compute(), self._elay, "wte")
            self._gemm(self.mode.act, 0, 0, T, d, V, dlogits, V, wte, d, dh, d)
        # the weight gradient runs on the side stream beside the blocks' backward
        # (joined at the end of the stage program, or before the embedding
        # backward adds into the same tied running sum)
        side = self._side() if _DEFER_JOIN else None
        sst = side.cuda_stream if side is not None else self.st
        if side is not None:
            self._fork()
        if acc is not None:
            # onto the running sum: the wte rows through the GEMM's TMA
            # reduce-add store (unsplit: one fp32 add per element); the head's
            # wpe part is zero, nothing to add
            self._gemm(torch.float32, 1, 0, V, d, T, dlogits, V, h, d,
                       self._slice(acc, self._elay, "wte"), d, _lib.EPI_ACCUM, st=sst)
            if side is not None:
                self._defer_side((dlogits, h))
            return (dh, acc)
        # wte gradient from the GEMM; wpe's part of the tied partial is zero.
        # Zero-fill only what the GEMM does not overwrite: all of wte when it
        # splits K (two halves reduce-added onto zeros), else just wpe.
        dw = self.empty((layout_size(self._elay),), torch.float32)
        bn, cg, ks = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        call("pc_gemm_tile_choice", 0, V, d, T, 1, ctypes.byref(bn), ctypes.byref(cg),
             ctypes.byref(ks))
        wte = self._slice(dw, self._elay, "wte")
        if ks.value > 1:
            call("pc_fill", _lib.PC_F32, dw.numel(), 0.0, dw.data_ptr(), sst)
        else:  # everything after wte: wpe and the alignment padding
            tail = dw[self._elay["wte"][0] + wte.numel():]
            call("pc_fill", _lib.PC_F32, tail.numel(), 0.0, tail.data_ptr(), sst)
        self._gemm(torch.float32, 1, 0, V, d, T, dlogits, V, h, d, wte, d, _lib.EPI_SPLITK_ZERO_C,
                   st=sst)
        if side is not None:
            self._defer_side((dlogits, h, dw))
        return (dh, dw)


    # ------------------------------------------------------- Llama pieces (C5)
    _LLAMA_MATS = ("w_qkv", "w_o", "w_gu", "w_down")

    def _zeros_cached(self, key: str, shape) -> torch.Tensor:
        t = getattr(self, key, None)
        if t is None or tuple(t.shape) != tuple(shape):
            t = self.zeros(shape, torch.float32)
            setattr(self, key, t)
        return t

    def _llama_embed(self, op, env):
        """h0 = wte[x] (oracle/llama.py llama_step); the embedding kernel with
        an all-zero position table."""
        cfg = self.gpt
        x = tensor_of(env[op.operands[0]])
        w0: Param = env[op.operands[1]]
        T, d = cfg.tokens, cfg.d_model
        out = self.empty((T, d), self.mode.act)
        zpe = self._zeros_cached("_llama_zpe", (cfg.seq_len, d))
        call("pc_embedding_fwd", self.mode.pc_act, T, d, cfg.seq_len, x.data_ptr(),
             self._slice(w0.master, self._elay, "wte").data_ptr(), zpe.data_ptr(),
             out.data_ptr(), self.st)
        return out

    def _llama_embed_bwd(self, op, env, acc=None):
        """Token-row sums of the embedding gradient, onto the running sum when
        fused (no [vocab, d] zero fill per microbatch), else onto zeros."""
        self._join_side()   # pending side-stream work may still write gradients
        cfg = self.gpt
        g = tensor_of(env[op.operands[0]])
        x = tensor_of(env[op.operands[1]])
        T, d = cfg.tokens, cfg.d_model
        dw = acc if acc is not None else self.zeros((layout_size(self._elay),), torch.float32)
        if self._emb_ws is None:
            nb = ctypes.c_int64(0)
            call("pc_embedding_bwd_workspace_bytes", T, ctypes.byref(nb))
            self._emb_ws = self.empty((nb.value,), torch.uint8)
        call("pc_embedding_bwd_acc", self.mode.pc_act, T, d, cfg.seq_len, cfg.vocab, x.data_ptr(),
             g.data_ptr(), self._slice(dw, self._elay, "wte").data_ptr(), None, 1,
             self._emb_ws.data_ptr(), self._emb_ws.numel(), self.st)
        self._emb_ws.record_stream(self.stream)
        return dw

    def _rms(self, x, g, T, d):
        y = self.empty((T, d), self.mode.act)
        rstd = self.empty((T,), torch.float32)
        call("pc_rmsnorm_fwd", self.mode.pc_act, T, d, x.data_ptr(), g.data_ptr(), y.data_ptr(),
             rstd.data_ptr(), RMS_EPS, self.st)
        return y, rstd

    def _native_gqa(self) -> bool:
        """Grouped-query heads go straight to the tcgen05 attention kernels (bf16,
        head_dim 64 / 128); other modes expand K/V heads (pc_gqa_kv)."""
        cfg = self.gpt
        return (self.mode.act == torch.bfloat16 and cfg.head_dim in (64, 128)
                and cfg.seq_len % 4 == 0)

    def _llama_block_fwd(self, op, env):
        """oracle/llama.py block_fwd: RMSNorm -> qkv GEMM -> RoPE(q, k) ->
        GQA causal attention -> o GEMM (+h) -> RMSNorm -> gate/up GEMM ->
        SwiGLU -> down GEMM (+h1) [-> final RMSNorm]."""
        cfg = self.gpt
        final = bool(op.attr("final_ln"))
        lay = self._blay[final]
        hv = env[op.operands[0]]
        if not isinstance(hv, Act):
            hv = env[op.operands[0]] = Act(tensor_of(hv))
        h = hv.t
        w: Param = env[op.operands[1]]
        pos = tensor_of(env[op.operands[2]])
        W, Mst = w.compute(), w.master
        T, d, f = cfg.tokens, cfg.d_model, cfg.d_ff
        H, Hkv, hd, qw = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.qkv_width
        act = self.mode.act
        sl = lambda name: self._slice(W, lay, name)
        ms = lambda name: self._slice(Mst, lay, name)
        a, rstd1 = self._rms(h, ms("rms1_g"), T, d)
        qkv = self.empty((T, qw), act)
        self._gemm(act, 0, 1, T, qw, d, a, d, sl("w_qkv"), d, qkv, qw)
        call("pc_rope", self.mode.pc_act, T, H + Hkv, hd, qkv.data_ptr(), qw, pos.data_ptr(),
             float(cfg.rope_theta), 0, self.st)
        if Hkv != H and not self._native_gqa():
            # grouped-query heads outside the tcgen05 kernels (fp32 parity mode):
            # expand K/V heads for the multi-head kernels
            qkv_att = self.empty((T, 3 * H * hd), act)
            call("pc_gqa_kv", self.mode.pc_act, T, H, Hkv, hd, qkv.data_ptr(), qw,
                 qkv_att.data_ptr(), 3 * H * hd, 0, self.st)
            Hk_att = H
        else:   # native: the kernels address kv head h / (H / Hkv) in qkv itself
            qkv_att, Hk_att = qkv, Hkv
        o = self.empty((T, H * hd), act)
        lse = self.empty((cfg.microbatch_size * H * cfg.seq_len,), torch.float32)
        call("pc_attention_gqa_fwd", self.mode.pc_act, cfg.microbatch_size, H, Hk_att,
             cfg.seq_len, hd, qkv_att.data_ptr(), qkv_att.shape[1], o.data_ptr(), H * hd,
             lse.data_ptr(), self.st)
        h1 = self.empty((T, d), act)
        self._gemm(act, 0, 1, T, d, H * hd, o, H * hd, sl("w_o"), H * hd, h1, d,
                   _lib.EPI_RESIDUAL, aux=h, ldaux=d)
        a2, rstd2 = self._rms(h1, ms("rms2_g"), T, d)
        gu = self.empty((T, 2 * f), act)
        self._gemm(act, 0, 1, T, 2 * f, d, a2, d, sl("w_gu"), d, gu, 2 * f)
        m = self.empty((T, f), act)
        call("pc_swiglu_fwd", self.mode.pc_act, T, f, gu.data_ptr(), 2 * f, m.data_ptr(), f,
             self.st)
        # the stage output: the down GEMM writes it into the next stage's slot when sent
        out = self.empty((T, d), act) if final else self._out(op.result, (T, d), act)
        self._gemm(act, 0, 1, T, d, f, m, f, sl("w_down"), f, out, d, _lib.EPI_RESIDUAL,
                   aux=h1, ldaux=d)
        saved = dict(a=a, rstd1=rstd1, qkv_att=qkv_att, o=o, lse=lse, h1=h1, a2=a2,
                     rstd2=rstd2, gu=gu, m=m)
        if final:
            z, rstdf = self._rms(out, ms("rmsf_g"), T, d)
            saved.update(out=out, rstdf=rstdf)
            out = z
        hv.saved[op.id] = saved
        env[op.result] = Act(out)

    def _llama_block_bwd(self, op, env, acc=None):
        """oracle/llama.py block_bwd; dX GEMMs read the transposed bf16 weight
        shadow (K-major B).  Weight and RMSNorm-gain gradients run on the side
        stream beside the dX chain and, when the plan allows (``acc``), add
        straight onto the fp32 running sum (TMA reduce-add / ordered split-K,
        accumulating reductions): no per-microbatch zero fill or add pass."""
        cfg = self.gpt
        final = bool(op.attr("final_ln"))
        lay = self._blay[final]
        dz = tensor_of(env[op.operands[0]])
        hv = env[op.operands[1]]
        h = tensor_of(hv)
        w: Param = env[op.operands[2]]
        pos = tensor_of(env[op.operands[3]])
        sv = hv.saved[f"block{op.attr('layer')}"]
        W, Mst = w.compute(), w.master
        T, d, f = cfg.tokens, cfg.d_model, cfg.d_ff
        H, Hkv, hd, qw = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.qkv_width
        act, f32 = self.mode.act, torch.float32
        sl = lambda name: self._slice(W, lay, name)
        ms = lambda name: self._slice(Mst, lay, name)
        if w.shadow is not None:
            Wt = self._shadow_t(w, lay, self._LLAMA_MATS)
            wB = lambda name: (1, self._slice_t(Wt, lay, name), lay[name][1][0])
        else:
            wB = lambda name: (0, sl(name), lay[name][1][1])
        fused = acc is not None
        dW = acc if fused else self.zeros((layout_size(lay),), f32)
        gs = lambda name: self._slice(dW, lay, name)
        self.red_ws(T, d, side=True)

        def rms_bwd(dy, x, gname, rstd, dres, dx=None):
            self._fork()   # gain gradient beside the dx chain
            call("pc_layernorm_param_grads", self.mode.pc_act, T, d, dy.data_ptr(), x.data_ptr(),
                 None, rstd.data_ptr(), gs(gname).data_ptr(), None, int(fused),
                 *self.red_ws(T, d, side=True), self._side().cuda_stream)
            if dx is None:
                dx = self.empty((T, d), act)
            call("pc_rmsnorm_bwd", self.mode.pc_act, T, d, dy.data_ptr(), x.data_ptr(),
                 ms(gname).data_ptr(), rstd.data_ptr(), ptr(dres), dx.data_ptr(), None, None, 0,
                 self.st)
            return dx

        def wgrad(M_, N_, A, lda, Bm, ldb, wname):
            self._fork()
            self._wgrad_into(M_, N_, T, A, lda, Bm, ldb, gs(wname), fused, self._side())

        dout = rms_bwd(dz, sv["out"], "rmsf_g", sv["rstdf"], None) if final else dz
        # MLP
        wgrad(d, f, dout, d, sv["m"], f, "w_down")
        dm = self.empty((T, f), act)
        tb, B, ldb = wB("w_down")
        self._gemm(act, 0, tb, T, f, d, dout, d, B, ldb, dm, f)
        dgu = self.empty((T, 2 * f), act)
        call("pc_swiglu_bwd", self.mode.pc_act, T, f, sv["gu"].data_ptr(), 2 * f, dm.data_ptr(),
             f, dgu.data_ptr(), 2 * f, self.st)
        wgrad(2 * f, d, dgu, 2 * f, sv["a2"], d, "w_gu")
        da2 = self.empty((T, d), act)
        tb, B, ldb = wB("w_gu")
        self._gemm(act, 0, tb, T, d, 2 * f, dgu, 2 * f, B, ldb, da2, d)
        dh1 = rms_bwd(da2, sv["h1"], "rms2_g", sv["rstd2"], dout)
        # attention
        wgrad(d, H * hd, dh1, d, sv["o"], H * hd, "w_o")
        do = self.empty((T, H * hd), act)
        tb, B, ldb = wB("w_o")
        self._gemm(act, 0, tb, T, H * hd, d, dh1, d, B, ldb, do, H * hd)
        qkv_att = sv["qkv_att"]
        ld_att = qkv_att.shape[1]
        Hk_att = Hkv if ld_att == qw else H
        dqkv_att = self.empty((T, ld_att), act)
        delta = self.empty((cfg.microbatch_size * H * cfg.seq_len,), f32)
        call("pc_attention_gqa_bwd", self.mode.pc_act, cfg.microbatch_size, H, Hk_att,
             cfg.seq_len, hd, qkv_att.data_ptr(), ld_att, sv["o"].data_ptr(), do.data_ptr(),
             H * hd, sv["lse"].data_ptr(), delta.data_ptr(), dqkv_att.data_ptr(), ld_att, self.st)
        if ld_att != qw:  # expanded heads: sum each kv head's group of query-head gradients
            dqkv = self.empty((T, qw), act)
            call("pc_gqa_kv", self.mode.pc_act, T, H, Hkv, hd, dqkv_att.data_ptr(), ld_att,
                 dqkv.data_ptr(), qw, 1, self.st)
        else:
            dqkv = dqkv_att
        call("pc_rope", self.mode.pc_act, T, H + Hkv, hd, dqkv.data_ptr(), qw, pos.data_ptr(),
             float(cfg.rope_theta), 1, self.st)
        wgrad(qw, d, dqkv, qw, sv["a"], d, "w_qkv")
        da = self.empty((T, d), act)
        tb, B, ldb = wB("w_qkv")
        self._gemm(act, 0, tb, T, d, qw, dqkv, qw, B, ldb, da, d)
        # the stage input gradient: into the previous stage's slot when sent
        dh = rms_bwd(da, h, "rms1_g", sv["rstd1"], dh1, self._placed_elem(op, 0, (T, d), act))
        if _DEFER_JOIN:   # as in _block_bwd
            self._defer_side((dz, dout, dgu, da2, dh1, dqkv, da, h, sv))
        else:
            self._join()
        return (dh, dW)

    def _llama_head_fwd(self, op, env):
        cfg = self.gpt
        hv = env[op.operands[0]]
        if not isinstance(hv, Act):
            hv = env[op.operands[0]] = Act(tensor_of(hv))
        h = hv.t
        wo: Param = env[op.operands[1]]
        x = tensor_of(env[op.operands[2]])
        T, d, V = cfg.tokens, cfg.d_model, cfg.vocab
        logits, rows = self._lmhead_xent(h, self._slice(wo.compute(), self._hlay, "w_head"), x)
        loss = self.empty((), torch.float32)
        call("pc_sum_f32", T, rows.data_ptr(), loss.data_ptr(), self.st)
        hv.saved[op.id] = dict(dlogits=logits)
        return loss

    def _llama_head_bwd(self, op, env, acc=None):
        cfg = self.gpt
        hv = env[op.operands[0]]
        h = tensor_of(hv)
        dlogits = hv.saved["head"]["dlogits"]
        wo: Param = env[op.operands[1]]
        T, d, V = cfg.tokens, cfg.d_model, cfg.vocab
        dh = self._placed_elem(op, 0, (T, d), self.mode.act)
        if wo.shadow is not None:
            wt = self._shadow_t(wo, self._hlay, ("w_head",))
            self._gemm(self.mode.act, 0, 1, T, d, V, dlogits, V,
                       self._slice_t(wt, self._hlay, "w_head"), V, dh, d)
        else:
            self._gemm(self.mode.act, 0, 0, T, d, V, dlogits, V,
                       self._slice(wo.compute(), self._hlay, "w_head"), d, dh, d)
        fused = acc is not None
        dw = acc if fused else self.zeros((layout_size(self._hlay),), torch.float32)
        self._fork()
        self._wgrad_into(V, d, T, dlogits, V, h, d, self._slice(dw, self._hlay, "w_head"), fused,
                         self._side())
        if _DEFER_JOIN:   # the blocks' backward does not wait for the head weight gradient
            self._defer_side((dlogits, h))
        else:
            self._join()
        return (dh, dw)


# ---------------------------------------------------------------- host <-> device


def to_device_param(value, mode: Mode, device, gpt: bool):
    """Step-input parameter on an actor: fp32/fp64 master (+ bf16 shadow)."""
    if isinstance(value, Param):
        return value
    if isinstance(value, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(value)).to(device=device, dtype=mode.master,
                                                             non_blocking=True)
    else:
        t = value.to(device=device, dtype=mode.master, non_blocking=True)
    if not gpt:
        return t
    if mode.act == torch.bfloat16:
        sh = torch.empty(t.shape, dtype=torch.bfloat16, device=device)
        call("pc_cast", _PC[t.dtype], _lib.PC_BF16, t.numel(), t.data_ptr(), sh.data_ptr(),
             torch.cuda.current_stream(device).cuda_stream)
        return Param(t, sh)
    return Param(t, None)


def to_device_input(value, mode: Mode, device, is_tokens: bool):
    if isinstance(value, np.ndarray):
        value = torch.from_numpy(np.ascontiguousarray(value))
    if is_tokens:
        return value.to(device=device, dtype=torch.int32, non_blocking=True)
    return value.to(device=device, dtype=mode.act, non_blocking=True)
