"""Float64 numpy restatement of the reference FFN path (TEST INFRASTRUCTURE ONLY).

Follows pkg/src/pipecraft/executor.py:
  _sum_to        :50-56
  eval_op        :59-96   (per-kind numpy expressions)
  split_batch    :110-114
  run_reference  :117-134 (grads summed from zeros in microbatch order, one SGD)
and the FFN model / gradient rules of pkg/src/pipecraft/ir.py:228-264 and
:519-543 (matmul backward via explicit transposes, relu-grad, the
sub-sample-loss seed aliased to h).  The same numpy expressions in the same
order make the results bit-identical to the reference (checked against
golden_seed0.json with rel == 0).
"""
from __future__ import annotations

import numpy as np


def sum_to(x: np.ndarray, dims) -> np.ndarray:
    """executor.py:50-56."""
    while x.ndim > len(dims):
        x = x.sum(axis=0)
    for ax, d in enumerate(dims):
        if x.shape[ax] != d:
            x = x.sum(axis=ax, keepdims=True)
    return x.reshape(dims)


def eval_op(kind: str, args: list, attrs: dict | None = None, result_dims=()) -> np.ndarray:
    """executor.py:59-96 for one op whose operand values are ``args``."""
    a = args[0] if args else None
    if kind == "matmul":
        return a @ args[1]
    if kind == "add":
        return a + args[1]
    if kind == "relu":
        return np.maximum(a, 0.0)
    if kind == "sub-sample-loss":
        return np.asarray(0.5 * np.sum(a * a))
    if kind == "broadcast":
        return np.broadcast_to(a, result_dims).copy()
    if kind == "transpose":
        return np.transpose(a)
    if kind in ("scale", "mul"):
        return a * args[1]
    if kind == "yield-marker":
        return a
    if kind == "concat":
        return np.concatenate([np.atleast_1d(v) for v in args], axis=0)
    if kind == "relu-grad":
        return a * (args[1] > 0.0)
    if kind == "sum-to":
        return sum_to(a, tuple(result_dims))
    if kind == "slice":
        off, ln = attrs["offset"], attrs["length"]
        return a[off:off + ln]
    raise ValueError(f"oracle has no rule for {kind!r}")


def split_batch(batch: np.ndarray, M: int) -> list[np.ndarray]:
    """executor.py:110-114."""
    if batch.shape[0] % M:
        raise ValueError(f"batch of {batch.shape[0]} rows does not split into {M} microbatches")
    step = batch.shape[0] // M
    return [batch[i * step:(i + 1) * step] for i in range(M)]


def ffn_step(params: dict, x: np.ndarray, layers: int, tied: bool):
    """Forward + backward of the FFN stack for one microbatch.

    Returns (loss, {param: grad}) computed with the expressions the reference's
    derived graph evaluates (ir.py:519-543): dX = g @ W^T, dW = X^T @ g with
    np.transpose views, relu-grad g * (z > 0), seed gradient = h.
    """
    wname = [("w0" if (tied and k == layers - 1) else f"w{k}") for k in range(layers)]
    hs, zs = [], []
    h = x
    for k in range(layers):
        hs.append(h)
        z = h @ params[wname[k]]
        zs.append(z)
        h = np.maximum(z, 0.0) if k < layers - 1 else z
    loss = float(np.asarray(0.5 * np.sum(h * h)))
    g = h  # seed alias (ir.py:537-541)
    partial: dict[str, list] = {}
    for k in reversed(range(layers)):
        if k < layers - 1:
            g = g * (zs[k] > 0.0)
        w = params[wname[k]]
        dx = g @ np.transpose(w)
        dw = np.transpose(hs[k]) @ g
        partial.setdefault(wname[k], []).append((k, dw))
        g = dx
    grads = {}
    for q, parts in partial.items():
        parts.sort(key=lambda kv: kv[0])   # fold in use order (ir.py:447-466)
        acc = parts[0][1]
        for _, v in parts[1:]:
            acc = acc + v
        grads[q] = acc
    return loss, grads


def ffn_step_skips(params: dict, x: np.ndarray, layers: int, tied: bool, skips) -> tuple:
    """ffn_step with differentiable skip connections (ir.ModelConfig.skips): block
    src's activation a_src = relu(z_src) is added to block dst's input.  The
    reference has no executor for them (its planner rejects the gradient merge,
    ir.py:568-571), so this restatement is pinned to torch float64 autograd
    (tests/test_oracle.py) rather than to reference outputs.  The gradient
    reaching a_src is the main-path gradient plus the skip partials in
    ascending destination order (the planner's use order)."""
    wname = [("w0" if (tied and k == layers - 1) else f"w{k}") for k in range(layers)]
    hs, zs, acts = [], [], {}
    h = x
    for k in range(layers):
        for src, dst in skips:
            if dst == k:
                h = h + acts[src]
        hs.append(h)
        z = h @ params[wname[k]]
        zs.append(z)
        if k < layers - 1:
            h = np.maximum(z, 0.0)
            acts[k] = h
        else:
            h = z
    loss = float(np.asarray(0.5 * np.sum(h * h)))
    g = h
    back: dict[int, list] = {}
    partial: dict[str, list] = {}
    for k in reversed(range(layers)):
        if k < layers - 1:
            for _, extra in sorted(back.get(k, []), key=lambda t: t[0]):
                g = g + extra
            g = g * (zs[k] > 0.0)
        w = params[wname[k]]
        dx = g @ np.transpose(w)
        partial.setdefault(wname[k], []).append((k, np.transpose(hs[k]) @ g))
        for src, dst in skips:
            if dst == k:
                back.setdefault(src, []).append((dst, dx))
        g = dx
    grads = {}
    for q, parts in partial.items():
        parts.sort(key=lambda kv: kv[0])
        acc = parts[0][1]
        for _, v in parts[1:]:
            acc = acc + v
        grads[q] = acc
    return loss, grads


def run_reference_ffn(params: dict, batch: np.ndarray, M: int, layers: int, tied: bool,
                      lr: float = 0.1, skips=()):
    """executor.py:117-134 on the FFN model: returns (grads, losses, new_params)."""
    grads = {q: np.zeros_like(v) for q, v in params.items()}
    losses = []
    for mb in split_batch(batch, M):
        loss, g = (ffn_step_skips(params, mb, layers, tied, skips) if skips
                   else ffn_step(params, mb, layers, tied))
        losses.append(loss)
        for q in params:
            grads[q] = grads[q] + g[q]
    new_params = {q: params[q] - lr * grads[q] for q in params}
    return grads, np.asarray(losses), new_params


def init_params(names_dims, rng: np.random.Generator, scale: float = 0.4) -> dict:
    """pkg/tests/helpers.py:91-94 (N(0,1) * 0.4 in sorted param order)."""
    return {q: rng.standard_normal(dims) * scale for q, dims in sorted(names_dims.items())}


def init_batch(M: int, mbs: int, width: int, rng: np.random.Generator) -> np.ndarray:
    """pkg/tests/helpers.py:97-99."""
    return rng.standard_normal((M * mbs, width))


def rel(a, b) -> float:
    """Max-normalised relative error (pkg/tests/test_executor.py:21-24, cli.py:257-259)."""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    scale = max(float(np.max(np.abs(a))), float(np.max(np.abs(b))), 1e-30)
    return float(np.max(np.abs(a - b)) / scale)
