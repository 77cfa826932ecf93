"""Float64 numpy Llama-style oracle (TEST INFRASTRUCTURE ONLY).

BASELINE config C5: RMSNorm, rotary position embeddings,
grouped-query attention, SwiGLU MLP, untied LM head, and the position ids as a
non-differentiable input that every block reads (so a pipelined plan sends it
from stage 0 to every later stage: the non-adjacent skip tensors of C5).

As for oracle/gpt.py, the reference (pipecraft) has no model vocabulary of
this kind: PARITY UNPINNED BY THE REFERENCE.  The arithmetic is pinned by
central finite differences (tests/test_oracle.py, the method of
pkg/tests/test_ir.py:32-49); the accumulation loop is the reference's
run_reference (pkg/src/pipecraft/executor.py:117-134).

Model (paper_2412_14374_b200.ir.LlamaConfig / build_llama):
  h0 = wte[x]
  block: a = RMS1(h); [q | k | v] = a Wqkv^T (q: H heads, k, v: Hkv heads)
         q, k = rope(q, pos), rope(k, pos); o = causal_gqa_attn(q, k, v)
         h1 = h + o Wo^T
         a2 = RMS2(h1); [g | u] = a2 Wgu^T; h2 = h1 + (silu(g) * u) Wdown^T
         (last block additionally applies RMS_f)
  loss = sum over positions t < S-1 of logsumexp(h_t Whead^T) - (h_t Whead^T)[x_{t+1}]
rope: rotate-half convention, angle(pos, i) = pos * theta^(-2i/hd), i < hd/2.
"""
from __future__ import annotations

import math

import numpy as np

from .gpt import _layout, unpack, head_loss as _tied_head_loss  # noqa: F401  (layout helper)

RMS_EPS = 1e-5


def embed_layout(cfg):
    return _layout([("wte", (cfg["vocab"], cfg["d"]))])


def head_layout(cfg):
    return _layout([("w_head", (cfg["vocab"], cfg["d"]))])


def block_layout(cfg, final: bool):
    d, f, H, Hkv = cfg["d"], cfg["ff"], cfg["heads"], cfg["kv_heads"]
    hd = d // H
    items = [("rms1_g", (d,)), ("w_qkv", ((H + 2 * Hkv) * hd, d)), ("w_o", (d, H * hd)),
             ("rms2_g", (d,)), ("w_gu", (2 * f, d)), ("w_down", (d, f))]
    if final:
        items += [("rmsf_g", (d,))]
    return _layout(items)


def param_sizes(cfg) -> dict:
    L = cfg["layers"]
    sizes = {"w0": embed_layout(cfg)[1], "wout": head_layout(cfg)[1]}
    for k in range(1, L + 1):
        sizes[f"w{k}"] = block_layout(cfg, k == L)[1]
    return sizes


def init_params(cfg, rng: np.random.Generator, std: float = 0.02) -> dict:
    """N(0, std) matrices, output projections (w_o, w_down) scaled 1/sqrt(2L),
    RMSNorm gains 1 (SURVEY.md §8(d) value distributions)."""
    L = cfg["layers"]
    out = {}
    for name, (lay, n) in (("w0", embed_layout(cfg)), ("wout", head_layout(cfg))):
        w = np.zeros(n)
        for _, (o, dims) in lay.items():
            w[o:o + math.prod(dims)] = rng.standard_normal(math.prod(dims)) * std
        out[name] = w
    for k in range(1, L + 1):
        lay, n = block_layout(cfg, k == L)
        w = np.zeros(n)
        for name, (o, dims) in lay.items():
            sz = math.prod(dims)
            if name.endswith("_g"):
                w[o:o + sz] = 1.0
            else:
                s = std / math.sqrt(2 * L) if name in ("w_o", "w_down") else std
                w[o:o + sz] = rng.standard_normal(sz) * s
        out[f"w{k}"] = w
    return out


def init_tokens(cfg, M: int, rng: np.random.Generator) -> np.ndarray:
    return rng.integers(0, cfg["vocab"], size=(M, cfg["mbs"], cfg["seq"])).astype(np.int32)


def positions(cfg, M: int) -> np.ndarray:
    """Position ids [M, mbs, seq] (0..seq-1 per sequence)."""
    return np.broadcast_to(np.arange(cfg["seq"], dtype=np.int32),
                           (M, cfg["mbs"], cfg["seq"])).copy()


# ---------------------------------------------------------------------------
# primitives


def rms_norm(x, g):
    rstd = 1.0 / np.sqrt((x * x).mean(-1, keepdims=True) + RMS_EPS)
    xh = x * rstd
    return xh * g, (xh, rstd)


def rms_norm_bwd(dy, g, cache):
    xh, rstd = cache
    dxh = dy * g
    dx = rstd * (dxh - xh * (dxh * xh).mean(-1, keepdims=True))
    return dx, (dy * xh).sum(0)


def rope_angles(pos, hd, theta):
    """cos, sin [T, hd/2] for position ids pos [T]."""
    inv = theta ** (-np.arange(0, hd // 2, dtype=np.float64) * 2.0 / hd)
    ang = pos.astype(np.float64)[:, None] * inv[None, :]
    return np.cos(ang), np.sin(ang)


def rope(t, cos, sin, inverse=False):
    """t [T, nh, hd] rotated per rotate-half: (t1, t2) -> (t1 c - t2 s, t2 c + t1 s).
    inverse=True applies the transpose rotation (the backward map)."""
    half = t.shape[-1] // 2
    t1, t2 = t[..., :half], t[..., half:]
    c, s = cos[:, None, :], sin[:, None, :]
    if inverse:
        s = -s
    return np.concatenate([t1 * c - t2 * s, t2 * c + t1 * s], axis=-1)


def silu(g):
    return g / (1.0 + np.exp(-g))


def silu_grad(g):
    sg = 1.0 / (1.0 + np.exp(-g))
    return sg * (1.0 + g * (1.0 - sg))


def gqa_attention(q, k, v):
    """q [B, H, S, hd], k, v [B, Hkv, S, hd]: causal softmax attention where
    query head h reads kv head h // (H / Hkv)."""
    from .gpt import attention
    G = q.shape[1] // k.shape[1]
    return attention(q, np.repeat(k, G, axis=1), np.repeat(v, G, axis=1))


def gqa_attention_bwd(do, q, k, v, p):
    from .gpt import attention_bwd
    B, Hkv, S, hd = k.shape
    G = q.shape[1] // Hkv
    dq, dk, dv = attention_bwd(do, q, np.repeat(k, G, axis=1), np.repeat(v, G, axis=1), p)
    return dq, dk.reshape(B, Hkv, G, S, hd).sum(2), dv.reshape(B, Hkv, G, S, hd).sum(2)


def _heads(t, B, S, nh):
    return t.reshape(B, S, nh, -1).transpose(0, 2, 1, 3)


def _merge(t):
    B, nh, S, hd = t.shape
    return t.transpose(0, 2, 1, 3).reshape(B * S, nh * hd)


# ---------------------------------------------------------------------------
# model


def block_fwd(h, P, pos, cfg, B, final):
    S, H, Hkv, d = cfg["seq"], cfg["heads"], cfg["kv_heads"], cfg["d"]
    hd, f = d // H, cfg["ff"]
    cos, sin = rope_angles(pos, hd, cfg["theta"])
    a, r1 = rms_norm(h, P["rms1_g"])
    qkv = a @ P["w_qkv"].T
    q = rope(qkv[:, :H * hd].reshape(-1, H, hd), cos, sin)
    k = rope(qkv[:, H * hd:(H + Hkv) * hd].reshape(-1, Hkv, hd), cos, sin)
    v = qkv[:, (H + Hkv) * hd:].reshape(-1, Hkv, hd)
    q4, k4, v4 = (_heads(t.reshape(B * S, -1), B, S, n) for t, n in ((q, H), (k, Hkv), (v, Hkv)))
    o4, p = gqa_attention(q4, k4, v4)
    o = _merge(o4)
    h1 = h + o @ P["w_o"].T
    a2, r2 = rms_norm(h1, P["rms2_g"])
    gu = a2 @ P["w_gu"].T
    g, u = gu[:, :f], gu[:, f:]
    m = silu(g) * u
    out = h1 + m @ P["w_down"].T
    rf = None
    if final:
        out, rf = rms_norm(out, P["rmsf_g"])
    cache = dict(h=h, a=a, r1=r1, q4=q4, k4=k4, v4=v4, p=p, o=o, h1=h1, a2=a2, r2=r2, g=g, u=u,
                 m=m, rf=rf, cos=cos, sin=sin)
    return out, cache


def block_bwd(dout, P, cfg, B, final, c):
    S, H, Hkv, d = cfg["seq"], cfg["heads"], cfg["kv_heads"], cfg["d"]
    hd = d // H
    G = {}
    if final:
        dout, G["rmsf_g"] = rms_norm_bwd(dout, P["rmsf_g"], c["rf"])
    dh1 = dout.copy()
    G["w_down"] = dout.T @ c["m"]
    dm = dout @ P["w_down"]
    dg = dm * c["u"] * silu_grad(c["g"])
    du = dm * silu(c["g"])
    dgu = np.concatenate([dg, du], axis=1)
    G["w_gu"] = dgu.T @ c["a2"]
    da2 = dgu @ P["w_gu"]
    dx, G["rms2_g"] = rms_norm_bwd(da2, P["rms2_g"], c["r2"])
    dh1 += dx
    G["w_o"] = dh1.T @ c["o"]
    do = _heads(dh1 @ P["w_o"], B, S, H)
    dq4, dk4, dv4 = gqa_attention_bwd(do, c["q4"], c["k4"], c["v4"], c["p"])
    dq = rope(_merge(dq4).reshape(-1, H, hd), c["cos"], c["sin"], inverse=True)
    dk = rope(_merge(dk4).reshape(-1, Hkv, hd), c["cos"], c["sin"], inverse=True)
    dqkv = np.concatenate([dq.reshape(B * S, -1), dk.reshape(B * S, -1), _merge(dv4)], axis=1)
    G["w_qkv"] = dqkv.T @ c["a"]
    da = dqkv @ P["w_qkv"]
    dx, G["rms1_g"] = rms_norm_bwd(da, P["rms1_g"], c["r1"])
    return dh1 + dx, G


def head_loss(h, w_head, tokens):
    """Summed next-token cross-entropy with an untied head: (loss, dh, dw_head)."""
    return _tied_head_loss(h, w_head, tokens)


def _pack(G: dict, layout, n) -> np.ndarray:
    flat = np.zeros(n)
    for k, (o, dims) in layout.items():
        if k in G:
            flat[o:o + math.prod(dims)] = np.asarray(G[k]).reshape(-1)
    return flat


def llama_step(params: dict, tokens: np.ndarray, pos: np.ndarray, cfg):
    """One microbatch: returns (loss, {param name: flat grad})."""
    B, L = tokens.shape[0], cfg["layers"]
    elay, en = embed_layout(cfg)
    hlay, hn = head_layout(cfg)
    wte = unpack(params["w0"], elay)["wte"]
    w_head = unpack(params["wout"], hlay)["w_head"]
    p = pos.reshape(-1)
    h = wte[tokens.reshape(-1)]
    caches, blays = [], []
    for k in range(1, L + 1):
        lay, n = block_layout(cfg, k == L)
        blays.append((lay, n))
        h, c = block_fwd(h, unpack(params[f"w{k}"], lay), p, cfg, B, k == L)
        caches.append(c)
    loss, dh, dw_head = head_loss(h, w_head, tokens)
    grads = {"wout": _pack({"w_head": dw_head}, hlay, hn)}
    for k in range(L, 0, -1):
        lay, n = blays[k - 1]
        dh, G = block_bwd(dh, unpack(params[f"w{k}"], lay), cfg, B, k == L, caches[k - 1])
        grads[f"w{k}"] = _pack(G, lay, n)
    dwte = np.zeros_like(wte)
    np.add.at(dwte, tokens.reshape(-1), dh)
    grads["w0"] = _pack({"wte": dwte}, elay, en)
    return loss, grads


def run_reference_llama(params: dict, tokens: np.ndarray, pos: np.ndarray, cfg, lr: float = 0.1):
    """Serial accumulation loop (executor.py:117-134) over microbatches
    tokens / pos [M, mbs, seq]: returns (grads, losses, new_params)."""
    grads = {q: np.zeros_like(v) for q, v in params.items()}
    losses = []
    for i in range(tokens.shape[0]):
        loss, g = llama_step(params, tokens[i], pos[i], cfg)
        losses.append(loss)
        for q in params:
            grads[q] = grads[q] + g[q]
    new = {q: params[q] - lr * grads[q] for q in params}
    return grads, np.asarray(losses), new
