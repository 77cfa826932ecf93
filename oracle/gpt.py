"""Float64 numpy GPT-2 oracle (TEST INFRASTRUCTURE ONLY).

The reference (pipecraft) has no GPT vocabulary (SURVEY.md key fact 5), so this
is a new CPU restatement that follows the reference's conventions:
per-microbatch forward + backward, gradients summed from zeros in microbatch
order and one SGD step (pkg/src/pipecraft/executor.py:117-134, the paper's
accumulate_grads loop).  PARITY UNPINNED BY THE REFERENCE:
it is pinned by central finite differences (tests/test_oracle.py, the method
of pkg/tests/test_ir.py:32-49) and torch float64 autograd.

Model (matches paper_2412_14374_b200.ir.GPTConfig / build_gpt semantics):
  h0 = wte[x] + wpe[pos]
  block: a = LN1(h); qkv = a Wqkv^T + bqkv; o = causal_attn(qkv) ; h1 = h + o Wo^T + bo
         a2 = LN2(h1); u = a2 W1^T + b1; h2 = h1 + gelu_tanh(u) W2^T + b2
         (last block additionally applies LN_f)
  loss = sum over positions t < S-1 of  logsumexp(h_t wte^T) - (h_t wte^T)[x_{t+1}]
Parameters are flat float vectors, one per block, laid out as below (offsets
rounded up to 64 elements).
"""
from __future__ import annotations

import math

import numpy as np

LN_EPS = 1e-5
_ALIGN = 64


def _layout(items):
    out, off = {}, 0
    for name, dims in items:
        out[name] = (off, dims)
        off += (math.prod(dims) + _ALIGN - 1) // _ALIGN * _ALIGN
    return out, off


def embed_layout(cfg):
    return _layout([("wte", (cfg["vocab"], cfg["d"])), ("wpe", (cfg["seq"], cfg["d"]))])


def block_layout(cfg, final: bool):
    d, f = cfg["d"], cfg["ff"]
    items = [("ln1_g", (d,)), ("ln1_b", (d,)), ("w_qkv", (3 * d, d)), ("b_qkv", (3 * d,)),
             ("w_o", (d, d)), ("b_o", (d,)), ("ln2_g", (d,)), ("ln2_b", (d,)),
             ("w_fc1", (f, d)), ("b_fc1", (f,)), ("w_fc2", (d, f)), ("b_fc2", (d,))]
    if final:
        items += [("lnf_g", (d,)), ("lnf_b", (d,))]
    return _layout(items)


def unpack(flat: np.ndarray, layout) -> dict:
    return {k: flat[o:o + math.prod(dims)].reshape(dims) for k, (o, dims) in layout.items()}


def param_sizes(cfg) -> dict:
    L = cfg["layers"]
    sizes = {"w0": embed_layout(cfg)[1]}
    for k in range(1, L + 1):
        sizes[f"w{k}"] = block_layout(cfg, k == L)[1]
    return sizes


def init_params(cfg, rng: np.random.Generator, std: float = 0.02) -> dict:
    """N(0, std) matrices, output projections scaled by 1/sqrt(2L), LN gamma=1,
    beta=0, biases 0 (SURVEY.md §8(d) value distributions)."""
    L = cfg["layers"]
    lay, n = embed_layout(cfg)
    w0 = np.zeros(n)
    for name, (o, dims) in lay.items():
        w0[o:o + math.prod(dims)] = rng.standard_normal(math.prod(dims)) * std
    out = {"w0": w0}
    for k in range(1, L + 1):
        lay, n = block_layout(cfg, k == L)
        w = np.zeros(n)
        for name, (o, dims) in lay.items():
            sz = math.prod(dims)
            if name.endswith("_g"):
                w[o:o + sz] = 1.0
            elif name.startswith("w_"):
                s = std / math.sqrt(2 * L) if name in ("w_o", "w_fc2") else std
                w[o:o + sz] = rng.standard_normal(sz) * s
        out[f"w{k}"] = w
    return out


def init_tokens(cfg, M: int, rng: np.random.Generator) -> np.ndarray:
    return rng.integers(0, cfg["vocab"], size=(M, cfg["mbs"], cfg["seq"])).astype(np.int32)


# ---------------------------------------------------------------------------
# primitives


def layer_norm(x, g, b):
    mu = x.mean(-1, keepdims=True)
    xc = x - mu
    var = (xc * xc).mean(-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + LN_EPS)
    xh = xc * rstd
    return xh * g + b, (xh, rstd)


def layer_norm_bwd(dy, g, cache):
    xh, rstd = cache
    dxh = dy * g
    dx = rstd * (dxh - dxh.mean(-1, keepdims=True) - xh * (dxh * xh).mean(-1, keepdims=True))
    return dx, (dy * xh).sum(0), dy.sum(0)


_K0, _K1 = 0.7978845608028654, 0.044715


def gelu(u):
    return 0.5 * u * (1.0 + np.tanh(_K0 * (u + _K1 * u ** 3)))


def gelu_grad(u):
    t = np.tanh(_K0 * (u + _K1 * u ** 3))
    return 0.5 * (1.0 + t) + 0.5 * u * (1.0 - t * t) * _K0 * (1.0 + 3.0 * _K1 * u * u)


def attention(q, k, v):
    """q,k,v: [B, H, S, hd]; causal softmax attention."""
    S = q.shape[2]
    scale = 1.0 / math.sqrt(q.shape[-1])
    s = (q @ np.swapaxes(k, -1, -2)) * scale
    s = np.where(np.tril(np.ones((S, S), dtype=bool)), s, -np.inf)
    s = s - s.max(-1, keepdims=True)
    p = np.exp(s)
    p /= p.sum(-1, keepdims=True)
    return p @ v, p


def attention_bwd(do, q, k, v, p):
    scale = 1.0 / math.sqrt(q.shape[-1])
    dv = np.swapaxes(p, -1, -2) @ do
    dp = do @ np.swapaxes(v, -1, -2)
    ds = p * (dp - (dp * p).sum(-1, keepdims=True))
    dq = (ds @ k) * scale
    dk = (np.swapaxes(ds, -1, -2) @ q) * scale
    return dq, dk, dv


def _split_heads(t, B, S, H):
    return t.reshape(B, S, H, -1).transpose(0, 2, 1, 3)


def _merge_heads(t):
    B, H, S, hd = t.shape
    return t.transpose(0, 2, 1, 3).reshape(B * S, H * hd)


# ---------------------------------------------------------------------------
# model


def block_fwd(h, P, cfg, B, final):
    S, H, d = cfg["seq"], cfg["heads"], cfg["d"]
    a, ln1 = layer_norm(h, P["ln1_g"], P["ln1_b"])
    qkv = a @ P["w_qkv"].T + P["b_qkv"]
    q, k, v = (_split_heads(qkv[:, i * d:(i + 1) * d], B, S, H) for i in range(3))
    o4, p = attention(q, k, v)
    o = _merge_heads(o4)
    h1 = h + o @ P["w_o"].T + P["b_o"]
    a2, ln2 = layer_norm(h1, P["ln2_g"], P["ln2_b"])
    u = a2 @ P["w_fc1"].T + P["b_fc1"]
    gu = gelu(u)
    out = h1 + gu @ P["w_fc2"].T + P["b_fc2"]
    lnf = None
    if final:
        out, lnf = layer_norm(out, P["lnf_g"], P["lnf_b"])
    cache = dict(h=h, a=a, ln1=ln1, q=q, k=k, v=v, p=p, o=o, h1=h1, a2=a2, ln2=ln2, u=u, gu=gu,
                 lnf=lnf)
    return out, cache


def block_bwd(dout, P, cfg, B, final, c):
    S, H, d = cfg["seq"], cfg["heads"], cfg["d"]
    G = {}
    if final:
        dout, G["lnf_g"], G["lnf_b"] = layer_norm_bwd(dout, P["lnf_g"], c["lnf"])
    dh1 = dout.copy()
    G["b_fc2"] = dout.sum(0)
    G["w_fc2"] = dout.T @ c["gu"]
    dgu = dout @ P["w_fc2"]
    du = dgu * gelu_grad(c["u"])
    G["b_fc1"] = du.sum(0)
    G["w_fc1"] = du.T @ c["a2"]
    da2 = du @ P["w_fc1"]
    dx, G["ln2_g"], G["ln2_b"] = layer_norm_bwd(da2, P["ln2_g"], c["ln2"])
    dh1 += dx
    G["b_o"] = dh1.sum(0)
    G["w_o"] = dh1.T @ c["o"]
    do = _split_heads(dh1 @ P["w_o"], B, S, H)
    dq, dk, dv = attention_bwd(do, c["q"], c["k"], c["v"], c["p"])
    dqkv = np.concatenate([_merge_heads(dq), _merge_heads(dk), _merge_heads(dv)], axis=1)
    G["b_qkv"] = dqkv.sum(0)
    G["w_qkv"] = dqkv.T @ c["a"]
    da = dqkv @ P["w_qkv"]
    dx, G["ln1_g"], G["ln1_b"] = layer_norm_bwd(da, P["ln1_g"], c["ln1"])
    return dh1 + dx, G


def head_loss(h, wte, tokens):
    """Summed next-token cross-entropy; returns (loss, dh, dwte)."""
    B, S = tokens.shape
    logits = h @ wte.T
    mx = logits.max(-1, keepdims=True)
    e = np.exp(logits - mx)
    z = e.sum(-1, keepdims=True)
    lse = (mx + np.log(z))[:, 0]
    tgt = np.zeros(B * S, dtype=np.int64)
    valid = np.zeros(B * S, dtype=bool)
    for b in range(B):
        tgt[b * S:b * S + S - 1] = tokens[b, 1:]
        valid[b * S:b * S + S - 1] = True
    rows = np.arange(B * S)
    loss = float(np.sum((lse - logits[rows, tgt])[valid]))
    dlog = e / z
    dlog[rows, tgt] -= 1.0
    dlog[~valid] = 0.0
    return loss, dlog @ wte, dlog.T @ h


def _pack(G: dict, layout, n) -> np.ndarray:
    flat = np.zeros(n)
    for k, (o, dims) in layout.items():
        if k in G:
            flat[o:o + math.prod(dims)] = np.asarray(G[k]).reshape(-1)
    return flat


def gpt_step(params: dict, tokens: np.ndarray, cfg):
    """One microbatch: returns (loss, {param name: flat grad})."""
    B, S, L = tokens.shape[0], cfg["seq"], cfg["layers"]
    elay, en = embed_layout(cfg)
    E = unpack(params["w0"], elay)
    pos = np.tile(np.arange(S), B)
    h = E["wte"][tokens.reshape(-1)] + E["wpe"][pos]
    caches, blays = [], []
    for k in range(1, L + 1):
        lay, n = block_layout(cfg, k == L)
        blays.append((lay, n))
        h, c = block_fwd(h, unpack(params[f"w{k}"], lay), cfg, B, k == L)
        caches.append(c)
    loss, dh, dwte_head = head_loss(h, E["wte"], tokens)
    grads = {}
    for k in range(L, 0, -1):
        lay, n = blays[k - 1]
        dh, G = block_bwd(dh, unpack(params[f"w{k}"], lay), cfg, B, k == L, caches[k - 1])
        grads[f"w{k}"] = _pack(G, lay, n)
    dwte = np.zeros_like(E["wte"])
    np.add.at(dwte, tokens.reshape(-1), dh)
    dwpe = np.zeros_like(E["wpe"])
    np.add.at(dwpe, pos, dh)
    # tied w0: embedding partial (stage 0) + head partial (last stage), ir fold order
    grads["w0"] = _pack({"wte": dwte, "wpe": dwpe}, elay, en) + _pack({"wte": dwte_head}, elay, en)
    return loss, grads


def run_reference_gpt(params: dict, tokens: np.ndarray, cfg, lr: float = 0.1):
    """Serial accumulation loop (executor.py:117-134) over microbatches
    tokens[M, mbs, seq]: returns (grads, losses, new_params)."""
    grads = {q: np.zeros_like(v) for q, v in params.items()}
    losses = []
    for i in range(tokens.shape[0]):
        loss, g = gpt_step(params, tokens[i], cfg)
        losses.append(loss)
        for q in params:
            grads[q] = grads[q] + g[q]
    new = {q: params[q] - lr * grads[q] for q in params}
    return grads, np.asarray(losses), new
