"""Float64 torch restatements of oracle/gpt.py pieces (TEST INFRASTRUCTURE ONLY).

The numpy oracle is exact but too slow on the CPU at BASELINE sizes (C2/C3
attention is 13 GFLOP per call, the LM-head cross-entropy reads 412 M logits).
These functions compute the same float64 math with torch so it can run on the
GPU box's device; `tests/test_torch_ref.py` pins each of them to the numpy
oracle (oracle/gpt.py, oracle/llama.py) on small inputs, rel < 1e-12, on the CPU.
"""
from __future__ import annotations

import math

import torch


def attention_fwd(q, k, v, causal: bool = True):
    """q [B,H,S,hd], k/v [B,Hkv,S,hd] float64 -> (o [B,H,S,hd], lse [B,H,S]).
    Query head h reads kv head h // (H / Hkv) (grouped-query attention; H == Hkv is
    plain multi-head).  Same math as oracle/gpt.py `attention`."""
    B, H, S, hd = q.shape
    g = H // k.shape[1]
    if g > 1:
        k = k.repeat_interleave(g, dim=1)
        v = v.repeat_interleave(g, dim=1)
    s = (q @ k.transpose(-1, -2)) / math.sqrt(hd)
    if causal:
        mask = torch.ones(S, S, dtype=torch.bool, device=q.device).tril()
        s = s.masked_fill(~mask, float("-inf"))
    lse = torch.logsumexp(s, -1)
    p = torch.exp(s - lse[..., None])
    return p @ v, lse


def attention_bwd(do, q, k, v, lse, causal: bool = True):
    """Gradients of attention_fwd: (dq [B,H,S,hd], dk, dv [B,Hkv,S,hd]).  The group
    sum of a kv head's gradient runs over its query heads (oracle/llama.py GQA)."""
    B, H, S, hd = q.shape
    Hkv = k.shape[1]
    g = H // Hkv
    ke = k.repeat_interleave(g, dim=1) if g > 1 else k
    ve = v.repeat_interleave(g, dim=1) if g > 1 else v
    scale = 1.0 / math.sqrt(hd)
    s = (q @ ke.transpose(-1, -2)) * scale
    if causal:
        mask = torch.ones(S, S, dtype=torch.bool, device=q.device).tril()
        s = s.masked_fill(~mask, float("-inf"))
    p = torch.exp(s - lse[..., None])
    dv = p.transpose(-1, -2) @ do
    dp = do @ ve.transpose(-1, -2)
    ds = p * (dp - (dp * p).sum(-1, keepdim=True))
    dq = (ds @ ke) * scale
    dk = (ds.transpose(-1, -2) @ q) * scale
    if g > 1:
        dk = dk.reshape(B, Hkv, g, S, hd).sum(2)
        dv = dv.reshape(B, Hkv, g, S, hd).sum(2)
    return dq, dk, dv


def xent_rows(logits, tokens):
    """Next-token cross-entropy of oracle/gpt.py `head_loss` given the logits:
    logits [B*S, V] float64, tokens [B, S] -> (row_loss [B*S], dlogits [B*S, V]).
    The last position of each sequence has no target: loss 0, dlogits 0."""
    B, S = tokens.shape
    lse = torch.logsumexp(logits, -1)
    tgt = torch.zeros(B, S, dtype=torch.long, device=logits.device)
    tgt[:, :-1] = tokens[:, 1:].long()
    tgt = tgt.reshape(-1)
    valid = torch.ones(B, S, dtype=torch.bool, device=logits.device)
    valid[:, -1] = False
    valid = valid.reshape(-1)
    rows = torch.arange(B * S, device=logits.device)
    loss = (lse - logits[rows, tgt]) * valid
    dl = torch.exp(logits - lse[:, None])
    dl[rows, tgt] -= 1.0
    dl[~valid] = 0.0
    return loss, dl


def embedding_bwd(tokens, dh, vocab: int, seq: int):
    """dwte[v] = sum of dh rows whose token is v; dwpe[p] = sum of rows at position p
    (oracle/gpt.py gpt_step's embedding gradient, np.add.at)."""
    T, d = dh.shape
    dwte = torch.zeros(vocab, d, dtype=dh.dtype, device=dh.device)
    dwte.index_add_(0, tokens.reshape(-1).long(), dh)
    dwpe = torch.zeros(seq, d, dtype=dh.dtype, device=dh.device)
    dwpe.index_add_(0, torch.arange(T, device=dh.device) % seq, dh)
    return dwte, dwpe


def rel(a, b) -> float:
    """The reference's max-normalised error (pkg/src/pipecraft/cli.py:257-259)."""
    a = a.double()
    b = b.double()
    den = max(a.abs().max().item(), b.abs().max().item(), 1e-30)
    return (a - b).abs().max().item() / den
