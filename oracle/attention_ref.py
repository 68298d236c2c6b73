"""ORACLE (test infrastructure only) — CPU fp32 restatement of vTensor attention.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this module, and only as the checker or
the CPU baseline. The product path (paper_2407_15309_b200) never imports it.

What it restates. The reference package (kvsim) has no attention: its compute
slot is a cost formula (pkg/src/kvsim/engine.py:499-511). The paper defines
the attention it runs on vTensor pointers by reference to FlashAttention
(PAPER.md:366-381 background; "integrate flash-attn-2.5.8 into
FlexInfer using vTensor"; "We adopt the v2.5.8 version of
FlashAttention"). So the algorithm lives in a third-party dependency that is
absent from /root/reference: flash-attn 2.5.8. Its published algorithm is
exact softmax attention,

    O[h] = softmax(scale * Q[h] . K[h // G]^T + mask) . V[h // G]

with GQA head grouping G = Hq / Hkv, scale = 1/sqrt(d), no mask for decode
(one query at the end of the sequence) and a causal mask for prefill where new
token i at absolute position start+i sees KV [0, start+i] (prefix reuse:
PAPER.md:743-749). Computed here in float32 (float64 softmax accumulation)
from the *same bf16 KV bytes* the kernels read, copied back from the vTensor
VAs.

Parity pinning. tests/golden/make_attention_golden.py runs the image's
flash-attn 2.8.3 (same library, later release) on seeded inputs on a B200 and
commits inputs + outputs; tests/test_oracle_attention.py checks this
restatement against those vectors. Tolerance: 2e-2 relative for bf16 inputs
with fp32 accumulation (BASELINE.json north_star).
"""

from __future__ import annotations

import numpy as np


def _as_f32(x) -> np.ndarray:
    try:  # torch tensor (any dtype, any device)
        import torch

        if isinstance(x, torch.Tensor):
            return x.detach().to("cpu", torch.float32).numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x, dtype=np.float32)


def decode_attention_ref(q, ks, vs, scale: float | None = None) -> np.ndarray:
    """Decode for a batch.

    q  : [B, Hq, d]
    ks : list of B arrays [Hkv, len_b, d]   (len_b may be 0 -> zero output)
    vs : list of B arrays [Hkv, len_b, d]
    returns [B, Hq, d] float32
    """
    q = _as_f32(q)
    B, Hq, d = q.shape
    scale = 1.0 / np.sqrt(d) if scale is None else scale
    out = np.zeros((B, Hq, d), dtype=np.float32)
    for b in range(B):
        k = _as_f32(ks[b])
        v = _as_f32(vs[b])
        hkv, n, _ = k.shape
        if n == 0:
            continue
        G = Hq // hkv
        for h in range(Hq):
            s = (k[h // G] @ q[b, h]).astype(np.float64) * scale  # [n]
            s -= s.max()
            p = np.exp(s)
            p /= p.sum()
            out[b, h] = (p @ v[h // G].astype(np.float64)).astype(np.float32)
    return out


def prefill_attention_ref(q, k, v, start: int, scale: float | None = None) -> np.ndarray:
    """Prefix-prefill for one request.

    q    : [n_new, Hq, d]  queries at absolute positions start .. start+n_new-1
    k, v : [Hkv, start + n_new, d]  full KV (shared prefix + new tokens)
    returns [n_new, Hq, d] float32 (new token i attends to KV [0, start+i])
    """
    q = _as_f32(q)
    k = _as_f32(k).astype(np.float64)
    v = _as_f32(v).astype(np.float64)
    n_new, Hq, d = q.shape
    hkv = k.shape[0]
    G = Hq // hkv
    scale = 1.0 / np.sqrt(d) if scale is None else scale
    out = np.zeros((n_new, Hq, d), dtype=np.float32)
    pos = start + np.arange(n_new)
    keys = np.arange(k.shape[1])
    mask = keys[None, :] <= pos[:, None]  # [n_new, L]
    for h in range(Hq):
        s = (q[:, h].astype(np.float64) @ k[h // G].T) * scale  # [n_new, L]
        s = np.where(mask, s, -np.inf)
        s -= s.max(axis=1, keepdims=True)
        p = np.exp(s)
        p /= p.sum(axis=1, keepdims=True)
        out[:, h] = (p @ v[h // G]).astype(np.float32)
    return out


def rel_err(got, want) -> float:
    """max |got - want| / max(|want|) — the 2e-2 criterion."""
    got = _as_f32(got).astype(np.float64)
    want = _as_f32(want).astype(np.float64)
    denom = max(np.abs(want).max(), 1e-6)
    return float(np.abs(got - want).max() / denom)


def decode_attention_torch_cpu(q, k, v, lens, scale: float | None = None):
    """Same math as :func:`decode_attention_ref`, vectorised per request with
    torch fp32 matmuls on all host threads — the timed CPU baseline.

    q : [B, Hq, d];  k, v : [B, Hkv, Lmax, d] (bf16 or fp32);  lens : B ints.
    """
    import torch

    B, Hq, d = q.shape
    hkv = k.shape[1]
    G = Hq // hkv
    scale = 1.0 / float(np.sqrt(d)) if scale is None else scale
    out = torch.zeros(B, Hq, d, dtype=torch.float32)
    for b in range(B):
        n = int(lens[b])
        if n == 0:
            continue
        kb = k[b, :, :n].float()
        vb = v[b, :, :n].float()
        qb = q[b].float().view(hkv, G, d)
        p = torch.softmax(torch.matmul(qb, kb.transpose(1, 2)) * scale, dim=-1)
        out[b] = torch.matmul(p, vb).reshape(Hq, d)
    return out
