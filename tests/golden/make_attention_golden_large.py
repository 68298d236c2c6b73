"""Attention golden vectors at the benchmarked shapes, from flash-attn (the
paper's attention library; the image has 2.8.3).

The committed fixture (attention_flash_attn_large.npz) holds only flash-attn's
OUTPUTS: the inputs are regenerated from a seeded CPU torch generator
(`inputs(case)`, used by the generator here and by
tests/test_oracle_attention.py), so 64 MiB-per-request KV never enters the
repo. Shapes: config 2's decode (Llama-3-8B heads, lengths 4096 / 4033 / 1 /
2049), config 4's 70B heads, config 5's 32,752-token request, and config 3's
prefix-prefill (2048 shared + 512 new; every 16th query row and the last).

    python tests/golden/make_attention_golden_large.py   # on a B200
"""

from __future__ import annotations

import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "attention_flash_attn_large.npz")

# tag: (kind, seed, B, hq, hkv, L or (start, n), lens)
CASES = {
    "dec_cfg2": ("decode", 11, 4, 32, 8, 4096, [4096, 4033, 1, 2049]),
    "dec_70b": ("decode", 12, 2, 64, 8, 4096, [4095, 3969]),
    "dec_32k": ("decode", 13, 1, 32, 8, 32752, [32752]),
    "pre_cfg3": ("prefill", 14, 1, 32, 8, (2048, 512), None),
}
PREFILL_ROWS = list(range(0, 512, 16)) + [511]


def inputs(tag: str):
    """Seeded bf16 inputs of a case (CPU, deterministic). Decode: q [B, hq, d],
    k / v [B, hkv, L, d]. Prefill: q [n, hq, d], k / v [hkv, start + n, d]."""
    kind, seed, B, hq, hkv, L, _ = CASES[tag]
    g = torch.Generator().manual_seed(seed)
    if kind == "decode":
        q = torch.randn(B, hq, 128, generator=g).bfloat16()
        k = torch.randn(B, hkv, L, 128, generator=g).bfloat16()
        v = torch.randn(B, hkv, L, 128, generator=g).bfloat16()
        return q, k, v
    start, n = L
    q = torch.randn(n, hq, 128, generator=g).bfloat16()
    k = torch.randn(hkv, start + n, 128, generator=g).bfloat16()
    v = torch.randn(hkv, start + n, 128, generator=g).bfloat16()
    return q, k, v


def main(path: str) -> None:
    from flash_attn import flash_attn_func, flash_attn_with_kvcache

    arrays = {}
    for tag, (kind, _, B, hq, hkv, L, lens) in CASES.items():
        q, k, v = (t.cuda() for t in inputs(tag))
        if kind == "decode":
            o = flash_attn_with_kvcache(q[:, None], k.transpose(1, 2).contiguous(),
                                        v.transpose(1, 2).contiguous(),
                                        cache_seqlens=torch.tensor(lens, dtype=torch.int32,
                                                                   device="cuda"),
                                        causal=True)[:, 0]
        else:
            o = flash_attn_func(q[None], k.transpose(0, 1).contiguous()[None],
                                v.transpose(0, 1).contiguous()[None], causal=True)[0]
            o = o[PREFILL_ROWS]
        arrays[f"{tag}__out"] = o.float().cpu().numpy()
    np.savez_compressed(path, **arrays)
    print("wrote", path, {k: v.shape for k, v in arrays.items()})


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else OUT)
