"""Generate attention golden vectors with flash-attn (the paper's attention
library: PAPER.md:666,689 use flash-attn 2.5.8; the image has 2.8.3).

Runs on a B200 (flash-attn needs CUDA). Inputs are seeded bf16; outputs are
flash-attn's. Saved as float32 arrays of the bf16 values so the CPU test
(tests/test_oracle_attention.py) can check oracle/attention_ref.py against
them without a GPU.

    python tests/golden/make_attention_golden.py [out.npz]
"""

from __future__ import annotations

import os
import sys

import numpy as np
import torch
from flash_attn import flash_attn_func, flash_attn_with_kvcache


def main(path: str) -> None:
    torch.manual_seed(20240721)
    dev = "cuda"
    arrays = {}

    def put(tag, kind, **kv):
        arrays[f"{tag}__kind"] = np.array(kind)
        for k, v in kv.items():
            arrays[f"{tag}__{k}"] = v.float().cpu().numpy() if torch.is_tensor(v) else np.asarray(v)

    # decode: one query per request at the end of its sequence, GQA 4 and 1
    for tag, (B, hq, hkv, L, lens) in {
        "dec_gqa4": (3, 8, 2, 160, [1, 77, 160]),
        "dec_mha": (2, 4, 4, 96, [96, 33]),
    }.items():
        q = torch.randn(B, hq, 128, device=dev).bfloat16()
        k = torch.randn(B, L, hkv, 128, device=dev).bfloat16()
        v = torch.randn(B, L, hkv, 128, device=dev).bfloat16()
        seqlens = torch.tensor(lens, dtype=torch.int32, device=dev)
        o = flash_attn_with_kvcache(q[:, None], k, v, cache_seqlens=seqlens, causal=True)[:, 0]
        put(tag, "decode", q=q, k=k.transpose(1, 2), v=v.transpose(1, 2), out=o, lens=np.array(lens))

    # prefix-prefill: n_new queries after a `start`-token prefix, causal
    # (bottom-right aligned: new token i sees KV [0, start+i])
    for tag, (B, hq, hkv, start, n) in {"pre_gqa4": (2, 8, 2, 64, 48)}.items():
        q = torch.randn(B, n, hq, 128, device=dev).bfloat16()
        k = torch.randn(B, start + n, hkv, 128, device=dev).bfloat16()
        v = torch.randn(B, start + n, hkv, 128, device=dev).bfloat16()
        o = flash_attn_func(q, k, v, causal=True)
        put(tag, "prefill", q=q, k=k.transpose(1, 2), v=v.transpose(1, 2), out=o,
            start=np.array(start))

    np.savez_compressed(path, **arrays)
    print("wrote", path, {k: v.shape for k, v in arrays.items()})


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else
         os.path.join(os.path.dirname(os.path.abspath(__file__)), "attention_flash_attn.npz"))
