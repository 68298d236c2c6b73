"""The paper's comparison point on B200: paged-KV decode kernels from the
libraries shipped in this image (BASELINE only — never the product path).

The paper compares vTensor against vLLM's PagedAttention and a paged
FlashAttention (ref: PAPER.md:715-720); kvsim's baselines.py:101-195 only
accounts for their memory. Here the same KV bytes are copied into each
library's own paged layout and its kernel is timed and oracle-checked:

* ``flashinfer`` — ``flashinfer.decode.trtllm_batch_decode_with_kv_cache``
  (flashinfer 0.6.11, sm100 trtllm-gen kernels, bf16, HND layout), page size
  16 = one 2 MiB vTensor chunk at the Llama-3-8B geometry;
* ``vllm`` — ``torch.ops._C.paged_attention_v2`` (vLLM 0.22 CUDA-core
  PagedAttention, block size 16; the kernel family the paper measured).

Each builder returns a closure ``run(q, out)`` for one layer, or raises if the
library is unavailable on this box (callers report the reason).
"""

from __future__ import annotations

import math

import torch

from paper_2407_15309_b200.kv_layout import read_kv


def gather_pages(st, kv_va, lens, layer, page: int = 16, seed: int = 0):
    """One layer's K/V of every request as pages of ``page`` tokens at shuffled
    page ids: K, V ``[num_pages, Hkv, page, d]`` bf16 + block table
    ``[B, max_pages]`` int32 (a paged cache holding the same bytes)."""
    H, d = st.geo.kv_heads, st.geo.head_dim
    npg = [-(-n // page) for n in lens]
    total = max(sum(npg), 1)
    perm = torch.randperm(total, generator=torch.Generator().manual_seed(seed)).tolist()
    K = torch.zeros(total, H, page, d, dtype=torch.bfloat16, device="cuda")
    V = torch.zeros_like(K)
    table = torch.zeros(len(lens), max(max(npg), 1), dtype=torch.int32)
    k = 0
    for b, (va, n) in enumerate(zip(kv_va.tolist(), lens)):
        if n == 0:
            continue
        kk, vv = read_kv(va, n, layer, st.geo)  # [H, n, d]
        pad = npg[b] * page - n
        kk = torch.nn.functional.pad(kk, (0, 0, 0, pad)).view(H, npg[b], page, d).transpose(0, 1)
        vv = torch.nn.functional.pad(vv, (0, 0, 0, pad)).view(H, npg[b], page, d).transpose(0, 1)
        ids = perm[k:k + npg[b]]
        k += npg[b]
        idx = torch.tensor(ids, device="cuda")
        K[idx] = kk
        V[idx] = vv
        table[b, :npg[b]] = torch.tensor(ids, dtype=torch.int32)
    return K, V, table.cuda()


def flashinfer_decode(K, V, table, lens, hq: int, scale: float | None = None):
    import flashinfer.decode as fd

    d = K.shape[-1]
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    ws = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")
    seq = torch.tensor(lens, dtype=torch.int32, device="cuda")
    mx = max(lens)

    def run(q, out):
        return fd.trtllm_batch_decode_with_kv_cache(
            q, (K, V), ws, table, seq, mx, bmm1_scale=scale, bmm2_scale=1.0, out=out,
            kv_layout="HND", backend="trtllm-gen")

    return run


def vllm_decode(K, V, table, lens, hq: int, scale: float | None = None):
    import vllm._C  # noqa: F401  (registers torch.ops._C)

    n_pages, H, page, d = K.shape
    x = 16 // K.element_size()
    # vLLM layout: key [blocks, H, d/x, page, x], value [blocks, H, d, page]
    kc = K.view(n_pages, H, page, d // x, x).permute(0, 1, 3, 2, 4).contiguous()
    vc = V.permute(0, 1, 3, 2).contiguous()
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    B = len(lens)
    part = 512
    max_parts = -(-max(lens) // part)
    exp_sums = torch.empty(B, hq, max_parts, dtype=torch.float32, device="cuda")
    max_logits = torch.empty_like(exp_sums)
    tmp = torch.empty(B, hq, max_parts, d, dtype=torch.bfloat16, device="cuda")
    seq = torch.tensor(lens, dtype=torch.int32, device="cuda")
    one = torch.tensor(1.0, dtype=torch.float32, device="cuda")
    mx = max(lens)

    def run(q, out):
        torch.ops._C.paged_attention_v2(out, exp_sums, max_logits, tmp, q, kc, vc, H, scale,
                                        table, seq, page, mx, None, "auto", one, one, 0, 0, 0,
                                        64, 0)
        return out

    return run


BUILDERS = {"flashinfer_trtllm_gen": flashinfer_decode, "vllm_paged_attention_v2": vllm_decode}
