"""The CPU attention oracle: internal consistency here, and (when the
flash-attn golden vectors exist) agreement with the paper's attention library."""

import os

import numpy as np
import pytest
import torch

from conftest import TESTS
from oracle.attention_ref import (decode_attention_ref, decode_attention_torch_cpu,
                                  prefill_attention_ref, rel_err)


def test_decode_loop_and_vectorised_agree():
    g = torch.Generator().manual_seed(0)
    B, hkv, hq, L = 3, 2, 8, 70
    q = torch.randn(B, hq, 128, generator=g).bfloat16()
    k = torch.randn(B, hkv, L, 128, generator=g).bfloat16()
    v = torch.randn(B, hkv, L, 128, generator=g).bfloat16()
    lens = [0, 1, 70]
    a = decode_attention_ref(q, [k[b, :, :n] for b, n in enumerate(lens)],
                             [v[b, :, :n] for b, n in enumerate(lens)])
    b = decode_attention_torch_cpu(q, k, v, lens)
    assert rel_err(b, a) < 1e-5
    assert np.all(a[0] == 0)


def test_decode_is_last_row_of_causal_prefill():
    """Decode of token n == prefill row for position n (same softmax)."""
    g = torch.Generator().manual_seed(1)
    hkv, hq, L = 2, 4, 33
    k = torch.randn(hkv, L, 128, generator=g)
    v = torch.randn(hkv, L, 128, generator=g)
    q = torch.randn(5, hq, 128, generator=g)
    pre = prefill_attention_ref(q, k, v, start=L - 5)
    dec = decode_attention_ref(q[-1:], [k], [v])
    assert rel_err(dec[0], pre[-1]) < 1e-6


def test_prefill_matches_torch_sdpa():
    g = torch.Generator().manual_seed(2)
    hkv, hq, start, n = 2, 8, 40, 24
    k = torch.randn(hkv, start + n, 128, generator=g)
    v = torch.randn(hkv, start + n, 128, generator=g)
    q = torch.randn(n, hq, 128, generator=g)
    ours = prefill_attention_ref(q, k, v, start)
    G = hq // hkv
    kk = k.repeat_interleave(G, 0)
    vv = v.repeat_interleave(G, 0)
    mask = torch.arange(start + n)[None, :] <= (start + torch.arange(n))[:, None]
    sd = torch.nn.functional.scaled_dot_product_attention(
        q.transpose(0, 1), kk, vv, attn_mask=mask)
    assert rel_err(ours, sd.transpose(0, 1)) < 1e-5


GOLDEN = os.path.join(TESTS, "golden", "attention_flash_attn.npz")


@pytest.mark.skipif(not os.path.exists(GOLDEN), reason="flash-attn golden not generated yet")
def test_oracle_matches_flash_attn_golden():
    z = np.load(GOLDEN)
    for tag in sorted({k.split("__")[0] for k in z.files}):
        kind = str(z[f"{tag}__kind"])
        q, k, v, o = (z[f"{tag}__{x}"].astype(np.float32) for x in ("q", "k", "v", "out"))
        if kind == "decode":
            lens = z[f"{tag}__lens"]
            ref = decode_attention_ref(q, [k[b, :, :n] for b, n in enumerate(lens)],
                                       [v[b, :, :n] for b, n in enumerate(lens)])
        else:
            start = int(z[f"{tag}__start"])
            ref = np.stack([prefill_attention_ref(q[b], k[b], v[b], start) for b in range(len(q))])
        assert rel_err(o, ref) < 2e-2, tag


GOLDEN_LARGE = os.path.join(TESTS, "golden", "attention_flash_attn_large.npz")


@pytest.mark.skipif(not os.path.exists(GOLDEN_LARGE), reason="large flash-attn golden not generated")
def test_oracle_matches_flash_attn_at_benchmarked_shapes():
    """The oracle against flash-attn at configs 2/4/5's decode shapes and
    config 3's prefill (inputs regenerated from the fixture's seeds)."""
    import sys

    sys.path.insert(0, os.path.join(TESTS, "golden"))
    from make_attention_golden_large import CASES, PREFILL_ROWS, inputs

    z = np.load(GOLDEN_LARGE)
    for tag, (kind, _, B, hq, hkv, L, lens) in CASES.items():
        q, k, v = inputs(tag)
        want = z[f"{tag}__out"]
        if kind == "decode":
            got = decode_attention_torch_cpu(q, k, v, lens)
        else:
            start, n = L
            G = hq // hkv
            rows = torch.tensor(PREFILL_ROWS)
            kf, vf = k.float(), v.float()
            qs = q[rows].float()  # [R, hq, d] at positions start + rows
            s = torch.einsum("rhd,hkd->hrk", qs, kf.repeat_interleave(G, 0)) / np.sqrt(128)
            mask = torch.arange(start + n)[None, :] <= (start + rows)[:, None]
            p = torch.softmax(s.masked_fill(~mask[None], float("-inf")), dim=-1)
            got = torch.einsum("hrk,hkd->rhd", p, vf.repeat_interleave(G, 0))
        assert rel_err(got, want) < 2e-2, tag
