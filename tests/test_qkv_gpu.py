"""Fused QKV projection + KV append on the B200.

The kernel computes qkv = x · W_qkvᵀ from the packed weight (bf16 in, fp32
accumulate; each feature tile's K halves on a 2-CTA cluster, the upper half's
partial added by the lower CTA through distributed shared memory) and writes
K/V of token t straight into the vTensor cache of request tok_req[t] at
tok_pos[t]. Cases cover one and two CTAs per tile, token tiles of 64/128/256
and several token tiles (more clusters than SMs). Checked against a torch fp32 GEMM
of the same bf16 inputs (the oracle for a floating-point kernel); tolerance
2e-2 relative (north_star), measured ~4e-3 (one bf16 rounding). Every other
KV row of the written layer and every other layer must be byte-identical.
"""

import pytest
import torch

from oracle.attention_ref import rel_err
from paper_2407_15309_b200.attention import decode_attention, pack_qkv_weight, qkv_append
from paper_2407_15309_b200.kv_layout import chunk_view
from vt_gpu_util import admit_with_lengths, cuda_stack

TOL = 2e-2

CASES = {
    # name: (layers, kv_heads, q_heads, hidden, lens, tokens_per_request, split_k)
    "llama8b_decode_b16": (32, 8, 32, 4096, [15, 16, 31, 200, 1, 0, 511, 77] * 2, 1, 0),
    "llama8b_decode_b64_nosplit": (32, 8, 32, 4096, list(range(3, 3 + 64 * 17, 17)), 1, 1),
    "prefill_chunks_300_tokens": (32, 8, 32, 4096, [16, 40, 0], 100, 0),
    "gqa8_hidden_1024_split2": (16, 2, 16, 1024, [5, 17, 33, 129], 3, 2),
    "gqa8_hidden_1024_auto": (16, 2, 16, 1024, [5, 17, 33, 129], 3, 0),
    "llama8b_b100_nt128": (32, 8, 32, 4096, list(range(7, 7 + 100 * 9, 9)), 1, 0),
    "prefill_1000_tokens_multi_segment": (32, 8, 32, 4096, [0, 16, 100, 333], 250, 0),
    "llama8b_decode_b64_split3": (32, 8, 32, 4096, list(range(3, 3 + 64 * 17, 17)), 1, 3),
    "gqa8_hidden_1024_split3": (16, 2, 16, 1024, [5, 17, 33, 129], 3, 3),
    "odd_tile_count_split3": (16, 1, 3, 1024, [5, 17, 300], 2, 3),
}


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_qkv_append_matches_torch(cuda_ok, name):
    layers, hkv, hq, hidden, lens, per_req, split_k = CASES[name]
    st = cuda_stack(layers, hkv, hq, 4096)
    kv_va, seq = admit_with_lengths(st, lens, seed=11)
    tpc = st.cfg.tokens_per_chunk
    for i, n in enumerate(lens):  # map the pages the new tokens land in
        st.sched.extend(f"req{i}", n + per_req)
    st.dev.wait()
    tok_req = torch.arange(len(lens), device="cuda", dtype=torch.int32).repeat_interleave(per_req)
    tok_pos = (seq.repeat_interleave(per_req) +
               torch.arange(per_req, device="cuda", dtype=torch.int32).repeat(len(lens)))
    T = tok_req.numel()
    gen = torch.Generator(device="cuda").manual_seed(len(name))
    feats = (hq + 2 * hkv) * 128
    x = torch.randn(T, hidden, generator=gen, device="cuda").to(torch.bfloat16)
    w = (torch.randn(feats, hidden, generator=gen, device="cuda") / hidden ** 0.5).to(torch.bfloat16)
    layer = layers - 2
    pages = [st.sched.mem[f"req{i}"].vt.space.mapped_pages for i in range(len(lens))]
    before = [chunk_view(va, p, st.geo).clone() for va, p in zip(kv_va.tolist(), pages)]

    q = qkv_append(x, pack_qkv_weight(w), tok_req, tok_pos, kv_va, st.geo, layer, split_k=split_k)
    torch.cuda.synchronize()

    ref = (x.float() @ w.float().T).view(T, hq + 2 * hkv, 128)
    assert rel_err(q.float().cpu(), ref[:, :hq].cpu()) <= TOL
    after = [chunk_view(va, p, st.geo).clone() for va, p in zip(kv_va.tolist(), pages)]
    for b in range(len(lens)):
        expect = before[b].clone()
        for t in torch.nonzero(tok_req == b).flatten().tolist():
            pos = int(tok_pos[t])
            c, r = divmod(pos, tpc)
            # compare the written rows with the oracle, then splice them in
            got_k = after[b][c, layer, 0, :, r].float().cpu()
            got_v = after[b][c, layer, 1, :, r].float().cpu()
            assert rel_err(got_k, ref[t, hq:hq + hkv].cpu()) <= TOL
            assert rel_err(got_v, ref[t, hq + hkv:].cpu()) <= TOL
            expect[c, layer, :, :, r] = after[b][c, layer, :, :, r]
        assert torch.equal(after[b], expect), f"request {b}: bytes outside the new rows changed"


@pytest.mark.gpu
def test_qkv_append_feeds_decode(cuda_ok):
    """The step order of a decode iteration: extend → fused QKV + append →
    decode over len+1 reading the K/V the projection just wrote."""
    from oracle.attention_ref import decode_attention_ref
    from vt_gpu_util import gather

    layers, hkv, hq, hidden = 32, 8, 32, 4096
    lens = [15, 16, 200, 1023]
    st = cuda_stack(layers, hkv, hq, 4096)
    kv_va, seq = admit_with_lengths(st, lens, seed=5)
    for i, n in enumerate(lens):
        st.sched.extend(f"req{i}", n + 1)
    st.dev.wait()
    gen = torch.Generator(device="cuda").manual_seed(9)
    x = torch.randn(len(lens), hidden, generator=gen, device="cuda").to(torch.bfloat16)
    w = (torch.randn((hq + 2 * hkv) * 128, hidden, generator=gen, device="cuda") / 64).to(torch.bfloat16)
    tok_req = torch.arange(len(lens), device="cuda", dtype=torch.int32)
    q = qkv_append(x, w, tok_req, seq.clone(), kv_va, st.geo, 7)
    for i in range(len(lens)):
        st.sched.append_token(f"req{i}", 1)
    new_lens = [n + 1 for n in lens]
    ks, vs = gather(st, kv_va, new_lens, 7)
    ref = decode_attention_ref(q.cpu(), ks, vs)
    out = decode_attention(q, kv_va, torch.tensor(new_lens, dtype=torch.int32, device="cuda"), 7,
                           st.geo, max(new_lens))
    assert rel_err(out.cpu(), ref) <= TOL


@pytest.mark.gpu
@pytest.mark.parametrize("split_k", [2, 3])
def test_qkv_append_back_to_back_launches(cuda_ok, split_k):
    """Eight PDL-chained launches on rotating weights (the layer stack's
    order): every launch's q matches torch — the split-3 helper flags reset
    inside each launch, and no launch reads another's partials."""
    layers, hkv, hq, hidden = 32, 8, 32, 4096
    lens = list(range(3, 3 + 64 * 17, 17))
    st = cuda_stack(layers, hkv, hq, 4096)
    kv_va, seq = admit_with_lengths(st, lens, seed=12)
    for i, n in enumerate(lens):
        st.sched.extend(f"req{i}", n + 1)
    st.dev.wait()
    tok_req = torch.arange(len(lens), device="cuda", dtype=torch.int32)
    tok_pos = seq.clone()
    gen = torch.Generator(device="cuda").manual_seed(5)
    feats = (hq + 2 * hkv) * 128
    ws = [(torch.randn(feats, hidden, generator=gen, device="cuda") / hidden ** 0.5).to(torch.bfloat16)
          for _ in range(3)]
    packed = [pack_qkv_weight(w) for w in ws]
    xs = [torch.randn(len(lens), hidden, generator=gen, device="cuda").to(torch.bfloat16) for _ in range(8)]
    outs = [qkv_append(xs[i], packed[i % 3], tok_req, tok_pos, kv_va, st.geo, i % layers, split_k=split_k)
            for i in range(8)]
    torch.cuda.synchronize()
    for i, q in enumerate(outs):
        ref = (xs[i].float() @ ws[i % 3].float().T).view(-1, hq + 2 * hkv, 128)[:, :hq]
        assert rel_err(q.float().cpu(), ref.cpu()) <= TOL, f"launch {i}"


@pytest.mark.gpu
def test_qkv_split3_two_streams_concurrently(cuda_ok):
    """Split 3 keeps its helper partials in a per-stream workspace: launches on
    two streams at once (different weights, same shape) both match torch."""
    layers, hkv, hq, hidden = 32, 8, 32, 4096
    lens = list(range(5, 5 + 48 * 11, 11))
    st = cuda_stack(layers, hkv, hq, 4096)
    kv_va, seq = admit_with_lengths(st, lens, seed=13)
    for i, n in enumerate(lens):
        st.sched.extend(f"req{i}", n + 1)
    st.dev.wait()
    tok_req = torch.arange(len(lens), device="cuda", dtype=torch.int32)
    gen = torch.Generator(device="cuda").manual_seed(6)
    feats = (hq + 2 * hkv) * 128
    ws = [(torch.randn(feats, hidden, generator=gen, device="cuda") / hidden ** 0.5).to(torch.bfloat16)
          for _ in range(2)]
    packed = [pack_qkv_weight(w) for w in ws]
    xs = [torch.randn(len(lens), hidden, generator=gen, device="cuda").to(torch.bfloat16) for _ in range(2)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    torch.cuda.synchronize()
    outs = [[], []]
    for rep in range(6):
        for j in range(2):
            with torch.cuda.stream(streams[j]):
                outs[j].append(qkv_append(xs[j], packed[j], tok_req, seq, kv_va, st.geo, 2 * rep + j,
                                          split_k=3, stream=streams[j]))
    torch.cuda.synchronize()
    for j in range(2):
        ref = (xs[j].float() @ ws[j].float().T).view(-1, hq + 2 * hkv, 128)[:, :hq]
        for q in outs[j]:
            assert rel_err(q.float().cpu(), ref.cpu()) <= TOL
