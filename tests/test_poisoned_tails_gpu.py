"""Stale-tail masking (VERDICT r01 "weak" item 2): bytes past a request's
``seq_len`` must never reach an accumulator.

A vTensor space maps whole 2 MiB chunks, so the last mapped chunk holds
``mapped*tpc - len`` rows that belong to no token yet, and chunks mapped ahead
(extend lookahead, scheduler.py:166-180) hold whatever the physical memory held
before (a recycled pSet chunk, ops.py:83-112, keeps its previous owner's KV).
The kernels read those rows (TMA boxes are whole chunks; the CUDA-core path
reads 16 B vectors of whole head blocks) and must mask them. Here every such
row is NaN / +-Inf / huge, and one chunk past the tail is either poisoned or
left exactly as the driver handed it out. The outputs must be finite and match
the oracle over the first ``len`` tokens (2e-2 relative, north_star).
"""

import pytest
import torch

from oracle.attention_ref import decode_attention_ref, prefill_attention_ref, rel_err
from paper_2407_15309_b200.attention import decode_attention, kv_tensor_maps, prefill_attention
from paper_2407_15309_b200.kv_layout import chunk_view, read_kv
from vt_gpu_util import admit_with_lengths, cuda_stack, gather

TOL = 2e-2

POISONS = {
    "nan": float("nan"),
    "inf": float("inf"),
    "neg_inf": float("-inf"),
    "huge": 3.0e38,  # finite in bf16 (max ~3.39e38): exp overflow if unmasked
}


def _poison_tail(st, va, n_tokens, mapped_pages, value):
    """Write `value` into every row >= n_tokens of the mapped chunks of one
    space (all layers, K and V, all kv heads)."""
    tpc = st.cfg.tokens_per_chunk
    if mapped_pages == 0:
        return
    v = chunk_view(va, mapped_pages, st.geo)  # [c, L, 2, H, tpc, d]
    full, rem = divmod(n_tokens, tpc)
    if rem:
        v[full, :, :, :, rem:, :].fill_(value)
        full += 1
    if full < mapped_pages:
        v[full:].fill_(value)


def _lookahead(st, lens, extra_chunks):
    """Map `extra_chunks` more chunks past each request's last token."""
    tpc = st.cfg.tokens_per_chunk
    for i, n in enumerate(lens):
        space = st.sched.mem[f"req{i}"].vt.space
        target = min(st.cfg.max_seq_len, (space.mapped_pages + extra_chunks) * tpc)
        st.sched.extend(f"req{i}", target)
    st.dev.wait()
    return [st.sched.mem[f"req{i}"].vt.space.mapped_pages for i in range(len(lens))]


CASES = {
    # name: (layers, kv_heads, q_heads, max_seq, lens)
    "llama8b_gqa4": (32, 8, 32, 4352, [1, 15, 17, 100, 1000, 4095, 4081]),
    "toy_mha_tpc512": (1, 8, 8, 4096, [1, 65, 513, 700, 3001]),
    "gqa8_tpc128": (16, 2, 16, 4096, [5, 129, 2049]),
}


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("poison", list(POISONS))
@pytest.mark.parametrize("path,split", [("cuda_core", 0), ("cuda_core", 64), ("tcgen05", 0),
                                        ("tcgen05", 128)])
def test_decode_ignores_poisoned_tail(cuda_ok, name, poison, path, split):
    layers, hkv, hq, max_seq, lens = CASES[name]
    st = cuda_stack(layers, hkv, hq, max_seq)
    kv_va, seq = admit_with_lengths(st, lens, seed=11)
    mapped = _lookahead(st, lens, 1)
    for i, n in enumerate(lens):
        _poison_tail(st, int(kv_va[i]), n, mapped[i], POISONS[poison])
    torch.cuda.synchronize()
    tpc = st.cfg.tokens_per_chunk
    maps = (kv_tensor_maps(kv_va.tolist(), [m * tpc for m in mapped], st.geo)
            if path == "tcgen05" else None)
    q = torch.randn(len(lens), hq, 128, device="cuda").to(torch.bfloat16)
    for layer in sorted({0, layers - 1}):
        out = decode_attention(q, kv_va, seq, layer, st.geo, max(lens), split_tokens=split,
                               kv_maps=maps)
        torch.cuda.synchronize()
        assert torch.isfinite(out.float()).all(), f"{poison} leaked into layer {layer}"
        ks, vs = gather(st, kv_va, lens, layer)
        err = rel_err(out.cpu(), decode_attention_ref(q.cpu(), ks, vs))
        assert err <= TOL, f"{name} {path} split={split} {poison}: rel err {err:.3e}"


@pytest.mark.gpu
@pytest.mark.parametrize("path", ["cuda_core", "tcgen05"])
def test_decode_ignores_unwritten_lookahead_chunks(cuda_ok, path):
    """Chunks mapped ahead and never written (whatever bytes the driver or a
    previous owner left: here a released request's NaN-filled chunks are
    recycled through the pSet free list) are read but masked."""
    layers, hkv, hq = 32, 8, 32
    st = cuda_stack(layers, hkv, hq, 4352)
    # a previous owner fills its chunks with NaN, then releases them (lazy free list)
    st.sched.create("old", [3] * 4096)
    st.dev.wait()
    chunk_view(st.dev.va(st.sched.mem["old"].vt.space.rng),
               st.sched.mem["old"].vt.space.mapped_pages, st.geo).fill_(float("nan"))
    torch.cuda.synchronize()
    st.sched.release("old")
    lens = [3, 40, 1000, 2047]
    kv_va, seq = admit_with_lengths(st, lens, seed=5, fill=False)
    gen = torch.Generator(device="cuda").manual_seed(6)
    for i, n in enumerate(lens):  # write exactly the valid rows, nothing else
        k = torch.randn(layers, 2, hkv, n, 128, generator=gen, device="cuda").to(torch.bfloat16)
        v = chunk_view(int(kv_va[i]), -(-n // 16), st.geo)
        for t0 in range(0, n, 16):
            c, m = t0 // 16, min(16, n - t0)
            v[c, :, :, :, :m] = k[:, :, :, t0:t0 + m]
    mapped = _lookahead(st, lens, 2)
    torch.cuda.synchronize()
    maps = (kv_tensor_maps(kv_va.tolist(), [m * 16 for m in mapped], st.geo)
            if path == "tcgen05" else None)
    q = torch.randn(len(lens), hq, 128, device="cuda").to(torch.bfloat16)
    out = decode_attention(q, kv_va, seq, 7, st.geo, max(lens), kv_maps=maps)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    ks, vs = gather(st, kv_va, lens, 7)
    assert rel_err(out.cpu(), decode_attention_ref(q.cpu(), ks, vs)) <= TOL


PF_CASES = {
    # name: (layers, kv_heads, q_heads, prefix, n_new, max_seq)
    "llama8b_ragged_100+200": (32, 8, 32, 100, 200, 1024),
    "llama8b_2048+509": (32, 8, 32, 2048, 509, 4096),
    "toy_mha_tpc512_300+77": (1, 8, 8, 300, 77, 4096),
}


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(PF_CASES))
@pytest.mark.parametrize("poison", ["nan", "inf", "huge"])
def test_prefill_ignores_poisoned_tail(cuda_ok, name, poison):
    layers, hkv, hq, prefix, n_new, max_seq = PF_CASES[name]
    st = cuda_stack(layers, hkv, hq, max_seq, capacity_chunks=2048)
    n = prefix + n_new
    lens = [n, n - 3]
    kv_va, _ = admit_with_lengths(st, lens, seed=21)
    mapped = _lookahead(st, lens, 1)
    for i, m in enumerate(lens):
        _poison_tail(st, int(kv_va[i]), m, mapped[i], POISONS[poison])
    torch.cuda.synchronize()
    tpc = st.cfg.tokens_per_chunk
    starts = [m - n_new for m in lens]
    maps = kv_tensor_maps(kv_va.tolist(), [m * tpc for m in mapped], st.geo)
    gen = torch.Generator(device="cuda").manual_seed(22)
    q = torch.randn(len(lens), n_new, hq, 128, generator=gen, device="cuda").to(torch.bfloat16)
    start_t = torch.tensor(starts, dtype=torch.int32, device="cuda")
    layer = layers - 1
    out = prefill_attention(q, maps, start_t, layer, st.geo)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all(), f"{poison} leaked into the prefill"
    for b, m in enumerate(lens):
        k, v = read_kv(int(kv_va[b]), m, layer, st.geo)
        ref = prefill_attention_ref(q[b].cpu(), k.cpu(), v.cpu(), starts[b])
        err = rel_err(out[b].cpu(), ref)
        assert err <= TOL, f"{name} {poison} request {b}: rel err {err:.3e}"
