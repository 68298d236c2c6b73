"""Prefix-prefill attention (tcgen05/TMEM/TMA) on the B200 vs the CPU oracle (row a28).

The config-3 path end to end: a finished conversation is recorded in the rTree
(prefix_record), the next turn's request prefix-matches it, so its space maps
the donor's chunks by identity (hard links) plus fresh chunks for the new
tokens; the kernel then reads the shared prefix *through the new request's own
VA*. Tolerance 2e-2 relative (bf16 in, fp32 accumulate).
"""

import pytest
import torch

from oracle.attention_ref import prefill_attention_ref, rel_err
from paper_2407_15309_b200.attention import kv_tensor_maps, prefill_attention
from paper_2407_15309_b200.kv_layout import chunk_view, read_kv
from vt_gpu_util import cuda_stack

TOL = 2e-2


def _fill(st, va, first_chunk, n_chunks, gen):
    if n_chunks <= 0:
        return
    v = chunk_view(va, first_chunk + n_chunks, st.geo)[first_chunk:]
    v.copy_(torch.randn(v.shape, generator=gen, device="cuda").to(torch.bfloat16))


def _turn(st, prefix, n_new, batch, gen, tokens_seed=5):
    """Record a `prefix`-token conversation, then admit `batch` follow-ups that
    share it. Returns (vas, starts)."""
    tpc = st.cfg.tokens_per_chunk
    base = [(i * 7 + tokens_seed) % 97 for i in range(prefix)]
    vas, starts = [], []
    if prefix:
        st.sched.create("donor", base)
        st.sched.mark_prefilled("donor")
        st.dev.wait()
        dva = st.dev.va(st.sched.mem["donor"].vt.space.rng)
        _fill(st, dva, 0, st.sched.mem["donor"].vt.space.mapped_pages, gen)
        assert st.sched.prefix_record("donor")
    for i in range(batch):
        rid = f"turn{i}"
        toks = base + [1000 + i * n_new + k for k in range(n_new)]
        hit = st.sched.prefix_match(rid, toks) if prefix else None
        if hit is None:
            st.sched.create(rid, toks)
            shared = 0
        else:
            _, stats = hit
            assert stats.identity_ok and stats.shared_tokens == prefix - prefix % tpc
            shared = stats.shared_tokens
        st.dev.wait()
        va = st.dev.va(st.sched.mem[rid].vt.space.rng)
        pages = st.sched.mem[rid].vt.space.mapped_pages
        _fill(st, va, shared // tpc, pages - shared // tpc, gen)  # the request's own chunks
        st.sched.mark_prefilled(rid)
        vas.append(va)
        starts.append(shared)
    torch.cuda.synchronize()
    return vas, starts


CASES = {
    # name: (layers, kv_heads, q_heads, prefix, n_new, batch, max_seq)
    "cfg3_llama8b_2048+512": (32, 8, 32, 2048, 512, 2, 4096),
    "no_prefix_plain_prefill": (32, 8, 32, 0, 384, 2, 1024),
    "ragged_prefix_100_new_200": (32, 8, 32, 100, 200, 2, 1024),
    "toy_mha_tpc512": (1, 8, 8, 1024, 300, 2, 4096),
    "gqa8_tpc128": (16, 2, 16, 640, 130, 1, 2048),
    # more work items than SMs: every persistent CTA walks several items, so
    # barrier phases and the K/V ring carry across items
    "persistent_multi_item_gqa4": (32, 8, 32, 300, 700, 12, 2048),
    "persistent_multi_item_mha": (1, 8, 8, 512, 1100, 8, 4096),
}


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_prefix_prefill_matches_oracle(cuda_ok, name):
    layers, hkv, hq, prefix, n_new, batch, max_seq = CASES[name]
    st = cuda_stack(layers, hkv, hq, max_seq, capacity_chunks=2048)
    gen = torch.Generator(device="cuda").manual_seed(len(name))
    vas, starts = _turn(st, prefix, n_new, batch, gen)
    # the n_new new tokens sit after the whole prefix; KV of any unshared
    # prefix tail (prefix % tpc tokens) lives in the request's own chunks
    starts = [prefix] * batch
    kv_len = [s + n_new for s in starts]
    layer = layers - 1
    q = torch.randn(batch, n_new, hq, 128, generator=gen, device="cuda").to(torch.bfloat16)
    maps = kv_tensor_maps(vas, kv_len, st.geo)
    start_t = torch.tensor(starts, dtype=torch.int32, device="cuda")
    out = prefill_attention(q, maps, start_t, layer, st.geo)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    for b in range(batch):
        k, v = read_kv(vas[b], kv_len[b], layer, st.geo)
        ref = prefill_attention_ref(q[b].cpu(), k.cpu(), v.cpu(), starts[b])
        err = rel_err(out[b].cpu(), ref)
        assert err <= TOL, f"{name} request {b}: rel err {err:.3e}"


@pytest.mark.gpu
def test_shared_prefix_is_the_same_physical_memory(cuda_ok):
    """Hard link, not copy: a write through the donor's VA is visible through
    the borrower's VA (same cuMemCreate handle mapped twice)."""
    st = cuda_stack(32, 8, 32, 4096, capacity_chunks=1024)
    gen = torch.Generator(device="cuda").manual_seed(0)
    vas, starts = _turn(st, 256, 64, 1, gen)
    donor = st.pool.tree.match(tuple((i * 7 + 5) % 97 for i in range(256)))[0]
    dva = st.dev.va(donor.space.rng)
    k_d, _ = read_kv(dva, 256, 3, st.geo)
    k_b, _ = read_kv(vas[0], 256, 3, st.geo)
    assert torch.equal(k_d, k_b)
    chunk_view(dva, 1, st.geo)[0, 3, 0].fill_(1.5)
    torch.cuda.synchronize()
    k_b2, _ = read_kv(vas[0], 16, 3, st.geo)
    assert torch.all(k_b2 == 1.5)


VARLEN_CASES = {
    # name: (layers, kv_heads, q_heads, max_seq, [(start, n_new), ...])
    "engine_step_mix_gqa4": (32, 8, 32, 4096, [(2048, 512), (0, 130), (100, 1), (2048, 37),
                                               (300, 700), (0, 128), (17, 129)]),
    "toy_mha_tpc512": (1, 8, 8, 4096, [(0, 256), (0, 3000), (512, 700), (1000, 1)]),
    "single_request": (16, 2, 16, 2048, [(640, 130)]),
}


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(VARLEN_CASES))
def test_varlen_prefill_matches_oracle(cuda_ok, name):
    """One launch prefills requests with different prefix lengths and
    different numbers of new tokens (the engine's admitted batch,
    kvsim/engine.py:422-484, 500-504), q/out packed cu_seqlens-style."""
    from paper_2407_15309_b200.attention import prefill_attention_varlen
    from vt_gpu_util import admit_with_lengths

    layers, hkv, hq, max_seq, reqs = VARLEN_CASES[name]
    st = cuda_stack(layers, hkv, hq, max_seq, capacity_chunks=4096)
    kv_len = [s + n for s, n in reqs]
    kv_va, _ = admit_with_lengths(st, kv_len, seed=len(name))
    offs = [0]
    for _, n in reqs:
        offs.append(offs[-1] + n)
    gen = torch.Generator(device="cuda").manual_seed(99)
    q = torch.randn(offs[-1], hq, 128, generator=gen, device="cuda").to(torch.bfloat16)
    maps = kv_tensor_maps(kv_va.tolist(), kv_len, st.geo)
    start = torch.tensor([s for s, _ in reqs], dtype=torch.int32, device="cuda")
    q_off = torch.tensor(offs, dtype=torch.int32, device="cuda")
    out = torch.full_like(q, float("nan"))  # every row must be written
    layer = layers - 1
    prefill_attention_varlen(q, maps, start, q_off, max(n for _, n in reqs), layer, st.geo, out=out)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    for b, (s, n) in enumerate(reqs):
        k, v = read_kv(int(kv_va[b]), s + n, layer, st.geo)
        ref = prefill_attention_ref(q[offs[b]:offs[b + 1]].cpu(), k.cpu(), v.cpu(), s)
        err = rel_err(out[offs[b]:offs[b + 1]].cpu(), ref)
        assert err <= TOL, f"{name} request {b} (start {s}, n {n}): rel err {err:.3e}"
