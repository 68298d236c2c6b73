"""Rows a25/a26 on the B200: a serving loop in the reference engine's step
order — admit (prefix match first), decode extends via ensure_capacity,
GpuCompute (KV append + tcgen05 decode over the batch), token progress,
finish (record or release, fenced), shutdown — with attention checked against
the CPU oracle and the driver having executed exactly the logged VMM calls."""

import pytest
import torch

import paper_2407_15309_b200 as vt
from oracle.attention_ref import decode_attention_ref, rel_err
from paper_2407_15309_b200.adapter import GpuCompute, VTensorAdapter
from paper_2407_15309_b200.kv_layout import chunk_view, read_kv

MIB = 1 << 20


@pytest.mark.gpu
def test_serving_loop_with_real_kernels(cuda_ok):
    L, hkv, hq = 4, 8, 32
    cfg = vt.SimConfig(capacity_bytes=512 * 2 * MIB, chunk_size_bytes=2 * MIB, weights_bytes=0,
                       geometry=vt.ModelGeometry(L, hkv, 128, 2), max_seq_len=2048,
                       initial_alloc_tokens=64, lookahead_chunks=1, max_batch=4)
    tpc = cfg.tokens_per_chunk  # 128 tokens per 2 MiB chunk at 4 layers
    dev = vt.VirtualMemoryDevice(vt.DeviceConfig(cfg.capacity_bytes, cfg.chunk_size_bytes),
                                 cuda_ordinal=0)
    ad = VTensorAdapter(dev, cfg)
    comp = GpuCompute(ad, hq, max_batch=4)
    gen = torch.Generator(device="cuda").manual_seed(11)
    stream = torch.cuda.current_stream()

    def fill_own(rid, first_token):
        space = ad.scheduler.mem[rid].vt.space
        va = dev.va(space.rng)
        c0 = first_token // tpc
        v = chunk_view(va, space.mapped_pages, comp.geo)[c0:]
        v.copy_(torch.randn(v.shape, generator=gen, device="cuda").to(torch.bfloat16))

    # conversation turn 1, recorded into the rTree
    conv = [i % 97 for i in range(300)]
    assert ad.can_admit(len(conv))
    ad.admit("c1", conv, try_prefix=False)
    ad.prefill_reserve("c1", len(conv))
    dev.wait()
    fill_own("c1", 0)
    ad.mark_prefilled("c1", len(conv))
    assert ad.finish("c1", record=True)
    # turn 2 shares the recorded prefix by identity; two unrelated requests
    stats = ad.admit("c2", conv + [5] * 40, try_prefix=True)
    assert stats.shared_tokens == 256 and stats.identity_ok
    ad.admit("a", [1] * 200, try_prefix=False)
    ad.admit("b", [2] * 333, try_prefix=False)
    dev.wait()
    fill_own("c2", 256)
    fill_own("a", 0)
    fill_own("b", 0)
    for r, n in (("c2", 340), ("a", 200), ("b", 333)):
        ad.mark_prefilled(r, n)

    batch = ["c2", "a", "b"]
    for step in range(160):  # crosses chunk boundaries: real extends on the worker
        for r in batch:
            ad.ensure_capacity(r, ad.scheduler.mem[r].vt.token_count + 1)
        q = torch.randn(L, len(batch), hq, 128, generator=gen, device="cuda").to(torch.bfloat16)
        k_new = torch.randn(L, len(batch), hkv, 128, generator=gen, device="cuda").to(torch.bfloat16)
        v_new = torch.randn_like(k_new)
        out = comp.step(batch, q, k_new, v_new, stream=stream)
        if step in (0, 77, 159):
            torch.cuda.synchronize()
            for layer in (0, L - 1):
                ks, vs = [], []
                for r in batch:
                    n = ad.scheduler.mem[r].vt.token_count + 1
                    k, v = read_kv(dev.va(ad.scheduler.mem[r].vt.space.rng), n, layer, comp.geo)
                    ks.append(k.cpu())
                    vs.append(v.cpu())
                ref = decode_attention_ref(q[layer].cpu(), ks, vs)
                assert rel_err(out[layer].cpu(), ref) <= 2e-2, (step, layer)
        for r in batch:
            ad.append_token(r, 9)
    # finish: record one, release the others (fenced unmaps), then shut down
    assert ad.finish("c2", record=True)
    ad.finish("a", record=False)
    ad.release("b")
    torch.cuda.synchronize()
    report = ad.shutdown()
    dev.wait()
    assert report["chunks_destroyed"] > 0
    log = list(dev.call_log)
    d = dev.driver_stats()
    assert d["map_calls"] == sum(c.op == "map_page" for c in log)
    assert d["unmap_calls"] == sum(c.op == "unmap_page" for c in log)
    assert d["create_calls"] == sum(c.op == "create_chunk" for c in log)
    assert d["destroy_calls"] == sum(c.op == "destroy_chunk" for c in log)
    assert dev.created_bytes == ad.pool.n_pinned * cfg.chunk_size_bytes  # only records remain
    dev.close()


@pytest.mark.gpu
def test_projection_prefill_then_decode_through_the_adapter(cuda_ok):
    """Every kernel of the path in one serving flow through the adapter:
    turn 1 prefills 300 tokens (fused QKV projection writes K/V into the
    cache, then prefill attention), is recorded into the rTree; turn 2 shares
    256 tokens by identity and prefills only its 84 new tokens over them; then
    decode steps whose new-token K/V also come from the projection. K/V in the
    cache and every attention output are checked against the oracle."""
    from oracle.attention_ref import prefill_attention_ref
    from paper_2407_15309_b200.attention import pack_qkv_weight

    L, hkv, hq, hidden = 4, 8, 32, 512
    cfg = vt.SimConfig(capacity_bytes=512 * 2 * MIB, chunk_size_bytes=2 * MIB, weights_bytes=0,
                       geometry=vt.ModelGeometry(L, hkv, 128, 2), max_seq_len=2048,
                       initial_alloc_tokens=64, lookahead_chunks=1, max_batch=4)
    dev = vt.VirtualMemoryDevice(vt.DeviceConfig(cfg.capacity_bytes, cfg.chunk_size_bytes),
                                 cuda_ordinal=0)
    ad = VTensorAdapter(dev, cfg)
    comp = GpuCompute(ad, hq, max_batch=4)
    gen = torch.Generator(device="cuda").manual_seed(5)
    feats = (hq + 2 * hkv) * 128
    W = [(torch.randn(feats, hidden, generator=gen, device="cuda") / hidden ** 0.5)
         .to(torch.bfloat16) for _ in range(L)]
    Wp = [pack_qkv_weight(w) for w in W]

    def proj(x, layer):  # fp32 reference of the projection, bf16-rounded like the kernel's output
        return (x.float() @ W[layer].float().T).to(torch.bfloat16).view(x.shape[0], hq + 2 * hkv, 128)

    def kv(rid, n, layer):
        k, v = read_kv(dev.va(ad.scheduler.mem[rid].vt.space.rng), n, layer, comp.geo)
        return k.cpu(), v.cpu()

    def check_prefill(rid, x, out, start):
        n_new = x.shape[1]
        for layer in (0, L - 1):
            ref = proj(x[layer], layer)
            k, v = kv(rid, start + n_new, layer)
            assert rel_err(k[:, start:].transpose(0, 1), ref[:, hq:hq + hkv].cpu()) <= 2e-2
            assert rel_err(v[:, start:].transpose(0, 1), ref[:, hq + hkv:].cpu()) <= 2e-2
            want = prefill_attention_ref(ref[:, :hq].cpu(), k, v, start)
            assert rel_err(out[layer].cpu(), want) <= 2e-2, (rid, layer)

    conv = [i % 97 for i in range(300)]
    ad.admit("c1", conv, try_prefix=False)
    ad.prefill_reserve("c1", len(conv))
    x1 = torch.randn(L, 300, hidden, generator=gen, device="cuda").to(torch.bfloat16)
    o1 = comp.prefill("c1", x1, Wp, start=0)
    torch.cuda.synchronize()
    check_prefill("c1", x1, o1, 0)
    ad.mark_prefilled("c1", len(conv))
    assert ad.finish("c1", record=True)

    stats = ad.admit("c2", conv + [5] * 40, try_prefix=True)
    assert stats.shared_tokens == 256 and stats.identity_ok
    ad.prefill_reserve("c2", 340)
    x2 = torch.randn(L, 84, hidden, generator=gen, device="cuda").to(torch.bfloat16)
    o2 = comp.prefill("c2", x2, Wp, start=256)
    torch.cuda.synchronize()
    check_prefill("c2", x2, o2, 256)
    ad.mark_prefilled("c2", 340)
    ad.admit("a", [1] * 200, try_prefix=False)
    ad.prefill_reserve("a", 200)
    xa = torch.randn(L, 200, hidden, generator=gen, device="cuda").to(torch.bfloat16)
    comp.prefill("a", xa, Wp, start=0)
    ad.mark_prefilled("a", 200)

    batch = ["c2", "a"]
    for _ in range(3):
        for r in batch:
            ad.ensure_capacity(r, ad.scheduler.mem[r].vt.token_count + 1)
        lens = [ad.scheduler.mem[r].vt.token_count for r in batch]
        xd = torch.randn(L, len(batch), hidden, generator=gen, device="cuda").to(torch.bfloat16)
        out = comp.step_from_hidden(batch, xd, Wp)
        torch.cuda.synchronize()
        for layer in (0, L - 1):
            ref = proj(xd[layer], layer)
            ks, vs = zip(*[kv(r, n + 1, layer) for r, n in zip(batch, lens)])
            for b, n in enumerate(lens):  # the projection's K/V landed at token_count
                assert rel_err(ks[b][:, n], ref[b, hq:hq + hkv].cpu()) <= 2e-2
            want = decode_attention_ref(ref[:, :hq].cpu(), list(ks), list(vs))
            assert rel_err(out[layer].cpu(), want) <= 2e-2, layer
        for r in batch:
            ad.append_token(r, 9)
    ad.finish("c2", record=False)
    ad.release("a")
    torch.cuda.synchronize()
    ad.shutdown()
    dev.wait()
    dev.close()
