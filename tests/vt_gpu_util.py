"""Helpers for GPU tests: a CUDA-backed manager stack with filled KV."""

from __future__ import annotations

from types import SimpleNamespace

import torch

import paper_2407_15309_b200 as vt
from paper_2407_15309_b200.kv_layout import KVGeometry, chunk_view, read_kv

MIB = 1 << 20


def cuda_stack(layers, kv_heads, q_heads, max_seq_len, capacity_chunks=4096,
               initial_alloc=0, lookahead=1):
    cfg = vt.SimConfig(
        capacity_bytes=capacity_chunks * 2 * MIB, chunk_size_bytes=2 * MIB, weights_bytes=0,
        geometry=vt.ModelGeometry(layers=layers, kv_heads=kv_heads, head_dim=128, elem_bytes=2),
        max_seq_len=max_seq_len, initial_alloc_tokens=initial_alloc, lookahead_chunks=lookahead)
    dev = vt.VirtualMemoryDevice(
        vt.DeviceConfig(capacity_bytes=cfg.capacity_bytes, chunk_size_bytes=cfg.chunk_size_bytes),
        cuda_ordinal=torch.cuda.current_device())
    pool = vt.TensorPool(cfg.tokens_per_chunk)
    ops = vt.VTensorOps(dev, pool, cfg)
    sched = vt.VTensorScheduler(ops)
    geo = KVGeometry.from_config(cfg, q_heads)
    return SimpleNamespace(cfg=cfg, dev=dev, pool=pool, ops=ops, sched=sched, geo=geo)


def admit_with_lengths(st, lens, seed=0, fill=True):
    """Create one request per length with exactly ceil(len/tpc) chunks mapped
    (no lookahead), mark the prompt prefilled, fill mapped chunks with seeded
    randn bf16 KV. Returns (kv_va int64 cuda tensor, seq_lens int32 cuda tensor)."""
    gen = torch.Generator(device="cuda").manual_seed(seed)
    vas = []
    for i, n in enumerate(lens):
        rid = f"req{i}"
        st.sched.create(rid, [7] * n)
        st.sched.mark_prefilled(rid)
        vas.append(st.dev.va(st.sched.mem[rid].vt.space.rng))
    st.dev.wait()
    if fill:
        for i, n in enumerate(lens):
            pages = st.sched.mem[f"req{i}"].vt.space.mapped_pages
            if pages:
                v = chunk_view(vas[i], pages, st.geo)
                v.copy_(torch.randn(v.shape, generator=gen, device="cuda", dtype=torch.float32)
                        .to(torch.bfloat16))
    torch.cuda.synchronize()
    return (torch.tensor(vas, dtype=torch.int64, device="cuda"),
            torch.tensor(lens, dtype=torch.int32, device="cuda"))


def gather(st, kv_va, lens, layer):
    ks, vs = [], []
    for va, n in zip(kv_va.tolist(), lens):
        k, v = read_kv(va, n, layer, st.geo)
        ks.append(k.cpu())
        vs.append(v.cpu())
    return ks, vs
