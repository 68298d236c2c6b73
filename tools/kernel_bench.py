"""Kernel-level timing of the two hot kernels on their BASELINE configs, and the
ncu target (use --iters 1 --warmup 1 under ncu).

  decode  : config 2 — Llama-3-8B decode, B=64, ctx 4096 (one layer launch)
  prefill : config 3 — 16 requests x (2048 rTree-shared prefix + 512 new),
            32 q / 8 kv heads (one layer launch), tcgen05 path

Prints one JSON line per kernel: duration (CUDA events, median of iters),
algorithmic bytes or FLOPs, achieved GB/s or TFLOP/s and fraction of the
measured peak (MEASURED_PEAKS.json).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

import paper_2407_15309_b200 as vt  # noqa: E402
from paper_2407_15309_b200.attention import (DecodeWorkspace, decode_attention,  # noqa: E402
                                             prefill_attention, kv_tensor_maps)
from paper_2407_15309_b200.kv_layout import KVGeometry, chunk_view  # noqa: E402

MIB = 1 << 20


def peaks():
    try:
        return json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def stack(layers, hkv, hq, max_seq, chunks):
    cfg = vt.SimConfig(capacity_bytes=chunks * 2 * MIB, chunk_size_bytes=2 * MIB, weights_bytes=0,
                       geometry=vt.ModelGeometry(layers, hkv, 128, 2), max_seq_len=max_seq,
                       initial_alloc_tokens=0)
    dev = vt.VirtualMemoryDevice(vt.DeviceConfig(cfg.capacity_bytes, cfg.chunk_size_bytes),
                                 cuda_ordinal=0)
    ops = vt.VTensorOps(dev, vt.TensorPool(cfg.tokens_per_chunk), cfg)
    return cfg, dev, ops, vt.VTensorScheduler(ops), KVGeometry.from_config(cfg, hq)


def fill(va, pages, geo, gen, first=0):
    if pages - first <= 0:
        return
    v = chunk_view(va, pages, geo)[first:]
    v.copy_(torch.randn(v.shape, generator=gen, device="cuda").to(torch.bfloat16))


def timed(fn, iters, warmup):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), ts


def timed_graph(fn, reps=20, iters=10):
    """Device time per call of `fn`, launched from a CUDA graph of `reps` calls
    (no host enqueue latency in the measurement)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / reps)
    return statistics.median(ts), ts


def bench_decode(args, pk):
    # 8b: Llama-3-8B (G=4, tpc 16); 70b: one 16-layer group of Llama-2-70B (G=8, tpc 32)
    L, hkv, hq, B, ctx = {"8b": (32, 8, 32, 64, 4096), "70b": (16, 8, 64, 64, 4096),
                          "toy": (1, 8, 8, 8, 4096), "mha64": (4, 8, 8, 64, 4096)}[args.shape]
    cfg, dev, ops, sched, geo = stack(L, hkv, hq, ctx + 256, 20000)
    gen = torch.Generator(device="cuda").manual_seed(0)
    vas = []
    for b in range(B):
        sched.create(f"r{b}", [1] * ctx)
        vas.append(dev.va(sched.mem[f"r{b}"].vt.space.rng))
    dev.wait()
    for b in range(B):
        fill(vas[b], sched.mem[f"r{b}"].vt.space.mapped_pages, geo, gen)
    kv_va = torch.tensor(vas, dtype=torch.int64, device="cuda")
    seq = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
    q = torch.randn(B, hq, 128, generator=gen, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    tpc = cfg.tokens_per_chunk
    maps = kv_tensor_maps(vas, [sched.mem[f"r{b}"].vt.space.mapped_pages * tpc for b in range(B)],
                          geo)
    res = []
    for path in args.paths:
        for split in args.splits:
            ws = DecodeWorkspace(geo, B, ctx, split)
            layer = [0]
            km = maps if path == "tcgen05" else None

            def fn(chained=False):
                decode_attention(q, kv_va, seq, layer[0] % L, geo, ctx, out=out, workspace=ws,
                                 split_tokens=split, kv_maps=km, chained=chained)
                layer[0] += 1  # rotate layers: 1 GiB per launch, never L2-resident

            if args.loop:  # 32 back-to-back layer launches, like one decode step
                def fn32():
                    for i in range(L):
                        fn(chained=args.chained and path == "tcgen05" and i > 0)
                ms, _ = timed(fn32, max(2, args.iters // 4), args.warmup)
                ms /= L
            else:
                ms, _ = timed(fn, args.iters, args.warmup)
            nbytes = 2 * B * ctx * hkv * 128 * 2 + 2 * B * hq * 128 * 2
            gbs = nbytes / (ms * 1e-3) / 1e9
            res.append({"kernel": f"decode[{path}]" + ("x32" if args.loop else "")
                        + ("_pdl" if args.loop and args.chained else ""),
                        "config": f"{args.shape} B64 ctx4096 G={hq // hkv}",
                        "split": split, "us": round(ms * 1e3, 2), "bytes": nbytes,
                        "GB/s": round(gbs, 1), "frac_of_hbm": round(gbs / pk["hbm_gbs"], 4)})
    dev.wait()
    return res


def bench_prefill(args, pk):
    L, hkv, hq, B, prefix, n_new = 32, 8, 32, args.pf_batch, args.pf_prefix, args.pf_new
    max_seq = max(4096, -(-(prefix + n_new) // 4096) * 4096)
    cfg, dev, ops, sched, geo = stack(L, hkv, hq, max_seq, max(4096, B * max_seq // 16 + max_seq // 16))
    gen = torch.Generator(device="cuda").manual_seed(1)
    tpc = cfg.tokens_per_chunk
    base = [i % 251 for i in range(prefix)]
    if prefix:
        sched.create("donor", base)
        sched.mark_prefilled("donor")
        dev.wait()
        fill(dev.va(sched.mem["donor"].vt.space.rng), sched.mem["donor"].vt.space.mapped_pages, geo, gen)
        assert sched.prefix_record("donor")
    vas = []
    for b in range(B):
        toks = base + [7000 + b * 600 + k for k in range(n_new)]
        if prefix:
            hit = sched.prefix_match(f"t{b}", toks)
            assert hit is not None and hit[1].shared_tokens == prefix
        else:
            sched.create(f"t{b}", toks)
        vas.append(dev.va(sched.mem[f"t{b}"].vt.space.rng))
    dev.wait()
    for b in range(B):
        fill(vas[b], sched.mem[f"t{b}"].vt.space.mapped_pages, geo, gen, first=prefix // tpc)
    maps = kv_tensor_maps(vas, [prefix + n_new] * B, geo)
    start = torch.full((B,), prefix, dtype=torch.int32, device="cuda")
    q = torch.randn(B, n_new, hq, 128, generator=gen, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    layer = [0]

    def fn():
        prefill_attention(q, maps, start, layer[0] % L, geo, out=out)
        layer[0] += 1

    ms, _ = timed(fn, args.iters, args.warmup)
    flops = 4 * hq * 128 * (n_new * prefix + n_new * (n_new + 1) // 2) * B
    tf = flops / (ms * 1e-3) / 1e12
    dev.wait()
    return [{"kernel": "prefill", "config": f"{B} x ({prefix} shared + {n_new} new)", "us": round(ms * 1e3, 2),
             "flops": flops, "TFLOP/s": round(tf, 1),
             "frac_of_bf16_burst": round(tf / pk["bf16_tflops"], 4),
             "frac_of_bf16_sustained": round(tf / pk["bf16_tflops_sustained"], 4)}]


def bench_qkv(args, pk):
    """Fused QKV projection + KV append, Llama-3-8B decode step shape (one
    layer): x [B, 4096] @ W_qkv[6144, 4096]^T, K/V written into the cache.
    Baseline in the same run: cuBLAS GEMM (torch) + vt_kv_append (unfused).
    Both timed as device time from a CUDA graph of 20 calls (4 weights of
    50 MB rotate, so W is never L2-resident)."""
    from paper_2407_15309_b200.attention import kv_append, pack_qkv_weight, qkv_append
    L, hkv, hq, hidden = 32, 8, 32, 4096
    res = []
    for B in args.qkv_batch:
        cfg, dev, ops, sched, geo = stack(L, hkv, hq, 4096, 4096)
        vas = []
        for b in range(B):
            sched.create(f"r{b}", [1] * 100)
            sched.mark_prefilled(f"r{b}")
            sched.extend(f"r{b}", 101)
            vas.append(dev.va(sched.mem[f"r{b}"].vt.space.rng))
        dev.wait()
        kv_va = torch.tensor(vas, dtype=torch.int64, device="cuda")
        tok_req = torch.arange(B, dtype=torch.int32, device="cuda")
        tok_pos = torch.full((B,), 100, dtype=torch.int32, device="cuda")
        feats = (hq + 2 * hkv) * 128
        ws = [(torch.randn(feats, hidden, device="cuda") / 64).to(torch.bfloat16) for _ in range(4)]
        packed = [pack_qkv_weight(w) for w in ws]
        x = torch.randn(B, hidden, device="cuda").to(torch.bfloat16)
        q = torch.empty(B, hq, 128, dtype=torch.bfloat16, device="cuda")
        nbytes = feats * hidden * 2 + B * hidden * 2 + B * feats * 2
        lay = [0]
        for split in args.qkv_split:
            def fn():
                qkv_append(x, packed[lay[0] % 4], tok_req, tok_pos, kv_va, geo, lay[0] % L, q_out=q,
                           split_k=split)
                lay[0] += 1  # 4 weights x 50 MB rotate: never L2-resident
            ms, _ = timed_graph(fn)
            gbs = nbytes / (ms * 1e-3) / 1e9
            res.append({"kernel": "qkv_append (fused)", "config": f"llama3-8b B{B}", "split_k": split,
                        "us": round(ms * 1e3, 2), "bytes": nbytes, "GB/s": round(gbs, 1),
                        "frac_of_hbm": round(gbs / pk["hbm_gbs"], 4)})

        def unfused():
            y = x @ ws[lay[0] % 4].T
            k = y[:, hq * 128:(hq + hkv) * 128].reshape(1, B, hkv, 128)
            v = y[:, (hq + hkv) * 128:].reshape(1, B, hkv, 128)
            kv_append(k.contiguous(), v.contiguous(), kv_va, tok_pos, geo, layer_begin=lay[0] % L)
            lay[0] += 1
        ms, _ = timed_graph(unfused)
        gbs = nbytes / (ms * 1e-3) / 1e9
        res.append({"kernel": "cuBLAS GEMM + vt_kv_append (unfused)", "config": f"llama3-8b B{B}",
                    "us": round(ms * 1e3, 2), "GB/s": round(gbs, 1),
                    "frac_of_hbm": round(gbs / pk["hbm_gbs"], 4)})
        dev.wait()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="decode,prefill")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--splits", type=lambda s: [int(x) for x in s.split(",")], default=[1024])
    ap.add_argument("--paths", type=lambda s: s.split(","), default=["tcgen05", "cuda_core"])
    ap.add_argument("--loop", action="store_true", help="time 32 back-to-back launches")
    ap.add_argument("--chained", action="store_true",
                    help="with --loop: layers after the first use programmatic dependent launch")
    ap.add_argument("--shape", choices=["8b", "70b", "toy", "mha64"], default="8b")
    ap.add_argument("--qkv-batch", type=lambda s: [int(x) for x in s.split(",")], default=[64])
    ap.add_argument("--qkv-split", type=lambda s: [int(x) for x in s.split(",")], default=[0])
    ap.add_argument("--pf-batch", type=int, default=16, help="prefill: requests (config 3: 16)")
    ap.add_argument("--pf-prefix", type=int, default=2048, help="prefill: shared prefix tokens")
    ap.add_argument("--pf-new", type=int, default=512, help="prefill: new tokens per request")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    pk = peaks()
    out = []
    if "decode" in args.which:
        out += bench_decode(args, pk)
    if "prefill" in args.which:
        out += bench_prefill(args, pk)
    if "qkv" in args.which:
        out += bench_qkv(args, pk)
    for r in out:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
