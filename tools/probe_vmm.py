"""Probe: cost of the CUDA VMM calls on B200 and whether they serialise with
running kernels (SURVEY.md §7.3.3 "unknown; probe it early").

Prints one JSON object. Run on the GPU box:  python tools/probe_vmm.py
"""

from __future__ import annotations

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2407_15309_b200 as vt  # noqa: E402

MIB = 1 << 20


def stack(pages=512):
    cfg = vt.SimConfig(capacity_bytes=8192 * 2 * MIB, chunk_size_bytes=2 * MIB, weights_bytes=0,
                       geometry=vt.ModelGeometry(32, 8, 128, 2), max_seq_len=16 * pages,
                       initial_alloc_tokens=0)
    dev = vt.VirtualMemoryDevice(vt.DeviceConfig(cfg.capacity_bytes, cfg.chunk_size_bytes),
                                 cuda_ordinal=0)
    ops = vt.VTensorOps(dev, vt.TensorPool(cfg.tokens_per_chunk), cfg)
    return cfg, dev, ops, vt.VTensorScheduler(ops)


def drv_delta(a, b):
    return {k: b[k] - a[k] for k in a}


def per_call(d):
    out = {}
    for op in ("map", "unmap", "create", "destroy"):
        n = d[f"{op}_calls"]
        out[f"{op}_us"] = round(d[f"{op}_ns_total"] / n / 1e3, 2) if n else None
    out["access_us_per_call"] = (round(d["access_ns_total"] / d["access_calls"] / 1e3, 2)
                                 if d["access_calls"] else None)
    out["access_calls"] = d["access_calls"]
    out["map_calls"] = d["map_calls"]
    return out


def main():
    torch.cuda.init()
    res = {}
    cfg, dev, ops, sched = stack()
    # 1) idle GPU, one page per extend (decode pattern), sync execution
    dev.set_async(False)
    s0 = dev.driver_stats()
    sched.create("a", [1] * 16)
    t0 = time.perf_counter()
    for n in range(2, 66):
        sched.extend("a", 16 * n)
    t1 = time.perf_counter()
    res["idle_1page_extend_us"] = round((t1 - t0) / 64 * 1e6, 2)
    res["idle_1page_driver"] = per_call(drv_delta(s0, dev.driver_stats()))
    # 2) idle GPU, 16 pages per extend: one cuMemSetAccess per run
    s0 = dev.driver_stats()
    sched.create("b", [1] * 16)
    t0 = time.perf_counter()
    for n in range(1, 9):
        sched.extend("b", 16 * (1 + 16 * n))
    t1 = time.perf_counter()
    res["idle_16page_extend_us_per_page"] = round((t1 - t0) / 128 * 1e6, 2)
    res["idle_16page_driver"] = per_call(drv_delta(s0, dev.driver_stats()))
    # 3) reuse path: release -> free list -> remap (no cuMemCreate)
    sched.release("b")
    dev.fence(torch.cuda.current_stream().cuda_stream)
    s0 = dev.driver_stats()
    sched.create("c", [1] * 16)
    t0 = time.perf_counter()
    for n in range(2, 66):
        sched.extend("c", 16 * n)
    t1 = time.perf_counter()
    res["idle_reuse_extend_us"] = round((t1 - t0) / 64 * 1e6, 2)
    res["idle_reuse_driver"] = per_call(drv_delta(s0, dev.driver_stats()))

    # 4) concurrency: GPU busy with a ~200 ms spin kernel, async maps meanwhile
    dev.set_async(True)
    st = torch.cuda.current_stream()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    torch.cuda._sleep(400_000_000)  # ~200 ms at 1.9 GHz
    ev1.record()
    t_launch = time.perf_counter()
    sched.create("d", [1] * 16)
    for n in range(2, 34):
        sched.extend("d", 16 * n)
    tk = dev.ticket()
    while not dev.ready(tk):
        time.sleep(1e-4)
    t_maps = time.perf_counter()
    gpu_done_early = ev1.query()
    torch.cuda.synchronize()
    t_gpu = time.perf_counter()
    res["busy_maps_done_after_ms"] = round((t_maps - t_launch) * 1e3, 2)
    res["busy_gpu_done_after_ms"] = round((t_gpu - t_launch) * 1e3, 2)
    res["busy_maps_finished_before_kernel"] = not gpu_done_early
    res["busy_kernel_ms"] = round(ev0.elapsed_time(ev1), 2)
    # 5) does a map issued during kernel A delay kernel B? (stream gap)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record()
    torch.cuda._sleep(100_000_000)
    e[1].record()
    for n in range(34, 42):
        sched.extend("d", 16 * n)
    e[2].record()
    torch.cuda._sleep(100_000_000)
    e[3].record()
    torch.cuda.synchronize()
    res["gap_between_kernels_with_concurrent_map_ms"] = round(e[1].elapsed_time(e[2]), 3)
    res["kernel_a_ms"] = round(e[0].elapsed_time(e[1]), 2)
    res["kernel_b_ms"] = round(e[2].elapsed_time(e[3]), 2)
    # 6) same, no maps, baseline gap
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record()
    torch.cuda._sleep(100_000_000)
    e[1].record()
    e[2].record()
    torch.cuda._sleep(100_000_000)
    e[3].record()
    torch.cuda.synchronize()
    res["gap_between_kernels_no_map_ms"] = round(e[1].elapsed_time(e[2]), 3)
    res["busy_driver_total"] = per_call(dev.driver_stats())
    print(json.dumps(res, indent=1))
    dev.wait()


if __name__ == "__main__":
    main()
