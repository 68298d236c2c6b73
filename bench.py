#!/usr/bin/env python
"""bench.py — vTensor decode step on B200 (BASELINE.json config 2 by default).

One *step* = one decode step of a Llama-3-8B-shaped batch (32 q / 8 kv heads,
d 128, bf16, 32 layers, batch 64 per GPU, ~4k context) through the product path:

  host : vTensor extend ahead of every request's next tokens (VTS.extend ->
         VTO.p_alloc/map_chunks -> libvtensor; cuMemCreate/cuMemMap/
         cuMemSetAccess run on the shim's worker thread, overlapping the GPU
         work already queued), wait(ticket) before the launch that writes the
         new pages, append_token bookkeeping;
  GPU  : vt_kv_append (new K/V of all 32 layers) + 32 x vt_decode_attention
         (tcgen05 split-KV kernel with the split merge fused in its epilogue;
         layers 2..32 chained with programmatic dependent launch).

Context lengths are staggered over one map-ahead window so that every step
some requests run low on headroom and extend by a run of real 2 MiB chunks.

Metric (BASELINE.json): decode-attn KV GB/s = algorithmic bytes
(KV read + q read + out write + appended K/V) / time; tokens/s and the extend
latency are reported beside it. ``value`` is device-timed with inputs resident
in HBM (KV working set 32 GiB >> 126 MB L2, so no flush is needed); ``e2e``
repeats the run through the public API with q / new-K/V copied from pinned host
memory and the outputs copied back inside the timed region (copies pipelined
on a side stream across steps, as a serving loop would).

Multi-GPU (torchrun, one process per GPU): requests are partitioned — each GPU
owns its own VMM chunk pool and its own 64 requests (weak scaling); there is no
collective on the data path, only a barrier and a max-over-ranks of the timings.

``--impl reference`` times the reference arm: the CPU fp32 restatement of the
same attention (oracle/attention_ref.py, the only CPU implementation of this
path — the reference package has none) on the host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

MIB = 1 << 20
GIB = 1 << 30

CONFIGS = {
    # name: (layers, kv_heads, q_heads, batch_per_gpu_or_total, ctx)
    "llama3-8b-decode": (32, 8, 32, 64, 4096),   # config 2 (request partition)
    "llama2-70b-decode": (80, 8, 64, 64, 4096),  # config 4 (kv-head partition)
    "toy-cfg1": (1, 8, 8, 8, 4096),              # config 1 shape
    "llama3-8b-32k": (32, 8, 32, 16, 32768 - 256),  # config 5: long context, batch 16
}
HEAD_PARTITIONED = {"llama2-70b-decode"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=list(CONFIGS), default="llama3-8b-decode")
    ap.add_argument("--split", type=int, default=0, help="split-KV tokens per CTA (0=auto)")
    ap.add_argument("--path", choices=["tcgen05", "cuda_core"], default="tcgen05",
                    help="decode kernel: tcgen05/TMEM (default) or CUDA-core FFMA2")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-chain", action="store_true",
                    help="launch every decode layer plainly (no programmatic dependent launch)")
    ap.add_argument("--premap", action="store_true",
                    help="map every chunk the run will need up front (config-5 comparison)")
    ap.add_argument("--no-prefill", action="store_true", help="skip the config-3 prefill probe")
    ap.add_argument("--no-qkv", action="store_true",
                    help="skip the fused QKV-projection + KV-append probe")
    ap.add_argument("--profile-steps", type=int, default=0,
                    help="run N untimed steps only (for ncu), print nothing")
    ap.add_argument("--growth", action="store_true",
                    help="config 5 growth trace: 16 requests decode from 256 to 32,752 tokens "
                         "(32,496 steps, every chunk mapped on demand); --steps is ignored "
                         "unless --growth-steps caps it")
    ap.add_argument("--growth-steps", type=int, default=0,
                    help="cap the growth trace at this many timed steps (0 = the full trace)")
    ap.add_argument("--phys-reserve", type=int, default=-1,
                    help="pre-created physical handles kept by the shim (-1 = auto: the chunks "
                         "the run will create, capped at 16 GiB; 0 = off)")
    ap.add_argument("--driver-threads", type=int, default=0,
                    help="shim threads executing driver VMM ops in parallel (0 = library default)")
    ap.add_argument("--lead-chunks", type=int, default=0,
                    help="extend this many chunks ahead of each request's next token (0 = 24: "
                         "covers the driver's cuMemSetAccess stalls, up to ~1.5 s)")
    ap.add_argument("--plain-every", type=int, default=0,
                    help="with chained decode layers, also launch every N-th layer of a run "
                         "plainly (a kernel boundary where queued cuMemMap/cuMemSetAccess "
                         "complete); 0 = only the run's first layer")
    ap.add_argument("--plain-adaptive", action="store_true",
                    help="apply --plain-every only to steps enqueued while the shim's driver "
                         "worker still has mapping work outstanding")
    ap.add_argument("--max-ahead", type=int, default=2,
                    help="steps the host may queue ahead of the GPU before waiting for the "
                         "oldest (a serving loop reads tokens back every step); 0 = unbounded")
    ap.add_argument("--clock-interval", type=float, default=0.05,
                    help="seconds between NVML clock samples in the timed region (each NVML "
                         "query enters the kernel driver, like the VMM calls)")
    ap.add_argument("--host-sync", choices=["spin", "poll", "block"], default="spin",
                    help="how the host waits for its oldest queued step: spin in the driver "
                         "(default), poll with short sleeps, or a blocking-sync event")
    ap.add_argument("--check", action="store_true",
                    help="after the timed region, compare sampled (request, layer) outputs of the "
                         "last step (and the config-3 prefill probe) with the CPU oracle")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """SM clocks + throttle reasons sampled in-process (NVML) every 50 ms
    during the timed region; nvidia-smi subprocesses are too slow/intrusive."""

    REASONS = {  # nvmlClocksEventReason* bits
        "sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40,
    }

    def __init__(self, index: int, interval: float = 0.05) -> None:
        self.index = index
        self.interval = interval
        self.samples: list[tuple[int, int, int]] = []
        self._stop = threading.Event()
        self._t = None
        self._nvml = None

    def _run(self) -> None:
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                try:
                    reasons = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                except AttributeError:  # older bindings
                    reasons = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append((sm, mx, reasons))
                self._stop.wait(self.interval)
        except Exception as exc:  # pragma: no cover - no NVML
            self._nvml = repr(exc)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.06)
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None,
                    "reasons": [f"nvml unavailable: {self._nvml}"]}
        reasons = sorted({name for _, _, r in self.samples for name, bit in self.REASONS.items()
                          if r & bit})
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------ dist plumbing --
_COLL_DEVICE = "cuda"


def dist_setup(args):
    """One process per GPU (torchrun). NCCL carries only the barrier and the
    max/sum of the timings. When more ranks than GPUs are launched (checking
    the N-rank mechanics on a 1-GPU box) ranks share devices round-robin, the
    timing reductions go over gloo (NCCL refuses two ranks on one GPU);
    numbers from such a run are not scaling numbers — a mechanics check only,
    never the driver's one-rank-per-GPU configuration. (Two ranks' tcgen05
    decode kernels time-sliced on one GPU used to deadlock on an mbarrier
    parity race, fixed in r02: tests/test_timeslice_gpu.py.)"""
    global _COLL_DEVICE
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        n_dev = torch.cuda.device_count()
        dev = local % n_dev
        torch.cuda.set_device(dev)
        if world <= n_dev:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
            _COLL_DEVICE = "cpu"
            args.oversubscribed = ("%d ranks share %d GPU(s): time-sliced, a mechanics check, "
                                   "not a scaling number" % (world, n_dev))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, torch.cuda.current_device() if torch.cuda.is_available() else local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def _reduce(x: float, world: int, op_name: str) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=_COLL_DEVICE)
    dist.all_reduce(t, op=getattr(dist.ReduceOp, op_name))
    return float(t.item())


def max_over_ranks(x: float, world: int) -> float:
    return _reduce(x, world, "MAX")


def sum_over_ranks(x: float, world: int) -> float:
    return _reduce(x, world, "SUM")


# ------------------------------------------------------------- the workload --
def staggered_lens(ctx: int, B: int, win: int) -> list[int]:
    """Context lengths staggered over one map-ahead window (`win` tokens):
    every step some request runs out of headroom and extends."""
    return [ctx - (win - 1) + (b * win // B) if ctx >= win else ctx for b in range(B)]


def workload_config(cfg_name: str, world: int, split: int = 0, path: str = "tcgen05",
                    growth: bool = False) -> dict:
    """The bench line's `config` (identical for both arms): the workload one
    GPU runs per step. Computed without a GPU so the reference arm reports
    exactly the same dict."""
    from paper_2407_15309_b200.sharding import head_shard, layer_groups

    L, hkv, hq, B, ctx = CONFIGS[cfg_name]
    head_partition = cfg_name in HEAD_PARTITIONED
    if head_partition:
        sh = head_shard(hkv, hq, world, 0)
        hkv, hq = sh.local_kv_heads, sh.local_q_heads
    groups = layer_groups(L, hkv)
    tpc = 2 * MIB // groups[0][1].bytes_per_token
    win = int(os.environ.get("VT_MAP_AHEAD", "4")) * tpc
    lens = [GROWTH_START] * B if growth else staggered_lens(ctx, B, win)
    span = (f"{GROWTH_START}..{GROWTH_END} (growth trace)" if growth
            else f"{min(lens)}..{max(lens)}")
    kv_gib = (GROWTH_END if growth else sum(lens) / B) * B * L * 2 * hkv * 128 * 2 / GIB
    return {
        "workload": f"{cfg_name}: decode step, {L} layers, {hq} q / {hkv} kv heads per GPU, "
                    f"d 128, batch {B}, ctx {span}",
        "batch_per_gpu": B, "context": ctx, "layers": L,
        "parallelism": (f"kv-head partition x{world} (no collective)" if head_partition
                        else f"request partition x{world} (no collective)"),
        "layer_groups": len(groups),
        "l2": "inputs larger than L2 (KV working set %.1f GiB)" % kv_gib,
        "split_tokens": split or "auto",
        "decode_path": path,
    }


class _Group:
    """One layer group: its own manager (pool/VTO/VTS) on the GPU's shared VMM
    device, geometry (layers_in_group, local kv heads), KV-map cache."""

    def __init__(self, wl, first_layer, geom, seed):
        import torch

        import paper_2407_15309_b200 as vt
        from paper_2407_15309_b200.attention import KVMapCache
        from paper_2407_15309_b200.kv_layout import KVGeometry, chunk_view

        self.first = first_layer
        self.n_layers = geom.layers
        self.cfg = vt.SimConfig(
            capacity_bytes=wl.dev.config.capacity_bytes, chunk_size_bytes=2 * MIB,
            weights_bytes=0, geometry=geom, max_seq_len=wl.max_seq, initial_alloc_tokens=0,
            lookahead_chunks=1, max_batch=wl.B)
        self.pool = vt.TensorPool(self.cfg.tokens_per_chunk)
        self.ops = vt.VTensorOps(wl.dev, self.pool, self.cfg)
        self.sched = vt.VTensorScheduler(self.ops)
        self.geo = KVGeometry.from_config(self.cfg, wl.hq)
        self.tpc = self.cfg.tokens_per_chunk
        gen = torch.Generator(device="cuda").manual_seed(seed)
        self.vas = []
        for rid, n in zip(wl.rids, wl.lens):
            self.sched.create(rid, [1] * n)
            self.sched.mark_prefilled(rid)
            self.vas.append(wl.dev.va(self.sched.mem[rid].vt.space.rng))
        wl.dev.wait()
        for va, rid in zip(self.vas, wl.rids):
            view = chunk_view(va, self.sched.mem[rid].vt.space.mapped_pages, self.geo)
            view.copy_(torch.randn(view.shape, generator=gen, device="cuda").to(torch.bfloat16))
        self.kv_va = torch.tensor(self.vas, dtype=torch.int64, device="cuda")
        self.maps = KVMapCache(self.geo, wl.B) if wl.path == "tcgen05" else None
        self.chunk_ticket: dict[tuple[int, int], int] = {}


class DecodeWorkload:
    """The requests one GPU serves, their vTensor spaces, and the step driver.

    Request partition (default configs): every rank serves its own `B`
    requests. KV-head partition (llama2-70b-decode): every rank serves all `B`
    requests for its slice of kv / q heads. Models whose per-token KV does not
    divide a 2 MiB chunk are managed as layer groups (sharding.layer_groups).
    """

    def __init__(self, cfg_name: str, split: int, seed: int, path: str = "tcgen05",
                 world: int = 1, rank: int = 0, premap_steps: int = 0, chain: bool = True,
                 total_steps: int = 64, start_len: int = 0, max_seq: int = 0,
                 phys_reserve: int = -1, driver_threads: int = 0, lead_chunks: int = 0):
        import torch

        import paper_2407_15309_b200 as vt
        from paper_2407_15309_b200.attention import DecodeWorkspace
        from paper_2407_15309_b200.sharding import head_shard, layer_groups

        L, hkv, hq, B, ctx = CONFIGS[cfg_name]
        self.head_partition = cfg_name in HEAD_PARTITIONED
        if self.head_partition:
            sh = head_shard(hkv, hq, world, rank)
            hkv, hq = sh.local_kv_heads, sh.local_q_heads
        self.L, self.hkv, self.hq, self.B, self.ctx = L, hkv, hq, B, ctx
        self.path = path
        # every request grows by one token per step: reserve for the whole run
        self.max_seq = max_seq or ctx + 1024 + total_steps
        self.dev = vt.VirtualMemoryDevice(
            vt.DeviceConfig(capacity_bytes=160 * GIB, chunk_size_bytes=2 * MIB),
            cuda_ordinal=torch.cuda.current_device())
        if driver_threads:
            self.dev.set_driver_threads(driver_threads)
        groups = layer_groups(L, hkv)
        tpc = 2 * MIB // groups[0][1].bytes_per_token
        self.map_ahead = int(os.environ.get("VT_MAP_AHEAD", "4"))  # chunks per extend call
        # extend once headroom drops below this many chunks. cuMemSetAccess
        # costs ~0.15-0.8 ms per chunk but stalls for 10-120 ms every ~1 s, in
        # windows of up to ~1.5 s, even on an idle GPU (tools/vmm_probe7.cu,
        # profiles/r02/vmm_probes): 24 chunks (384 tokens at 8B, ~2 s of
        # config-2 decode) rode out every stall in the sustained runs
        # (profiles/r02/vmm_sustained/r2w_*: 0 host waits; 3 or 12 chunks did not)
        self.chain = chain
        self.lead_chunks = lead_chunks or int(os.environ.get("VT_LEAD_CHUNKS", "24"))
        win = self.map_ahead * tpc
        self.rids = [f"r{b}" for b in range(B)]
        if start_len:  # growth trace: every request starts at the same length
            self.lens = [start_len] * B
        else:
            # staggered lengths over one map-ahead window: every step some
            # request runs out of headroom and extends by a `map_ahead` run
            self.lens = staggered_lens(ctx, B, win)
        self.groups = [_Group(self, first, geom, seed + 17 * i)
                       for i, (first, geom) in enumerate(groups)]
        gen = torch.Generator(device="cuda").manual_seed(seed)
        self.q = torch.randn(L, B, hq, 128, generator=gen, device="cuda").to(torch.bfloat16)
        self.k_new = torch.randn(L, B, hkv, 128, generator=gen, device="cuda").to(torch.bfloat16)
        self.v_new = torch.randn_like(self.k_new)
        self.out = torch.empty_like(self.q)
        self.split = split
        self.ws = DecodeWorkspace(self.groups[0].geo, B, self.max_seq, split)
        self.stream = torch.cuda.current_stream()
        self.seq = torch.tensor(self.lens, dtype=torch.int32, device="cuda")
        self.seq1 = torch.empty_like(self.seq)
        self.host_lens = list(self.lens)
        self.stalls = 0
        self.host_waits = 0
        self.host_wait_ns = 0
        self.chained_steps = 0
        self.plain_every = 0  # see --plain-every
        self.plain_adaptive = False
        self.boundaries = 0  # plain decode launches (kernel boundaries) enqueued
        self.max_ahead = 2  # steps the host may have queued ahead of the GPU (0 = unbounded)
        self.host_sync = "spin"  # how the host waits for the oldest queued step (--host-sync)
        self.inflight: list = []
        self.last_done = None
        self.gap_events: list | None = None  # (previous step's end, this step's start)
        self.extend_ns: list[int] = []
        # time-based lead: keep at least `lead_s` seconds of decode mapped
        # ahead (host step period, EWMA), between lead_chunks and lead_max
        # chunks — short early steps of the growth trace need more chunks
        # than config 2's 5 ms steps to cover the same driver stall
        self.lead_s = 0.0 if premap_steps else float(os.environ.get("VT_LEAD_SECONDS", "2.0"))
        self.lead_max = int(os.environ.get("VT_LEAD_MAX_CHUNKS", "128"))
        self.step_s = 0.0
        self._t_last = None
        self.lead_eff_max = 0
        self.chunks_mapped = 0
        self._prewarm(1024)
        if phys_reserve < 0:  # auto: the chunks this run will still have to create
            grow = sum(-(-(n + total_steps + (self.map_ahead + self.lead_chunks + 1) * tpc) // tpc)
                       for n in self.lens) * len(groups)
            phys_reserve = min(max(0, grow - 1024), 8192)
        self.phys_reserve = phys_reserve
        if phys_reserve:
            self.dev.set_phys_reserve(phys_reserve)
        for grp in self.groups:  # staggered initial headroom (0..win-1 tokens)
            for b, rid in enumerate(self.rids):
                # premap: every token the run appends plus the extend
                # headroom, so no extend is issued inside the timed region
                extra = (premap_steps + win + self.lead_chunks * tpc if premap_steps
                         else (self.lead_chunks - 1) * tpc + (b * win) // B)
                grp.sched.extend(rid, min(self.max_seq, self.lens[b] + 1 + extra))
        self.dev.wait()
        torch.cuda.synchronize()

    @property
    def kv_bytes_per_token(self) -> int:
        return self.L * 2 * self.hkv * 128 * 2

    # -- manager half ---------------------------------------------------------
    def _prewarm(self, chunks: int):
        """Warm each group's pSet free list (lazy deallocation, ops.py:150-178):
        admit and release placeholder requests one after another so steady
        state extends reuse parked chunks instead of paying cuMemCreate under
        load. Each placeholder reuses its predecessor's chunks, so the list
        ends at one space's worth (e.g. 320 chunks at 8B) while `chunks` are
        cycled through the driver. (Holding all placeholders before releasing
        them — 1024 parked chunks — was measured to make the worker's
        cuMemSetAccess 5-10x slower in the timed region, so it stays this way.)"""
        for grp in self.groups:
            per = self.max_seq // grp.tpc
            left, i = chunks // len(self.groups), 0
            while left > 0:
                n = min(per, left)
                grp.sched.create(f"prewarm{i}", [0] * (n * grp.tpc))
                grp.sched.release(f"prewarm{i}")
                left -= n
                i += 1
        self.dev.wait()

    def _issue_extends(self):
        """VTS extend with map-ahead: when a request has less than one chunk of
        headroom past its next token, extend by `map_ahead` chunks (one
        contiguous run -> one cuMemSetAccess). Each newly mapped chunk records
        the worker ticket that makes it valid; a launch waits only for the
        chunks it touches, which were issued steps earlier."""
        for grp in self.groups:
            tpc = grp.tpc
            lead = self.lead_chunks
            if self.step_s > 0:
                lead = min(max(lead, math.ceil(self.lead_s / self.step_s / tpc)),
                           max(self.lead_max, self.lead_chunks))
            self.lead_eff_max = max(self.lead_eff_max, lead)
            for b, (rid, length) in enumerate(zip(self.rids, self.host_lens)):
                space = grp.sched.mem[rid].vt.space
                if space.mapped_pages * tpc >= min(self.max_seq, length + 1 + lead * tpc):
                    continue
                first = space.mapped_pages
                target = min(self.max_seq, length + 1 + (self.map_ahead + lead - 1) * tpc)
                t0 = time.perf_counter_ns()
                n = grp.sched.extend(rid, target)
                if n:
                    self.extend_ns.append(time.perf_counter_ns() - t0)
                    tk = self.dev.ticket()
                    for c in range(first, first + n):
                        grp.chunk_ticket[(b, c)] = tk
                self.chunks_mapped += n

    def algorithmic_bytes_per_step(self) -> int:
        """KV read (all layers, len+1 tokens incl. the new one) + q + out + appended K/V."""
        kv = sum(n + 1 for n in self.host_lens) * self.kv_bytes_per_token
        return kv + 2 * self.q.numel() * 2 + 2 * self.k_new.numel() * 2

    def decode_bytes_per_launch(self) -> int:
        return (sum(2 * (n + 1) * self.hkv * 128 * 2 for n in self.host_lens)
                + 2 * self.B * self.hq * 128 * 2)

    # -- one step -------------------------------------------------------------
    def step(self, q=None, k_new=None, v_new=None, out=None, run_events=None):
        import torch

        from paper_2407_15309_b200.attention import decode_attention, kv_append, last_launches

        q = self.q if q is None else q
        k_new = self.k_new if k_new is None else k_new
        v_new = self.v_new if v_new is None else v_new
        out = self.out if out is None else out
        # Bounded run-ahead: a serving loop reads each step's tokens back, so
        # the host never queues more than `max_ahead` steps beyond the GPU.
        # (Unbounded, the host queued ~30 steps of chained launches, and the
        # driver's cuMemSetAccess tails grew to 100-350 ms: profiles/r02.)
        while self.max_ahead and len(self.inflight) >= self.max_ahead:
            ev = self.inflight.pop(0)
            if self.host_sync == "poll":  # short driver calls: never block inside the driver
                while not ev.query():
                    time.sleep(2e-5)
            else:
                ev.synchronize()
        # the only pages this step touches: the chunk of each request's new token
        ticket = 0
        for grp in self.groups:
            for b, n in enumerate(self.host_lens):
                if n % grp.tpc == 0:
                    ticket = max(ticket, grp.chunk_ticket.pop((b, n // grp.tpc), 0))
        if ticket and not self.dev.ready(ticket):
            self.host_waits += 1
            t0 = time.perf_counter_ns()
            self.dev.wait(ticket)
            self.host_wait_ns += time.perf_counter_ns() - t0
            # queried after the wait: the GPU ran dry while this step's pages
            # were still mapping (the previous step's work had all finished)
            if self.last_done is not None and self.last_done.query():
                self.stalls += 1
        elif ticket:
            self.dev.wait(ticket)
        if self.gap_events is not None and self.last_done is not None:
            # device-side idle gap between the previous step's last kernel and
            # this step's first one (events at the step boundary only, where
            # the stream has a plain launch anyway)
            st = torch.cuda.Event(enable_timing=True)
            st.record(self.stream)
            self.gap_events.append((self.last_done, st))
        mx = max(self.host_lens) + 1
        launches = 1
        # Decode layers after the first are chained (programmatic dependent
        # launch, vt_decode_attention_chained): +3-4% per step. The worker's
        # concurrent cuMemMap / cuMemSetAccess complete while the chain runs
        # (probe 6: chained or plain, same per-call cost); their latency tail
        # is covered by extending `lead_chunks` chunks ahead.
        chain = self.chain
        self.chained_steps += int(chain)
        pe = self.plain_every
        if pe and self.plain_adaptive and self.dev.ready(self.dev.ticket()):
            pe = 0  # nothing queued on the driver worker: keep the whole chain
        torch.add(self.seq, 1, out=self.seq1)  # lengths including this step's token
        for gi, grp in enumerate(self.groups):
            kv_maps = None
            if grp.maps is not None:
                # TMA chunk extent = chunks holding valid tokens (all waited
                # for); chunks mapped ahead may still be in flight on the worker
                kv_maps = grp.maps.update(
                    grp.vas, [-(-(n + 1) // grp.tpc) * grp.tpc for n in self.host_lens])
            lo = grp.first
            kv_append(k_new[lo:lo + grp.n_layers], v_new[lo:lo + grp.n_layers], grp.kv_va,
                      self.seq, grp.geo)
            launches += 1
            # events bracket each group's run of decode layers only: the run
            # starts with a plain launch after the KV append, so they do not
            # break the chain of programmatic dependent launches inside it
            if run_events is not None:
                run_events[gi][0].record(self.stream)
            for li in range(grp.n_layers):
                layer = lo + li
                chained = chain and li > 0 and not (pe and li % pe == 0)
                self.boundaries += not chained
                decode_attention(q[layer], grp.kv_va, self.seq1, li, grp.geo, mx,
                                 out=out[layer], workspace=self.ws, split_tokens=self.split,
                                 kv_maps=kv_maps, chained=chained)
                launches += last_launches()
            if run_events is not None:
                run_events[gi][1].record(self.stream)
        self.seq, self.seq1 = self.seq1, self.seq
        self.dev.fence(self.stream.cuda_stream)
        self.last_done = torch.cuda.Event(enable_timing=self.gap_events is not None,
                                          blocking=self.host_sync == "block")
        self.last_done.record(self.stream)
        self.inflight.append(self.last_done)
        for grp in self.groups:
            for rid in self.rids:
                grp.sched.append_token(rid, 1)
        self.host_lens = [n + 1 for n in self.host_lens]
        now = time.perf_counter()
        if self._t_last is not None:  # host step period (= GPU step once run-ahead is bounded)
            dt = now - self._t_last
            self.step_s = dt if self.step_s == 0 else 0.9 * self.step_s + 0.1 * dt
        self._t_last = now
        self._issue_extends()  # next steps' pages: overlap with this step's kernels
        return launches


GROWTH_START, GROWTH_END = 256, 32752  # config 5: 32,496 decode steps


def check_decode(wl, samples: int = 8, tol: float = 2e-2) -> dict:
    """--check: the last timed step's outputs for `samples` (request, layer)
    pairs — spread over the batch, the layers and the layer groups — against
    the CPU oracle (oracle/attention_ref.py) over the same bf16 KV bytes read
    back from the request VAs. Run after the timed region, outside it. The
    tolerance is north_star's 2e-2 relative (bf16 in, fp32 accumulate)."""
    import torch

    from oracle.attention_ref import decode_attention_ref, rel_err
    from paper_2407_15309_b200.kv_layout import read_kv

    torch.cuda.synchronize()
    picks = []
    for i in range(samples):
        b = (i * 37 + 5) % wl.B
        layer = (i * (wl.L // samples) + i) % wl.L
        picks.append((b, layer))
    picks.append((wl.B - 1, wl.L - 1))
    worst, rows = 0.0, []
    for b, layer in picks:
        gi = max(i for i, g in enumerate(wl.groups) if g.first <= layer)
        grp = wl.groups[gi]
        n = wl.host_lens[b]  # valid tokens the last step attended (incl. its own)
        k, v = read_kv(grp.vas[b], n, layer - grp.first, grp.geo)
        ref = decode_attention_ref(wl.q[layer, b:b + 1].cpu(), [k.cpu()], [v.cpu()])
        err = rel_err(wl.out[layer, b:b + 1].cpu(), ref)
        worst = max(worst, err)
        rows.append({"request": b, "layer": layer, "len": n, "rel_err": round(err, 5)})
    return {"oracle": "oracle/attention_ref.py decode_attention_ref (fp32/fp64 CPU)",
            "samples": rows, "max_rel_err": round(worst, 5), "tol": tol, "ok": worst <= tol,
            "split_tokens": wl.split or "auto"}


def run_ours(args, world, rank, local):
    import torch

    if args.growth:
        args.config = "llama3-8b-32k"
        trace = GROWTH_END - GROWTH_START
        args.steps = min(trace - args.warmup, args.growth_steps or trace)
        args.no_e2e = True  # the e2e pass would need a second growth trace
        total_steps = args.warmup + args.steps
        wl = DecodeWorkload(args.config, args.split, seed=1234 + rank, path=args.path,
                            world=world, rank=rank,
                            premap_steps=total_steps if args.premap else 0,
                            chain=not args.no_chain, total_steps=total_steps,
                            start_len=GROWTH_START, max_seq=32768,
                            phys_reserve=0 if args.premap else args.phys_reserve,
                            driver_threads=args.driver_threads,
                            lead_chunks=args.lead_chunks)
    else:
        total_steps = args.warmup + 2 * args.steps + 2
        wl = DecodeWorkload(args.config, args.split, seed=1234 + rank, path=args.path,
                            world=world, rank=rank,
                            premap_steps=total_steps if args.premap else 0,
                            chain=not args.no_chain, total_steps=total_steps,
                            phys_reserve=0 if args.premap else args.phys_reserve,
                            driver_threads=args.driver_threads, lead_chunks=args.lead_chunks)
    wl.plain_every, wl.plain_adaptive = args.plain_every, args.plain_adaptive
    wl.max_ahead = args.max_ahead
    wl.host_sync = args.host_sync
    wl.dev.wait()  # the physical reserve (if any) is filled before any timing
    if args.profile_steps:
        for _ in range(args.profile_steps):
            wl.step()
        torch.cuda.synchronize()
        return
    wl.gap_events = []
    for _ in range(args.warmup):
        wl.step()
    torch.cuda.synchronize()
    barrier(world)
    wl.gap_events = []
    # the warm-up's last step ended before the synchronize/barrier above: its
    # event would turn that host-side pause into a "gap" (and an idle GPU into
    # a "stall") of the first timed step
    wl.last_done = None

    # ---- device-resident timed region ----
    run_ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in wl.groups] for _ in range(args.steps)]
    bytes_total = 0
    decode_bytes = 0
    launches = 0
    stalls0 = wl.stalls
    waits0 = wl.host_waits
    wait_ns0 = wl.host_wait_ns
    chained0 = wl.chained_steps
    bounds0 = wl.boundaries
    drv0 = wl.dev.driver_stats()
    wl.dev.driver_latencies("map_page", reset=True)
    wl.dev.driver_latencies("cuMemMap", reset=True)
    wl.dev.driver_latencies("cuMemSetAccess", reset=True)
    wl.extend_ns.clear()
    mapped0 = wl.chunks_mapped
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local, args.clock_interval) as clocks:
        torch.cuda.synchronize()
        barrier(world)
        start.record()
        for i in range(args.steps):
            bytes_total += wl.algorithmic_bytes_per_step()
            # Decode launch durations: CUDA events on the launch stream around
            # each group's run of decode layers in every timed step (an event
            # between two chained launches would serialise them; these sit
            # where the chain starts and ends anyway).
            decode_bytes += wl.decode_bytes_per_launch() * wl.L
            launches += wl.step(run_events=run_ev[i])
        stop.record()
        torch.cuda.synchronize()
    elapsed_ms = start.elapsed_time(stop)
    kern_ms = sum(a.elapsed_time(b) for evs in run_ev for a, b in evs)
    gaps = [a.elapsed_time(b) for a, b in wl.gap_events]
    wl.gap_events = None
    check = None
    if args.check:
        check = check_decode(wl)
    n_decode = wl.L * args.steps  # decode launches inside the bracketed runs
    stalls = wl.stalls - stalls0
    chained = wl.chained_steps - chained0
    plain_per_step = (wl.boundaries - bounds0) / max(args.steps, 1)
    elapsed_max = max_over_ranks(elapsed_ms, world)
    bytes_all = sum_over_ranks(bytes_total, world)
    tokens_all = wl.B * args.steps * (1 if wl.head_partition else world)
    value = bytes_all / (elapsed_max * 1e-3) / 1e9

    # ---- e2e: host buffers through the public API ----
    # Serving-loop pipeline: the copy engine moves step i+1's q / new K/V in
    # (pinned host -> HBM) and step i's attention output out (HBM -> pinned
    # host) on a side stream while step i's kernels run; device buffers are
    # double-buffered and every hand-off is an event, so no step reads an
    # input before its copy lands and no output is overwritten before it has
    # been read back. The timed region closes after the last read-back.
    e2e = None
    if not args.no_e2e:
        host_q = torch.empty(wl.q.shape, dtype=torch.bfloat16, pin_memory=True).copy_(wl.q)
        host_k = torch.empty(wl.k_new.shape, dtype=torch.bfloat16, pin_memory=True).copy_(wl.k_new)
        host_v = torch.empty(wl.v_new.shape, dtype=torch.bfloat16, pin_memory=True).copy_(wl.v_new)
        host_o = torch.empty(wl.out.shape, dtype=torch.bfloat16, pin_memory=True)
        bufs = [(torch.empty_like(wl.q), torch.empty_like(wl.k_new), torch.empty_like(wl.v_new),
                 torch.empty_like(wl.out)) for _ in range(2)]
        comp = torch.cuda.current_stream()
        cs = torch.cuda.Stream()
        in_ready = [torch.cuda.Event() for _ in range(2)]   # H2D into buffer b landed
        in_free = [torch.cuda.Event() for _ in range(2)]    # step done reading buffer b
        out_free = [torch.cuda.Event() for _ in range(2)]   # D2H of buffer b's output done

        def h2d(b):
            dq, dk, dv, _ = bufs[b]
            with torch.cuda.stream(cs):
                dq.copy_(host_q, non_blocking=True)
                dk.copy_(host_k, non_blocking=True)
                dv.copy_(host_v, non_blocking=True)
                in_ready[b].record(cs)

        e_bytes = 0
        torch.cuda.synchronize()
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(comp)
        cs.wait_event(e0)
        h2d(0)
        for i in range(args.steps):
            b = i & 1
            e_bytes += wl.algorithmic_bytes_per_step()
            if i + 1 < args.steps:
                if i >= 1:
                    cs.wait_event(in_free[b ^ 1])  # step i-1 has finished reading it
                h2d(b ^ 1)
            dq, dk, dv, do = bufs[b]
            comp.wait_event(in_ready[b])
            if i >= 2:
                comp.wait_event(out_free[b])       # step i-2's output has been read back
            wl.step(q=dq, k_new=dk, v_new=dv, out=do)
            in_free[b].record(comp)
            cs.wait_event(in_free[b])
            with torch.cuda.stream(cs):
                host_o.copy_(do, non_blocking=True)
                out_free[b].record(cs)
        comp.wait_stream(cs)
        e1.record(comp)
        torch.cuda.synchronize()
        e_ms = max_over_ranks(e0.elapsed_time(e1), world)
        e_all = sum_over_ranks(e_bytes, world)
        e2e = {"value": round(e_all / (e_ms * 1e-3) / 1e9, 2), "unit": "GB/s",
               "tokens_per_s": round(wl.B * args.steps * world / (e_ms * 1e-3), 1),
               "ms_per_step": round(e_ms / args.steps, 4),
               "h2d_bytes_per_step": int((host_q.numel() + host_k.numel() + host_v.numel()) * 2),
               "d2h_bytes_per_step": int(host_o.numel() * 2),
               "pipeline": "copies on a side stream overlap the previous/next step (double-buffered)"}

    map_lat = sorted(wl.dev.driver_latencies("map_page")) or [0]

    def call_stats(name):  # raw driver call durations inside the timed region
        v = sorted(wl.dev.driver_latencies(name)) or [0]
        return {"calls": len(v) if v != [0] else 0, "us_p50": round(v[len(v) // 2] / 1e3, 1),
                "us_p99": round(v[min(len(v) - 1, int(len(v) * 0.99))] / 1e3, 1),
                "us_max": round(v[-1] / 1e3, 1)}
    raw_calls = {"cuMemMap": call_stats("cuMemMap"), "cuMemSetAccess": call_stats("cuMemSetAccess")}
    drv_end = wl.dev.driver_stats()
    drv = {k: drv_end[k] - drv0[k] for k in drv_end}  # timed region only
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    per_launch_s = kern_ms * 1e-3 / n_decode
    achieved = (decode_bytes / n_decode) / per_launch_s / 1e9
    traffic = None
    traffic_key = f"{'growth' if args.growth else args.config}/{args.path}"
    try:  # the committed ncu --set full capture of THIS config's kernel (per launch), if any
        prof = json.load(open(os.path.join(REPO, "profiles", "decode_traffic.json")))
        traffic = prof[traffic_key]["dram_bytes_per_launch"]
    except Exception:
        pass

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, budget_s=8.0)
    prefill = None
    if rank == 0 and not args.no_prefill and args.config == "llama3-8b-decode":
        prefill = prefill_probe(check=args.check, cpu=not args.no_cpu_baseline)
    qkv = None
    if rank == 0 and not args.no_qkv and args.config == "llama3-8b-decode":
        qkv = qkv_probe()

    if rank == 0:
        ext = sorted(wl.extend_ns) or [0]
        line = {
            "metric": "decode-attn KV GB/s (% of HBM peak) and tokens/s; vTensor extend latency",
            "value": round(value, 2),
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(elapsed_max / args.steps, 4),
            "higher_is_better": True,
            "scaling": "strong" if wl.head_partition else "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic (seeded randn bf16 KV in real cuMemMap'd 2 MiB chunks)",
            "config": dict(workload_config(args.config, world, args.split, args.path, args.growth),
                           **({"oversubscribed": args.oversubscribed}
                              if getattr(args, "oversubscribed", None) else {})),
            "tokens_per_s": round(tokens_all / (elapsed_max * 1e-3), 1),
            "hbm_frac_of_step": round(value / hbm_peak, 4),
            "roofline": {
                "bound": "hbm",
                "kernel": ("vt::dtc::decode_tc_kernel" if args.path == "tcgen05"
                           else "vt::decode_splitkv_kernel<4>"),
                "achieved": round(achieved, 1),
                "peak": hbm_peak,
                "peak_source": peak_src,
                "peak_note": ("MEASURED_PEAKS hbm_gbs is a device copy (read + write); the "
                              "read-dominated decode stream can exceed it (ncu: one launch "
                              "moves 1.004x its algorithmic bytes)"),
                "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 4),
                "traffic": traffic,
                "per_launch_us": round(per_launch_s * 1e6, 2),
                "launch_timing": ("CUDA events on the launch stream around each run of chained "
                                  "decode layers, every timed step; per launch = run time / "
                                  "launches in the run"),
                "algorithmic_bytes_per_launch": int(decode_bytes / n_decode),
            },
            "extend": {
                "chunks_mapped": wl.chunks_mapped - mapped0,
                "extend_calls": len(wl.extend_ns),
                "ready_latency_us_p50": round(map_lat[len(map_lat) // 2] / 1e3, 1),
                "ready_latency_us_p99": round(map_lat[min(len(map_lat) - 1, int(len(map_lat) * 0.99))] / 1e3, 1),
                "ready_latency_note": "per mapped chunk, submit -> cuMemMap+cuMemSetAccess done on the worker",
                "chunks_per_extend": wl.map_ahead,
                "host_submit_us_p50": round(ext[len(ext) // 2] / 1e3, 2),
                "host_submit_us_p99": round(ext[min(len(ext) - 1, int(len(ext) * 0.99))] / 1e3, 2),
                "driver_map_us_mean": round(drv["map_ns_total"] / max(drv["map_calls"], 1) / 1e3, 2),
                "driver_create_us_mean": round(drv["create_ns_total"] / max(drv["create_calls"], 1) / 1e3, 2),
                "driver_access_us_mean": round(drv["access_ns_total"] / max(drv["access_calls"], 1) / 1e3, 2),
                "driver_calls": raw_calls,
                "gpu_stalled_steps": stalls,
                "gpu_idle_between_steps_ms": round(sum(gaps), 3),
                "gpu_idle_gap_ms_max": round(max(gaps), 3) if gaps else 0.0,
                "host_wait_ms_total": round((wl.host_wait_ns - wait_ns0) / 1e6, 3),
                "chained_steps": chained,
                "plain_decode_launches_per_step": round(plain_per_step, 2),
                "plain_every": args.plain_every,
                "max_steps_ahead": args.max_ahead,
                "host_sync": args.host_sync,
                "plain_adaptive": args.plain_adaptive,
                "lead_chunks": wl.lead_chunks,
                "lead_seconds": wl.lead_s,
                "lead_chunks_max_used": wl.lead_eff_max,
                "ready_note": ("cuMemSetAccess costs 0.15-0.8 ms per chunk with 10-120 ms "
                               "stalls (even on an idle GPU, tools/vmm_probe7.cu): ready latency "
                               "tails are covered by extending lead_chunks ahead"),
                "host_waited_steps": wl.host_waits - waits0,
                "hidden": stalls == 0 and wl.host_waits - waits0 == 0,
                "hidden_rule": ("no step waited on the host for a mapping and the GPU never ran "
                                "dry behind one; compare ms_per_step with the --premap twin"),
                "driver_threads": drv_end.get("driver_threads"),
                "phys_reserve_chunks": wl.phys_reserve,
                "creates_from_reserve": drv["reserve_hits"],
                "driver_creates": drv["create_calls"],
                "phys_reserve_note": ("pre-created physical handles (cuMemCreate before the timed "
                                      "region; the logical create_chunk + cuMemMap/SetAccess of "
                                      "every extend still happen on demand inside it)"),
            },
            "check": check,
            "growth": ({"from_tokens": GROWTH_START, "to_tokens": max(wl.host_lens),
                        "timed_steps": args.steps} if args.growth else None),
            "gpu_launches": launches + 0,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "prefill_cfg3": prefill,
            "qkv_append": qkv,
            "premapped": bool(args.premap),
            "clocks": dict(clocks.summary(), interval_s=args.clock_interval),
        }
        print(json.dumps(line))
    wl.dev.wait()
    torch.cuda.synchronize()


# ------------------------------------------------------- config-3 prefill --
def prefill_probe(iters: int = 8, check: bool = False, cpu: bool = True) -> dict:
    """Config 3 through the manager: a 2048-token conversation is recorded in
    the rTree, 16 follow-up turns prefix-match it (128 shared chunks mapped by
    identity + 32 new chunks each), and the tcgen05 prefix-prefill kernel runs
    the 512 new tokens of all 16 requests per layer (32 back-to-back layers)."""
    import torch

    import paper_2407_15309_b200 as vt
    from paper_2407_15309_b200.attention import kv_tensor_maps, last_launches, prefill_attention
    from paper_2407_15309_b200.kv_layout import KVGeometry, chunk_view

    L, hkv, hq, B, prefix, n_new = 32, 8, 32, 16, 2048, 512
    cfg = vt.SimConfig(capacity_bytes=16 * GIB, chunk_size_bytes=2 * MIB, weights_bytes=0,
                       geometry=vt.ModelGeometry(L, hkv, 128, 2), max_seq_len=4096,
                       initial_alloc_tokens=0)
    dev = vt.VirtualMemoryDevice(vt.DeviceConfig(cfg.capacity_bytes, cfg.chunk_size_bytes),
                                 cuda_ordinal=torch.cuda.current_device())
    sched = vt.VTensorScheduler(vt.VTensorOps(dev, vt.TensorPool(cfg.tokens_per_chunk), cfg))
    geo = KVGeometry.from_config(cfg, hq)
    tpc = cfg.tokens_per_chunk
    gen = torch.Generator(device="cuda").manual_seed(3)
    base = [i % 251 for i in range(prefix)]
    sched.create("conv", base)
    sched.mark_prefilled("conv")
    dev.wait()
    v = chunk_view(dev.va(sched.mem["conv"].vt.space.rng), prefix // tpc, geo)
    v.copy_(torch.randn(v.shape, generator=gen, device="cuda").to(torch.bfloat16))
    sched.prefix_record("conv")
    vas, shared_ok = [], True
    for b in range(B):
        rm, st = sched.prefix_match(f"t{b}", base + [9000 + b * n_new + k for k in range(n_new)])
        shared_ok &= st.identity_ok and st.shared_tokens == prefix
        vas.append(dev.va(rm.vt.space.rng))
    dev.wait()
    for va in vas:
        w = chunk_view(va, (prefix + n_new) // tpc, geo)[prefix // tpc:]
        w.copy_(torch.randn(w.shape, generator=gen, device="cuda").to(torch.bfloat16))
    maps = kv_tensor_maps(vas, [prefix + n_new] * B, geo)
    start = torch.full((B,), prefix, dtype=torch.int32, device="cuda")
    q = torch.randn(B, n_new, hq, 128, generator=gen, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    for layer in range(3):
        prefill_attention(q, maps, start, layer, geo, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        for layer in range(L):
            prefill_attention(q, maps, start, layer, geo, out=out)
    e1.record()
    torch.cuda.synchronize()
    per = e0.elapsed_time(e1) / (iters * L) * 1e-3
    flops = 4 * hq * 128 * (n_new * prefix + n_new * (n_new + 1) // 2) * B
    try:
        pk = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
    except Exception:
        pk = {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
    tf = flops / per / 1e12
    res = {"workload": "config 3: 16 x (2048 rTree-shared + 512 new), Llama-3-8B heads, per layer",
           "prefix_shared_by_identity": bool(shared_ok), "us_per_layer": round(per * 1e6, 1),
           "tflops": round(tf, 1), "frac_of_bf16_burst": round(tf / pk["bf16_tflops"], 4),
           "frac_of_bf16_sustained": round(tf / pk["bf16_tflops_sustained"], 4),
           "frac_note": "a ~70 ms probe of back-to-back launches: burst is the denominator",
           "kernel": "vt::pf::prefill_kernel (tcgen05/TMEM/TMA)", "launches": last_launches()}
    if check:
        # the last launch was layer L-1: sampled (request, kv head) slices vs the oracle
        from oracle.attention_ref import prefill_attention_ref, rel_err
        from paper_2407_15309_b200.kv_layout import read_kv

        G = hq // hkv
        rows, worst = [], 0.0
        for b, h in ((0, 0), (7, 3), (15, 7)):
            k, v = read_kv(vas[b], prefix + n_new, L - 1, geo)
            qs = q[b, :, h * G:(h + 1) * G].cpu()
            ref = prefill_attention_ref(qs, k[h:h + 1].cpu(), v[h:h + 1].cpu(), prefix)
            err = rel_err(out[b, :, h * G:(h + 1) * G].cpu(), ref)
            worst = max(worst, err)
            rows.append({"request": b, "kv_head": h, "rel_err": round(err, 5)})
        res["check"] = {"samples": rows, "max_rel_err": round(worst, 5), "tol": 2e-2,
                        "ok": worst <= 2e-2, "batch": B}
    if cpu:
        res["cpu_baseline"] = prefill_cpu_baseline(q, vas, geo, prefix, n_new, L - 1)
    dev.wait()
    return res


def prefill_cpu_baseline(q, vas, geo, prefix: int, n_new: int, layer: int,
                         budget_s: float = 6.0) -> dict:
    """CPU causal prefix-prefill (torch fp32 matmuls on all host threads) over
    the same KV bytes: one request's 512 new tokens x 32 q heads against its
    2048 + 512 tokens, repeated for about `budget_s`."""
    import torch

    from paper_2407_15309_b200.kv_layout import read_kv

    k, v = read_kv(vas[0], prefix + n_new, layer, geo)
    k, v, qq = k.cpu().float(), v.cpu().float(), q[0].cpu().float()  # [Hkv, L, d], [n, Hq, d]
    hkv, G = geo.kv_heads, geo.group
    pos = prefix + torch.arange(n_new)
    mask = torch.arange(prefix + n_new)[None, :] > pos[:, None]
    scale = 1.0 / math.sqrt(geo.head_dim)

    def once():
        qh = qq.permute(1, 0, 2).reshape(hkv, G * n_new, geo.head_dim)
        sc = torch.matmul(qh, k.transpose(1, 2)).view(hkv, G, n_new, -1) * scale
        sc.masked_fill_(mask, float("-inf"))
        return torch.matmul(torch.softmax(sc, dim=-1).view(hkv, G * n_new, -1), v)

    once()
    t0, reps = time.perf_counter(), 0
    while time.perf_counter() - t0 < budget_s and reps < 50:
        once()
        reps += 1
    dt = (time.perf_counter() - t0) / reps
    flops = 4 * geo.q_heads * geo.head_dim * (n_new * prefix + n_new * (n_new + 1) // 2)
    return {"value": round(flops / dt / 1e12, 4), "unit": "TFLOP/s",
            "cores": torch.get_num_threads(), "kind": "port",
            "sample": f"1 request x 1 layer ({n_new} new over {prefix} prefix, 32q/8kv), {reps} reps"}


# ---------------------------------------------- fused QKV + KV append probe --
def qkv_probe(layers: int = 32) -> dict:
    """SURVEY.md §8(f) row 2 at the config-2 shape: per layer, the new token
    of each of 64 requests goes through the fused QKV projection
    (x [64, 4096] . W_qkv[6144, 4096]^T, tcgen05) whose epilogue writes K/V
    straight into each request's vTensor VA at token_count. Timed as device
    time of a CUDA graph of 32 layers (32 distinct 50 MB weights: never
    L2-resident), next to the unfused path (cuBLAS GEMM + vt_kv_append)."""
    import torch

    import paper_2407_15309_b200 as vt
    from paper_2407_15309_b200.attention import kv_append, pack_qkv_weight, qkv_append
    from paper_2407_15309_b200.kv_layout import KVGeometry

    hkv, hq, hidden, B = 8, 32, 4096, 64
    cfg = vt.SimConfig(capacity_bytes=8 * GIB, chunk_size_bytes=2 * MIB, weights_bytes=0,
                       geometry=vt.ModelGeometry(layers, hkv, 128, 2), max_seq_len=4096,
                       initial_alloc_tokens=0)
    dev = vt.VirtualMemoryDevice(vt.DeviceConfig(cfg.capacity_bytes, cfg.chunk_size_bytes),
                                 cuda_ordinal=torch.cuda.current_device())
    sched = vt.VTensorScheduler(vt.VTensorOps(dev, vt.TensorPool(cfg.tokens_per_chunk), cfg))
    geo = KVGeometry.from_config(cfg, hq)
    vas = []
    for b in range(B):
        sched.create(f"r{b}", [1] * (100 + b))
        sched.mark_prefilled(f"r{b}")
        sched.extend(f"r{b}", 101 + b)
        vas.append(dev.va(sched.mem[f"r{b}"].vt.space.rng))
    dev.wait()
    kv_va = torch.tensor(vas, dtype=torch.int64, device="cuda")
    tok_req = torch.arange(B, dtype=torch.int32, device="cuda")
    tok_pos = torch.arange(100, 100 + B, dtype=torch.int32, device="cuda")
    feats = (hq + 2 * hkv) * 128
    gen = torch.Generator(device="cuda").manual_seed(4)
    ws = [(torch.randn(feats, hidden, generator=gen, device="cuda") / 64).to(torch.bfloat16)
          for _ in range(layers)]
    packed = [pack_qkv_weight(w) for w in ws]  # once, at weight-load time
    x = torch.randn(B, hidden, generator=gen, device="cuda").to(torch.bfloat16)
    q = torch.empty(B, hq, 128, dtype=torch.bfloat16, device="cuda")

    def fused():
        for l in range(layers):
            qkv_append(x, packed[l], tok_req, tok_pos, kv_va, geo, l, q_out=q)

    def unfused():
        for l in range(layers):
            y = x @ ws[l].T
            kv_append(y[:, hq * 128:(hq + hkv) * 128].reshape(1, B, hkv, 128).contiguous(),
                      y[:, (hq + hkv) * 128:].reshape(1, B, hkv, 128).contiguous(),
                      kv_va, tok_pos, geo, layer_begin=l)

    def graph_ms(fn):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        g.replay()
        torch.cuda.synchronize()
        best = float("inf")
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best

    t_f = graph_ms(fused) / layers * 1e-3
    t_u = graph_ms(unfused) / layers * 1e-3
    nbytes = feats * hidden * 2 + B * hidden * 2 + B * feats * 2
    try:
        pk = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
        hbm = pk["hbm_gbs"]
    except Exception:
        hbm = 6549.1
    dev.wait()
    return {"workload": "Llama-3-8B decode: 64 new tokens, x[64,4096] . W_qkv[6144,4096]^T per layer, "
                        "K/V into the vTensor cache at token_count",
            "us_per_layer": round(t_f * 1e6, 2), "GBps": round(nbytes / t_f / 1e9, 1),
            "frac_of_hbm": round(nbytes / t_f / 1e9 / hbm, 4), "bytes_per_layer": nbytes,
            "unfused_us_per_layer": round(t_u * 1e6, 2),
            "speedup_vs_unfused": round(t_u / t_f, 3),
            "unfused": "cuBLAS GEMM (torch) + vt_kv_append",
            "kernel": "vt::qkv::qkv_append_kernel<64,3> (tcgen05, packed weight; per feature tile a 2-CTA cluster (K halves, DSMEM reduction) + a helper CTA (first K quarter, partial through L2); 144 CTAs)",
            "weight_layout": "packed once (vt_qkv_pack_weight) outside the timed region"}


# --------------------------------------------------------- CPU / reference --
def cpu_baseline(cfg_name: str, budget_s: float = 8.0) -> dict:
    """The oracle's fp32 attention on the host cores over a bounded sample of
    the same workload (a few requests of one layer), GB/s of bf16 KV bytes."""
    import torch

    from oracle.attention_ref import decode_attention_torch_cpu

    L, hkv, hq, B, ctx = CONFIGS[cfg_name]
    threads = torch.get_num_threads()
    gen = torch.Generator().manual_seed(0)
    nb = min(B, 8)
    k = torch.randn(nb, hkv, ctx, 128, generator=gen).to(torch.bfloat16)
    v = torch.randn(nb, hkv, ctx, 128, generator=gen).to(torch.bfloat16)
    q = torch.randn(nb, hq, 128, generator=gen).to(torch.bfloat16)
    lens = [ctx] * nb
    decode_attention_torch_cpu(q, k, v, lens)  # warm
    t0 = time.perf_counter()
    reps = 0
    while time.perf_counter() - t0 < budget_s and reps < 200:
        decode_attention_torch_cpu(q, k, v, lens)
        reps += 1
    dt = (time.perf_counter() - t0) / reps
    kv_bytes = 2 * nb * hkv * ctx * 128 * 2 + 2 * nb * hq * 128 * 2
    cpu_name = ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                cpu_name = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"value": round(kv_bytes / dt / 1e9, 3), "unit": "GB/s", "cores": threads,
            "kind": "port",
            "sample": f"{nb} requests x 1 layer x {ctx} tokens ({hq}q/{hkv}kv heads), {reps} reps",
            "tokens_per_s_equiv": round(nb / (dt * L), 2),
            "manager": manager_cpu_baseline(),
            "host_cpus": os.cpu_count(), "cpu_model": cpu_name}


def manager_cpu_baseline(reference_only: bool = False) -> dict:
    """vTensor extend / append on the host, 1 core: the reference's algorithm
    (oracle/vtm_ref.py, reference cost model) vs this package's manager on the
    simulated shim (same op stream, Llama-3-8B geometry, 64 requests at ~4k)."""
    from oracle import vtm_ref as R

    arms = [("reference_port", R)]
    kv = _reference_kvsim()
    if kv is not None:
        arms.insert(0, ("reference_kvsim", kv))
    if not reference_only:
        import paper_2407_15309_b200 as vt

        arms.append(("ours_host_side", vt))
    out = {}
    for rep, (name, ns) in ((r, a) for r in range(3) for a in arms):
        # arms interleaved over 3 rounds, best p50 kept per arm: one arm run
        # after the others must not pay for their heap / allocator state
        cfg = ns.SimConfig(capacity_bytes=160 * GIB, chunk_size_bytes=2 * MIB, weights_bytes=0,
                           geometry=ns.ModelGeometry(32, 8, 128, 2), max_seq_len=8192,
                           initial_alloc_tokens=0)
        dev = ns.VirtualMemoryDevice(ns.DeviceConfig(cfg.capacity_bytes, cfg.chunk_size_bytes))
        sched = ns.VTensorScheduler(ns.VTensorOps(dev, ns.TensorPool(cfg.tokens_per_chunk), cfg))
        for b in range(64):
            sched.create(f"r{b}", [1] * 4080)
            sched.mark_prefilled(f"r{b}")
        ext, app = [], []
        for k in range(1, 9):
            for b in range(64):
                t0 = time.perf_counter_ns()
                sched.extend(f"r{b}", 4080 + 16 * k)  # +1 chunk
                ext.append(time.perf_counter_ns() - t0)
            for b in range(64):
                for _ in range(16):
                    t0 = time.perf_counter_ns()
                    sched.append_token(f"r{b}", 7)
                    app.append(time.perf_counter_ns() - t0)
        ext.sort()
        app.sort()
        # config 3's manager ops: record a 2048-token conversation prefix, then
        # admit turns that rTree-match it (2048 shared + 512 new tokens)
        rec, match = [], []
        for c in range(4):
            conv = [(c * 7919 + i) % 32000 for i in range(2048)]
            sched.create(f"c{c}", conv)
            sched.mark_prefilled(f"c{c}")
            t0 = time.perf_counter_ns()
            sched.prefix_record(f"c{c}")
            rec.append(time.perf_counter_ns() - t0)
            for t in range(4):
                rid = f"c{c}t{t}"
                t0 = time.perf_counter_ns()
                sched.prefix_match(rid, conv + [(t * 31 + i) % 32000 for i in range(512)])
                match.append(time.perf_counter_ns() - t0)
                sched.release(rid)
        rec.sort()
        match.sort()
        got = {"extend_1chunk_us_p50": round(ext[len(ext) // 2] / 1e3, 2),
               "extend_1chunk_us_p99": round(ext[int(len(ext) * 0.99)] / 1e3, 2),
               "append_token_us_p50": round(app[len(app) // 2] / 1e3, 2),
               "prefix_record_2048_us_p50": round(rec[len(rec) // 2] / 1e3, 1),
               "prefix_match_2048_512_us_p50": round(match[len(match) // 2] / 1e3, 1)}
        prev = out.get(name)
        out[name] = got if prev is None else {k: min(prev[k], got[k]) for k in got}
    out["cores"] = 1
    out["rounds"] = "3 interleaved rounds per arm, best p50/p99 of each"
    out["kind"] = "reference" if kv is not None else "port"
    return out


def _reference_kvsim():
    """The unmodified reference package (kvsim) from baseline/_ref, installed
    with `pip install --no-index ... --target baseline/_ref`;
    None when it is not there."""
    ref = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "kvsim")):
        return None
    if ref not in sys.path:
        sys.path.append(ref)
    try:
        import kvsim
    except Exception:
        return None
    return kvsim


def _first(d: dict) -> dict:
    name = "reference_kvsim" if "reference_kvsim" in d else "reference_port"
    return dict(d[name], impl=name, kind=d["kind"], cores=1)


def run_reference(args, world, rank):
    if rank != 0:
        return
    import torch

    torch.set_num_threads(os.cpu_count() or 1)
    if args.growth:
        args.config = "llama3-8b-32k"
    L, hkv, hq, B, ctx = CONFIGS[args.config]
    from oracle.attention_ref import decode_attention_torch_cpu

    gen = torch.Generator().manual_seed(0)
    nb = B  # the whole batch of one layer (1 GiB of KV at config 2) per step
    k = torch.randn(nb, hkv, ctx, 128, generator=gen).to(torch.bfloat16)
    v = torch.randn(nb, hkv, ctx, 128, generator=gen).to(torch.bfloat16)
    q = torch.randn(nb, hq, 128, generator=gen).to(torch.bfloat16)
    lens = [ctx] * nb
    # exactly K timed steps after W warm-up steps; each step is a bounded
    # sample (one layer of the whole batch: ~0.1-0.2 s on the box's 16 cores)
    steps, warm = args.steps, args.warmup
    for _ in range(warm):
        decode_attention_torch_cpu(q, k, v, lens)
    t0 = time.perf_counter()
    for _ in range(steps):
        decode_attention_torch_cpu(q, k, v, lens)
    dt = time.perf_counter() - t0
    kv_bytes = (2 * nb * hkv * ctx * 128 * 2 + 2 * nb * hq * 128 * 2) * steps
    value = kv_bytes / dt / 1e9
    sample = (f"all {nb} requests x 1 of {L} layers x {ctx} tokens per step ({hq}q/{hkv}kv "
              f"heads); {steps} timed steps after {warm} warm-up")
    line = {
        "impl": "reference",
        "metric": "decode-attn KV GB/s (% of HBM peak) and tokens/s; vTensor extend latency",
        "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": steps,
        "warmup": warm, "ms_per_step": round(dt / steps * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": workload_config(args.config, world, args.split, args.path,
                                                       args.growth),
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s",
                         "cores": torch.get_num_threads(), "kind": "port", "sample": sample},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        # the metric's other half: vTensor extend / token append through the
        # reference's own manager (kvsim from baseline/_ref; else the port), 1 host core
        "extend": _first(manager_cpu_baseline(reference_only=True)),
    }
    print(json.dumps(line))


def self_launch(n: int) -> None:
    """`python bench.py --gpus N` without torchrun: re-run this command under
    torch.distributed.run with N ranks on this node (127.0.0.1 rendezvous), so
    --gpus N always measures N processes. Exits with the launcher's code."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def main():
    args = parse()
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        self_launch(args.gpus)
    if env_world is not None and int(env_world) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}")
    hang_s = float(os.environ.get("VT_BENCH_HANG_DUMP_S", "0"))
    if hang_s > 0:  # diagnostics: dump every thread's stack if the run wedges
        import faulthandler

        faulthandler.dump_traceback_later(hang_s, exit=True)
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, world, rank)
        return
    world, rank, local = dist_setup(args)
    run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
