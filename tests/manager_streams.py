"""Seeded manager op streams + canonical state dumps (test infrastructure).

The same stream is fed to any kvsim-API namespace (the reference ``kvsim``
here in the CPU container, this package with the simulated or the CUDA-driver
shim anywhere). ``dump()`` canonicalises the whole manager state — spaces,
page tables (by chunk id), pSet entries, class counters, rTree records, device
accounting, the full device call log and the VTO journal — the §7.1 dump of
SURVEY.md. Parity = identical digests after every op.
"""

from __future__ import annotations

import hashlib
import json
import random
from types import SimpleNamespace


def make_stack(ns, cfg, device_kwargs=None):
    dev = ns.VirtualMemoryDevice(
        ns.DeviceConfig(
            capacity_bytes=cfg.capacity_bytes,
            chunk_size_bytes=cfg.chunk_size_bytes,
            weights_bytes=cfg.weights_bytes,
        ),
        **(device_kwargs or {}),
    )
    pool = ns.TensorPool(cfg.tokens_per_chunk)
    ops = ns.VTensorOps(dev, pool, cfg)
    sched = ns.VTensorScheduler(ops)
    return SimpleNamespace(dev=dev, pool=pool, ops=ops, sched=sched, cfg=cfg)


def dump(st) -> dict:
    pool, dev, ops = st.pool, st.dev, st.ops
    spaces = []
    for sid in sorted(pool.spaces):
        s = pool.spaces[sid]
        spaces.append([sid, s.state.value, s.mapped_pages, s.recorded, s.owner,
                       [h.id if h is not None else None for h in s.page_table]])
    entries = []
    for hid in sorted(pool.entries):
        e = pool.entries[hid]
        entries.append([hid, e.state.value, sorted(e.referrers), e.tokens_stored, e.cls,
                        e.handle.map_count])
    recs = [[list(map(int, seq))] for seq in pool.tree.recorded_sequences()]
    rec_spaces = sorted(vt.space.space_id for _, vt in pool.tree.records())
    stats = dev.stats()
    return {
        "spaces": spaces,
        "entries": entries,
        "counters": [pool.n_request, pool.n_pinned, pool.n_free, pool.used_tokens],
        "free": [h.id for h in pool.free_handles()],
        "avail": [s.space_id for s in pool.available_spaces()],
        "tree": recs,
        "tree_spaces": rec_spaces,
        "device": [stats.created_bytes, stats.reserved_virtual_bytes,
                   stats.mapped_page_count, stats.free_bytes],
        "log": [[c.seq, c.op, c.detail, c.created_bytes_after] for c in dev.call_log],
        "journal": [[r.name, r.call_start, r.call_end, sorted(r.detail.items())]
                    for r in ops.journal],
        "mem": {rid: [rm.vt.token_count, rm.vt.space.space_id, rm.shared_prefix_tokens]
                for rid, rm in sorted(st.sched.mem.items())},
    }


def digest(d: dict) -> str:
    return hashlib.sha256(json.dumps(d, sort_keys=True).encode()).hexdigest()[:16]


def run_stream(ns, cfg, seed: int, steps: int, on_step=None, device_kwargs=None,
               alphabet: int = 4, fence=None):
    """A serving-like lifecycle: admit (prefix-match first), prefill, decode with
    extends, record or release, probe matches, empty memory. Returns the stack
    and the list of (step, action, result) events."""
    st = make_stack(ns, cfg, device_kwargs)
    rng = random.Random(seed)
    tpc = cfg.tokens_per_chunk
    sched, ops = st.sched, st.ops
    active: list[str] = []
    serial = 0
    events = []
    OOM = ns.DeviceOutOfMemory
    shared_roots = [[rng.randrange(alphabet) for _ in range(3 * tpc)] for _ in range(3)]
    for step in range(steps):
        roll = rng.random()
        action = "noop"
        result = None
        try:
            if roll < 0.30:
                action = "admit"
                serial += 1
                rid = f"r{serial}"
                if rng.random() < 0.5:
                    root = rng.choice(shared_roots)
                    cut = rng.randint(0, len(root))
                    tokens = root[:cut]
                else:
                    tokens = []
                tokens = tokens + [rng.randrange(alphabet)
                                   for _ in range(rng.randint(1, 2 * tpc + 3))]
                tokens = tokens[: cfg.max_seq_len - 2 * tpc]
                hit = sched.prefix_match(rid, tokens) if rng.random() < 0.7 else None
                if hit is None:
                    _, stats = sched.create(rid, tokens)
                else:
                    _, stats = hit
                result = [stats.shared_tokens, stats.chunks_reused, stats.chunks_created,
                          stats.identity_ok]
                target = min(sched.lookahead_target(len(tokens)), cfg.max_seq_len)
                try:
                    result.append(sched.extend(rid, target))
                except OOM:
                    result.append("oom")
                sched.mark_prefilled(rid)
                active.append(rid)
            elif roll < 0.62 and active:
                action = "decode"
                rid = rng.choice(active)
                n = rng.randint(1, 2 * tpc)
                grown = 0
                for _ in range(n):
                    rm = sched.mem[rid]
                    if rm.vt.token_count + 1 > cfg.max_seq_len:
                        break
                    grown += sched.extend(rid, rm.vt.token_count + 1)
                    sched.append_token(rid, rng.randrange(alphabet))
                result = grown
            elif roll < 0.74 and active:
                action = "record"
                rid = active.pop(rng.randrange(len(active)))
                if fence:
                    fence(st)
                result = sched.prefix_record(rid)
                if not result:
                    sched.release(rid)
            elif roll < 0.86 and active:
                action = "release"
                rid = active.pop(rng.randrange(len(active)))
                if fence:
                    fence(st)
                sched.release(rid)
            elif roll < 0.95:
                action = "match"
                root = rng.choice(shared_roots)
                got = ops.r_prefix_match(root[: rng.randint(0, len(root))])
                result = None if got is None else got[1]
            else:
                action = "empty"
                if fence:
                    fence(st)
                r = ops.empty_memory(evict_prefix=rng.random() < 0.5)
                result = [r.chunks_destroyed, r.spaces_released, r.records_evicted]
        except OOM:
            result = "oom"
            if active:
                if fence:
                    fence(st)
                sched.release(active.pop(0))
            else:
                ops.empty_memory(evict_prefix=True)
        events.append([step, action, result])
        if on_step is not None:
            on_step(step, st)
    if fence:
        fence(st)
    sched.release_all()
    ops.empty_memory(evict_prefix=True)
    if on_step is not None:
        on_step(steps, st)
    return st, events


# Stream configurations. Every one uses 2 MiB chunks so the CUDA-driver
# backend can replay it on a B200; capacities are small to force OOM paths.
def stream_configs(ns):
    MIB = 1 << 20
    return {
        # config 1 geometry: 1 layer, 8 heads, d 128 -> 4 KiB/token, tpc 512, P 8
        "toy": ns.SimConfig(
            capacity_bytes=24 * 2 * MIB, chunk_size_bytes=2 * MIB, weights_bytes=0,
            geometry=ns.ModelGeometry(layers=1, kv_heads=8, head_dim=128, elem_bytes=2),
            max_seq_len=4096, initial_alloc_tokens=256, lookahead_chunks=1,
            prefix_cache_max_chunks=None),
        # Llama-3-8B geometry: 32 layers, 8 kv heads -> 128 KiB/token, tpc 16
        "llama8b": ns.SimConfig(
            capacity_bytes=96 * 2 * MIB, chunk_size_bytes=2 * MIB, weights_bytes=0,
            geometry=ns.ModelGeometry(layers=32, kv_heads=8, head_dim=128, elem_bytes=2),
            max_seq_len=512, initial_alloc_tokens=32, lookahead_chunks=1,
            prefix_cache_max_chunks=40),
        # 70B layer-group geometry (16 layers, 2 kv heads per GPU at N=4): tpc 256
        "llama70b_g16_h2": ns.SimConfig(
            capacity_bytes=40 * 2 * MIB, chunk_size_bytes=2 * MIB, weights_bytes=0,
            geometry=ns.ModelGeometry(layers=16, kv_heads=2, head_dim=128, elem_bytes=2),
            max_seq_len=2048, initial_alloc_tokens=128, lookahead_chunks=2,
            prefix_cache_max_chunks=12),
    }


STREAMS = [("toy", 0, 300), ("toy", 1, 300), ("llama8b", 2, 400), ("llama8b", 3, 400),
           ("llama70b_g16_h2", 4, 300)]
