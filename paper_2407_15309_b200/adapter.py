"""Engine seam (rows a25/a26): the allocator adapter the serving loop drives,
and the GPU compute that replaces the reference's cost formula.

``VTensorAdapter`` keeps the duck-typed allocator protocol of
kvsim/engine.py:176-250 (startup / can_admit / admit / prefill_reserve /
ensure_capacity / mark_prefilled / append_token / finish / release / shutdown /
kv_stats / extra_summary) with identical manager calls, so the reference's
``ServingEngine`` runs unchanged on top of it (tests/test_adapter.py).

``GpuCompute`` is the compute slot (kvsim/engine.py:499-511 prices a step as
``prefill_cost * prefill_tokens + decode_cost * batch``): it owns the per-step
launch sequence on the B200 — wait for exactly the worker tickets a launch
needs, refresh the TMA descriptors of requests that mapped a chunk, KV append,
tcgen05 decode over the batch, and a fence so later unmaps never tear pages
down under an in-flight kernel.
"""

from __future__ import annotations

import torch

from .geometry import SimConfig
from .tensor_pool import TensorPool
from .vto import VTensorOps
from .vts import VTensorScheduler


class VTensorAdapter:
    """Engine-facing wrapper around the chunked virtual-memory stack."""

    name = "vtensor"

    def __init__(self, device, config: SimConfig) -> None:
        self.device = device
        self.config = config
        self.pool = TensorPool(config.tokens_per_chunk)
        self.ops = VTensorOps(device, self.pool, config)
        self.scheduler = VTensorScheduler(self.ops)
        # worker ticket that makes each request's latest mappings valid (the
        # driver half of admit / reserve / extend runs asynchronously)
        self._ticket: dict[str, int] = {}

    def _note(self, rid: str, log_before: int) -> None:
        if len(self.device.call_log) != log_before:
            self._ticket[rid] = self.device.ticket()

    def ticket_for(self, rids) -> int:
        """The worker ticket a launch over ``rids`` must wait for: their own
        mappings only — unmaps of other requests are fenced on the GPU."""
        return max((self._ticket.get(r, 0) for r in rids), default=0)

    def startup(self) -> None:
        pass

    def can_admit(self, prompt_len: int) -> bool:
        cfg = self.config
        tpc = cfg.tokens_per_chunk
        need = -(-max(prompt_len, cfg.initial_alloc_tokens) // tpc) + cfg.lookahead_chunks
        have = self.device.free_bytes // cfg.chunk_size_bytes + self.pool.free_count()
        return need <= have

    def admit(self, request_id: str, tokens: list[int], try_prefix: bool):
        n0 = len(self.device.call_log)
        try:
            if try_prefix:
                hit = self.scheduler.prefix_match(request_id, tokens)
                if hit is not None:
                    return hit[1]
            return self.scheduler.create(request_id, tokens)[1]
        finally:
            self._note(request_id, n0)

    def prefill_reserve(self, request_id: str, prompt_len: int) -> int:
        from .vmm import DeviceOutOfMemory

        target = min(self.scheduler.lookahead_target(prompt_len), self.config.max_seq_len)
        n0 = len(self.device.call_log)
        try:
            return self.scheduler.extend(request_id, target)
        except DeviceOutOfMemory:
            return 0  # headroom only; the decode-path extend competes for memory later
        finally:
            self._note(request_id, n0)

    def ensure_capacity(self, request_id: str, target_tokens: int) -> None:
        n0 = len(self.device.call_log)
        try:
            self.scheduler.extend(request_id, target_tokens)
        finally:
            self._note(request_id, n0)

    def mark_prefilled(self, request_id: str, prompt_len: int) -> None:
        self.scheduler.mark_prefilled(request_id)

    def append_token(self, request_id: str, token: int) -> None:
        self.scheduler.append_token(request_id, token)

    def finish(self, request_id: str, record: bool) -> bool:
        if record and self.scheduler.prefix_record(request_id):
            return True
        self.scheduler.release(request_id)
        return False

    def release(self, request_id: str) -> None:
        self.scheduler.release(request_id)
        self._ticket.pop(request_id, None)

    def shutdown(self) -> dict:
        self.scheduler.release_all()
        rep = self.ops.empty_memory(evict_prefix=self.config.evict_prefix_on_empty)
        return {
            "chunks_destroyed": rep.chunks_destroyed,
            "spaces_released": rep.spaces_released,
            "records_evicted": rep.records_evicted,
        }

    def kv_stats(self):
        """Chunk classes from the pool counters (kvsim/metrics.py:91-123)."""
        from types import SimpleNamespace

        cfg, pool = self.config, self.pool
        chunk, bpt, tpc = cfg.chunk_size_bytes, cfg.bytes_per_token, cfg.tokens_per_chunk
        look = 0
        for rid in sorted(self.scheduler.mem):
            rm = self.scheduler.mem[rid]
            look += min(max(rm.provisioned_tokens - rm.vt.token_count, 0),
                        cfg.lookahead_chunks * tpc)
        used = pool.used_tokens * bpt
        allocated = (pool.n_request + pool.n_pinned + pool.n_free) * chunk
        pinned, retained = pool.n_pinned * chunk, pool.n_free * chunk
        lookahead = min(look * bpt, pool.n_request * chunk - used)
        reserved = retained + pinned + lookahead
        return SimpleNamespace(kv_allocated=allocated, kv_used=used, reserved=reserved,
                               pinned=pinned, retained=retained, lookahead=lookahead,
                               fragmentation=allocated - used - reserved)

    def extra_summary(self) -> dict:
        return {"prefix_records": len(self.pool.tree.records()),
                "pinned_chunks": self.pool.n_pinned}


class GpuCompute:
    """The compute slot on the B200 for a batch of decoding requests.

    ``step(rids, q, k_new, v_new)`` runs one decode step for the requests in
    ``rids`` (their KV already holds ``token_count`` tokens): the new token's
    K/V are appended at ``token_count`` for every layer, then every layer's
    attention reads ``token_count + 1`` tokens. The caller advances the manager
    (``append_token``) afterwards, as the reference engine does.
    """

    def __init__(self, adapter: VTensorAdapter, q_heads: int, max_batch: int,
                 split_tokens: int = 0) -> None:
        from .attention import DecodeWorkspace, KVMapCache
        from .kv_layout import KVGeometry

        self.adapter = adapter
        self.dev = adapter.device
        self.geo = KVGeometry.from_config(adapter.config, q_heads)
        self.max_batch = max_batch
        self.ws = DecodeWorkspace(self.geo, max_batch, adapter.config.max_seq_len, split_tokens)
        self.maps = KVMapCache(self.geo, max_batch)
        self.split = split_tokens
        self.launches = 0

    def _va(self, rid: str) -> int:
        return self.dev.va(self.adapter.scheduler.mem[rid].vt.space.rng)

    def _batch(self, rids: list[str], device, stream):
        """Device-side tables of a decode batch: VAs, positions of the new
        token (= token_count), lengths including it, TMA descriptors."""
        sched = self.adapter.scheduler
        tpc = self.adapter.config.tokens_per_chunk
        B = len(rids)
        if B > self.max_batch:
            raise ValueError("batch exceeds max_batch")
        lens = [sched.mem[r].vt.token_count for r in rids]
        for r, n in zip(rids, lens):
            if sched.mem[r].vt.space.mapped_pages * tpc < n + 1:
                raise RuntimeError(f"{r}: no capacity for token {n}; call ensure_capacity first")
        # the pages this step touches were mapped by the worker (unrelated
        # teardown is fenced on the GPU, not waited for here)
        self.dev.wait(self.adapter.ticket_for(rids))
        vas = [self._va(r) for r in rids]
        kv_va = torch.tensor(vas, dtype=torch.int64).to(device, non_blocking=True)
        pos = torch.tensor(lens, dtype=torch.int32).to(device, non_blocking=True)
        pad = self.max_batch - B
        maps = self.maps.update(vas + [vas[0]] * pad,
                                [-(-(n + 1) // tpc) * tpc for n in lens] + [lens[0] + 1] * pad,
                                stream)[: B * 128]
        return kv_va, pos, pos + 1, maps, max(lens) + 1

    def step(self, rids: list[str], q: torch.Tensor, k_new: torch.Tensor, v_new: torch.Tensor,
             out: torch.Tensor | None = None, stream: torch.cuda.Stream | None = None):
        from .attention import decode_attention, kv_append, last_launches

        stream = stream or torch.cuda.current_stream()
        kv_va, pos, seq, maps, mx = self._batch(rids, q.device, stream)
        kv_append(k_new, v_new, kv_va, pos, self.geo, stream=stream)
        self.launches += 1
        if out is None:
            out = torch.empty_like(q)
        for layer in range(q.shape[0]):
            decode_attention(q[layer], kv_va, seq, layer, self.geo, mx, out=out[layer],
                             workspace=self.ws, split_tokens=self.split, kv_maps=maps,
                             stream=stream, chained=layer > 0)
            self.launches += last_launches()
        self.dev.fence(stream.cuda_stream)
        return out

    def step_from_hidden(self, rids: list[str], x: torch.Tensor, w_qkv: list,
                         out: torch.Tensor | None = None,
                         stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """A decode step whose new token's q / K / V come from the fused QKV
        projection: per layer, ``x[l]`` ``[B, hidden]`` through
        ``w_qkv[l]`` (:class:`PackedQKVWeight`) writes K/V at ``token_count``
        straight into the cache (vt_qkv_append), then attention reads
        ``token_count + 1`` tokens. Returns ``[L, B, Hq, d]``."""
        from .attention import decode_attention, last_launches, qkv_append

        stream = stream or torch.cuda.current_stream()
        L, B, _ = x.shape
        kv_va, pos, seq, maps, mx = self._batch(rids, x.device, stream)
        tok_req = torch.arange(B, dtype=torch.int32, device=x.device)
        if out is None:
            out = torch.empty(L, B, self.geo.q_heads, self.geo.head_dim, dtype=torch.bfloat16,
                              device=x.device)
        for layer in range(L):
            q = qkv_append(x[layer], w_qkv[layer], tok_req, pos, kv_va, self.geo, layer,
                           stream=stream)
            # plain launch: it reads the K/V the projection just wrote
            decode_attention(q, kv_va, seq, layer, self.geo, mx, out=out[layer],
                             workspace=self.ws, split_tokens=self.split, kv_maps=maps,
                             stream=stream)
            self.launches += 1 + last_launches()
        self.dev.fence(stream.cuda_stream)
        return out

    def prefill(self, rid: str, x: torch.Tensor, w_qkv: list, start: int,
                stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """Prefill / prefix-prefill of request ``rid``: its new tokens sit at
        ``[start, start + n_new)`` (``start`` = tokens already in the cache,
        e.g. an rTree-shared prefix mapped by identity). Per layer, ``x[l]``
        ``[n_new, hidden]`` goes through the fused projection, which writes the
        new tokens' K/V into the cache (vt_qkv_append), then the new tokens
        attend causally to ``[0, start + i]`` (vt_prefill_attention). The pages
        of ``[0, start + n_new)`` must be mapped (admission / prefill_reserve).
        Returns ``[L, n_new, Hq, d]``; the caller then ``mark_prefilled``."""
        from .attention import kv_tensor_maps, last_launches, prefill_attention, qkv_append

        stream = stream or torch.cuda.current_stream()
        L, n_new, _ = x.shape
        rm = self.adapter.scheduler.mem[rid]
        tpc = self.adapter.config.tokens_per_chunk
        if rm.vt.space.mapped_pages * tpc < start + n_new:
            raise RuntimeError(f"{rid}: tokens [0, {start + n_new}) are not all mapped")
        self.dev.wait(self.adapter.ticket_for([rid]))
        va = self._va(rid)
        dev = x.device
        kv_va = torch.tensor([va], dtype=torch.int64, device=dev)
        tok_req = torch.zeros(n_new, dtype=torch.int32, device=dev)
        tok_pos = torch.arange(start, start + n_new, dtype=torch.int32, device=dev)
        maps = kv_tensor_maps([va], [start + n_new], self.geo)
        st = torch.tensor([start], dtype=torch.int32, device=dev)
        out = torch.empty(L, n_new, self.geo.q_heads, self.geo.head_dim, dtype=torch.bfloat16,
                          device=dev)
        for layer in range(L):
            q = qkv_append(x[layer], w_qkv[layer], tok_req, tok_pos, kv_va, self.geo, layer,
                           stream=stream)
            prefill_attention(q.unsqueeze(0), maps, st, layer, self.geo, out=out[layer].unsqueeze(0),
                              stream=stream)
            self.launches += 1 + last_launches()
        self.dev.fence(stream.cuda_stream)
        return out


# ----------------------------------------------------------------------------
# The reference engine with the real compute slot.
# ----------------------------------------------------------------------------
_M31 = (1 << 31) - 1


def _mix(x: torch.Tensor) -> torch.Tensor:
    """31-bit integer hash (int64 arithmetic, exact on any device)."""
    x = x & _M31
    x = (x ^ (x >> 15)) * 0x2C1B3C6D & _M31
    x = (x ^ (x >> 12)) * 0x297A2D39 & _M31
    return x ^ (x >> 15)


class HashedTokenSource:
    """Synthetic, weight-free stand-in for the model's QKV projection.

    K/V of the token at position ``p`` is a pure function of ``(token id, p)``
    — so a request that hard-links a donor's prefix chunks through the rTree
    (scheduler.py:104-162; same tokens at the same positions) finds exactly the
    K/V it would have written itself — and the query of a request at position
    ``p`` is a function of ``(request id, p)``. Values are uniform in
    ``[-2, 2)`` with a 16-bit grid, generated with integer arithmetic only, so
    the same call on the CPU reproduces the device bytes bit for bit (the
    tests' oracle mirror relies on that)."""

    def __init__(self, geo, seed: int = 0) -> None:
        self.geo = geo
        self.seed = seed

    def _vals(self, key: torch.Tensor, lanes: int, salt: int, first_lane: int = 0) -> torch.Tensor:
        lane = torch.arange(first_lane, first_lane + lanes, dtype=torch.int64, device=key.device)
        h = _mix(key[:, None] * 0x01000193 + lane[None, :] * 0x5BD1E995 + salt + self.seed)
        return ((h & 0xFFFF).to(torch.float32) * (4.0 / 65536.0) - 2.0).to(torch.bfloat16)

    def kv(self, tokens: torch.Tensor, positions: torch.Tensor, layer: int | None = None):
        """K, V ``[layers, n, kv_heads, head_dim]`` bf16 for n (token, position);
        with ``layer``, that layer only (``[n, kv_heads, head_dim]``)."""
        g = self.geo
        key = _mix(tokens.to(torch.int64) * 0x3C6EF372 + positions.to(torch.int64))
        per_layer = 2 * g.kv_heads * g.head_dim
        if layer is None:
            v = self._vals(key, g.layers * per_layer, 0x1234567)
            v = v.view(-1, g.layers, 2, g.kv_heads, g.head_dim).permute(1, 2, 0, 3, 4)
            return v[:, 0].contiguous(), v[:, 1].contiguous()  # [L, n, H, d]
        v = self._vals(key, per_layer, 0x1234567, first_lane=layer * per_layer)
        v = v.view(-1, 2, g.kv_heads, g.head_dim)
        return v[:, 0].contiguous(), v[:, 1].contiguous()

    def q(self, request_keys: torch.Tensor, positions: torch.Tensor,
          layer: int | None = None) -> torch.Tensor:
        """q ``[layers, n, q_heads, head_dim]`` bf16 for n (request key,
        position); with ``layer``, that layer only (``[n, q_heads, head_dim]``)."""
        g = self.geo
        key = _mix(request_keys.to(torch.int64) * 0x7FEB352D + positions.to(torch.int64))
        per_layer = g.q_heads * g.head_dim
        if layer is not None:
            v = self._vals(key, per_layer, 0x7654321, first_lane=layer * per_layer)
            return v.view(-1, g.q_heads, g.head_dim)
        v = self._vals(key, g.layers * per_layer, 0x7654321)
        return v.view(-1, g.layers, g.q_heads, g.head_dim).permute(1, 0, 2, 3).contiguous()

    @staticmethod
    def request_key(rid: str) -> int:
        import zlib

        return zlib.crc32(rid.encode()) & _M31


class GpuServingAdapter(VTensorAdapter):
    """``VTensorAdapter`` that runs the step's attention on the B200 in the
    compute slot of the reference ``ServingEngine`` (engine.py:499-511),
    with the engine itself unmodified.

    The engine calls, per step: extends (``ensure_capacity``), admissions
    (``admit`` / ``prefill_reserve``), then token progress for every request
    of the batch (``mark_prefilled`` for the ones admitted this step,
    ``append_token`` for the decoding ones), then ``finish`` / ``release`` and
    ``kv_stats`` (engine.py:384-560). Progress calls are exactly the batch, so
    the adapter collects them and launches the step's kernels at the first
    call after them — before any page of the batch can be released:

    * wait on the host for the worker tickets of the batch's own mappings
      only (admit / reserve / extend of these requests), never for unrelated
      teardown (that is fenced on the GPU);
    * prefill: new tokens' K/V of every admitted request written at
      ``[shared, len)`` (rTree-shared prefix chunks are read in place), then
      one variable-length tcgen05 prefill launch per layer for all of them;
    * decode: the new token's K/V appended at ``token_count``, then the
      tcgen05 decode over ``token_count + 1`` tokens per layer (layers after
      the first chained with programmatic dependent launch);
    * a fence, so later unmaps (finish, preemption) wait for these kernels.

    The manager calls and their order are the base adapter's, so the
    engine's CSV / summary / admissions stay byte-identical to the
    reference's (tests/test_engine_gpu.py). The memory lane is measured, not
    modelled: ``lane`` counts steps whose launch waited on the host for a
    mapping and steps where the GPU ran dry during that wait.
    ``on_step(record)`` (optional) receives each step's inputs and outputs.
    """

    def __init__(self, device, config: SimConfig, q_heads: int, source=None,
                 split_tokens: int = 0, on_step=None) -> None:
        from .attention import DecodeWorkspace, KVMapCache
        from .kv_layout import KVGeometry

        super().__init__(device, config)
        self.geo = KVGeometry.from_config(config, q_heads)
        self.source = source or HashedTokenSource(self.geo)
        self.max_batch = config.max_batch
        self.ws = DecodeWorkspace(self.geo, self.max_batch, config.max_seq_len, split_tokens)
        self.maps = KVMapCache(self.geo, self.max_batch)
        self.split = split_tokens
        self.on_step = on_step
        self.stream = torch.cuda.current_stream()
        self._tokens: dict[str, list[int]] = {}
        self._shared: dict[str, int] = {}
        self._prefill: list[str] = []
        self._decode: list[tuple[str, int, int]] = []  # (rid, position, token)
        self._last_done: torch.cuda.Event | None = None
        self.steps = 0
        self.launches = 0
        self.lane = {"steps": 0, "host_waited_steps": 0, "gpu_stalled_steps": 0,
                     "host_wait_ms": 0.0, "prefill_tokens": 0, "decode_tokens": 0}

    # -- manager calls (the base adapter notes each request's worker ticket)
    def admit(self, request_id: str, tokens: list[int], try_prefix: bool):
        self._flush()
        stats = super().admit(request_id, tokens, try_prefix)
        self._tokens[request_id] = list(tokens)
        self._shared[request_id] = stats.shared_tokens
        return stats

    def ensure_capacity(self, request_id: str, target_tokens: int) -> None:
        self._flush()
        super().ensure_capacity(request_id, target_tokens)

    def can_admit(self, prompt_len: int) -> bool:
        self._flush()
        return super().can_admit(prompt_len)

    # -- token progress = the batch of this step
    def mark_prefilled(self, request_id: str, prompt_len: int) -> None:
        self._prefill.append(request_id)
        super().mark_prefilled(request_id, prompt_len)

    def append_token(self, request_id: str, token: int) -> None:
        pos = self.scheduler.mem[request_id].vt.token_count
        self._decode.append((request_id, pos, token))
        self._tokens[request_id].append(token)
        super().append_token(request_id, token)

    # -- anything after progress flushes the step's compute first
    def finish(self, request_id: str, record: bool) -> bool:
        self._flush()
        return super().finish(request_id, record)

    def release(self, request_id: str) -> None:
        self._flush()
        super().release(request_id)

    def kv_stats(self):
        self._flush()
        return super().kv_stats()

    def shutdown(self) -> dict:
        self._flush()
        torch.cuda.synchronize()
        return super().shutdown()

    # -- the compute slot
    def _va(self, rid: str) -> int:
        return self.device.va(self.scheduler.mem[rid].vt.space.rng)

    def _wait_for(self, rids) -> None:
        import time

        t = self.ticket_for(rids)
        if not t or self.device.ready(t):
            return
        self.lane["host_waited_steps"] += 1
        t0 = time.perf_counter()
        self.device.wait(t)
        self.lane["host_wait_ms"] += (time.perf_counter() - t0) * 1e3
        if self._last_done is not None and self._last_done.query():
            self.lane["gpu_stalled_steps"] += 1  # the GPU ran dry behind the mapping

    def _flush(self) -> None:
        if not self._prefill and not self._decode:
            return
        from .attention import (decode_attention, kv_append, kv_tensor_maps, last_launches,
                                prefill_attention_varlen)

        prefill, decode = self._prefill, self._decode
        self._prefill, self._decode = [], []
        geo, src, st = self.geo, self.source, self.stream
        dev = torch.device("cuda", torch.cuda.current_device())
        self._wait_for([r for r in prefill] + [r for r, _, _ in decode])
        rec = {"step": self.steps, "tokens": self._tokens}
        with torch.cuda.stream(st):
            if prefill and sum(len(self._tokens[r]) - self._shared[r] for r in prefill) == 0:
                prefill = []  # whole prompts matched in the rTree: nothing to compute
            if prefill:
                starts = [self._shared[r] for r in prefill]
                lens = [len(self._tokens[r]) for r in prefill]
                vas = [self._va(r) for r in prefill]
                tok, pos, req, keys, offs = [], [], [], [], [0]
                for i, (r, s, n) in enumerate(zip(prefill, starts, lens)):
                    tok += self._tokens[r][s:n]
                    pos += range(s, n)
                    req += [vas[i]] * (n - s)
                    keys += [HashedTokenSource.request_key(r)] * (n - s)
                    offs.append(offs[-1] + n - s)
                tok_t = torch.tensor(tok, dtype=torch.int64).to(dev, non_blocking=True)
                pos_t = torch.tensor(pos, dtype=torch.int64).to(dev, non_blocking=True)
                k, v = src.kv(tok_t, pos_t)  # [L, T, Hkv, d]
                q = src.q(torch.tensor(keys, dtype=torch.int64).to(dev, non_blocking=True), pos_t)
                kv_append(k, v, torch.tensor(req, dtype=torch.int64).to(dev, non_blocking=True),
                          pos_t.to(torch.int32), geo, stream=st)
                maps = kv_tensor_maps(vas, lens, geo)
                start_t = torch.tensor(starts, dtype=torch.int32).to(dev, non_blocking=True)
                off_t = torch.tensor(offs, dtype=torch.int32).to(dev, non_blocking=True)
                out = torch.empty_like(q)
                mx = max(n - s for s, n in zip(starts, lens))
                for layer in range(geo.layers):
                    prefill_attention_varlen(q[layer], maps, start_t, off_t, mx, layer, geo,
                                             out=out[layer], stream=st)
                self.launches += 1 + geo.layers
                self.lane["prefill_tokens"] += offs[-1]
                rec["prefill"] = {"rids": prefill, "starts": starts, "lens": lens,
                                  "q_offsets": offs, "q": q, "out": out}
            if decode:
                rids = [r for r, _, _ in decode]
                B = len(rids)
                vas = [self._va(r) for r in rids]
                pos = [p for _, p, _ in decode]
                tok_t = torch.tensor([t for _, _, t in decode], dtype=torch.int64).to(
                    dev, non_blocking=True)
                pos_t = torch.tensor(pos, dtype=torch.int64).to(dev, non_blocking=True)
                k, v = src.kv(tok_t, pos_t)  # [L, B, Hkv, d]
                keys = torch.tensor([HashedTokenSource.request_key(r) for r in rids],
                                    dtype=torch.int64).to(dev, non_blocking=True)
                q = src.q(keys, pos_t)
                kv_va = torch.tensor(vas, dtype=torch.int64).to(dev, non_blocking=True)
                pos32 = pos_t.to(torch.int32)
                kv_append(k, v, kv_va, pos32, geo, stream=st)
                seq = pos32 + 1
                tpc = geo.tokens_per_chunk
                pad = self.max_batch - B
                maps = self.maps.update(vas + [vas[0]] * pad,
                                        [-(-(p + 1) // tpc) * tpc for p in pos] + [pos[0] + 1] * pad,
                                        st)[: B * 128]
                out = torch.empty_like(q)
                mx = max(pos) + 1
                for layer in range(geo.layers):
                    decode_attention(q[layer], kv_va, seq, layer, geo, mx, out=out[layer],
                                     workspace=self.ws, split_tokens=self.split, kv_maps=maps,
                                     stream=st, chained=layer > 0)
                    self.launches += last_launches()
                self.launches += 1
                self.lane["decode_tokens"] += B
                rec["decode"] = {"rids": rids, "positions": pos, "q": q, "out": out}
            self.device.fence(st.cuda_stream)
            self._last_done = torch.cuda.Event()
            self._last_done.record(st)
        self.steps += 1
        self.lane["steps"] += 1
        if self.on_step is not None:
            self.on_step(rec)
