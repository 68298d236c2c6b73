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

    def startup(self) -> None:
        pass

    def can_admit(self, prompt_len: int) -> bool:
        cfg = self.config
        tpc = cfg.tokens_per_chunk
        need = -(-max(prompt_len, cfg.initial_alloc_tokens) // tpc) + cfg.lookahead_chunks
        have = self.device.free_bytes // cfg.chunk_size_bytes + self.pool.free_count()
        return need <= have

    def admit(self, request_id: str, tokens: list[int], try_prefix: bool):
        if try_prefix:
            hit = self.scheduler.prefix_match(request_id, tokens)
            if hit is not None:
                return hit[1]
        return self.scheduler.create(request_id, tokens)[1]

    def prefill_reserve(self, request_id: str, prompt_len: int) -> int:
        from .vmm import DeviceOutOfMemory

        target = min(self.scheduler.lookahead_target(prompt_len), self.config.max_seq_len)
        try:
            return self.scheduler.extend(request_id, target)
        except DeviceOutOfMemory:
            return 0  # headroom only; the decode-path extend competes for memory later

    def ensure_capacity(self, request_id: str, target_tokens: int) -> None:
        self.scheduler.extend(request_id, target_tokens)

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
        self.dev.wait()  # every page this step touches has been mapped by the worker
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
        self.dev.wait()
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
