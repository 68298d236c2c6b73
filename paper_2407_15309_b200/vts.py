"""Layer L3: vTensor Scheduler, VTS — request actions (rows a19-a23).

create / prefix_match / extend / mark_prefilled / append_token /
prefix_record / release, with kvsim/scheduler.py semantics:

* create provisions ``ceil(max(prompt, initial_alloc) / tpc)`` chunks and
  unwinds the space on OOM (scheduler.py:70-102);
* prefix_match maps the donor's leading handles *by identity* (hard links, no
  copies), then provisions the suffix with **no** initial_alloc floor
  (scheduler.py:104-162 — the code, not SPEC.md:356, is the parity target);
* extend is ``ceil(target / tpc) - mapped_pages`` chunks (scheduler.py:166-180)
  — the "vTensor extend" whose latency the bench reports; on the CUDA shim the
  driver half of it runs on the worker thread and is fenced before launch;
* progress tracking advances per-chunk ``tokens_stored`` (scheduler.py:195-205).
"""

from __future__ import annotations

import dataclasses

from .geometry import SimConfig
from .tensor_pool import VirtualTensor
from .vmm import DeviceOutOfMemory
from .vto import VTensorOps


class ExceedsMaxSeqLen(Exception):
    pass


@dataclasses.dataclass
class AdmitStats:
    """How a request's memory came to be: sharing and chunk acquisition."""

    shared_tokens: int = 0
    chunks_reused: int = 0
    chunks_created: int = 0
    donor_space: int | None = None
    identity_ok: bool = True

    @property
    def chunks_acquired(self) -> int:
        return self.chunks_reused + self.chunks_created


@dataclasses.dataclass
class RequestMem:
    request_id: str
    vt: VirtualTensor
    shared_prefix_tokens: int = 0

    @property
    def provisioned_tokens(self) -> int:
        return self.vt.space.mapped_pages * self._tpc

    _tpc: int = 32


def _ceil_div(a: int, b: int) -> int:
    return -(-a // b)


class VTensorScheduler:
    def __init__(self, ops: VTensorOps) -> None:
        self.ops = ops
        self.config: SimConfig = ops.config
        self.mem: dict[str, RequestMem] = {}

    # -- helpers --------------------------------------------------------------

    def _alloc_counts(self, since: int) -> tuple[int, int]:
        reused = created = 0
        for rec in self.ops.journal[since:]:
            if rec.name == "p_alloc" and not rec.detail.get("failed"):
                reused += rec.detail.get("reused", 0)
                created += rec.detail.get("created", 0)
        return reused, created

    def _check_new(self, request_id: str, tokens: list[int]) -> None:
        if request_id in self.mem:
            raise ValueError(f"request {request_id} already has memory")
        if len(tokens) > self.config.max_seq_len:
            raise ExceedsMaxSeqLen(
                f"prompt of {len(tokens)} tokens exceeds max_seq_len {self.config.max_seq_len}"
            )

    def _register(self, request_id, space, tokens, shared: int) -> RequestMem:
        tpc = self.config.tokens_per_chunk
        space.owner = request_id
        vt = VirtualTensor(
            space=space,
            tokens=list(tokens),
            token_count=0,
            capacity_tokens=space.page_count * tpc,
            owner=request_id,
        )
        rm = RequestMem(request_id, vt, shared_prefix_tokens=shared)
        rm._tpc = tpc
        self.mem[request_id] = rm
        return rm

    # -- admission ------------------------------------------------------------

    def create(self, request_id: str, tokens: list[int]) -> tuple[RequestMem, AdmitStats]:
        self._check_new(request_id, tokens)
        tpc = self.config.tokens_per_chunk
        want = _ceil_div(max(len(tokens), self.config.initial_alloc_tokens), tpc)
        mark = len(self.ops.journal)
        space = self.ops.v_alloc(self.config.max_seq_len)
        try:
            handles = self.ops.p_alloc(want)
        except DeviceOutOfMemory:
            self.ops.unmap_space(space)
            raise
        self.ops.map_chunks(space, handles)
        rm = self._register(request_id, space, tokens, 0)
        reused, created = self._alloc_counts(mark)
        return rm, AdmitStats(chunks_reused=reused, chunks_created=created)

    def prefix_match(self, request_id: str, tokens: list[int]) -> tuple[RequestMem, AdmitStats] | None:
        self._check_new(request_id, tokens)
        hit = self.ops.r_prefix_match(tokens)
        if hit is None:
            return None
        donor, matched = hit
        tpc = self.config.tokens_per_chunk
        shared_pages = matched // tpc
        mark = len(self.ops.journal)
        space = self.ops.v_alloc(self.config.max_seq_len)
        donor_table = donor.space.page_table
        try:
            self.ops.map_chunks(space, donor_table[:shared_pages])
            deficit = _ceil_div(len(tokens), tpc) - shared_pages
            if deficit > 0:
                self.ops.map_chunks(space, self.ops.p_alloc(deficit))
        except DeviceOutOfMemory:
            self.ops.unmap_space(space)
            raise
        rm = self._register(request_id, space, tokens, matched)
        self._advance_stored(rm, matched)  # shared KV is already materialised
        rm.vt.token_count = matched
        reused, created = self._alloc_counts(mark)
        table = space.page_table
        identity = all(table[p] is donor_table[p] for p in range(shared_pages))
        return rm, AdmitStats(
            shared_tokens=matched,
            chunks_reused=reused,
            chunks_created=created,
            donor_space=donor.space.space_id,
            identity_ok=identity,
        )

    # -- growth ---------------------------------------------------------------

    def extend(self, request_id: str, target_tokens: int) -> int:
        rm = self.mem[request_id]
        if target_tokens > self.config.max_seq_len:
            raise ExceedsMaxSeqLen(
                f"extend to {target_tokens} exceeds max_seq_len {self.config.max_seq_len}"
            )
        deficit = _ceil_div(target_tokens, self.config.tokens_per_chunk) - rm.vt.space.mapped_pages
        if deficit <= 0:
            return 0
        self.ops.extend_space(rm.vt.space, deficit)  # p_alloc + map_chunks, one shim call
        return deficit

    def mark_prefilled(self, request_id: str) -> None:
        rm = self.mem[request_id]
        n = len(rm.vt.tokens)
        self._advance_stored(rm, n)
        rm.vt.token_count = n

    def append_token(self, request_id: str, token: int) -> None:
        rm = self.mem[request_id]
        rm.vt.tokens.append(token)
        rm.vt.token_count += 1
        self._advance_stored(rm, rm.vt.token_count)

    def _advance_stored(self, rm: RequestMem, token_count: int) -> None:
        if token_count <= 0:
            return
        tpc = self.config.tokens_per_chunk
        prev = rm.vt.token_count
        first = max(0, (prev - 1) // tpc) if prev else 0
        last = (token_count - 1) // tpc
        table, pool = rm.vt.space.page_table, self.ops.pool
        for page in range(first, last + 1):
            handle = table[page]
            if handle is None:
                raise RuntimeError("token progress ran past mapped capacity")
            pool.note_stored(handle, min(tpc, token_count - page * tpc))

    # -- teardown -------------------------------------------------------------

    def prefix_record(self, request_id: str) -> bool:
        rm = self.mem.get(request_id)
        if rm is None or not self.ops.r_push(rm.vt):
            return False
        del self.mem[request_id]
        return True

    def release(self, request_id: str) -> None:
        rm = self.mem.pop(request_id, None)
        if rm is not None:
            self.ops.unmap_space(rm.vt.space)

    def release_all(self) -> None:
        for request_id in sorted(self.mem):
            self.release(request_id)

    # -- queries --------------------------------------------------------------

    def provisioned_tokens(self, request_id: str) -> int:
        return self.mem[request_id].provisioned_tokens

    def lookahead_target(self, token_count: int) -> int:
        return token_count + self.config.lookahead_chunks * self.config.tokens_per_chunk
