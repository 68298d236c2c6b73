"""Cross-device prefix sharing.

The reference shares a recorded prefix inside one pool by hard link: the
borrower's space maps the donor's chunk handles (kvsim/scheduler.py:104-162,
identity at :128-130). With one pool per GPU (request partition, §8(e)) a
conversation whose prefix was recorded on GPU A could only be reused on A.
Here the donor exports the matched chunks' physical memory as POSIX file
descriptors (cuMemExportToShareableHandle) and the borrower — another
manager, in this process or another one (fds travel over a Unix socket with
SCM_RIGHTS) — imports them (cuMemImportFromShareableHandle) and maps them
into its own VA by identity, exactly like a local hard link. On a different
GPU the mapping's cuMemSetAccess grants peer access over NVLink 5, so the
prefill kernel reads the shared prefix in place through the borrower's VA;
nothing is copied.

A donor pool opts in with ``device.set_shareable(True)`` before it creates
the chunks it may share (shareable allocations cost more per cuMemCreate, so
it is off by default).

Lifetime: the CUDA allocation lives until every device has released its
handle, so a donor may evict its record while borrowers still read it.
Imported chunks are outside the borrower's budget (created_bytes) and are
never parked in its free list; when the last borrowing space unmaps them the
borrower drops its reference (vto.VTensorOps._reap_imports).
"""

from __future__ import annotations

import array
import dataclasses
import json
import socket

from .vmm import DeviceOutOfMemory
from .vts import AdmitStats, RequestMem, VTensorScheduler, _ceil_div


@dataclasses.dataclass
class SharedPrefix:
    """What a donor hands to a borrower: the matched token count and one fd per
    shared chunk (page order), plus the geometry both sides must agree on."""

    matched_tokens: int
    fds: list[int]
    tokens_per_chunk: int
    chunk_bytes: int

    def close(self) -> None:
        import os

        for fd in self.fds:
            os.close(fd)
        self.fds = []


def export_prefix(sched: VTensorScheduler, tokens: list[int]) -> SharedPrefix | None:
    """Donor side: rTree match of ``tokens`` (touches the record's LRU clock
    like any match) and an exported fd for each chunk of the matched prefix."""
    hit = sched.ops.r_prefix_match(tokens)
    if hit is None:
        return None
    donor, matched = hit
    cfg = sched.config
    pages = matched // cfg.tokens_per_chunk
    dev = sched.ops.device
    fds = [dev.export_chunk(h) for h in donor.space.page_table[:pages]]
    return SharedPrefix(matched, fds, cfg.tokens_per_chunk, cfg.chunk_size_bytes)


def import_prefix(sched: VTensorScheduler, request_id: str, tokens: list[int],
                  shared: SharedPrefix) -> tuple[RequestMem, AdmitStats]:
    """Borrower side of a prefix hit (scheduler.py:104-162 with the donor in
    another pool): import the shared chunks, map them by identity at the head
    of a fresh space, provision ``ceil(len/tpc) - shared`` local chunks (no
    initial_alloc floor, as in the reference's prefix hit) and start the
    request at ``matched`` tokens. Consumes ``shared.fds``."""
    cfg = sched.config
    if shared.tokens_per_chunk != cfg.tokens_per_chunk or shared.chunk_bytes != cfg.chunk_size_bytes:
        raise ValueError("donor and borrower geometries differ")
    sched._check_new(request_id, tokens)
    ops = sched.ops
    tpc = cfg.tokens_per_chunk
    matched = shared.matched_tokens
    if matched > len(tokens) or matched % tpc:
        raise ValueError("shared prefix must be chunk-aligned and within the prompt")
    handles = [ops.device.import_chunk(fd) for fd in shared.fds]
    shared.fds = []
    for h in handles:
        ops.pool.add_entry(h)
    mark = len(ops.journal)
    space = ops.v_alloc(cfg.max_seq_len)
    try:
        ops.map_chunks(space, handles)
        deficit = _ceil_div(len(tokens), tpc) - len(handles)
        if deficit > 0:
            ops.map_chunks(space, ops.p_alloc(deficit))
    except DeviceOutOfMemory:
        ops.unmap_space(space)
        raise
    rm = sched._register(request_id, space, tokens, matched)
    sched._advance_stored(rm, matched)  # the donor's KV is already materialised
    rm.vt.token_count = matched
    reused, created = sched._alloc_counts(mark)
    table = space.page_table
    return rm, AdmitStats(shared_tokens=matched, chunks_reused=reused, chunks_created=created,
                          donor_space=None,
                          identity_ok=all(table[p] is handles[p] for p in range(len(handles))))


def send_shared_prefix(sock: socket.socket, shared: SharedPrefix) -> None:
    """Send to another process over a Unix socket (fds via SCM_RIGHTS); the
    local fds are closed afterwards (the receiver owns duplicates)."""
    header = json.dumps({"matched_tokens": shared.matched_tokens, "n": len(shared.fds),
                         "tokens_per_chunk": shared.tokens_per_chunk,
                         "chunk_bytes": shared.chunk_bytes}).encode()
    sock.sendall(len(header).to_bytes(4, "little") + header)
    for i in range(0, len(shared.fds), 200):  # stay under SCM_MAX_FD (253)
        batch = shared.fds[i:i + 200]
        socket.send_fds(sock, [len(batch).to_bytes(4, "little")], batch)
    shared.close()


def recv_shared_prefix(sock: socket.socket) -> SharedPrefix:
    n = int.from_bytes(_recv_exact(sock, 4), "little")
    meta = json.loads(_recv_exact(sock, n))
    fds: list[int] = []
    while len(fds) < meta["n"]:
        msg, got, _, _ = socket.recv_fds(sock, 4, 200)
        fds.extend(got)
    return SharedPrefix(meta["matched_tokens"], fds, meta["tokens_per_chunk"], meta["chunk_bytes"])


def _recv_exact(sock: socket.socket, n: int) -> bytes:
    buf = b""
    while len(buf) < n:
        part = sock.recv(n - len(buf))
        if not part:
            raise ConnectionError("peer closed")
        buf += part
    return buf
