"""ORACLE (test infrastructure only) — CPU restatement of the reference's
vTensor manager state machine (layers L0-L3 of kvsim).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module, as the checker or the timed CPU baseline; the product
(paper_2407_15309_b200) never imports it.

It restates, in one flat module and deliberately different structure from the
product (plain dicts + sorted scans, exactly the reference's cost model):
  * device VMM model  — kvsim/device.py:118-295 (ordinals never reused
    :199-201/:212-213, accounting :141-182, call log :184-187, errors :18-55)
  * vSet/pSet/rTree   — kvsim/pool.py:251-427 / :115-248
  * VTO ops + journal — kvsim/ops.py:72-303
  * VTS actions       — kvsim/scheduler.py:51-240
Parity pinned: tests/test_oracle_manager.py replays every golden stream in
tests/golden/manager_streams.json (generated from the reference itself by
tests/golden/make_manager_golden.py) through this module and requires the same
per-op state digests. It exposes the small object surface the stream driver
and dump in tests/manager_streams.py read.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass, field
from enum import Enum
from types import SimpleNamespace


# ----------------------------------------------------------------- errors --
class DeviceError(Exception):
    pass


class InvalidSize(DeviceError):
    pass


class DeviceOutOfMemory(DeviceError):
    pass


class PageAlreadyMapped(DeviceError):
    pass


class PageNotMapped(DeviceError):
    pass


class StaleHandle(DeviceError):
    pass


class IndexOutOfRange(DeviceError):
    pass


class RangeStillMapped(DeviceError):
    pass


class UnknownRange(DeviceError):
    pass


class ChunkStillMapped(DeviceError):
    pass


class PoolStateError(Exception):
    pass


class UnknownReferrer(Exception):
    pass


class CapacityExceeded(Exception):
    pass


class ExceedsMaxSeqLen(Exception):
    pass


# ----------------------------------------------------------------- config --
@dataclass
class ModelGeometry:  # config.py:38-50
    layers: int = 32
    kv_heads: int = 4
    head_dim: int = 128
    elem_bytes: int = 2

    @property
    def bytes_per_token(self) -> int:
        return 2 * self.layers * self.kv_heads * self.head_dim * self.elem_bytes


@dataclass
class SimConfig:  # config.py:53-117 (only the manager fields)
    capacity_bytes: int = 80 << 30
    chunk_size_bytes: int = 2 << 20
    weights_bytes: int = 12 << 30
    activation_bytes_per_request: int = 0
    geometry: ModelGeometry = field(default_factory=ModelGeometry)
    max_seq_len: int = 4096
    initial_alloc_tokens: int = 256
    lookahead_chunks: int = 1
    max_batch: int = 8
    prefix_cache_max_chunks: int | None = None

    def __post_init__(self):
        if self.chunk_size_bytes % self.geometry.bytes_per_token:
            raise ValueError("chunk is not a multiple of bytes_per_token")

    @property
    def bytes_per_token(self) -> int:
        return self.geometry.bytes_per_token

    @property
    def tokens_per_chunk(self) -> int:
        return self.chunk_size_bytes // self.bytes_per_token

    @property
    def pages_per_space(self) -> int:
        return -(-self.max_seq_len // self.tokens_per_chunk)


@dataclass
class DeviceConfig:
    capacity_bytes: int
    chunk_size_bytes: int
    weights_bytes: int = 0
    activation_bytes_per_request: int = 0


# ----------------------------------------------------------------- device --
@dataclass(frozen=True)
class VirtualRange:
    base: int
    length_bytes: int
    page_count: int


@dataclass
class PhysicalHandle:
    id: int
    map_count: int = 0


class VirtualMemoryDevice:
    """device.py:118-295 as one dict of ranges and one of handles."""

    def __init__(self, config: DeviceConfig):
        self.config = config
        self.r: dict[int, tuple[VirtualRange, dict[int, int]]] = {}
        self.h: dict[int, PhysicalHandle] = {}
        self.nb = self.nh = self.mapped = 0
        self.call_log: list[SimpleNamespace] = []

    @property
    def created_bytes(self):
        return len(self.h) * self.config.chunk_size_bytes

    @property
    def free_bytes(self):
        return self.config.capacity_bytes - self.config.weights_bytes - self.created_bytes

    def stats(self):
        return SimpleNamespace(created_bytes=self.created_bytes,
                               reserved_virtual_bytes=sum(v.length_bytes for v, _ in self.r.values()),
                               mapped_page_count=self.mapped, free_bytes=self.free_bytes)

    def _log(self, op, detail):
        self.call_log.append(SimpleNamespace(seq=len(self.call_log), op=op, detail=detail,
                                             created_bytes_after=self.created_bytes))

    def reserve_address(self, size):
        page = self.config.chunk_size_bytes
        if size <= 0 or size % page:
            raise InvalidSize(size)
        rng = VirtualRange(self.nb, size, size // page)
        self.nb += rng.page_count
        self.r[rng.base] = (rng, {})
        self._log("reserve_address", f"base={rng.base} pages={rng.page_count}")
        return rng

    def create_chunk(self):
        if self.free_bytes < self.config.chunk_size_bytes:
            raise DeviceOutOfMemory()
        h = PhysicalHandle(self.nh)
        self.nh += 1
        self.h[h.id] = h
        self._log("create_chunk", f"handle={h.id}")
        return h

    def map_page(self, rng, page, h):
        if rng.base not in self.r:
            raise UnknownRange(rng.base)
        if not 0 <= page < rng.page_count:
            raise IndexOutOfRange(page)
        if h.id not in self.h:
            raise StaleHandle(h.id)
        m = self.r[rng.base][1]
        if page in m:
            raise PageAlreadyMapped(page)
        m[page] = h.id
        h.map_count += 1
        self.mapped += 1
        self._log("map_page", f"base={rng.base} page={page} handle={h.id}")

    def unmap_page(self, rng, page):
        if rng.base not in self.r:
            raise UnknownRange(rng.base)
        m = self.r[rng.base][1]
        if page not in m:
            raise PageNotMapped(page)
        h = self.h[m.pop(page)]
        h.map_count -= 1
        self.mapped -= 1
        self._log("unmap_page", f"base={rng.base} page={page} handle={h.id}")
        return h

    def release_address(self, rng):
        if rng.base not in self.r:
            raise UnknownRange(rng.base)
        if self.r[rng.base][1]:
            raise RangeStillMapped(rng.base)
        del self.r[rng.base]
        self._log("release_address", f"base={rng.base}")

    def destroy_chunk(self, h):
        if h.id not in self.h:
            raise StaleHandle(h.id)
        if h.map_count:
            raise ChunkStillMapped(h.id)
        del self.h[h.id]
        self._log("destroy_chunk", f"handle={h.id}")


# ------------------------------------------------------------------- pool --
class SpaceState(Enum):
    AVAILABLE = "available"
    IN_USE = "in_use"


class ChunkState(Enum):
    FREE = "free"
    ACTIVE = "active"


@dataclass
class VirtualSpace:
    rng: VirtualRange
    page_table: list = field(default_factory=list)
    mapped_pages: int = 0
    state: SpaceState = SpaceState.AVAILABLE
    owner: str | None = None
    recorded: bool = False

    def __post_init__(self):
        self.page_table = self.page_table or [None] * self.rng.page_count

    @property
    def space_id(self):
        return self.rng.base

    @property
    def page_count(self):
        return self.rng.page_count


@dataclass
class PhysicalEntry:
    handle: PhysicalHandle
    state: ChunkState = ChunkState.ACTIVE
    referrers: set = field(default_factory=set)
    tokens_stored: int = 0
    cls: str = "request"


@dataclass
class VirtualTensor:
    space: VirtualSpace
    tokens: list
    token_count: int = 0
    capacity_tokens: int = 0
    owner: str | None = None


class _Node:
    def __init__(self, key, parent=None):
        self.key, self.parent, self.children, self.record, self.last_touch = key, parent, {}, None, 0


class PrefixTree:
    """pool.py:115-248 — chunk-wise slice compares, as in the reference."""

    def __init__(self, tpc):
        self.tpc, self.root, self.clock = tpc, _Node(()), itertools.count(1)

    def _cm(self, a, b):
        n, t = 0, self.tpc
        for i in range(0, min(len(a), len(b)) // t * t, t):
            if a[i:i + t] != b[i:i + t]:
                break
            n = i + t
        return n

    def insert(self, key, vt):
        node, rest = self.root, key
        while True:
            child = node.children.get(rest[:self.tpc])
            if child is None:
                leaf = _Node(rest, node)
                leaf.record, leaf.last_touch = vt, next(self.clock)
                node.children[rest[:self.tpc]] = leaf
                return []
            m = self._cm(child.key, rest)
            if m < len(child.key):
                up = _Node(child.key[:m], node)
                node.children[rest[:self.tpc]] = up
                child.key, child.parent = child.key[m:], up
                up.children[child.key[:self.tpc]] = child
                node = up
            else:
                node = child
            rest = rest[m:]
            if not rest:
                out = [node.record] if node.record is not None and node.record is not vt else []
                node.record, node.last_touch = vt, next(self.clock)
                return out

    def match(self, tokens):
        node, n = self.root, 0
        while True:
            child = node.children.get(tokens[n:][:self.tpc])
            if child is None:
                break
            m = self._cm(child.key, tokens[n:])
            n += m
            node = child
            if m < len(child.key):
                break
        if n == 0 or node is self.root:
            return None
        while node.record is None:
            if not node.children:
                return None
            node = node.children[min(node.children)]
        node.last_touch = next(self.clock)
        return node.record, n

    def remove(self, node):
        node.record = None
        while node is not self.root and node.record is None and not node.children:
            del node.parent.children[node.key[:self.tpc]]
            node = node.parent

    def records(self):
        out, st = [], [self.root]
        while st:
            x = st.pop()
            if x.record is not None:
                out.append((x, x.record))
            st.extend(x.children[k] for k in sorted(x.children))
        return out

    def recorded_sequences(self):
        out = []

        def walk(x, pre):
            full = pre + x.key
            if x.record is not None:
                out.append(full)
            for k in sorted(x.children):
                walk(x.children[k], full)

        walk(self.root, ())
        return out


class TensorPool:
    """pool.py:251-427 with the reference's sorted scans."""

    def __init__(self, tpc):
        self.tokens_per_chunk = tpc
        self.spaces, self.entries, self.avail, self.free = {}, {}, set(), set()
        self.tree = PrefixTree(tpc)
        self.n_request = self.n_pinned = self.n_free = self.used_tokens = 0

    def _cls(self, e):
        if e.state is ChunkState.FREE:
            return "free"
        ok = e.referrers and all(self.spaces.get(s) is not None and self.spaces[s].recorded
                                 for s in e.referrers)
        return "pinned" if ok else "request"

    def _re(self, e):
        new = self._cls(e)
        if new == e.cls:
            return
        for c, sign in ((e.cls, -1), (new, +1)):
            if c == "free":
                self.n_free += sign
            elif c == "pinned":
                self.n_pinned += sign
            else:
                self.n_request += sign
                self.used_tokens += sign * e.tokens_stored
        e.cls = new

    def set_space_recorded(self, sp, flag):
        sp.recorded = flag
        for p in range(sp.mapped_pages):
            if sp.page_table[p] is not None:
                self._re(self.entries[sp.page_table[p].id])

    def add_space(self, sp):
        self.spaces[sp.space_id] = sp
        if sp.state is SpaceState.AVAILABLE:
            self.avail.add(sp.space_id)

    def acquire_space(self, pages):
        for sid in sorted(self.avail):
            if self.spaces[sid].page_count >= pages:
                self.avail.discard(sid)
                self.spaces[sid].state = SpaceState.IN_USE
                return self.spaces[sid]
        return None

    def return_space(self, sp):
        if sp.mapped_pages:
            raise PoolStateError()
        sp.state, sp.owner, sp.recorded = SpaceState.AVAILABLE, None, False
        self.avail.add(sp.space_id)

    def drop_space(self, sp):
        self.avail.discard(sp.space_id)
        del self.spaces[sp.space_id]

    def available_spaces(self):
        return [self.spaces[s] for s in sorted(self.avail)]

    def add_entry(self, h):
        self.entries[h.id] = PhysicalEntry(h)
        self.n_request += 1

    def take_free(self, n):
        out = []
        for hid in sorted(self.free):
            if len(out) == n:
                break
            e = self.entries[hid]
            self.free.discard(hid)
            e.state = ChunkState.ACTIVE
            self._re(e)
            out.append(e.handle)
        return out

    def _park(self, e):
        e.state = ChunkState.FREE
        self._re(e)
        e.tokens_stored = 0
        self.free.add(e.handle.id)

    def incref(self, h, sid):
        e = self.entries[h.id]
        if sid in e.referrers:
            raise PoolStateError()
        e.referrers.add(sid)
        e.state = ChunkState.ACTIVE
        self.free.discard(h.id)
        self._re(e)

    def decref(self, h, sid):
        e = self.entries[h.id]
        if sid not in e.referrers:
            raise UnknownReferrer()
        e.referrers.discard(sid)
        if e.referrers:
            self._re(e)
        else:
            self._park(e)

    def note_stored(self, h, n):
        e = self.entries[h.id]
        if n > e.tokens_stored:
            if e.cls == "request":
                self.used_tokens += n - e.tokens_stored
            e.tokens_stored = n

    def drop_entry(self, h):
        self.free.discard(h.id)
        self.n_free -= 1
        del self.entries[h.id]

    def free_handles(self):
        return [self.entries[i].handle for i in sorted(self.free)]


# -------------------------------------------------------------------- VTO --
class VTensorOps:
    """ops.py:72-303; each op journals its slice of the call log (ops.py:37-69)."""

    def __init__(self, device, pool, config):
        self.device, self.pool, self.config, self.journal = device, pool, config, []

    def _j(self, name, start, detail):
        self.journal.append(SimpleNamespace(name=name, call_start=start,
                                            call_end=len(self.device.call_log), detail=detail))

    def p_alloc(self, n):
        start, reused, made = len(self.device.call_log), self.pool.take_free(n), []
        try:
            while len(reused) + len(made) < n:
                h = self.device.create_chunk()
                self.pool.add_entry(h)
                made.append(h)
        except DeviceOutOfMemory:
            for h in made:
                self.pool._park(self.pool.entries[h.id])
                self.pool.drop_entry(h)
                self.device.destroy_chunk(h)
            for h in reused:
                self.pool._park(self.pool.entries[h.id])
            self._j("p_alloc", start, {"requested": n, "failed": True})
            raise
        self._j("p_alloc", start, {"requested": n, "reused": len(reused), "created": len(made)})
        return reused + made

    def v_alloc(self, size):
        start, pages = len(self.device.call_log), self.config.pages_per_space
        sp = self.pool.acquire_space(pages)
        if sp is not None:
            self._j("v_alloc", start, {"reused": True, "space": sp.space_id})
            return sp
        sp = VirtualSpace(self.device.reserve_address(pages * self.config.chunk_size_bytes),
                          state=SpaceState.IN_USE)
        self.pool.add_space(sp)
        self._j("v_alloc", start, {"reused": False, "space": sp.space_id})
        return sp

    def map_chunks(self, sp, hs):
        if sp.mapped_pages + len(hs) > sp.page_count:
            raise CapacityExceeded()
        start = len(self.device.call_log)
        for h in hs:
            p = sp.mapped_pages
            self.device.map_page(sp.rng, p, h)
            self.pool.incref(h, sp.space_id)
            sp.page_table[p] = h
            sp.mapped_pages += 1
        self._j("map", start, {"space": sp.space_id, "chunks": len(hs)})

    def _tail(self, sp, keep):
        for p in range(sp.mapped_pages - 1, keep - 1, -1):
            h = sp.page_table[p]
            self.device.unmap_page(sp.rng, p)
            self.pool.decref(h, sp.space_id)
            sp.page_table[p] = None
        sp.mapped_pages = min(sp.mapped_pages, keep)

    def unmap_space(self, sp):
        start = len(self.device.call_log)
        if sp.state is SpaceState.AVAILABLE or sp.recorded:
            self._j("unmap_space", start, {"space": sp.space_id, "noop": True})
            return
        self._tail(sp, 0)
        self.pool.return_space(sp)
        self._j("unmap_space", start, {"space": sp.space_id})

    def empty_memory(self, evict_prefix=False):
        start, rep = len(self.device.call_log), SimpleNamespace(
            chunks_destroyed=0, spaces_released=0, records_evicted=0)
        if evict_prefix:
            for node, vt in self.pool.tree.records():
                self.pool.tree.remove(node)
                self._unpin(vt)
                rep.records_evicted += 1
        for h in self.pool.free_handles():
            self.pool.drop_entry(h)
            self.device.destroy_chunk(h)
            rep.chunks_destroyed += 1
        for sp in self.pool.available_spaces():
            self.pool.drop_space(sp)
            self.device.release_address(sp.rng)
            rep.spaces_released += 1
        self._j("empty_memory", start, {"evict_prefix": evict_prefix,
                                         "chunks": rep.chunks_destroyed,
                                         "spaces": rep.spaces_released})
        return rep

    def r_push(self, vt):
        tpc = self.config.tokens_per_chunk
        aligned = vt.token_count // tpc * tpc
        if aligned < tpc or vt.space.recorded:
            return False
        start, key = len(self.device.call_log), tuple(vt.tokens[:aligned])
        self._tail(vt.space, aligned // tpc)
        vt.tokens, vt.token_count = list(key), aligned
        self.pool.set_space_recorded(vt.space, True)
        vt.space.owner = None
        for old in self.pool.tree.insert(key, vt):
            self._unpin(old)
        self._cap(vt)
        self._j("r_push", start, {"space": vt.space.space_id, "tokens": aligned})
        return True

    def r_prefix_match(self, tokens):
        return self.pool.tree.match(tuple(tokens))

    def _unpin(self, vt):
        self.pool.set_space_recorded(vt.space, False)
        if vt.space.state is SpaceState.IN_USE:
            self._tail(vt.space, 0)
            self.pool.return_space(vt.space)

    def _cap(self, keep):
        cap, tpc = self.config.prefix_cache_max_chunks, self.config.tokens_per_chunk
        if cap is None:
            return

        def flen(x):
            n = 0
            while x is not None:
                n, x = n + len(x.key), x.parent
            return n

        while sum(flen(n) for n, _ in self.pool.tree.records()) // tpc > cap:
            victims = [(n.last_touch, n) for n, v in self.pool.tree.records() if v is not keep]
            if not victims:
                return
            _, node = min(victims, key=lambda t: t[0])
            vt = node.record
            self.pool.tree.remove(node)
            self._unpin(vt)


# -------------------------------------------------------------------- VTS --
@dataclass
class AdmitStats:
    shared_tokens: int = 0
    chunks_reused: int = 0
    chunks_created: int = 0
    donor_space: int | None = None
    identity_ok: bool = True


class VTensorScheduler:
    """scheduler.py:51-240."""

    def __init__(self, ops):
        self.ops, self.config, self.mem = ops, ops.config, {}

    def _counts(self, mark):
        r = c = 0
        for rec in self.ops.journal[mark:]:
            if rec.name == "p_alloc" and not rec.detail.get("failed"):
                r += rec.detail.get("reused", 0)
                c += rec.detail.get("created", 0)
        return r, c

    def _new(self, rid, sp, tokens, shared):
        tpc = self.config.tokens_per_chunk
        sp.owner = rid
        vt = VirtualTensor(sp, list(tokens), 0, sp.page_count * tpc, rid)
        self.mem[rid] = SimpleNamespace(vt=vt, shared_prefix_tokens=shared)
        return self.mem[rid]

    def create(self, rid, tokens):
        if len(tokens) > self.config.max_seq_len:
            raise ExceedsMaxSeqLen()
        tpc, mark = self.config.tokens_per_chunk, len(self.ops.journal)
        sp = self.ops.v_alloc(self.config.max_seq_len)
        try:
            hs = self.ops.p_alloc(-(-max(len(tokens), self.config.initial_alloc_tokens) // tpc))
        except DeviceOutOfMemory:
            self.ops.unmap_space(sp)
            raise
        self.ops.map_chunks(sp, hs)
        rm = self._new(rid, sp, tokens, 0)
        r, c = self._counts(mark)
        return rm, AdmitStats(chunks_reused=r, chunks_created=c)

    def prefix_match(self, rid, tokens):
        if len(tokens) > self.config.max_seq_len:
            raise ExceedsMaxSeqLen()
        hit = self.ops.r_prefix_match(tokens)
        if hit is None:
            return None
        donor, matched = hit
        tpc, mark = self.config.tokens_per_chunk, len(self.ops.journal)
        shared = matched // tpc
        sp = self.ops.v_alloc(self.config.max_seq_len)
        table = [donor.space.page_table[p] for p in range(shared)]
        try:
            self.ops.map_chunks(sp, table)
            deficit = -(-len(tokens) // tpc) - shared
            if deficit > 0:
                self.ops.map_chunks(sp, self.ops.p_alloc(deficit))
        except DeviceOutOfMemory:
            self.ops.unmap_space(sp)
            raise
        rm = self._new(rid, sp, tokens, matched)
        self._stored(rm, matched)
        rm.vt.token_count = matched
        r, c = self._counts(mark)
        ok = all(sp.page_table[p] is donor.space.page_table[p] for p in range(shared))
        return rm, AdmitStats(matched, r, c, donor.space.space_id, ok)

    def extend(self, rid, target):
        if target > self.config.max_seq_len:
            raise ExceedsMaxSeqLen()
        sp = self.mem[rid].vt.space
        deficit = -(-target // self.config.tokens_per_chunk) - sp.mapped_pages
        if deficit <= 0:
            return 0
        self.ops.map_chunks(sp, self.ops.p_alloc(deficit))
        return deficit

    def mark_prefilled(self, rid):
        rm = self.mem[rid]
        self._stored(rm, len(rm.vt.tokens))
        rm.vt.token_count = len(rm.vt.tokens)

    def append_token(self, rid, tok):
        rm = self.mem[rid]
        rm.vt.tokens.append(tok)
        rm.vt.token_count += 1
        self._stored(rm, rm.vt.token_count)

    def _stored(self, rm, n):
        tpc = self.config.tokens_per_chunk
        if n <= 0:
            return
        first = max(0, (rm.vt.token_count - 1) // tpc) if rm.vt.token_count else 0
        for p in range(first, (n - 1) // tpc + 1):
            self.ops.pool.note_stored(rm.vt.space.page_table[p], min(tpc, n - p * tpc))

    def prefix_record(self, rid):
        rm = self.mem.get(rid)
        if rm is None or not self.ops.r_push(rm.vt):
            return False
        del self.mem[rid]
        return True

    def release(self, rid):
        rm = self.mem.pop(rid, None)
        if rm is not None:
            self.ops.unmap_space(rm.vt.space)

    def release_all(self):
        for rid in sorted(self.mem):
            self.release(rid)

    def lookahead_target(self, n):
        return n + self.config.lookahead_chunks * self.config.tokens_per_chunk
