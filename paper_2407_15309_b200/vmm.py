"""Layer L0: the device facade over libvtensor.so (rows a1-a6).

``VirtualMemoryDevice`` keeps the reference device's Python surface
(kvsim/device.py:118-295) so VTO, the engine adapter and the reference's own
verify scanners run unchanged on top of it, while every primitive is one call
into the C-ABI shim (include/vtensor.h). With ``cuda_ordinal`` set, the shim
also drives the CUDA driver VMM on its worker thread; the extra methods
``va``, ``ticket``, ``wait``, ``fence`` and the batched ``map_pages`` /
``unmap_tail`` are the async contract of SPEC.md:303-304.

Identity rules the tests rely on (test_device.py:109,192): the facade interns
exactly one :class:`PhysicalHandle` per chunk id and mirrors ``map_count`` on
it; ``resolve``/``unmap_page``/``live_handles`` return those same objects.
"""

from __future__ import annotations

import ctypes
import dataclasses
from collections.abc import Sequence

from . import _native as N


class DeviceError(Exception):
    """Base class for device (driver) failures."""


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


class DriverFailure(DeviceError):
    """The CUDA driver refused an op the budget had already admitted (fatal)."""


_RAISE = {
    N.VT_E_INVALID_SIZE: InvalidSize,
    N.VT_E_OUT_OF_MEMORY: DeviceOutOfMemory,
    N.VT_E_PAGE_ALREADY_MAPPED: PageAlreadyMapped,
    N.VT_E_PAGE_NOT_MAPPED: PageNotMapped,
    N.VT_E_STALE_HANDLE: StaleHandle,
    N.VT_E_INDEX_OUT_OF_RANGE: IndexOutOfRange,
    N.VT_E_RANGE_STILL_MAPPED: RangeStillMapped,
    N.VT_E_UNKNOWN_RANGE: UnknownRange,
    N.VT_E_CHUNK_STILL_MAPPED: ChunkStillMapped,
    N.VT_E_CUDA: DriverFailure,
    N.VT_E_ARG: ValueError,
}


@dataclasses.dataclass(frozen=True)
class VirtualRange:
    """A contiguous reserved span of virtual address space (ordinal base)."""

    base: int
    length_bytes: int
    page_count: int


@dataclasses.dataclass(slots=True)
class PhysicalHandle:
    """One physical chunk; shared by identity between device, pool and tables."""

    id: int
    map_count: int = 0
    # True for a chunk imported from another device's pool (export_chunk /
    # import_chunk): it maps like a local chunk but is never reused for this
    # pool's own allocations.
    imported: bool = False


@dataclasses.dataclass(frozen=True)
class DeviceStats:
    created_bytes: int
    reserved_virtual_bytes: int
    mapped_page_count: int
    free_bytes: int


@dataclasses.dataclass(frozen=True)
class DeviceCall:
    """One call-log entry (device.py:83-90)."""

    seq: int
    op: str
    detail: str
    created_bytes_after: int


@dataclasses.dataclass
class DeviceConfig:
    capacity_bytes: int
    chunk_size_bytes: int
    page_size_bytes: int = 0
    weights_bytes: int = 0
    activation_bytes_per_request: int = 0

    def __post_init__(self) -> None:
        if not self.page_size_bytes:
            self.page_size_bytes = self.chunk_size_bytes
        if self.page_size_bytes != self.chunk_size_bytes:
            raise ValueError("page size must equal chunk size")
        if self.capacity_bytes <= 0 or self.chunk_size_bytes <= 0:
            raise ValueError("capacity and chunk size must be positive")
        if not 0 <= self.weights_bytes <= self.capacity_bytes:
            raise ValueError("weights must fit in capacity")


def _detail(c: N.VtCall) -> str:
    op = c.op
    if op == 0:
        return f"base={c.base} pages={c.pages}"
    if op in (1, 5):
        return f"handle={c.handle}"
    if op in (2, 3):
        return f"base={c.base} page={c.page} handle={c.handle}"
    return f"base={c.base}"


class CallLog(Sequence):
    """Read-only list view of the shim's call log, materialised lazily.

    Entries are immutable once logged, so converted ``DeviceCall`` objects are
    cached; ``len()`` is one C call (the engine prices memory ops by call-log
    deltas, engine.py:377).
    """

    def __init__(self, dev: "VirtualMemoryDevice") -> None:
        self._dev = dev
        self._cache: list[DeviceCall] = []

    def __len__(self) -> int:
        # every primitive appends exactly one entry per processed page and
        # goes through the facade, so the length is tracked on the Python
        # side (no C call on the engine's hot "calls since" arithmetic)
        return self._dev._log_len

    def _fill(self, upto: int) -> None:
        have = len(self._cache)
        if upto <= have:
            return
        want = upto - have
        buf = (N.VtCall * want)()
        got = ctypes.c_int64()
        self._dev._lib.vt_call_log_read(self._dev._h, have, buf, want, ctypes.byref(got))
        names = N.OP_NAMES
        self._cache.extend(
            DeviceCall(c.seq, names[c.op], _detail(c), c.created_bytes_after)
            for c in buf[: got.value]
        )

    def __getitem__(self, index):
        n = len(self)
        if isinstance(index, slice):
            start, stop, step = index.indices(n)
            self._fill(max(start, stop))
            return self._cache[start:stop:step]
        if index < 0:
            index += n
        if not 0 <= index < n:
            raise IndexError("call log index out of range")
        self._fill(index + 1)
        return self._cache[index]

    def __iter__(self):
        self._fill(len(self))
        return iter(list(self._cache))

    def __eq__(self, other) -> bool:
        return list(self) == list(other)

    def __repr__(self) -> str:
        return f"CallLog({len(self)} calls)"


class VirtualMemoryDevice:
    """Driver VMM API facade: simulated (``cuda_ordinal=None``) or CUDA-backed."""

    def __init__(self, config: DeviceConfig, cuda_ordinal: int | None = None) -> None:
        self.config = config
        self._lib = N.vtensor_lib()
        self._fast = N.vtfast()
        cfg = N.VtConfig(
            config.capacity_bytes,
            config.chunk_size_bytes,
            config.weights_bytes,
            config.activation_bytes_per_request,
        )
        handle = ctypes.c_void_p()
        ordinal = -1 if cuda_ordinal is None else int(cuda_ordinal)
        rc = self._lib.vt_dev_open(ctypes.byref(cfg), ordinal, ctypes.byref(handle))
        if rc != N.VT_OK:
            raise _RAISE.get(rc, DeviceError)(
                f"vt_dev_open(ordinal={ordinal}) failed with code {rc}"
            )
        self._h = handle
        self.cuda_ordinal = cuda_ordinal
        self._interned: dict[int, PhysicalHandle] = {}
        self._ranges: dict[int, VirtualRange] = {}
        self.call_log = CallLog(self)
        self._log_len = 0
        self._i64 = ctypes.c_int64()
        self._i64b = ctypes.c_int64()
        self._hv = handle.value  # the vt_device* as an int, for the fast-call module

    # -- lifetime -------------------------------------------------------------

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._hv = 0
            self._lib.vt_dev_close(self._h)
            self._h = None

    def __del__(self) -> None:  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:
            pass

    def _raise(self, rc: int, done: int = 0):
        msg = self._lib.vt_last_error(self._h)
        exc = _RAISE.get(rc, DeviceError)(msg.decode() if msg else f"code {rc}")
        exc.done = done  # pages processed by a batched call before the failure
        raise exc

    # -- accounting -----------------------------------------------------------

    def _stats(self) -> N.VtStats:
        s = N.VtStats()
        self._lib.vt_get_stats(self._h, ctypes.byref(s))
        return s

    @property
    def created_bytes(self) -> int:
        return self._stats().created_bytes

    @property
    def reserved_virtual_bytes(self) -> int:
        return self._stats().reserved_virtual_bytes

    @property
    def activation_bytes(self) -> int:
        return self._stats().activation_bytes

    @property
    def free_bytes(self) -> int:
        return self._stats().free_bytes

    @property
    def active_requests(self) -> int:
        return self._stats().active_requests

    def set_active_requests(self, n: int) -> None:
        rc = self._lib.vt_set_active_requests(self._h, n)
        if rc:
            self._raise(rc)

    def stats(self) -> DeviceStats:
        s = self._stats()
        return DeviceStats(
            created_bytes=s.created_bytes,
            reserved_virtual_bytes=s.reserved_virtual_bytes,
            mapped_page_count=s.mapped_page_count,
            free_bytes=s.free_bytes,
        )

    # -- primitives (device.py:191-268) ---------------------------------------

    def reserve_address(self, size_bytes: int) -> VirtualRange:
        base, pages = ctypes.c_int64(), ctypes.c_int64()
        rc = self._lib.vt_reserve(self._h, size_bytes, ctypes.byref(base), ctypes.byref(pages))
        if rc:
            self._raise(rc)
        rng = VirtualRange(base=base.value, length_bytes=size_bytes, page_count=pages.value)
        self._ranges[rng.base] = rng
        self._log_len += 1
        return rng

    def create_chunk(self) -> PhysicalHandle:
        rc = self._lib.vt_create_chunk(self._h, ctypes.byref(self._i64))
        if rc:
            self._raise(rc)
        handle = PhysicalHandle(id=self._i64.value)
        self._interned[handle.id] = handle
        self._log_len += 1
        return handle

    def map_page(self, rng: VirtualRange, page_index: int, handle: PhysicalHandle) -> None:
        rc = self._lib.vt_map_page(self._h, rng.base, page_index, handle.id)
        if rc:
            self._raise(rc)
        handle.map_count += 1
        self._log_len += 1

    def map_pages(self, rng: VirtualRange, first_page: int, handles: list[PhysicalHandle]) -> None:
        """Batched ``map_page`` over consecutive slots: one shim call, same log."""
        n = len(handles)
        if n == 0:
            return
        if n == 1:
            rc = self._lib.vt_map_page(self._h, rng.base, first_page, handles[0].id)
            done = 0 if rc else 1
        else:
            ids = (ctypes.c_int64 * n)(*[h.id for h in handles])
            rc = self._lib.vt_map_pages(self._h, rng.base, first_page, ids, n,
                                        ctypes.byref(self._i64))
            done = self._i64.value
        self._log_len += done
        for h in handles[:done]:
            h.map_count += 1
        if rc:
            self._raise(rc, done)

    def extend_pages(self, rng: VirtualRange, first_page: int, reused: list[PhysicalHandle],
                     n_create: int) -> list[PhysicalHandle] | None:
        """``create_chunk`` x n_create then ``map_pages(reused + created)`` in one
        shim call (``vt_extend``; same call log). All-or-nothing: returns None,
        with nothing changed, when any precondition fails — the caller then
        runs the per-op sequence, which raises exactly as the reference does."""
        ids = self._fast.extend(self._hv, rng.base, first_page, [h.id for h in reused], n_create)
        if ids is None:
            return None
        interned = self._interned
        fresh = []
        for hid in ids:
            h = PhysicalHandle(id=hid)
            interned[hid] = h
            fresh.append(h)
        handles = reused + fresh if reused else fresh
        for h in handles:
            h.map_count += 1
        self._log_len += n_create + len(handles)
        return handles

    def unmap_page(self, rng: VirtualRange, page_index: int) -> PhysicalHandle:
        rc = self._lib.vt_unmap_page(self._h, rng.base, page_index, ctypes.byref(self._i64))
        if rc:
            self._raise(rc)
        handle = self._interned[self._i64.value]
        handle.map_count -= 1
        self._log_len += 1
        return handle

    def unmap_tail(self, rng: VirtualRange, from_page: int, down_to: int) -> list[PhysicalHandle]:
        """Batched tail-first ``unmap_page`` for pages from_page..down_to."""
        n = from_page - down_to + 1
        if n <= 0:
            return []
        rc, ids = self._fast.unmap_tail(self._hv, rng.base, from_page, down_to)
        done = len(ids)
        self._log_len += done
        interned = self._interned
        out = []
        for hid in ids:
            h = interned[hid]
            h.map_count -= 1
            out.append(h)
        if rc:
            self._raise(rc, done)
        return out

    def release_address(self, rng: VirtualRange) -> None:
        rc = self._lib.vt_release(self._h, rng.base)
        if rc:
            self._raise(rc)
        self._ranges.pop(rng.base, None)
        self._log_len += 1

    def destroy_chunk(self, handle: PhysicalHandle) -> None:
        rc = self._lib.vt_destroy_chunk(self._h, handle.id)
        if rc:
            self._raise(rc)
        self._interned.pop(handle.id, None)
        if not handle.imported:  # dropping an imported reference is not logged
            self._log_len += 1

    # -- cross-device sharing (include/vtensor.h vt_export_chunk) -------------

    def set_shareable(self, enabled: bool = True) -> None:
        """Chunks created from now on can be exported (a donor pool opts in)."""
        rc = self._lib.vt_dev_set_shareable(self._h, int(bool(enabled)))
        if rc:
            self._raise(rc)

    def export_chunk(self, handle: PhysicalHandle) -> int:
        """POSIX fd naming this chunk's physical memory (caller owns it)."""
        fd = ctypes.c_int(-1)
        rc = self._lib.vt_export_chunk(self._h, handle.id, ctypes.byref(fd))
        if rc:
            self._raise(rc)
        return fd.value

    def import_chunk(self, fd: int) -> PhysicalHandle:
        """Map-able handle of another device's chunk; consumes ``fd``."""
        rc = self._lib.vt_import_chunk(self._h, int(fd), ctypes.byref(self._i64))
        if rc:
            self._raise(rc)
        handle = PhysicalHandle(id=self._i64.value, imported=True)
        self._interned[handle.id] = handle
        return handle

    # -- inspection (device.py:272-295) ---------------------------------------

    def resolve(self, rng: VirtualRange, page_index: int) -> PhysicalHandle:
        rc = self._lib.vt_resolve(self._h, rng.base, page_index, ctypes.byref(self._i64))
        if rc:
            self._raise(rc)
        return self._interned[self._i64.value]

    def live_handles(self) -> list[PhysicalHandle]:
        n = len(self._interned)
        buf = (ctypes.c_int64 * max(n, 1))()
        self._lib.vt_live_handles(self._h, buf, n, ctypes.byref(self._i64))
        return [self._interned[buf[i]] for i in range(self._i64.value)]

    def live_ranges(self) -> list[VirtualRange]:
        n = len(self._ranges)
        bases = (ctypes.c_int64 * max(n, 1))()
        pages = (ctypes.c_int64 * max(n, 1))()
        self._lib.vt_live_ranges(self._h, bases, pages, n, ctypes.byref(self._i64))
        return [self._ranges[bases[i]] for i in range(self._i64.value)]

    def mapped_pages_of(self, rng: VirtualRange) -> dict[int, int]:
        cap = max(rng.page_count, 1)
        pages = (ctypes.c_int64 * cap)()
        ids = (ctypes.c_int64 * cap)()
        rc = self._lib.vt_range_mappings(self._h, rng.base, pages, ids, cap,
                                         ctypes.byref(self._i64))
        if rc:
            self._raise(rc)
        return {pages[i]: ids[i] for i in range(self._i64.value)}

    # -- CUDA-backend extensions (async contract) ------------

    @property
    def is_cuda(self) -> bool:
        return bool(self._lib.vt_dev_is_cuda(self._h))

    def va(self, rng: VirtualRange) -> int:
        """CUdeviceptr of the range; fixed for the range's whole life."""
        out = ctypes.c_uint64()
        rc = self._lib.vt_va(self._h, rng.base, ctypes.byref(out))
        if rc:
            self._raise(rc)
        return out.value

    def ticket(self) -> int:
        return int(self._lib.vt_ticket(self._h))

    def wait(self, ticket: int | None = None) -> None:
        """Block until every driver op up to ``ticket`` (default: all) ran."""
        t = self.ticket() if ticket is None else ticket
        rc = self._lib.vt_wait(self._h, t)
        if rc:
            self._raise(rc)

    def ready(self, ticket: int) -> bool:
        done = ctypes.c_int()
        rc = self._lib.vt_poll(self._h, ticket, ctypes.byref(done))
        if rc:
            self._raise(rc)
        return bool(done.value)

    def fence(self, stream_handle: int) -> None:
        """Later unmap/destroy/release wait for work queued on this stream."""
        rc = self._lib.vt_fence(self._h, ctypes.c_void_p(stream_handle))
        if rc:
            self._raise(rc)

    def set_async(self, enabled: bool) -> None:
        self._lib.vt_set_async(self._h, int(bool(enabled)))

    def set_driver_threads(self, threads: int) -> None:
        """Threads executing independent driver ops of a batch in parallel."""
        rc = self._lib.vt_set_driver_threads(self._h, int(threads))
        if rc:
            self._raise(rc)

    def set_phys_reserve(self, chunks: int) -> None:
        """Keep up to `chunks` pre-created physical handles (cuMemCreate off
        the extend path); purely physical, invisible to the call log and the
        byte budget. ``wait()`` returns once the reserve is full."""
        rc = self._lib.vt_set_phys_reserve(self._h, int(chunks))
        if rc:
            self._raise(rc)

    def driver_latencies(self, op: str = "map_page", reset: bool = False) -> list[int]:
        """Submit->completed latency (ns) of the driver ops of one kind, or
        (op "cuMemMap" / "cuMemSetAccess") the duration of each raw call."""
        code = {"cuMemMap": 6, "cuMemSetAccess": 7}.get(op)
        if code is None:
            code = N.OP_NAMES.index(op)
        n = ctypes.c_int64()
        self._lib.vt_driver_latencies(self._h, code, None, 0, ctypes.byref(n), 0)
        buf = (ctypes.c_int64 * max(n.value, 1))()
        self._lib.vt_driver_latencies(self._h, code, buf, n.value, ctypes.byref(n), int(reset))
        return list(buf[: n.value])

    def driver_stats(self) -> dict:
        s = N.VtDriverStats()
        self._lib.vt_driver_stats_get(self._h, ctypes.byref(s))
        return {name: getattr(s, name) for name, _ in N.VtDriverStats._fields_}
