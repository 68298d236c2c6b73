"""ctypes bindings to the in-tree native libraries (declared in include/*.h).

``libvtensor.so`` is the C-ABI VMM shim (include/vtensor.h) and
``libvtattn.so`` holds the sm_100a attention kernels (include/vt_attention.h).
Both are built in-tree by ``__graft_entry__.build()``; there is no fallback:
if a library is missing the import fails loudly.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_int, c_int32, c_int64, c_uint32, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))

VT_OK = 0
VT_E_INVALID_SIZE = 1
VT_E_OUT_OF_MEMORY = 2
VT_E_PAGE_ALREADY_MAPPED = 3
VT_E_PAGE_NOT_MAPPED = 4
VT_E_STALE_HANDLE = 5
VT_E_INDEX_OUT_OF_RANGE = 6
VT_E_RANGE_STILL_MAPPED = 7
VT_E_UNKNOWN_RANGE = 8
VT_E_CHUNK_STILL_MAPPED = 9
VT_E_CUDA = 10
VT_E_ARG = 11

OP_NAMES = (
    "reserve_address",
    "create_chunk",
    "map_page",
    "unmap_page",
    "release_address",
    "destroy_chunk",
)


class VtConfig(ctypes.Structure):
    _fields_ = [
        ("capacity_bytes", c_int64),
        ("chunk_bytes", c_int64),
        ("weights_bytes", c_int64),
        ("activation_bytes_per_request", c_int64),
    ]


class VtStats(ctypes.Structure):
    _fields_ = [
        ("created_bytes", c_int64),
        ("reserved_virtual_bytes", c_int64),
        ("mapped_page_count", c_int64),
        ("free_bytes", c_int64),
        ("activation_bytes", c_int64),
        ("active_requests", c_int64),
        ("live_handles", c_int64),
        ("live_ranges", c_int64),
    ]


class VtCall(ctypes.Structure):
    _fields_ = [
        ("seq", c_int64),
        ("op", c_int32),
        ("_pad", c_int32),
        ("base", c_int64),
        ("page", c_int64),
        ("handle", c_int64),
        ("pages", c_int64),
        ("created_bytes_after", c_int64),
    ]


class VtDriverStats(ctypes.Structure):
    _fields_ = [
        ("ops_completed", c_int64),
        ("map_calls", c_int64),
        ("unmap_calls", c_int64),
        ("create_calls", c_int64),
        ("destroy_calls", c_int64),
        ("access_calls", c_int64),
        ("map_ns_total", c_int64),
        ("unmap_ns_total", c_int64),
        ("create_ns_total", c_int64),
        ("destroy_ns_total", c_int64),
        ("access_ns_total", c_int64),
        ("fence_waits", c_int64),
        ("fence_wait_ns_total", c_int64),
        ("max_op_ns", c_int64),
        ("reserve_hits", c_int64),
        ("reserve_chunks", c_int64),
        ("driver_threads", c_int64),
    ]


def _load(name: str) -> ctypes.CDLL:
    path = os.path.join(_HERE, name)
    # A/B experiments only (tools/): load a variant build of the same library
    override = os.environ.get("VT_LIB_" + name.split(".")[0].upper())
    if override:
        path = override
    if not os.path.exists(path):
        raise ImportError(
            f"{name} is not built ({path} missing); run __graft_entry__.build() "
            "— there is no CPU or Python fallback for the native path"
        )
    return ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)


_vt = None


def vtensor_lib() -> ctypes.CDLL:
    """libvtensor.so with argtypes declared (mirrors include/vtensor.h)."""
    global _vt
    if _vt is not None:
        return _vt
    lib = _load("libvtensor.so")
    P64 = POINTER(c_int64)
    sig = {
        "vt_dev_open": (c_int, [POINTER(VtConfig), c_int, POINTER(c_void_p)]),
        "vt_dev_close": (c_int, [c_void_p]),
        "vt_dev_is_cuda": (c_int, [c_void_p]),
        "vt_last_error": (ctypes.c_char_p, [c_void_p]),
        "vt_reserve": (c_int, [c_void_p, c_int64, P64, P64]),
        "vt_create_chunk": (c_int, [c_void_p, P64]),
        "vt_map_page": (c_int, [c_void_p, c_int64, c_int64, c_int64]),
        "vt_unmap_page": (c_int, [c_void_p, c_int64, c_int64, P64]),
        "vt_release": (c_int, [c_void_p, c_int64]),
        "vt_destroy_chunk": (c_int, [c_void_p, c_int64]),
        "vt_dev_set_shareable": (c_int, [c_void_p, c_int]),
        "vt_export_chunk": (c_int, [c_void_p, c_int64, POINTER(c_int)]),
        "vt_import_chunk": (c_int, [c_void_p, c_int, P64]),
        "vt_chunk_is_imported": (c_int, [c_void_p, c_int64]),
        "vt_map_pages": (c_int, [c_void_p, c_int64, c_int64, P64, c_int64, P64]),
        "vt_unmap_tail": (c_int, [c_void_p, c_int64, c_int64, c_int64, P64, P64]),
        "vt_extend": (c_int, [c_void_p, c_int64, c_int64, P64, c_int64, c_int64, P64]),
        "vt_set_active_requests": (c_int, [c_void_p, c_int64]),
        "vt_get_stats": (c_int, [c_void_p, POINTER(VtStats)]),
        "vt_resolve": (c_int, [c_void_p, c_int64, c_int64, P64]),
        "vt_handle_alive": (c_int, [c_void_p, c_int64, P64]),
        "vt_live_handles": (c_int, [c_void_p, P64, c_int64, P64]),
        "vt_live_ranges": (c_int, [c_void_p, P64, P64, c_int64, P64]),
        "vt_range_mappings": (c_int, [c_void_p, c_int64, P64, P64, c_int64, P64]),
        "vt_call_log_len": (c_int64, [c_void_p]),
        "vt_call_log_read": (c_int, [c_void_p, c_int64, POINTER(VtCall), c_int64, P64]),
        "vt_ticket": (c_uint64, [c_void_p]),
        "vt_wait": (c_int, [c_void_p, c_uint64]),
        "vt_poll": (c_int, [c_void_p, c_uint64, POINTER(c_int)]),
        "vt_fence": (c_int, [c_void_p, c_void_p]),
        "vt_set_async": (c_int, [c_void_p, c_int]),
        "vt_set_driver_threads": (c_int, [c_void_p, c_int]),
        "vt_set_phys_reserve": (c_int, [c_void_p, c_int64]),
        "vt_driver_stats_get": (c_int, [c_void_p, POINTER(VtDriverStats)]),
        "vt_driver_latencies": (c_int, [c_void_p, c_int32, P64, c_int64, P64, c_int]),
        "vt_va": (c_int, [c_void_p, c_int64, POINTER(c_uint64)]),
        "vt_encode_tensor_map": (
            c_int,
            [c_void_p, c_uint64, c_int, POINTER(c_uint64), POINTER(c_uint64),
             POINTER(c_uint32), c_int, c_void_p],
        ),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _vt = lib
    return lib


def vtfast():
    """The CPython fast-call module for the manager's hot shim calls
    (csrc/vt_pyfast.c); its symbols bind to the libvtensor.so loaded above."""
    vtensor_lib()
    from . import _vtfast

    return _vtfast


VTENSOR_SYMBOLS = (
    "vt_dev_open", "vt_dev_close", "vt_dev_is_cuda", "vt_last_error",
    "vt_reserve", "vt_create_chunk", "vt_map_page", "vt_unmap_page",
    "vt_release", "vt_destroy_chunk", "vt_map_pages", "vt_unmap_tail", "vt_extend",
    "vt_set_active_requests", "vt_get_stats", "vt_resolve", "vt_handle_alive",
    "vt_live_handles", "vt_live_ranges", "vt_range_mappings",
    "vt_call_log_len", "vt_call_log_read", "vt_ticket", "vt_wait", "vt_poll",
    "vt_fence", "vt_set_async", "vt_set_driver_threads", "vt_set_phys_reserve", "vt_driver_stats_get", "vt_driver_latencies", "vt_va",
    "vt_encode_tensor_map", "vt_dev_set_shareable", "vt_export_chunk", "vt_import_chunk", "vt_chunk_is_imported",
)
