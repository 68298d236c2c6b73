"""The C-ABI libraries load on a CPU-only host and export every symbol their
public headers declare (no compute calls: there is no GPU here)."""

import ctypes
import os
import re

import pytest

from conftest import REPO

PKG = os.path.join(REPO, "paper_2407_15309_b200")
HEADERS = {
    "vtensor.h": "libvtensor.so",
    "vt_attention.h": "libvtattn.so",
}


def declared(header: str) -> list[str]:
    text = open(os.path.join(REPO, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*[A-Za-z_][\w\s\*]*?\b(vt_\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


@pytest.mark.parametrize("header,lib", list(HEADERS.items()))
def test_library_exports_every_declared_symbol(header, lib):
    names = declared(header)
    assert len(names) >= 5, names
    so = ctypes.CDLL(os.path.join(PKG, lib))
    missing = [n for n in names if not hasattr(so, n)]
    assert not missing, f"{lib} lacks {missing}"


def test_python_bindings_cover_the_headers():
    from paper_2407_15309_b200 import _native
    from paper_2407_15309_b200.attention import ATTN_SYMBOLS

    assert set(declared("vtensor.h")) == set(_native.VTENSOR_SYMBOLS)
    assert set(declared("vt_attention.h")) == set(ATTN_SYMBOLS)


def test_cuda_backend_fails_loudly_without_a_driver():
    """No libcuda here: opening a CUDA-backed device must raise, never fall
    back to the simulated backend."""
    import paper_2407_15309_b200 as vt

    if os.path.exists("/dev/nvidia0"):
        pytest.skip("GPU present")
    with pytest.raises(vt.DeviceError):
        vt.VirtualMemoryDevice(vt.DeviceConfig(1 << 30, 2 << 20), cuda_ordinal=0)


def test_attention_rejects_cpu_tensors():
    import torch

    from paper_2407_15309_b200.attention import _need_cuda

    with pytest.raises(RuntimeError):
        _need_cuda(torch.zeros(4))


def test_fused_extend_is_all_or_nothing_and_logs_like_the_two_ops():
    """vt_extend (one scheduler extend = p_alloc creates + map_chunks maps in
    one shim call): the call log equals create_chunk x n then map_page per
    page, and a rejected call (budget, occupied page) changes nothing."""
    import paper_2407_15309_b200 as vt

    dev = vt.VirtualMemoryDevice(vt.DeviceConfig(capacity_bytes=8 << 21, chunk_size_bytes=2 << 20))
    rng = dev.reserve_address(6 << 21)
    parked = dev.create_chunk()
    got = dev.extend_pages(rng, 0, [parked], 2)
    assert [h.id for h in got] == [parked.id, parked.id + 1, parked.id + 2]
    assert [c.op for c in dev.call_log] == ["reserve_address", "create_chunk", "create_chunk",
                                            "create_chunk", "map_page", "map_page", "map_page"]
    assert all(h.map_count == 1 for h in got)
    n = len(dev.call_log)
    stats = dev.stats()
    assert dev.extend_pages(rng, 2, [], 1) is None  # page 2 is mapped
    assert dev.extend_pages(rng, 3, [], 6) is None  # over the 8-chunk budget
    assert dev.extend_pages(rng, 5, [], 2) is None  # past the range's 6 pages
    assert len(dev.call_log) == n and dev._lib.vt_call_log_len(dev._h) == n
    assert dev.stats() == stats
    assert [h.id for h in dev.extend_pages(rng, 3, [], 3)] == [parked.id + 3, parked.id + 4,
                                                                parked.id + 5]
