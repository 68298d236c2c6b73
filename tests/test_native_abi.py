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
