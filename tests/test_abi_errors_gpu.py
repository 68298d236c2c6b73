"""Error behaviour of the attention C ABI on the B200 (include/vt_attention.h):
contract violations return a non-zero status (raised by the Python wrappers)
and never launch, crash or silently compute something else."""

import ctypes

import pytest
import torch

from paper_2407_15309_b200.attention import (_Geo, attn_lib, decode_attention,
                                             pack_qkv_weight, qkv_append, qkv_workspace)
from paper_2407_15309_b200.kv_layout import KVGeometry
from vt_gpu_util import admit_with_lengths, cuda_stack


def _geo(head_dim=128, q_heads=32, kv_heads=8):
    return _Geo(32, kv_heads, head_dim, q_heads, 16, 0, 2 << 20)


@pytest.mark.gpu
def test_decode_rejects_bad_geometry(cuda_ok):
    lib = attn_lib()
    dummy = torch.zeros(1 << 16, dtype=torch.bfloat16, device="cuda")
    p = dummy.data_ptr()
    for g in (_geo(head_dim=64), _geo(q_heads=30)):
        rc = lib.vt_decode_attention(ctypes.byref(g), 0, p, p, None, p, 1, 16, 1.0, p, p,
                                     1 << 20, 0, None)
        assert rc != 0
    # split not a multiple of the 16-token stage
    rc = lib.vt_decode_attention(ctypes.byref(_geo()), 0, p, p, None, p, 1, 16, 1.0, p, p,
                                 1 << 20, 24, None)
    assert rc != 0
    # workspace smaller than vt_decode_workspace_bytes
    rc = lib.vt_decode_attention(ctypes.byref(_geo()), 0, p, p, None, p, 4, 4096, 1.0, p, p,
                                 16, 0, None)
    assert rc != 0
    torch.cuda.synchronize()


@pytest.mark.gpu
def test_qkv_rejects_contract_violations(cuda_ok):
    lib = attn_lib()
    w = torch.zeros(6144, 4096, dtype=torch.bfloat16, device="cuda")
    packed = torch.empty_like(w)
    # feature count not a multiple of 128 / hidden not a multiple of 64
    assert lib.vt_qkv_pack_weight(w.data_ptr(), 6100, 4096, packed.data_ptr(), None) != 0
    assert lib.vt_qkv_pack_weight(w.data_ptr(), 6144, 4000, packed.data_ptr(), None) != 0
    # misaligned packed weight pointer
    assert lib.vt_qkv_pack_weight(w.data_ptr(), 6144, 4096, packed.data_ptr() + 2, None) != 0
    st = cuda_stack(32, 8, 32, 4096)
    kv_va, seq = admit_with_lengths(st, [17, 40])
    x = torch.zeros(2, 4096, dtype=torch.bfloat16, device="cuda")
    tok = torch.arange(2, dtype=torch.int32, device="cuda")
    pw = pack_qkv_weight(w)
    with pytest.raises(RuntimeError):  # split_k > 3 is not a supported split
        qkv_append(x, pw, tok, seq, kv_va, st.geo, 0, split_k=4)
    q = torch.empty(2, 32, 128, dtype=torch.bfloat16, device="cuda")
    geo = ctypes.byref(_geo())  # the 8B geometry of `st`
    # split 3 needs a workspace (the plain entry point has none) ...
    assert lib.vt_qkv_append(geo, 0, x.data_ptr(), pw.data.data_ptr(), 4096, 2, tok.data_ptr(),
                             seq.data_ptr(), kv_va.data_ptr(), q.data_ptr(), 3, None) != 0
    # ... and at most 64 tokens
    x80 = torch.zeros(80, 4096, dtype=torch.bfloat16, device="cuda")
    ws = qkv_workspace(st.geo)
    assert lib.vt_qkv_append_ws(geo, 0, x80.data_ptr(), pw.data.data_ptr(), 4096, 80, tok.data_ptr(),
                                seq.data_ptr(), kv_va.data_ptr(), q.data_ptr(), 3, ws.data_ptr(),
                                None) != 0
    with pytest.raises(ValueError):  # weight shape does not match the geometry
        qkv_append(x, pack_qkv_weight(torch.zeros(128 * 40, 4096, dtype=torch.bfloat16,
                                                  device="cuda")), tok, seq, kv_va, st.geo, 0)
    torch.cuda.synchronize()


@pytest.mark.gpu
def test_decode_rejects_cpu_tensors(cuda_ok):
    st = cuda_stack(32, 8, 32, 4096)
    kv_va, seq = admit_with_lengths(st, [5])
    q = torch.zeros(1, 32, 128, dtype=torch.bfloat16)
    with pytest.raises(RuntimeError):
        decode_attention(q, kv_va, seq, 0, st.geo, 5)
    geo = KVGeometry(32, 8, 128, 32, 16, 2 << 20)
    assert geo.group == 4
