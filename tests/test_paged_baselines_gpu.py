"""The paper's paged-KV comparison kernels (flashinfer trtllm-gen, vLLM
PagedAttention v2; tests/paged_libs.py) oracle-checked on the same KV bytes
as the vTensor kernels (the paged side must be checked against
the oracle itself, not only against this package's own paged variant)."""

import pytest
import torch

from oracle.attention_ref import decode_attention_ref, rel_err
from paged_libs import BUILDERS, gather_pages
from paper_2407_15309_b200.attention import decode_attention, kv_tensor_maps
from vt_gpu_util import admit_with_lengths, cuda_stack, gather


@pytest.mark.gpu
@pytest.mark.parametrize("lib", list(BUILDERS))
def test_paged_library_decode_matches_oracle(cuda_ok, lib):
    lens = [1, 15, 16, 17, 300, 1000, 2049, 4096]
    st = cuda_stack(32, 8, 32, 4352)
    kv_va, seq = admit_with_lengths(st, lens, seed=31)
    layer = 13
    K, V, table = gather_pages(st, kv_va, lens, layer)
    q = torch.randn(len(lens), 32, 128, device="cuda").to(torch.bfloat16)
    try:
        run = BUILDERS[lib](K, V, table, lens, 32)
        out = run(q, torch.empty_like(q))
        torch.cuda.synchronize()
    except (ImportError, OSError, RuntimeError) as exc:  # library not usable on this box
        pytest.skip(f"{lib} unavailable: {str(exc).splitlines()[0][:200]}")
    ks, vs = gather(st, kv_va, lens, layer)
    ref = decode_attention_ref(q.cpu(), ks, vs)
    assert rel_err(out.cpu(), ref) <= 2e-2
    # and the vTensor tcgen05 kernel on the very same bytes agrees with it
    tpc = st.cfg.tokens_per_chunk
    maps = kv_tensor_maps(kv_va.tolist(), [-(-n // tpc) * tpc for n in lens], st.geo)
    ours = decode_attention(q, kv_va, seq, layer, st.geo, max(lens), kv_maps=maps)
    torch.cuda.synchronize()
    assert rel_err(ours.cpu(), out.float().cpu().numpy()) <= 2e-2
