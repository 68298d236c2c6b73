"""The synthetic K/V / q source the engine integration feeds the kernels
(adapter.HashedTokenSource): integer-only, so the CPU mirror the GPU tests
check against reproduces the device bytes; per-layer slices equal the
all-layer tensors; K/V depend only on (token, position)."""

import torch

from paper_2407_15309_b200.adapter import HashedTokenSource
from paper_2407_15309_b200.kv_layout import KVGeometry


def _src():
    return HashedTokenSource(KVGeometry(layers=3, kv_heads=2, head_dim=128, q_heads=8,
                                        tokens_per_chunk=16, chunk_bytes=2 << 20))


def test_layer_slices_match_full_tensors():
    s = _src()
    tok = torch.tensor([5, 17, 31999, 0, 5], dtype=torch.int64)
    pos = torch.tensor([0, 1, 2, 3, 4], dtype=torch.int64)
    k, v = s.kv(tok, pos)
    assert k.shape == (3, 5, 2, 128) and k.dtype == torch.bfloat16
    for layer in range(3):
        kl, vl = s.kv(tok, pos, layer=layer)
        assert torch.equal(kl, k[layer]) and torch.equal(vl, v[layer])
    q = s.q(torch.tensor([7, 7, 9]), torch.tensor([0, 1, 0]))
    assert q.shape == (3, 3, 8, 128)
    assert torch.equal(s.q(torch.tensor([7, 7, 9]), torch.tensor([0, 1, 0]), layer=2), q[2])


def test_kv_is_a_function_of_token_and_position():
    s = _src()
    a = s.kv(torch.tensor([5, 6]), torch.tensor([10, 11]))[0]
    b = s.kv(torch.tensor([9, 5, 6]), torch.tensor([3, 10, 11]))[0]
    assert torch.equal(a, b[:, 1:])
    assert not torch.equal(a[:, 0], a[:, 1])
    vals = s.kv(torch.arange(1000), torch.arange(1000))[0].float()
    assert vals.abs().max() <= 2.0 and abs(vals.mean()) < 0.05 and 0.9 < vals.std() < 1.4
