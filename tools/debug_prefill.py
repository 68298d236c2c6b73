"""Debug aid: per-head / per-row error map of the prefill kernel vs the oracle."""
import sys
import numpy as np
import torch

sys.path[:0] = [".", "tests"]
from oracle.attention_ref import prefill_attention_ref
from paper_2407_15309_b200.attention import kv_tensor_maps, prefill_attention
from paper_2407_15309_b200.kv_layout import read_kv
from test_prefill_gpu import _turn
from vt_gpu_util import cuda_stack

for (layers, hkv, hq, prefix, n_new, batch, max_seq) in [(32, 8, 32, 0, 128, 1, 1024),
                                                          (32, 8, 32, 0, 256, 1, 1024),
                                                          (32, 8, 32, 128, 128, 1, 1024)]:
    st = cuda_stack(layers, hkv, hq, max_seq, capacity_chunks=2048)
    gen = torch.Generator(device="cuda").manual_seed(3)
    vas, starts = _turn(st, prefix, n_new, batch, gen)
    starts = [prefix] * batch
    q = torch.randn(batch, n_new, hq, 128, generator=gen, device="cuda").to(torch.bfloat16)
    maps = kv_tensor_maps(vas, [s + n_new for s in starts], st.geo)
    out = prefill_attention(q, maps, torch.tensor(starts, dtype=torch.int32, device="cuda"), 1, st.geo)
    torch.cuda.synchronize()
    k, v = read_kv(vas[0], starts[0] + n_new, 1, st.geo)
    ref = prefill_attention_ref(q[0].cpu(), k.cpu(), v.cpu(), starts[0])
    got = out[0].float().cpu().numpy()
    err = np.abs(got - ref).max(axis=2) / np.abs(ref).max()  # [n_new, Hq]
    print("case", prefix, n_new, "max", err.max())
    print(" per head:", np.round(err.max(axis=0), 3))
    rows = err.max(axis=1)
    bad = np.nonzero(rows > 2e-2)[0]
    print(" bad rows:", len(bad), bad[:20], bad[-5:] if len(bad) else "")
