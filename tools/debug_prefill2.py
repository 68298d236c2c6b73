"""Debug aid: host-side numbers for row 70 of head 0/1, case (0,128), to compare with VT_PF_DUMP."""
import sys
import numpy as np
import torch
sys.path[:0] = [".", "tests"]
from paper_2407_15309_b200.attention import kv_tensor_maps, prefill_attention
from paper_2407_15309_b200.kv_layout import read_kv
from test_prefill_gpu import _turn
from vt_gpu_util import cuda_stack

st = cuda_stack(32, 8, 32, 1024, capacity_chunks=2048)
gen = torch.Generator(device="cuda").manual_seed(3)
vas, starts = _turn(st, 0, 128, 1, gen)
q = torch.randn(1, 128, 32, 128, generator=gen, device="cuda").to(torch.bfloat16)
maps = kv_tensor_maps(vas, [128], st.geo)
out = prefill_attention(q, maps, torch.tensor([0], dtype=torch.int32, device="cuda"), 1, st.geo)
torch.cuda.synchronize()
k, v = read_kv(vas[0], 128, 1, st.geo)
k = k.float().cpu().numpy(); v = v.float().cpu().numpy(); qq = q[0].float().cpu().numpy()
for h in (0, 1):
    s = qq[70, h] @ k[0].T
    print("host head", h, "S[64:68]", s[64:68], "S[127]", s[127], "S[0:4]", s[0:4], "S[63]", s[63])
    sc = s[:71] / np.sqrt(128)
    p = np.exp(sc - sc.max())
    o = (p / p.sum()) @ v[0][:71]
    print("host head", h, "O", o[:4], "gpu", out[0, 70, h, :4].float().cpu().numpy())
