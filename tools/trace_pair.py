"""Debug aid: per-block timeline of pair 0 of the CTA-pair prefill kernel
(libvtattn built with -DVT_PF2_TRACE, VT_PREFILL_PAIR=1). Config 3 shape."""
import ctypes
import sys

import numpy as np

sys.path[:0] = [".", "tools"]
import kernel_bench as kb
from paper_2407_15309_b200.attention import attn_lib


class A:
    pass


args = A()
args.pf_batch, args.pf_prefix, args.pf_new = 16, 2048, 512
args.iters, args.warmup = 3, 1
print(kb.bench_prefill(args, {"bf16_tflops": 1, "bf16_tflops_sustained": 1}))
buf = (ctypes.c_longlong * (256 * 8))()
attn_lib().vt_prefill_pair_trace(buf)
a = np.frombuffer(buf, dtype=np.int64).reshape(256, 8).copy()
n = int((a[:, 0] > 0).sum())
t0 = a[0, 0]
r = np.where(a > 0, a - t0, -1)
print("   g   SA_rdy   PA    SB_rdy   PB  |  iS_A(g+1) iPV_A  iS_B(g+1) iPV_B")
for g in range(min(n, 60)):
    print(" ".join(f"{v:7d}" for v in [g, *r[g]]))
d = np.diff(r[:n, 0])
print("period (SA ready) p50", int(np.median(d)), "mean", int(d.mean()))
print("half A S->P p50", int(np.median(r[:n, 1] - r[:n, 0])), "half B", int(np.median(r[:n, 3] - r[:n, 2])))
print("B wait after A (SB_rdy - PA) p50", int(np.median(r[:n, 2] - r[:n, 1])))
