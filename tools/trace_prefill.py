"""Debug aid: per-key-block timeline of CTA 0 of the persistent prefill kernel
(libvtattn.so built with -DVT_PF_TRACE; tools/gpu_trace_pf.sh). Config 3
shape by default; clock64 cycles relative to the first S."""
import ctypes
import sys

import numpy as np

sys.path[:0] = [".", "tools"]
import kernel_bench as kb
from paper_2407_15309_b200.attention import attn_lib


class A:
    pass


args = A()
args.pf_batch, args.pf_prefix, args.pf_new = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3
                                                                 else (16, 2048, 512)))
args.iters, args.warmup = 3, 1
print(kb.bench_prefill(args, {"bf16_tflops": 1, "bf16_tflops_sustained": 1}))
buf = (ctypes.c_longlong * (256 * 12))()
attn_lib().vt_prefill_trace(buf)
allv = np.frombuffer(buf, dtype=np.int64).copy()
a = allv[:256 * 8].reshape(256, 8)
sub = allv[256 * 8:].reshape(256, 4)
n = int((a[:, 0] > 0).sum())
t0 = a[0, 0]
r = np.where(a > 0, a - t0, -1)
print("blocks traced", n)
print("   g  S0rdy   P0   S1rdy   P1  | mma0   mma1 | epi0 start/end | sm0 sm1 (S->P cycles)")
for g in range(n):
    sm0 = r[g, 1] - r[g, 0]
    sm1 = r[g, 3] - r[g, 2]
    ep = f"{r[g, 6]:7d} {r[g, 7]:7d}" if r[g, 6] >= 0 and a[g, 6] >= a[0, 0] else ""
    print(f"{g:4d} {r[g,0]:7d} {r[g,1]:7d} {r[g,2]:7d} {r[g,3]:7d} | {r[g,4]:7d} {r[g,5]:7d} | "
          f"{ep:15s} | {sm0:5d} {sm1:5d}")
d = np.diff(r[:n, 0])
print("S0-ready period: p50", int(np.median(d)), "mean", int(d.mean()))
print("softmax S->P p50 slot0", int(np.median(r[:n, 1] - r[:n, 0])), "slot1", int(np.median(r[:n, 3] - r[:n, 2])))
sd = np.stack([sub[:n, 0] - a[:n, 0], sub[:n, 1] - sub[:n, 0], sub[:n, 2] - sub[:n, 1],
               sub[:n, 3] - sub[:n, 2], a[:n, 1] - sub[:n, 3]], axis=1)
print("slot0 softmax phases p50 [S-ready->ld done, ->max, ->exp loop, ->P stored, ->arrive]:",
      [int(v) for v in np.median(sd, axis=0)])
