"""Debug aid: per-key-block timeline of CTA (0,0,0) of the prefill kernel
(libvtattn.so built with -DVT_PF_TRACE; tools/gpu_trace_pf.sh). Config 3 shape."""
import ctypes
import sys
import numpy as np
sys.path[:0] = [".", "tools"]
import kernel_bench as kb
from paper_2407_15309_b200.attention import attn_lib

class A: pass
args = A(); args.pf_batch, args.pf_prefix, args.pf_new, args.iters, args.warmup = 16, 2048, 512, 3, 1
kb.bench_prefill(args, {"bf16_tflops": 1, "bf16_tflops_sustained": 1})
buf = (ctypes.c_longlong * (2 * 64 * 2 + 64 * 2))()
attn_lib().vt_prefill_trace(buf)
a = np.frombuffer(buf, dtype=np.int64)
smx = a[:256].reshape(2, 64, 2); mma = a[256:].reshape(64, 2)
t0 = smx[0, 0, 0]
n = int((smx[0, :, 1] > 0).sum())
r = lambda v: int(v - t0) if v else -1
print("n_kv", n)
for j in range(n):
    print(f"{j:3d} grp0 {r(mma[j,0]):7d} grp1 {r(mma[j,1]):7d} | s0 S {r(smx[0,j,0]):7d} P {r(smx[0,j,1]):7d}"
          f" | s1 S {r(smx[1,j,0]):7d} P {r(smx[1,j,1]):7d}")
