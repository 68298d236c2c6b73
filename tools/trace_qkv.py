"""Debug aid: per-CTA timeline of the fused QKV kernel (libvtattn.so built with
-DVT_QKV_TRACE; tools/gpu_trace_qkv.sh). Llama-3-8B, B tokens.

  python tools/trace_qkv.py B SPLIT          one launch after warm-up (cold W)
  python tools/trace_qkv.py B SPLIT chain    9 back-to-back PDL launches over 6
                                             rotating weights; the last two
                                             launches on one clock (steady state)
"""
import ctypes
import sys

import numpy as np
import torch

sys.path[:0] = [".", "tools"]
import kernel_bench as kb
from paper_2407_15309_b200.attention import attn_lib, pack_qkv_weight, qkv_append

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
split = int(sys.argv[2]) if len(sys.argv) > 2 else 0
chain = len(sys.argv) > 3 and sys.argv[3] == "chain"
L, hkv, hq, hidden = 32, 8, 32, 4096
cfg, dev, ops, sched, geo = kb.stack(L, hkv, hq, 4096, 4096)
vas = []
for b in range(B):
    sched.create(f"r{b}", [1] * 100)
    sched.mark_prefilled(f"r{b}")
    sched.extend(f"r{b}", 101)
    vas.append(dev.va(sched.mem[f"r{b}"].vt.space.rng))
dev.wait()
kv_va = torch.tensor(vas, dtype=torch.int64, device="cuda")
tok_req = torch.arange(B, dtype=torch.int32, device="cuda")
tok_pos = torch.full((B,), 100, dtype=torch.int32, device="cuda")
feats = (hq + 2 * hkv) * 128
NW = 6
ws = [pack_qkv_weight((torch.randn(feats, hidden, device="cuda") / 64).to(torch.bfloat16)) for _ in range(NW)]
x = torch.randn(B, hidden, device="cuda").to(torch.bfloat16)
q = torch.empty(B, hq, 128, dtype=torch.bfloat16, device="cuda")
for i in range(3):
    qkv_append(x, ws[i], tok_req, tok_pos, kv_va, geo, i, q_out=q, split_k=split)
torch.cuda.synchronize()
graph = len(sys.argv) > 4 and sys.argv[4] == "graph"
same = len(sys.argv) > 4 and sys.argv[4] == "same"   # graph, one weight (L2 / TLB warm)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n_launch = 9 if chain else 1


def run():
    for i in range(n_launch):
        lay = 3 + i
        qkv_append(x, ws[0 if same else lay % NW], tok_req, tok_pos, kv_va, geo, lay, q_out=q,
                   split_k=split)


if graph or same:
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        run()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run()
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
else:
    e0.record()
    run()
    e1.record()
torch.cuda.synchronize()
print(f"B={B} split={split} launches {n_launch} event time {e0.elapsed_time(e1)*1e3:.1f} us"
      f" ({e0.elapsed_time(e1)*1e3/n_launch:.2f} per launch)")
buf = (ctypes.c_longlong * (2 * 256 * 16))()
lib = attn_lib()
lib.vt_qkv_trace(buf)
full = np.frombuffer(buf, dtype=np.int64).reshape(2, 256, 16)
last = (3 + n_launch - 1) & 1
slots = [1 - last, last] if chain else [last]
names = ["entry", "setup", "w_issue", "first_land", "last_land", "last_commit", "acc_ready",
         "peer_ready", "partial", "end", "helper_flag", "ring_issued", "tmem_alloc",
         "cluster_sync", "dep_wait"]
t0 = None
for s in slots:
    a = full[s]
    n_all = int((a[:, 0] > 0).sum())
    a = a[:n_all]
    if t0 is None:
        t0 = a[:, 0].min()
    r = a - t0
    r[a == 0] = -1
    print(f"--- launch slot {s}: ctas {len(a)} (times from the first traced launch's first entry)")
    idx = np.arange(len(a))
    n_help = 2 * ((48 + 1) // 2) if split == 3 else 0  # split 3: helper clusters come first
    groups = [("helper", idx < n_help)] if n_help else []
    groups += [("lower", (idx >= n_help) & (idx % 2 == 0)), ("upper", (idx >= n_help) & (idx % 2 == 1))]
    for lab, sel in groups:
        for j, n in enumerate(names):
            col = r[sel, j]
            col = col[col >= 0]
            if len(col):
                print(f"{lab} {n:12s} min {col.min():7d} p50 {int(np.median(col)):7d} max {col.max():7d} ns")
