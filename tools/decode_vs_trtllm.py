"""Config-2 decode (B 64, ctx 4096, 32 q / 8 kv heads): this package's tcgen05
vTensor kernel and flashinfer's trtllm-gen paged decode on the same bytes,
for ncu (`--launches N` launches of each on layer 0) or plain timing
(`--time`). Both arms' outputs are oracle-checked on sampled requests.

  python tools/decode_vs_trtllm.py [--launches 4] [--time]
"""

import argparse
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
sys.path.insert(0, os.path.join(REPO, "tools"))

import torch  # noqa: E402

from oracle.attention_ref import decode_attention_ref, rel_err  # noqa: E402
from paged_libs import flashinfer_decode, gather_pages  # noqa: E402
from paged_vs_vtensor import timed32  # noqa: E402
from paper_2407_15309_b200.attention import DecodeWorkspace, decode_attention, kv_tensor_maps  # noqa: E402
from vt_gpu_util import admit_with_lengths, cuda_stack, gather  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches", type=int, default=4)
    ap.add_argument("--time", action="store_true")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    B, ctx = 64, 4096
    st = cuda_stack(32, 8, 32, ctx + 256, capacity_chunks=20000)
    kv_va, seq = admit_with_lengths(st, [ctx] * B, seed=5)
    q = torch.randn(B, 32, 128, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    tpc = st.cfg.tokens_per_chunk
    maps = kv_tensor_maps(kv_va.tolist(), [st.sched.mem[f"req{i}"].vt.space.mapped_pages * tpc
                                           for i in range(B)], st.geo)
    ws = DecodeWorkspace(st.geo, B, ctx)
    picks = [0, 21, 42, 63]
    ks, vs = gather(st, kv_va, [ctx] * B, 0)
    ref = decode_attention_ref(q[picks].cpu(), [ks[i] for i in picks], [vs[i] for i in picks])
    del ks, vs
    K, V, table = gather_pages(st, kv_va, [ctx] * B, 0)
    run = flashinfer_decode(K, V, table, [ctx] * B, 32)
    res = {}
    o = decode_attention(q, kv_va, seq, 0, st.geo, ctx, workspace=ws, kv_maps=maps)
    res["err_vtensor"] = rel_err(o[picks].cpu(), ref)
    o2 = run(q, torch.empty_like(q))
    torch.cuda.synchronize()
    res["err_trtllm"] = rel_err(o2[picks].cpu(), ref)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("cmp")  # ncu --nvtx --nvtx-include "cmp/"
    for _ in range(args.launches):  # layer 0 for both arms (same bytes)
        decode_attention(q, kv_va, seq, 0, st.geo, ctx, out=out, workspace=ws, kv_maps=maps)
        run(q, out)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    if args.time:
        nbytes = 2 * B * ctx * 8 * 128 * 2 + 2 * B * 32 * 128 * 2
        t_vt_l0 = timed32(lambda l: decode_attention(q, kv_va, seq, 0, st.geo, ctx, out=out,
                                                     workspace=ws, kv_maps=maps))
        t_vt = timed32(lambda l: decode_attention(q, kv_va, seq, l, st.geo, ctx, out=out,
                                                  workspace=ws, kv_maps=maps))
        t_tr = timed32(lambda l: run(q, out))
        res.update({"us_vtensor_32_layers": round(t_vt, 2), "us_vtensor_layer0_only": round(t_vt_l0, 2),
                    "us_trtllm_layer0": round(t_tr, 2),
                    "GB/s": {k: round(nbytes / (v * 1e-6) / 1e9, 1) for k, v in
                             (("vtensor", t_vt), ("vtensor_l0", t_vt_l0), ("trtllm", t_tr))}})
    print(json.dumps(res))


if __name__ == "__main__":
    main()
