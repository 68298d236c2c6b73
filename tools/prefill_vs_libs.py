"""Config-3 prefix prefill (16 requests x (2048 rTree-shared prefix + 512 new
tokens), Llama-3-8B heads: 32 q / 8 kv, d 128, bf16) — this package's tcgen05
kernel beside the prefill kernels shipped in the image, on the same K/V bytes:

* ``flashinfer.prefill.trtllm_batch_context_with_kv_cache`` (flashinfer
  0.6.11, sm100 trtllm-gen FMHA cubins, paged KV, HND layout); the 128 prefix
  pages are shared by every request's block table, as a paged prefix cache
  would share them; page size 16 = one 2 MiB vTensor chunk and 64;
* ``flash_attn.flash_attn_varlen_func`` (flash-attn 2.8.3, the family the
  paper ran; sm80 code on sm_100), contiguous per-request K/V.

Library kernels are a BASELINE only, never the product path. Every arm's output
is checked against the CPU oracle (oracle/attention_ref.py) on two requests.
Timing: CUDA events around 20 back-to-back launches, median of 5. Prints one
JSON line per arm."""

import json
import math
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tools"))

import torch  # noqa: E402

from kernel_bench import fill, peaks, stack  # noqa: E402
from oracle.attention_ref import prefill_attention_ref, rel_err  # noqa: E402
from paper_2407_15309_b200.attention import kv_tensor_maps, prefill_attention  # noqa: E402
from paper_2407_15309_b200.kv_layout import read_kv  # noqa: E402


def timed(fn, n=20, reps=5):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / n)
    return statistics.median(ts) * 1e3  # us


def main():
    torch.cuda.set_device(0)
    pk = peaks()
    L, hkv, hq, d, B, prefix, n_new = 32, 8, 32, 128, 16, 2048, 512
    kv_len = prefix + n_new
    cfg, dev, ops, sched, geo = stack(L, hkv, hq, 4096, 4096)
    gen = torch.Generator(device="cuda").manual_seed(3)
    tpc = cfg.tokens_per_chunk
    base = [i % 251 for i in range(prefix)]
    sched.create("donor", base)
    sched.mark_prefilled("donor")
    dev.wait()
    fill(dev.va(sched.mem["donor"].vt.space.rng), sched.mem["donor"].vt.space.mapped_pages, geo, gen)
    assert sched.prefix_record("donor")
    vas = []
    for b in range(B):
        hit = sched.prefix_match(f"t{b}", base + [7000 + b * 600 + k for k in range(n_new)])
        assert hit is not None and hit[1].shared_tokens == prefix
        vas.append(dev.va(sched.mem[f"t{b}"].vt.space.rng))
    dev.wait()
    for b in range(B):
        fill(vas[b], sched.mem[f"t{b}"].vt.space.mapped_pages, geo, gen, first=prefix // tpc)
    layer = 5
    maps = kv_tensor_maps(vas, [kv_len] * B, geo)
    start = torch.full((B,), prefix, dtype=torch.int32, device="cuda")
    q = (torch.randn(B, n_new, hq, d, generator=gen, device="cuda")).to(torch.bfloat16)
    scale = 1.0 / math.sqrt(d)
    flops = 4 * hq * d * (n_new * prefix + n_new * (n_new + 1) // 2) * B
    kv = [read_kv(va, kv_len, layer, geo) for va in vas]  # [Hkv, kv_len, d] each
    check_b = (0, B - 1)
    want = {b: prefill_attention_ref(q[b].cpu(), kv[b][0].cpu(), kv[b][1].cpu(), prefix)
            for b in check_b}
    lines = []

    def report(name, us, got, extra=None):
        errs = [rel_err(got[b].float().cpu(), want[b]) for b in check_b]
        tf = flops / (us * 1e-6) / 1e12
        r = {"kernel": name, "config": f"{B} x ({prefix} shared + {n_new} new), 32q/8kv d128 bf16",
             "us": round(us, 2), "TFLOP/s": round(tf, 1),
             "frac_of_bf16_burst": round(tf / pk["bf16_tflops"], 4),
             "oracle_rel_err_max": float(f"{max(errs):.3e}"), "parity_ok": max(errs) < 2e-2}
        r.update(extra or {})
        lines.append(r)
        print(json.dumps(r), flush=True)

    out = torch.empty_like(q)
    us = timed(lambda: prefill_attention(q, maps, start, layer, geo, out=out))
    report("vtensor tcgen05 prefill (this package)", us, out)

    qf = q.reshape(B * n_new, hq, d).contiguous()
    cu_q = torch.arange(0, (B + 1) * n_new, n_new, dtype=torch.int32, device="cuda")
    cu_k = torch.arange(0, (B + 1) * kv_len, kv_len, dtype=torch.int32, device="cuda")
    try:
        import flashinfer.prefill as fp
        for page in (16, 64):
            npre, nnew = prefix // page, n_new // page
            kp = torch.empty(npre + B * nnew, hkv, page, d, dtype=torch.bfloat16, device="cuda")
            vp = torch.empty_like(kp)
            kp[:npre] = kv[0][0][:, :prefix].reshape(hkv, npre, page, d).transpose(0, 1)
            vp[:npre] = kv[0][1][:, :prefix].reshape(hkv, npre, page, d).transpose(0, 1)
            table = torch.empty(B, npre + nnew, dtype=torch.int32, device="cuda")
            for b in range(B):
                assert torch.equal(kv[b][0][:, :prefix], kv[0][0][:, :prefix])  # rTree-shared bytes
                lo = npre + b * nnew
                kp[lo:lo + nnew] = kv[b][0][:, prefix:].reshape(hkv, nnew, page, d).transpose(0, 1)
                vp[lo:lo + nnew] = kv[b][1][:, prefix:].reshape(hkv, nnew, page, d).transpose(0, 1)
                table[b, :npre] = torch.arange(npre, device="cuda")
                table[b, npre:] = torch.arange(lo, lo + nnew, device="cuda")
            seq = torch.full((B,), kv_len, dtype=torch.int32, device="cuda")
            ws = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")
            o2 = torch.empty_like(qf)

            def run():
                fp.trtllm_batch_context_with_kv_cache(
                    qf, (kp, vp), ws, table, seq, n_new, kv_len, scale, 1.0, B, cu_q, cu_k,
                    out=o2, kv_layout="HND", causal=True)
            try:
                us = timed(run)
                report(f"flashinfer trtllm-gen context (paged, page {page})", us,
                       o2.view(B, n_new, hq, d))
            except Exception as e:  # noqa: BLE001
                print(json.dumps({"kernel": f"flashinfer trtllm-gen page {page}",
                                  "unavailable": f"{type(e).__name__}: {str(e)[:200]}"}), flush=True)
    except ImportError as e:
        print(json.dumps({"kernel": "flashinfer", "unavailable": str(e)[:200]}))

    try:
        from flash_attn import flash_attn_varlen_func
        kc = torch.cat([kv[b][0].transpose(0, 1) for b in range(B)]).contiguous()  # [B*kv_len, Hkv, d]
        vc = torch.cat([kv[b][1].transpose(0, 1) for b in range(B)]).contiguous()
        o3 = [None]

        def run_fa():
            o3[0] = flash_attn_varlen_func(qf, kc, vc, cu_q, cu_k, n_new, kv_len, softmax_scale=scale,
                                           causal=True)
        us = timed(run_fa)
        report("flash-attn 2.8.3 varlen (contiguous KV)", us, o3[0].view(B, n_new, hq, d))
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"kernel": "flash-attn", "unavailable": f"{type(e).__name__}: {str(e)[:200]}"}))
    dev.wait()


if __name__ == "__main__":
    main()
