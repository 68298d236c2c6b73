"""Run the REFERENCE ServingEngine (unmodified kvsim engine.py) on a trace,
either on the reference's own CPU stack (mode=reference) or on this package
with the B200 in the compute slot (mode=gpu: kvsim overlay whose L0-L3 are
this package, CUDA-driver device, GpuServingAdapter). Prints one JSON object.

mode=gpu also checks attention against the CPU oracle (oracle/attention_ref.py)
through a CPU mirror of the K/V: every prefill, and every decode step whose
index is a multiple of --check-every (1 = every step), for --check-layers
layers; and every --bytes-every steps the cache bytes of sampled requests are
read back from their VAs and compared bit-exactly with the mirror.

Usage: python tests/engine_gpu_run.py {reference|gpu} TRACE [--check-every N]
TRACE: toy_cfg1 | multi_turn | reduced_preempt | prefix_share
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
GIB, MIB = 1 << 30, 1 << 20


def traces(kvsim):
    TR = kvsim.trace.TraceRequest if hasattr(kvsim, "trace") else None
    if TR is None:
        from kvsim.trace import TraceRequest as TR
    prompts = [256, 512, 700, 1024, 1500, 2000, 2600, 3000]
    toy = [TR(id=f"t{i}", arrival_step=0, prompt_len=p, output_len=4096 - p - 1, seq=i)
           for i, p in enumerate(prompts)]
    return {
        # 1 layer, 8 kv heads (MHA), tpc 512, P 8
        "toy_cfg1": (dict(capacity_bytes=1 * GIB, weights_bytes=0,
                          geometry=kvsim.ModelGeometry(1, 8, 128, 2), max_seq_len=4096,
                          initial_alloc_tokens=256, lookahead_chunks=1, max_batch=8),
                     8, toy),
        "multi_turn": (dict(max_seq_len=12288), 32,
                       kvsim.generate_trace("multi_turn", seed=7, conversations=3, turns=2)),
        "reduced_preempt": (dict(capacity_bytes=13 * GIB, weights_bytes=12 * GIB,
                                 max_seq_len=12288, max_batch=4), 32,
                            kvsim.generate_trace("single_gen", seed=3, requests=4)),
        "prefix_share": (dict(max_seq_len=16384), 32,
                         kvsim.generate_trace("prefix_share", seed=5, requests=8)),
    }


class Checker:
    """CPU mirror of every request's K/V (HashedTokenSource on the CPU, one
    layer at a time) and the oracle comparisons."""

    def __init__(self, ad, layers, check_every, bytes_every):
        self.ad, self.layers = ad, layers
        self.every, self.bytes_every = check_every, bytes_every
        self.mirror: dict[tuple[str, int], tuple] = {}  # (rid, layer) -> (tokens, K, V)
        self.worst = 0.0
        self.checked_decode = self.checked_prefill = self.byte_checks = 0
        self.fail: list[str] = []

    def _kv(self, rid, layer, tokens):
        """Mirror K/V ``[n, H, d]`` of ``tokens`` (positions 0..n-1), grown in
        place: K/V of a position depends only on (token, position), so the
        prefix of a longer or restarted request is reused as long as its
        tokens agree."""
        import torch

        n = len(tokens)
        ent = self.mirror.get((rid, layer))
        if ent is None or ent[1].shape[0] < n:
            cap = max(n, 1024) if ent is None else max(n, 2 * ent[1].shape[0])
            H, d = self.ad.geo.kv_heads, self.ad.geo.head_dim
            K = torch.empty(cap, H, d, dtype=torch.bfloat16)
            V = torch.empty_like(K)
            have, toks = 0, []
            if ent is not None:
                have, toks = ent[0], ent[3]
                K[:have], V[:have] = ent[1][:have], ent[2][:have]
            ent = [have, K, V, toks]
            self.mirror[(rid, layer)] = ent
        have, K, V, toks = ent
        # keep the longest prefix whose tokens agree (a preempted request restarts)
        have = min(have, n)
        if have and toks[have - 1] != tokens[have - 1]:
            have = 0
            while have < n and have < len(toks) and toks[have] == tokens[have]:
                have += 1
        if have < n:
            t = torch.tensor(tokens[have:n], dtype=torch.int64)
            p = torch.arange(have, n, dtype=torch.int64)
            k, v = self.ad.source.kv(t, p, layer=layer)  # [n - have, H, d]
            K[have:n], V[have:n] = k, v
        ent[0] = n
        ent[3] = list(tokens) if len(tokens) != len(toks) or have < n else toks
        return K[:n], V[:n]

    def __call__(self, rec):
        import numpy as np
        import torch

        from oracle.attention_ref import decode_attention_ref, prefill_attention_ref, rel_err
        from paper_2407_15309_b200.adapter import HashedTokenSource
        from paper_2407_15309_b200.kv_layout import read_kv

        step = rec["step"]
        toks = rec["tokens"]
        need = "prefill" in rec or (self.every and step % self.every == 0)
        if not need:
            return
        torch.cuda.synchronize()
        for layer in self.layers:
            if "prefill" in rec:
                pf = rec["prefill"]
                out = pf["out"][layer].cpu()
                for i, r in enumerate(pf["rids"]):
                    s, n = pf["starts"][i], pf["lens"][i]
                    a, b = pf["q_offsets"][i], pf["q_offsets"][i + 1]
                    K, V = self._kv(r, layer, toks[r][:n])
                    q = self.ad.source.q(
                        torch.full((n - s,), HashedTokenSource.request_key(r), dtype=torch.int64),
                        torch.arange(s, n), layer=layer)
                    assert torch.equal(q, pf["q"][layer, a:b].cpu())
                    if n - s <= 256:  # whole causal block
                        ref = prefill_attention_ref(q, K.permute(1, 0, 2), V.permute(1, 0, 2), s)
                        got = out[a:b]
                    else:  # sampled query rows: row i is a decode over keys [0, s + i]
                        rows = sorted({0, 1, 127, 128, (n - s) // 2, n - s - 2, n - s - 1}
                                      | {(i * 7919) % (n - s) for i in range(9)})
                        ref = np.concatenate([
                            decode_attention_ref(q[i:i + 1], [K[:s + i + 1].permute(1, 0, 2)],
                                                 [V[:s + i + 1].permute(1, 0, 2)])
                            for i in rows])
                        got = out[a:b][rows]
                    self._note(rel_err(got, ref), f"step {step} prefill {r} layer {layer}")
                    self.checked_prefill += 1
            if "decode" in rec and self.every and step % self.every == 0:
                dc = rec["decode"]
                ks, vs = [], []
                for r, p in zip(dc["rids"], dc["positions"]):
                    K, V = self._kv(r, layer, toks[r][:p + 1])
                    ks.append(K.permute(1, 0, 2))
                    vs.append(V.permute(1, 0, 2))
                q = dc["q"][layer].cpu()
                ref = decode_attention_ref(q, ks, vs)
                self._note(rel_err(dc["out"][layer].cpu(), ref), f"step {step} decode layer {layer}")
                self.checked_decode += 1
        if self.bytes_every and step % self.bytes_every == 0 and "decode" in rec:
            # the cache bytes themselves, through the request VA (donor chunks included)
            dc = rec["decode"]
            for r, p in list(zip(dc["rids"], dc["positions"]))[:2]:
                va = self.ad.device.va(self.ad.scheduler.mem[r].vt.space.rng)
                layer = self.layers[-1]
                k, v = read_kv(va, p + 1, layer, self.ad.geo)
                K, V = self._kv(r, layer, toks[r][:p + 1])
                if not (torch.equal(k.cpu(), K.permute(1, 0, 2))
                        and torch.equal(v.cpu(), V.permute(1, 0, 2))):
                    self.fail.append(f"step {step}: cache bytes of {r} differ from the mirror")
                self.byte_checks += 1

    def _note(self, err, what):
        self.worst = max(self.worst, err)
        if not err <= 2e-2:
            self.fail.append(f"{what}: rel err {err:.3e}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["reference", "gpu"])
    ap.add_argument("trace")
    ap.add_argument("--check-every", type=int, default=1)
    ap.add_argument("--bytes-every", type=int, default=256)
    ap.add_argument("--kvsim", default=None, help="kvsim source dir (default: auto)")
    args = ap.parse_args()
    sys.path.insert(0, HERE)
    sys.path.insert(0, REPO)
    from ref_suite import build_kvsim_overlay, kvsim_source

    src = args.kvsim or kvsim_source()
    if src is None:
        print(json.dumps({"unavailable": "no kvsim source (/root/reference or baseline/_ref)"}))
        return
    if args.mode == "reference":
        sys.path.insert(0, os.path.dirname(src))
    else:
        sys.path.insert(0, build_kvsim_overlay(tempfile.mkdtemp(), src))
    import kvsim
    import kvsim.engine as eng

    cfg_kw, q_heads, trace = traces(kvsim)[args.trace]
    cfg = kvsim.SimConfig(**cfg_kw)
    res = {"trace": args.trace}
    t0 = time.perf_counter()
    if args.mode == "reference":
        rep = eng.run_trace(trace, cfg)
    else:
        import torch

        import paper_2407_15309_b200 as vt
        from paper_2407_15309_b200.adapter import GpuServingAdapter

        # engine.py:253-261 build_device, on the CUDA driver
        dev = vt.VirtualMemoryDevice(
            vt.DeviceConfig(capacity_bytes=cfg.capacity_bytes,
                            chunk_size_bytes=cfg.chunk_size_bytes,
                            weights_bytes=cfg.weights_bytes,
                            activation_bytes_per_request=cfg.activation_bytes_per_request),
            cuda_ordinal=torch.cuda.current_device())
        holder = {}
        L = cfg.geometry.layers
        layers = sorted({0, L - 1})

        def build(name, device, config):
            ad = GpuServingAdapter(device, config, q_heads)
            ad.on_step = Checker(ad, layers, args.check_every, args.bytes_every)
            holder["ad"] = ad
            return ad

        eng.build_allocator = build
        rep = eng.ServingEngine(cfg, trace, allocator="vtensor", device=dev).run()
        torch.cuda.synchronize()
        dev.wait()  # the shutdown's unmaps / destroys have run on the driver
        ad = holder["ad"]
        chk = ad.on_step
        logged = {}
        for c in dev.call_log:
            logged[c.op] = logged.get(c.op, 0) + 1
        res["gpu"] = {"lane": ad.lane, "launches": ad.launches, "steps": ad.steps,
                      "check": {"max_rel_err": chk.worst, "decode_checks": chk.checked_decode,
                                "prefill_checks": chk.checked_prefill,
                                "byte_checks": chk.byte_checks, "fail": chk.fail[:20],
                                "layers": layers, "every": args.check_every},
                      "driver": dev.driver_stats(), "logged_calls": logged}
    res["wall_s"] = round(time.perf_counter() - t0, 2)
    res.update({"csv": rep.to_csv(), "summary": rep.summary(), "admissions": rep.admissions,
                "stalls": rep.stall_count, "preemptions": rep.preemption_count})
    print(json.dumps(res, sort_keys=True, default=str))


if __name__ == "__main__":
    main()
