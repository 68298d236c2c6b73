"""Partitioned decode at world sizes 2 / 4 / 8 on the B200 vs the CPU oracle
(north_star: "results matching the CPU oracle at 1/2/4/8 GPUs").

One process per rank, exactly as `bench.py` runs under torchrun: every rank
owns its own ``VirtualMemoryDevice`` (its own VMM chunk pool and VA ranges),
manager and kernel launches; no collective touches the data path — gloo only
gathers the per-rank outputs so rank 0 can check them. The round-end box has
one GPU, so ranks map onto ``cuda:(rank % device_count)`` and take turns on it
(concurrent time-sliced ranks are covered, under a hard timeout, by
test_timeslice_gpu.py);
the N pools share its HBM, which changes nothing on the path under test
(every pool, VA and launch is still private to its rank).

* KV-head partition (config 4, Llama-2-70B shape): rank r holds kv heads
  ``[r*8/N, (r+1)*8/N)`` and the matching q heads of every request, in
  16-layer-group managers (80 x 8 x 128 x 2 x 2 B per token does not divide a
  2 MiB chunk); the gathered head slices must equal the unsharded oracle.
* Request partition (configs 2 / 5): rank r serves its block of requests with
  the Llama-3-8B geometry; the gathered rows must equal the oracle.

Tolerance: max|got - ref| / max|ref| <= 2e-2 (north_star), both decode paths.
"""

import os
import socket
import tempfile

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

TOL = 2e-2
D = 128


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _global_kv(seed, lens, hkv):
    g = torch.Generator().manual_seed(seed)
    ks = [torch.randn(hkv, n, D, generator=g).to(torch.bfloat16) for n in lens]
    vs = [torch.randn(hkv, n, D, generator=g).to(torch.bfloat16) for n in lens]
    return ks, vs


def _write_layer(st, va, layer, k, v):
    """Store dense K/V [H, n, d] of one layer into a request's mapped chunks."""
    from paper_2407_15309_b200.kv_layout import chunk_view

    tpc = st.geo.tokens_per_chunk
    n = k.shape[1]
    c = -(-n // tpc)
    if c == 0:
        return
    view = chunk_view(va, c, st.geo)[:, layer]  # [c, 2, H, tpc, d]
    for kv, t in ((0, k), (1, v)):
        pad = torch.zeros(t.shape[0], c * tpc, D, dtype=torch.bfloat16)
        pad[:, :n] = t
        view[:, kv].copy_(pad.view(t.shape[0], c, tpc, D).permute(1, 0, 2, 3).cuda())


def _decode_both(st, q, kv_va, seq, layer, lens):
    from paper_2407_15309_b200.attention import decode_attention, kv_tensor_maps

    tpc = st.geo.tokens_per_chunk
    mapped = [st.sched.mem[f"req{i}"].vt.space.mapped_pages * tpc for i in range(len(lens))]
    maps = kv_tensor_maps(kv_va.tolist(), mapped, st.geo)
    outs = {}
    for path in ("tcgen05", "cuda_core"):
        o = decode_attention(q, kv_va, seq, layer, st.geo, max(lens),
                             kv_maps=maps if path == "tcgen05" else None)
        torch.cuda.synchronize()
        outs[path] = o.cpu()
    return outs


def _rank_main(rank, world, port, tmp):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(rank % torch.cuda.device_count())
        from oracle.attention_ref import decode_attention_ref, rel_err
        from paper_2407_15309_b200.sharding import head_shard, layer_groups, partition_requests
        from vt_gpu_util import admit_with_lengths, cuda_stack

        # the global (unsharded) inputs, identical on every rank (seeded, CPU)
        lens = [1, 255, 256, 257, 1500, 4096]
        ks, vs = _global_kv(70, lens, 8)
        q = torch.randn(len(lens), 64, D, generator=torch.Generator().manual_seed(71)).to(torch.bfloat16)
        rlens = [0, 15, 16, 17, 333, 1024, 2047, 4096]
        rks, rvs = _global_kv(80, rlens, 8)
        rq = torch.randn(len(rlens), 32, D, generator=torch.Generator().manual_seed(81)).to(torch.bfloat16)

        def gpu_work():
            out = {}
            # ---- KV-head partition, Llama-2-70B shape (80 layers, 64 q / 8 kv heads)
            sh = head_shard(8, 64, world, rank)
            kl, kh = sh.kv_heads
            ql, qh = sh.q_heads
            layer = 37  # inside the third 16-layer group
            first, geom = next((f, g) for f, g in layer_groups(80, sh.local_kv_heads)
                               if f <= layer < f + g.layers)
            st = cuda_stack(geom.layers, sh.local_kv_heads, sh.local_q_heads, 4096)
            kv_va, seq = admit_with_lengths(st, lens, fill=False)
            for b, va in enumerate(kv_va.tolist()):
                _write_layer(st, va, layer - first, ks[b][kl:kh], vs[b][kl:kh])
            torch.cuda.synchronize()
            out["heads"] = _decode_both(st, q[:, ql:qh].cuda(), kv_va, seq, layer - first, lens)
            # ---- request partition, Llama-3-8B shape (32 layers, 32 q / 8 kv heads)
            mine = partition_requests([f"r{i}" for i in range(len(rlens))], world, rank)
            if mine:
                sub = [rlens[i] for i in mine]
                st8 = cuda_stack(32, 8, 32, 4352)
                kv8, seq8 = admit_with_lengths(st8, sub, fill=False)
                for j, va in enumerate(kv8.tolist()):
                    _write_layer(st8, va, 5, rks[mine[j]], rvs[mine[j]])
                torch.cuda.synchronize()
                out["requests"] = (mine, _decode_both(st8, rq[mine].cuda(), kv8, seq8, 5, sub))
            else:
                out["requests"] = (mine, None)
            st.dev.wait()
            torch.cuda.synchronize()
            return out

        # Ranks share the one GPU here: they run their GPU sections one after
        # another (gloo barriers) so a spawn without a timeout can never wait
        # on a wedged peer; everything else (process, VMM pool, VA ranges,
        # manager, launches) stays private to each rank.
        results = None
        for turn in range(world):
            if turn == rank:
                results = gpu_work()
            dist.barrier()

        gathered = [None] * world
        dist.all_gather_object(gathered, (rank, results))
        if rank == 0:
            report = []
            parts = sorted(gathered, key=lambda t: t[0])
            full = decode_attention_ref(q, ks, vs)
            rfull = decode_attention_ref(rq, rks, rvs)
            for path in ("tcgen05", "cuda_core"):
                cat = torch.cat([r["heads"][path] for _, r in parts], dim=1)
                report.append(("heads", path, rel_err(cat, full)))
                got = torch.zeros(len(rlens), 32, D)
                seen = []
                for _, r in parts:
                    idx, outs = r["requests"]
                    if outs is not None:
                        got[idx] = outs[path].float()
                        seen += idx
                assert sorted(seen) == list(range(len(rlens))), seen
                report.append(("requests", path, rel_err(got, rfull)))
            torch.save(report, os.path.join(tmp, "report.pt"))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4, 8])
def test_partitioned_decode_matches_oracle(cuda_ok, world):
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_rank_main, args=(world, _free_port(), tmp), nprocs=world, join=True)
        report = torch.load(os.path.join(tmp, "report.pt"))
    assert len(report) == 4
    for kind, path, err in report:
        assert err <= TOL, f"world={world} {kind} {path}: rel err {err:.3e}"
