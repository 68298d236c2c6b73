"""Multi-rank (world_size 2, gloo, CPU) coverage of the partitioned path.

* request partition: each rank serves its own requests with its own manager
  (own device / chunk pool); per-rank state equals an oracle run on the same
  sub-stream, the partitions are disjoint and cover every request, and
  conversations never straddle ranks;
* KV-head partition (70B shape): each rank computes attention for its head
  slice only (oracle math on CPU); the gathered slices equal the unsharded
  result; 80 layers are grouped into 16-layer managers that fit 2 MiB chunks.
No collective is used on the data path — gloo only gathers results to check.
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import manager_streams as ms
import paper_2407_15309_b200 as vt
from oracle import vtm_ref
from oracle.attention_ref import decode_attention_ref
from paper_2407_15309_b200.sharding import head_shard, layer_groups, partition_requests

WORLD = 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, port, tmp):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        # --- request partition: ranks run disjoint sub-streams on their own pools
        ids = [f"req{i}" for i in range(12)]
        convs = [None] * 8 + ["c0", "c0", "c1", "c1"]
        mine = partition_requests(ids, WORLD, rank, conversation=convs)
        digests = []
        for ns in (vt, vtm_ref):
            cfg = ms.stream_configs(ns)["llama8b"]
            st, _ = ms.run_stream(ns, cfg, seed=100 + rank, steps=120)
            digests.append(ms.digest(ms.dump(st)))
        same = digests[0] == digests[1]
        gathered = [None] * WORLD
        dist.all_gather_object(gathered, (rank, mine, same))

        # --- head partition of a 70B-shaped decode (oracle math, CPU)
        g = torch.Generator().manual_seed(7)
        hkv, hq, B, n = 8, 64, 3, 96
        q = torch.randn(B, hq, 128, generator=g)
        k = torch.randn(B, hkv, n, 128, generator=g)
        v = torch.randn(B, hkv, n, 128, generator=g)
        sh = head_shard(hkv, hq, WORLD, rank)
        kl, kh = sh.kv_heads
        ql, qh = sh.q_heads
        part = decode_attention_ref(q[:, ql:qh], [k[b, kl:kh] for b in range(B)],
                                    [v[b, kl:kh] for b in range(B)])
        parts = [None] * WORLD
        dist.all_gather_object(parts, (rank, part))
        if rank == 0:
            full = decode_attention_ref(q, [k[b] for b in range(B)], [v[b] for b in range(B)])
            cat = np.concatenate([p for _, p in sorted(parts, key=lambda t: t[0])], axis=1)
            np.save(os.path.join(tmp, "heads_ok.npy"), np.array([np.allclose(cat, full, atol=1e-6)]))
            with open(os.path.join(tmp, "req.txt"), "w") as f:
                f.write(repr(gathered))
    finally:
        dist.destroy_process_group()


def test_partitioned_ranks_over_gloo():
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_rank_main, args=(_free_port(), tmp), nprocs=WORLD, join=True)
        assert bool(np.load(os.path.join(tmp, "heads_ok.npy"))[0])
        gathered = eval(open(os.path.join(tmp, "req.txt")).read())
    covered = sorted(i for _, mine, _ in gathered for i in mine)
    assert covered == list(range(12)), "partitions must be disjoint and complete"
    assert all(same for _, _, same in gathered), "per-rank manager != oracle"
    by_rank = {r: set(m) for r, m, _ in gathered}
    for a, b in ((8, 9), (10, 11)):  # one conversation, one rank
        assert any({a, b} <= s for s in by_rank.values())


def test_70b_layer_groups_fit_2mib_chunks():
    for world in (1, 2, 4, 8):
        sh = head_shard(8, 64, world, 0)
        groups = layer_groups(80, sh.local_kv_heads)
        assert sum(g.layers for _, g in groups) == 80
        for _, geo in groups:
            assert (2 << 20) % geo.bytes_per_token == 0
        with pytest.raises(ValueError):  # the ungrouped geometry is rejected, as in config.py
            vt.SimConfig(geometry=vt.ModelGeometry(80, sh.local_kv_heads, 128, 2))
