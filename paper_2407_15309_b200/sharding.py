"""Multi-GPU partitioning of the vTensor path.

Nothing on the attention path needs a collective: every GPU owns its own VMM
chunk pool (its own ``VirtualMemoryDevice(cuda_ordinal=rank)``) and manager.

* Request partition (configs 2, 3, 5 and 4-by-request): requests are assigned
  to ranks in contiguous blocks or round-robin; every request of one
  conversation stays on one rank because rTree records are per pool
  (prefix reuse is pool-local, scheduler.py:104-162).
* KV-head partition (config 4, Llama-2-70B): rank r owns kv heads
  ``[r*Hkv/N, (r+1)*Hkv/N)`` and the matching q heads for *all* requests; its
  manager geometry uses ``Hkv/N`` heads. Outputs are disjoint head slices.
* Layer groups (config 4): 80 layers x 8 kv heads x 128 x 2 B x 2 = 320 KiB per
  token, which does not divide a 2 MiB chunk (config.py:103-107 rejects it), so
  the 70B cache is managed as 16-layer groups (64 KiB/token at 8 heads, tpc 32),
  each an independent manager over the same op stream.
"""

from __future__ import annotations

import dataclasses
import zlib
from collections.abc import Sequence

from .geometry import ModelGeometry


def owner_of(key: str, world: int) -> int:
    """Stable rank for a conversation / request id (crc32, like trace seeds)."""
    return zlib.crc32(key.encode("utf-8")) % world


def partition_requests(ids: Sequence[str], world: int, rank: int, policy: str = "block",
                       conversation: Sequence[str | None] | None = None) -> list[int]:
    """Indices of the requests rank `rank` serves.

    ``block``: contiguous blocks of ceil(n/world); ``round_robin``: i % world;
    requests with a conversation id always go to ``owner_of(conversation)``.
    """
    n = len(ids)
    per = -(-n // world) if n else 0
    out = []
    for i, rid in enumerate(ids):
        conv = conversation[i] if conversation is not None else None
        if conv is not None:
            r = owner_of(conv, world)
        elif policy == "round_robin":
            r = i % world
        else:
            r = i // per if per else 0
        if r == rank:
            out.append(i)
    return out


@dataclasses.dataclass(frozen=True)
class HeadShard:
    rank: int
    world: int
    kv_heads: tuple[int, int]  # [lo, hi) of the global kv heads
    q_heads: tuple[int, int]   # [lo, hi) of the global q heads

    @property
    def local_kv_heads(self) -> int:
        return self.kv_heads[1] - self.kv_heads[0]

    @property
    def local_q_heads(self) -> int:
        return self.q_heads[1] - self.q_heads[0]


def head_shard(kv_heads: int, q_heads: int, world: int, rank: int) -> HeadShard:
    if kv_heads % world:
        raise ValueError(f"{kv_heads} kv heads do not split over {world} ranks")
    g = q_heads // kv_heads
    per = kv_heads // world
    lo = rank * per
    return HeadShard(rank, world, (lo, lo + per), (lo * g, (lo + per) * g))


def layer_groups(layers: int, kv_heads: int, head_dim: int = 128, elem_bytes: int = 2,
                 chunk_bytes: int = 2 << 20) -> list[tuple[int, ModelGeometry]]:
    """Split `layers` into the fewest equal groups whose per-token bytes divide
    the chunk. Returns [(first_layer, group_geometry), ...]."""
    for n_groups in range(1, layers + 1):
        if layers % n_groups:
            continue
        per = layers // n_groups
        g = ModelGeometry(layers=per, kv_heads=kv_heads, head_dim=head_dim, elem_bytes=elem_bytes)
        if chunk_bytes % g.bytes_per_token == 0:
            return [(i * per, g) for i in range(n_groups)]
    raise ValueError("no layer grouping tiles the chunk")
