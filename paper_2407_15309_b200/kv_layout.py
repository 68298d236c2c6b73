"""KV layout inside a vTensor space, and torch views over a request's VA.

The reference prices one token as ``2 * L * Hkv * d * elem`` bytes spanning
every layer (kvsim/config.py:48-50), so chunk ``c`` of a space holds tokens
``[c*tpc, (c+1)*tpc)`` of all layers (config.py:86-88). We lay those bytes out
*chunk-blocked*: inside a chunk, block ``(layer, kv, head)`` is a dense
``[tpc][head_dim]`` bf16 tile at byte offset
``((layer*2 + kv)*Hkv + head) * tpc*head_dim*2``. For Llama-3-8B (tpc 16) a
block is 4 KiB contiguous, and all 16 tokens x 128 dims of one head of one
layer arrive in one bulk copy. Addresses are pure arithmetic off the request's
VA; the VA and strides never change while a request grows, which is what lets
the kernels run without a block table.
"""

from __future__ import annotations

import dataclasses

import torch

from .geometry import SimConfig


@dataclasses.dataclass(frozen=True)
class KVGeometry:
    layers: int
    kv_heads: int
    head_dim: int
    q_heads: int
    tokens_per_chunk: int
    chunk_bytes: int

    @classmethod
    def from_config(cls, cfg: SimConfig, q_heads: int) -> "KVGeometry":
        g = cfg.geometry
        if g.elem_bytes != 2:
            raise ValueError("the CUDA path stores bf16 KV (elem_bytes == 2)")
        if q_heads % g.kv_heads:
            raise ValueError("q_heads must be a multiple of kv_heads")
        return cls(g.layers, g.kv_heads, g.head_dim, q_heads, cfg.tokens_per_chunk,
                   cfg.chunk_size_bytes)

    @property
    def group(self) -> int:
        return self.q_heads // self.kv_heads

    @property
    def head_block_bytes(self) -> int:
        return self.tokens_per_chunk * self.head_dim * 2

    def block_offset(self, layer: int, kv: int, head: int) -> int:
        return ((layer * 2 + kv) * self.kv_heads + head) * self.head_block_bytes

    def token_offset(self, pos: int, layer: int, kv: int, head: int) -> int:
        c, t = divmod(pos, self.tokens_per_chunk)
        return c * self.chunk_bytes + self.block_offset(layer, kv, head) + t * self.head_dim * 2

    def kv_bytes(self, n_tokens: int, layers: int | None = None) -> int:
        """Algorithmic K+V bytes for n_tokens of `layers` layers (default: 1)."""
        return 2 * n_tokens * self.kv_heads * self.head_dim * 2 * (1 if layers is None else layers)


class _CudaArray:
    """Minimal __cuda_array_interface__ exporter for a raw device pointer."""

    def __init__(self, ptr: int, shape: tuple[int, ...], typestr: str = "<i2") -> None:
        self.__cuda_array_interface__ = {
            "shape": shape,
            "typestr": typestr,
            "data": (int(ptr), False),
            "version": 3,
            "strides": None,
        }


def chunk_view(va: int, n_chunks: int, geo: KVGeometry) -> torch.Tensor:
    """bf16 view ``[n_chunks, layers, 2, kv_heads, tpc, head_dim]`` of the first
    ``n_chunks`` chunks of a space. Only mapped chunks may be touched."""
    shape = (n_chunks, geo.layers, 2, geo.kv_heads, geo.tokens_per_chunk, geo.head_dim)
    n = 1
    for s in shape:
        n *= s
    if n * 2 != n_chunks * geo.chunk_bytes:
        raise ValueError("geometry does not tile the chunk exactly")
    raw = torch.as_tensor(_CudaArray(va, (n,)), device="cuda")
    return raw.view(torch.bfloat16).view(shape)


def read_kv(va: int, n_tokens: int, layer: int, geo: KVGeometry) -> tuple[torch.Tensor, torch.Tensor]:
    """Dense ``K, V: [kv_heads, n_tokens, head_dim]`` copies of one layer."""
    n_chunks = -(-n_tokens // geo.tokens_per_chunk)
    if n_chunks == 0:
        z = torch.zeros(geo.kv_heads, 0, geo.head_dim, dtype=torch.bfloat16, device="cuda")
        return z, z.clone()
    v = chunk_view(va, n_chunks, geo)[:, layer]  # [c, 2, H, tpc, d]
    kv = v.permute(1, 2, 0, 3, 4).reshape(2, geo.kv_heads, n_chunks * geo.tokens_per_chunk,
                                          geo.head_dim)
    return kv[0, :, :n_tokens].clone(), kv[1, :, :n_tokens].clone()
