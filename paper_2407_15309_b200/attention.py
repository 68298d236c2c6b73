"""Attention over a vTensor KV cache (rows a27-a29) — calls into libvtattn.so.

These functions are the compute slot the reference leaves as a cost formula
(kvsim/engine.py:499-511). Every tensor must already be on the GPU; there is
no CPU or eager-PyTorch fallback — a missing library or a CPU tensor raises.
"""

from __future__ import annotations

import ctypes
import math
from ctypes import POINTER, c_float, c_int, c_int32, c_int64, c_size_t, c_uint64, c_void_p

import torch

from ._native import _load
from .kv_layout import KVGeometry


class _Geo(ctypes.Structure):
    _fields_ = [
        ("layers", c_int32),
        ("kv_heads", c_int32),
        ("head_dim", c_int32),
        ("q_heads", c_int32),
        ("tokens_per_chunk", c_int32),
        ("_pad", c_int32),
        ("chunk_bytes", c_int64),
    ]


_lib = None


def attn_lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        lib = _load("libvtattn.so")
        P = c_void_p
        lib.vt_decode_attention.argtypes = [POINTER(_Geo), c_int32, P, P, P, P, c_int32, c_int32,
                                            c_float, P, P, c_size_t, c_int32, P]
        lib.vt_decode_attention.restype = c_int
        lib.vt_decode_attention_chained.argtypes = lib.vt_decode_attention.argtypes
        lib.vt_decode_attention_chained.restype = c_int
        lib.vt_decode_attention_paged.argtypes = [POINTER(_Geo), c_int32, P, P, P, c_int32, P,
                                                  c_int32, c_int32, c_float, P, P, c_size_t,
                                                  c_int32, P]
        lib.vt_decode_attention_paged.restype = c_int
        lib.vt_decode_workspace_bytes.argtypes = [POINTER(_Geo), c_int32, c_int32, c_int32]
        lib.vt_decode_workspace_bytes.restype = c_size_t
        lib.vt_kv_append.argtypes = [POINTER(_Geo), c_int32, c_int32, P, P, P, P, c_int32, P]
        lib.vt_kv_append.restype = c_int
        lib.vt_prefill_attention.argtypes = [POINTER(_Geo), c_int32, P, P, P, c_int32, c_int32,
                                             c_float, P, P]
        lib.vt_prefill_attention.restype = c_int
        lib.vt_prefill_attention_varlen.argtypes = [POINTER(_Geo), c_int32, P, P, P, P, c_int32,
                                                    c_int32, c_int64, c_float, P, P]
        lib.vt_prefill_attention_varlen.restype = c_int
        lib.vt_kv_tensor_maps.argtypes = [POINTER(_Geo), P, P, c_int32, P]
        lib.vt_kv_tensor_maps.restype = c_int
        lib.vt_qkv_append.argtypes = [POINTER(_Geo), c_int32, P, P, c_int32, c_int32, P, P, P, P,
                                      c_int32, P]
        lib.vt_qkv_append.restype = c_int
        lib.vt_qkv_append_ws.argtypes = [POINTER(_Geo), c_int32, P, P, c_int32, c_int32, P, P, P,
                                         P, c_int32, P, P]
        lib.vt_qkv_append_ws.restype = c_int
        lib.vt_qkv_workspace_bytes.argtypes = [POINTER(_Geo)]
        lib.vt_qkv_workspace_bytes.restype = c_size_t
        lib.vt_qkv_pack_weight.argtypes = [P, c_int32, c_int32, P, P]
        lib.vt_qkv_pack_weight.restype = c_int
        lib.vt_attn_last_launches.argtypes = []
        lib.vt_attn_last_launches.restype = c_int32
        _lib = lib
    return _lib


ATTN_SYMBOLS = ("vt_decode_attention", "vt_decode_attention_chained", "vt_decode_attention_paged",
                "vt_decode_workspace_bytes", "vt_kv_append",
                "vt_kv_tensor_maps", "vt_prefill_attention", "vt_prefill_attention_varlen",
                "vt_qkv_append", "vt_qkv_append_ws", "vt_qkv_workspace_bytes",
                "vt_qkv_pack_weight",
                "vt_attn_last_launches")


def _geo(g: KVGeometry) -> _Geo:
    return _Geo(g.layers, g.kv_heads, g.head_dim, g.q_heads, g.tokens_per_chunk, 0, g.chunk_bytes)


def _need_cuda(*tensors: torch.Tensor) -> None:
    for t in tensors:
        if not t.is_cuda:
            raise RuntimeError("vTensor attention runs on the GPU only; got a CPU tensor")
        if not t.is_contiguous():
            raise RuntimeError("vTensor attention needs contiguous tensors")


def _check(rc: int, what: str) -> None:
    if rc != 0:
        raise RuntimeError(f"{what} failed: cudaError {rc}")


def _stream(stream: torch.cuda.Stream | None) -> int:
    return (stream or torch.cuda.current_stream()).cuda_stream


class DecodeWorkspace:
    """Split-KV partials buffer sized for (batch, max_seq_len)."""

    def __init__(self, geo: KVGeometry, batch: int, max_seq_len: int, split_tokens: int = 0,
                 device: str = "cuda") -> None:
        self.geo, self.split_tokens = geo, split_tokens
        nbytes = attn_lib().vt_decode_workspace_bytes(ctypes.byref(_geo(geo)), batch,
                                                       max_seq_len, split_tokens)
        # zeroed: the tail holds the self-resetting split-arrival counters
        self.buf = torch.zeros(max(nbytes, 16), dtype=torch.uint8, device=device)
        self.batch, self.max_seq_len = batch, max_seq_len


def decode_attention(q: torch.Tensor, kv_va: torch.Tensor, seq_lens: torch.Tensor, layer: int,
                     geo: KVGeometry, max_seq_len: int, out: torch.Tensor | None = None,
                     workspace: DecodeWorkspace | None = None, scale: float | None = None,
                     split_tokens: int = 0, stream: torch.cuda.Stream | None = None,
                     kv_maps: torch.Tensor | None = None, chained: bool = False) -> torch.Tensor:
    """q ``[B, Hq, d]`` bf16 -> out ``[B, Hq, d]`` bf16 for one layer.

    ``kv_va`` is an int64 CUDA tensor of request VAs (``device.va(space.rng)``),
    ``seq_lens`` an int32 CUDA tensor; ``max_seq_len`` a host bound on it.
    With ``kv_maps`` (:class:`KVMapCache`) the tcgen05/TMEM kernel runs;
    without, the CUDA-core cp.async.bulk kernel. ``chained=True`` for a layer
    launched right after another decode layer on the same stream
    (``vt_decode_attention_chained``: programmatic dependent launch)."""
    B = q.shape[0]
    if q.dtype != torch.bfloat16 or q.shape[1:] != (geo.q_heads, geo.head_dim):
        raise ValueError(f"q must be bf16 [B, {geo.q_heads}, {geo.head_dim}]")
    if out is None:
        out = torch.empty_like(q)
    if workspace is None or workspace.batch < B or workspace.max_seq_len < max_seq_len:
        workspace = DecodeWorkspace(geo, B, max_seq_len, split_tokens)
    _need_cuda(q, kv_va, seq_lens, out)
    if scale is None:
        scale = 1.0 / math.sqrt(geo.head_dim)
    maps_ptr = None
    if kv_maps is not None:
        _need_cuda(kv_maps)
        maps_ptr = kv_maps.data_ptr()
    fn = attn_lib().vt_decode_attention_chained if chained else attn_lib().vt_decode_attention
    rc = fn(
        ctypes.byref(_geo(geo)), layer, q.data_ptr(), kv_va.data_ptr(), maps_ptr,
        seq_lens.data_ptr(), B,
        max_seq_len, scale, out.data_ptr(), workspace.buf.data_ptr(), workspace.buf.numel(),
        workspace.split_tokens or split_tokens, _stream(stream))
    _check(rc, "vt_decode_attention")
    return out


def decode_attention_paged(q: torch.Tensor, pool: torch.Tensor, block_table: torch.Tensor,
                           seq_lens: torch.Tensor, layer: int, geo: KVGeometry, max_seq_len: int,
                           out: torch.Tensor | None = None,
                           workspace: DecodeWorkspace | None = None, scale: float | None = None,
                           split_tokens: int = 0,
                           stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """BASELINE (paper's comparison point): the CUDA-core decode over a paged
    KV pool addressed through ``block_table`` [B, max_blocks] int32."""
    B = q.shape[0]
    if out is None:
        out = torch.empty_like(q)
    if workspace is None:
        workspace = DecodeWorkspace(geo, B, max_seq_len, split_tokens)
    _need_cuda(q, pool, block_table, seq_lens, out)
    if scale is None:
        scale = 1.0 / math.sqrt(geo.head_dim)
    rc = attn_lib().vt_decode_attention_paged(
        ctypes.byref(_geo(geo)), layer, q.data_ptr(), pool.data_ptr(), block_table.data_ptr(),
        block_table.shape[1], seq_lens.data_ptr(), B, max_seq_len, scale, out.data_ptr(),
        workspace.buf.data_ptr(), workspace.buf.numel(), split_tokens, _stream(stream))
    _check(rc, "vt_decode_attention_paged")
    return out


def kv_append(k_new: torch.Tensor, v_new: torch.Tensor, kv_va: torch.Tensor,
              positions: torch.Tensor, geo: KVGeometry, layer_begin: int = 0,
              stream: torch.cuda.Stream | None = None) -> None:
    """Write ``[n_layers, B, Hkv, d]`` new-token K/V at ``positions[b]``."""
    _need_cuda(k_new, v_new, kv_va, positions)
    n_layers, B = k_new.shape[0], k_new.shape[1]
    rc = attn_lib().vt_kv_append(ctypes.byref(_geo(geo)), layer_begin, n_layers, k_new.data_ptr(),
                                 v_new.data_ptr(), kv_va.data_ptr(), positions.data_ptr(), B,
                                 _stream(stream))
    _check(rc, "vt_kv_append")


class PackedQKVWeight:
    """A QKV weight rewritten once into the streaming layout of the fused
    kernel (include/vt_attention.h vt_qkv_pack_weight): 128 x 64 blocks of 16
    KiB, [feature tile][k block], pre-swizzled for the MMA. Same byte size as
    the ``[(Hq + 2 Hkv) * d, hidden]`` nn.Linear weight it came from."""

    def __init__(self, w_qkv: torch.Tensor, stream: torch.cuda.Stream | None = None) -> None:
        if w_qkv.dtype != torch.bfloat16 or w_qkv.dim() != 2 or not w_qkv.is_contiguous():
            raise ValueError("w_qkv must be a contiguous bf16 [features, hidden] tensor")
        _need_cuda(w_qkv)
        self.shape = tuple(w_qkv.shape)
        self.data = torch.empty_like(w_qkv)
        rc = attn_lib().vt_qkv_pack_weight(w_qkv.data_ptr(), self.shape[0], self.shape[1],
                                           self.data.data_ptr(), _stream(stream))
        _check(rc, "vt_qkv_pack_weight")


def pack_qkv_weight(w_qkv: torch.Tensor,
                    stream: torch.cuda.Stream | None = None) -> PackedQKVWeight:
    return PackedQKVWeight(w_qkv, stream)


_QKV_WS: dict = {}


def qkv_workspace(geo: KVGeometry, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """The split-3 workspace of ``stream`` (include/vt_attention.h
    vt_qkv_workspace_bytes): zero-filled once, private to the stream, reused by
    every launch on it (its flags reset inside each launch)."""
    s = stream or torch.cuda.current_stream()
    nbytes = attn_lib().vt_qkv_workspace_bytes(ctypes.byref(_geo(geo)))
    key = (s.device.index, s.cuda_stream)
    ws = _QKV_WS.get(key)
    if ws is None or ws.numel() < nbytes:
        with torch.cuda.stream(s):
            ws = torch.zeros(nbytes, dtype=torch.uint8, device=s.device)
        _QKV_WS[key] = ws
    return ws


def qkv_append(x: torch.Tensor, w_qkv: "PackedQKVWeight | torch.Tensor", tok_req: torch.Tensor,
               tok_pos: torch.Tensor, kv_va: torch.Tensor, geo: KVGeometry, layer: int,
               q_out: torch.Tensor | None = None, split_k: int = 0,
               stream: torch.cuda.Stream | None = None,
               workspace: torch.Tensor | None = None) -> torch.Tensor:
    """Fused QKV projection + KV append (include/vt_attention.h vt_qkv_append).

    x ``[T, hidden]`` bf16; w_qkv a :class:`PackedQKVWeight` of the
    ``[(Hq + 2 Hkv) * d, hidden]`` bf16 weight (a plain tensor is packed on
    every call — an extra pass over the weight, for one-off use only). Returns
    q ``[T, Hq, d]``; K/V of token t land in the cache of request
    ``tok_req[t]`` at position ``tok_pos[t]`` of ``layer`` (its page must
    already be mapped). ``split_k`` = CTAs per 128-feature tile: 1, 2
    (the K halves on a 2-CTA cluster, reduced through distributed shared
    memory), or 3 (that pair plus a helper CTA whose partial of the first
    k blocks reaches the pair through L2; T <= 64 only); 0 picks
    automatically. ``workspace`` defaults to :func:`qkv_workspace` of the
    stream."""
    T, hidden = x.shape
    feats = (geo.q_heads + 2 * geo.kv_heads) * geo.head_dim
    if isinstance(w_qkv, torch.Tensor):
        w_qkv = PackedQKVWeight(w_qkv, stream)
    if x.dtype != torch.bfloat16 or w_qkv.shape != (feats, hidden):
        raise ValueError(f"x must be bf16 [T, hidden], w_qkv [{feats}, hidden]")
    if not x.is_contiguous():
        raise ValueError("x must be contiguous")
    if q_out is None:
        q_out = torch.empty(T, geo.q_heads, geo.head_dim, dtype=torch.bfloat16, device=x.device)
    _need_cuda(x, w_qkv.data, tok_req, tok_pos, kv_va, q_out)
    if workspace is None:
        workspace = qkv_workspace(geo, stream)
    rc = attn_lib().vt_qkv_append_ws(ctypes.byref(_geo(geo)), layer, x.data_ptr(),
                                     w_qkv.data.data_ptr(), hidden, T, tok_req.data_ptr(),
                                     tok_pos.data_ptr(), kv_va.data_ptr(), q_out.data_ptr(),
                                     split_k, workspace.data_ptr(), _stream(stream))
    _check(rc, "vt_qkv_append_ws")
    return q_out


def kv_tensor_maps(va: list[int], n_tokens: list[int], geo: KVGeometry,
                   device: str = "cuda") -> torch.Tensor:
    """Per-request TMA descriptors over the request VAs (host encode, one H2D
    copy). Chunk extent = ceil(n_tokens/tpc) — pass valid or mapped tokens."""
    B = len(va)
    raw = ctypes.create_string_buffer(B * 128 + 64)
    addr = (ctypes.addressof(raw) + 63) & ~63
    vas = (c_uint64 * B)(*va)
    lens = (c_int32 * B)(*n_tokens)
    rc = attn_lib().vt_kv_tensor_maps(ctypes.byref(_geo(geo)), ctypes.addressof(vas),
                                      ctypes.addressof(lens), B, addr)
    _check(rc, "vt_kv_tensor_maps")
    host = torch.frombuffer(bytearray(ctypes.string_at(addr, B * 128)), dtype=torch.uint8)
    return host.to(device)


prefill_kv_maps = kv_tensor_maps


class KVMapCache:
    """Device array of per-request TMA descriptors, re-encoded only for the
    requests whose mapped-chunk count changed (the VA never moves, so a
    request's descriptor changes once per newly mapped 2 MiB chunk).

    Uploads go through a ring of pinned staging buffers guarded by CUDA
    events, so an update never blocks the host on in-flight GPU work."""

    RING = 4

    def __init__(self, geo: KVGeometry, batch: int, device: str = "cuda") -> None:
        self.geo, self.batch = geo, batch
        self._raw = ctypes.create_string_buffer(batch * 128 + 64)
        self._addr = (ctypes.addressof(self._raw) + 63) & ~63
        self._key: list[tuple[int, int] | None] = [None] * batch
        self._host = [torch.empty(batch * 128, dtype=torch.uint8, pin_memory=True)
                      for _ in range(self.RING)]
        self._done: list[torch.cuda.Event | None] = [None] * self.RING
        self._slot = 0
        self.dev = torch.empty(batch * 128, dtype=torch.uint8, device=device)
        self.encodes = 0

    def update(self, va: list[int], mapped_tokens: list[int],
               stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        changed = [i for i in range(self.batch) if self._key[i] != (va[i], mapped_tokens[i])]
        if not changed:
            return self.dev
        g = ctypes.byref(_geo(self.geo))
        for i in changed:
            vas = (c_uint64 * 1)(va[i])
            n = (c_int32 * 1)(mapped_tokens[i])
            rc = attn_lib().vt_kv_tensor_maps(g, ctypes.addressof(vas), ctypes.addressof(n), 1,
                                              self._addr + 128 * i)
            _check(rc, "vt_kv_tensor_maps")
            self._key[i] = (va[i], mapped_tokens[i])
        self.encodes += len(changed)
        slot = self._slot
        self._slot = (slot + 1) % self.RING
        if self._done[slot] is not None:
            self._done[slot].synchronize()  # copy issued RING updates ago
        host = self._host[slot]
        ctypes.memmove(host.data_ptr(), self._addr, self.batch * 128)
        st = stream or torch.cuda.current_stream()
        with torch.cuda.stream(st):
            self.dev.copy_(host, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(st)
        self._done[slot] = ev
        return self.dev


def prefill_attention(q: torch.Tensor, kv_maps: torch.Tensor, start: torch.Tensor, layer: int,
                      geo: KVGeometry, out: torch.Tensor | None = None, scale: float | None = None,
                      stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """q ``[B, n_new, Hq, d]``: new tokens at ``[start_b, start_b + n_new)``
    attend causally to the KV already in the cache (shared prefix included);
    ``kv_maps`` from :func:`prefill_kv_maps` with kv_len = start + n_new."""
    B, n_new = q.shape[0], q.shape[1]
    if q.dtype != torch.bfloat16 or q.shape[2:] != (geo.q_heads, geo.head_dim):
        raise ValueError(f"q must be bf16 [B, n_new, {geo.q_heads}, {geo.head_dim}]")
    if out is None:
        out = torch.empty_like(q)
    _need_cuda(q, kv_maps, start, out)
    if scale is None:
        scale = 1.0 / math.sqrt(geo.head_dim)
    rc = attn_lib().vt_prefill_attention(ctypes.byref(_geo(geo)), layer, q.data_ptr(),
                                         kv_maps.data_ptr(), start.data_ptr(), B, n_new, scale,
                                         out.data_ptr(), _stream(stream))
    _check(rc, "vt_prefill_attention")
    return out


def prefill_attention_varlen(q: torch.Tensor, kv_maps: torch.Tensor, start: torch.Tensor,
                             q_offsets: torch.Tensor, max_n_new: int, layer: int, geo: KVGeometry,
                             out: torch.Tensor | None = None, scale: float | None = None,
                             stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Variable-length prefill in one launch: q packed ``[T, Hq, d]``, request
    b's ``n_b = q_offsets[b+1] - q_offsets[b]`` new tokens (rows
    ``[q_offsets[b], q_offsets[b+1])``) sit at positions
    ``[start_b, start_b + n_b)`` and attend causally to the cache. ``kv_maps``
    chunk extent must cover ``start_b + n_b``; ``max_n_new`` >= every n_b."""
    T = q.shape[0]
    B = start.shape[0]
    if q.dtype != torch.bfloat16 or q.shape[1:] != (geo.q_heads, geo.head_dim):
        raise ValueError(f"q must be bf16 [T, {geo.q_heads}, {geo.head_dim}]")
    if q_offsets.dtype != torch.int32 or q_offsets.shape != (B + 1,):
        raise ValueError("q_offsets must be int32 [batch + 1]")
    if out is None:
        out = torch.empty_like(q)
    _need_cuda(q, kv_maps, start, q_offsets, out)
    if scale is None:
        scale = 1.0 / math.sqrt(geo.head_dim)
    rc = attn_lib().vt_prefill_attention_varlen(
        ctypes.byref(_geo(geo)), layer, q.data_ptr(), kv_maps.data_ptr(), start.data_ptr(),
        q_offsets.data_ptr(), B, max_n_new, T, scale, out.data_ptr(), _stream(stream))
    _check(rc, "vt_prefill_attention_varlen")
    return out


def last_launches() -> int:
    return int(attn_lib().vt_attn_last_launches())
