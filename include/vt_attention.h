/*
 * vt_attention.h — C ABI of libvtattn.so: attention over a vTensor KV cache.
 *
 * The reference (kvsim) has no attention: its compute slot is the cost
 * formula at engine.py:499-511 (`prefill_cost_per_token * prefill_tokens +
 * decode_cost_per_request * batch`). These entry points are what that slot
 * calls instead (SURVEY.md §8(b) seam 2): decode over the batch, prefill /
 * prefix-prefill for admitted requests, and the KV append of new tokens.
 *
 * KV layout (kv_layout.py): every request owns one contiguous VA reserved for
 * max_seq_len (vt_reserve); chunk c of that VA (vt_map_page) holds tokens
 * [c*tpc, (c+1)*tpc) of ALL layers (config.py:48-50, 86-88). Inside a chunk,
 * block (layer, K|V, kv_head) is a dense [tpc][head_dim] bf16 tile at byte
 * offset ((layer*2 + kv)*kv_heads + head) * tpc*head_dim*2. Kernels address
 * K/V by arithmetic off the request's VA — there is no block table.
 *
 * All pointers are device pointers unless stated; every call is asynchronous
 * on `stream` (a cudaStream_t) and returns 0 or a cudaError_t value.
 */
#ifndef VT_ATTENTION_H_
#define VT_ATTENTION_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vt_kv_geometry {
  int32_t layers;           /* ModelGeometry.layers (config.py:42) */
  int32_t kv_heads;         /* ModelGeometry.kv_heads (config.py:43) */
  int32_t head_dim;         /* ModelGeometry.head_dim, must be 128 */
  int32_t q_heads;          /* query heads; q_heads / kv_heads = GQA group */
  int32_t tokens_per_chunk; /* SimConfig.tokens_per_chunk (config.py:86-88) */
  int32_t _pad;
  int64_t chunk_bytes;      /* SimConfig.chunk_size_bytes (2 MiB) */
} vt_kv_geometry;

/* Decode attention for one layer (row a27): for each request b and q head h,
 * out[b,h,:] = softmax(scale * q[b,h,:] . K[b, 0:len_b, h/G]^T) V[b, 0:len_b, h/G].
 *   q, out   : [batch, q_heads, head_dim] bf16
 *   kv_va    : [batch] u64 request VAs;  seq_lens : [batch] i32
 *   kv_maps  : NULL -> CUDA-core path (cp.async.bulk ring, FFMA2);
 *              else device copy of vt_kv_tensor_maps(...) -> tcgen05/TMEM path
 *   max_seq_len: host upper bound of seq_lens (sizes the split grid)
 *   workspace: >= vt_decode_workspace_bytes(...) bytes (fp32 split partials)
 *   split_tokens: KV tokens per work unit (multiple of 128), 0 = default */
int vt_decode_attention(const vt_kv_geometry* g, int32_t layer, const void* q,
                        const uint64_t* kv_va, const void* kv_maps, const int32_t* seq_lens,
                        int32_t batch, int32_t max_seq_len, float scale, void* out,
                        void* workspace, size_t workspace_bytes, int32_t split_tokens,
                        void* stream);

/* Same as vt_decode_attention, for a layer launched right after another
 * decode layer on the same stream (the layers of one step after its KV
 * append): the tcgen05 kernel then uses programmatic dependent launch, so its
 * first K/V tiles stream while the previous layer drains. Contract: the K/V
 * this call reads were written by kernels that completed before the previous
 * kernel on the stream started. Same arguments and errors. */
int vt_decode_attention_chained(const vt_kv_geometry* g, int32_t layer, const void* q,
                                const uint64_t* kv_va, const void* kv_maps,
                                const int32_t* seq_lens, int32_t batch, int32_t max_seq_len,
                                float scale, void* out, void* workspace, size_t workspace_bytes,
                                int32_t split_tokens, void* stream);
size_t vt_decode_workspace_bytes(const vt_kv_geometry* g, int32_t batch, int32_t max_seq_len,
                                 int32_t split_tokens);

/* BASELINE, not the product path: the same CUDA-core decode kernel reading a
 * paged KV cache (the layout the paper compares vTensor against, vLLM
 * PagedAttention / FA_paged). Block j of request b is
 * block_table[b*max_blocks + j] of a flat pool (block = one chunk-sized
 * [layers][K|V][kv_heads][tpc][head_dim] tile), i.e. one dependent table
 * lookup per block instead of VA arithmetic. */
int vt_decode_attention_paged(const vt_kv_geometry* g, int32_t layer, const void* q,
                              const void* pool_base, const int32_t* block_table,
                              int32_t max_blocks, const int32_t* seq_lens, int32_t batch,
                              int32_t max_seq_len, float scale, void* out, void* workspace,
                              size_t workspace_bytes, int32_t split_tokens, void* stream);

/* KV append (row a29): write the K/V of one new token per request at token
 * position positions[b], for layers [layer_begin, layer_begin + n_layers).
 *   k_new, v_new : [n_layers, batch, kv_heads, head_dim] bf16 */
int vt_kv_append(const vt_kv_geometry* g, int32_t layer_begin, int32_t n_layers,
                 const void* k_new, const void* v_new, const uint64_t* kv_va,
                 const int32_t* positions, int32_t batch, void* stream);

/* TMA descriptors over the request VAs (HOST function): one 128-byte
 * CUtensorMap per request, written to maps_host (batch*128 bytes, 64-byte
 * aligned), viewing va_host[b] as (d, token-in-chunk, (layer,K|V,head) block,
 * chunk) with chunk extent ceil(n_tokens_host[b] / tpc) — pass the mapped
 * token capacity (mapped_pages*tpc) or the valid length: the TMA never reads
 * unmapped VA. The caller copies the maps to device memory. A map only
 * changes when its request maps a new chunk (the VA itself never moves). */
int vt_kv_tensor_maps(const vt_kv_geometry* g, const uint64_t* va_host,
                      const int32_t* n_tokens_host, int32_t batch, void* maps_host);

/* Prefill / prefix-prefill (row a28), tcgen05/TMEM/TMA: n_new query tokens per
 * request at positions [start_b, start_b + n_new) attend causally to KV
 * [0, start_b + i] already in the cache (prefix chunks shared through the
 * rTree are mapped into the request's own VA, so they are read in place).
 *   q, out : [batch, n_new, q_heads, head_dim] bf16
 *   kv_maps: device copy of vt_kv_tensor_maps output;  start : [batch] i32 */
int vt_prefill_attention(const vt_kv_geometry* g, int32_t layer, const void* q,
                         const void* kv_maps, const int32_t* start, int32_t batch,
                         int32_t n_new, float scale, void* out, void* stream);

/* Variable-length prefill of the requests one engine step admits (the engine
 * charges sum(len - shared) prefill tokens, kvsim/engine.py:422-484, 500-504):
 * request b has n_b = q_offsets[b+1] - q_offsets[b] new tokens at positions
 * [start_b, start_b + n_b), one launch for the whole batch.
 *   q, out    : packed [total_tokens, q_heads, head_dim] bf16, request b's rows
 *               at [q_offsets[b], q_offsets[b+1])
 *   q_offsets : [batch + 1] i32 device, q_offsets[0] = 0, non-decreasing,
 *               q_offsets[batch] = total_tokens (cu_seqlens convention)
 *   max_n_new : host upper bound of n_b (sizes the tile grid)
 *   kv_maps   : chunk extent >= start_b + n_b;  start : [batch] i32 device
 * Same errors as vt_prefill_attention; q_offsets == NULL is an error. */
int vt_prefill_attention_varlen(const vt_kv_geometry* g, int32_t layer, const void* q,
                                const void* kv_maps, const int32_t* start,
                                const int32_t* q_offsets, int32_t batch, int32_t max_n_new,
                                int64_t total_tokens, float scale, void* out, void* stream);

/* Fused QKV projection + KV append, tcgen05:
 *   qkv = x . W^T    x [n_tokens, hidden] bf16, W [(Hq+2Hkv)*head_dim, hidden]
 *                    bf16 (nn.Linear layout) passed PACKED (vt_qkv_pack_weight),
 *                    fp32 accumulate
 * Q rows -> q_out [n_tokens, q_heads, head_dim] bf16; K and V rows are written
 * straight into request tok_req[t]'s VA (kv_va[tok_req[t]]) at token position
 * tok_pos[t] of `layer`, in the vt_kv_append layout (the page must be mapped:
 * the manager's extend ticket was waited on, kvsim/scheduler.py:189-205).
 * hidden % 64 == 0.  tok_req, tok_pos : [n_tokens] i32 (device);
 * kv_va : [n_req] u64 (device).
 * split_k = CTAs per 128-feature tile:
 *   1  one CTA streams the whole hidden dimension;
 *   2  the K halves on a 2-CTA cluster, reduced through distributed shared
 *      memory (no workspace);
 *   3  that pair plus a helper CTA streaming the first quarter of K, its fp32
 *      partial handed to the pair through L2 (1.5x the SMs streaming);
 *      n_tokens <= 64 and hidden >= 1024 only, needs `workspace`;
 *   0  auto: 3 when a workspace is given and the shape allows it, else 2
 *      unless the tile grid alone fills the SMs twice over, else 1.
 * workspace: vt_qkv_workspace_bytes(g) bytes, 256-byte aligned, zero-filled
 * once before first use (its flags reset themselves inside every launch),
 * private to one stream (launches on that stream may reuse it); NULL allowed
 * for split_k 0/1/2. vt_qkv_append == vt_qkv_append_ws with workspace NULL. */
size_t vt_qkv_workspace_bytes(const vt_kv_geometry* g);
int vt_qkv_append_ws(const vt_kv_geometry* g, int32_t layer, const void* x, const void* w_packed,
                     int32_t hidden, int32_t n_tokens, const int32_t* tok_req,
                     const int32_t* tok_pos, const uint64_t* kv_va, void* q_out, int32_t split_k,
                     void* workspace, void* stream);
int vt_qkv_append(const vt_kv_geometry* g, int32_t layer, const void* x, const void* w_packed,
                  int32_t hidden, int32_t n_tokens, const int32_t* tok_req,
                  const int32_t* tok_pos, const uint64_t* kv_va, void* q_out, int32_t split_k,
                  void* stream);

/* Rewrite a QKV weight W [feats, hidden] bf16 (row-major) once into the
 * streaming layout vt_qkv_append reads: [feats/128][hidden/64] blocks of
 * 128 x 64 bf16 (16 KiB, SWIZZLE_128B K-major), so each CTA's share of the
 * weight is one contiguous byte range. Same size as W; feats % 128 == 0,
 * hidden % 64 == 0, 16-byte aligned pointers. Stream-ordered. */
int vt_qkv_pack_weight(const void* w, int32_t feats, int32_t hidden, void* w_packed,
                       void* stream);

/* Number of kernel launches the last call on this thread issued (bench
 * accounting of "gpu_launches"). */
int32_t vt_attn_last_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* VT_ATTENTION_H_ */
