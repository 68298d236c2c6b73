// KV append (row a29): write one new token's K and V per request straight into
// the request's vTensor VA at position positions[b], for a range of layers.
// The page holding that position must be mapped (the manager's extend ran and
// its ticket was waited on before this launch).
//
// One warp per (layer, request, kv head) row pair: 16 lanes move the K row and
// 16 the V row, 16 B each (row = head_dim * 2 = 256 B).

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/vt_attention.h"

namespace {

__global__ void kv_append_kernel(const uint4* __restrict__ k_new, const uint4* __restrict__ v_new,
                                 const uint64_t* __restrict__ kv_va,
                                 const int32_t* __restrict__ positions, int batch, int hkv,
                                 int layer_begin, int n_layers, int tpc, int64_t chunk_bytes) {
  const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t rows = static_cast<int64_t>(n_layers) * batch * hkv;
  if (row >= rows) return;
  const int h = static_cast<int>(row % hkv);
  const int b = static_cast<int>((row / hkv) % batch);
  const int l = static_cast<int>(row / (static_cast<int64_t>(hkv) * batch));
  const int pos = positions[b];
  const int c = pos / tpc;
  const int64_t head_bytes = static_cast<int64_t>(tpc) * 256;
  const int kv = lane >> 4;  // 0: K, 1: V
  const int64_t off = static_cast<int64_t>(c) * chunk_bytes +
                      (static_cast<int64_t>((layer_begin + l) * 2 + kv) * hkv + h) * head_bytes +
                      static_cast<int64_t>(pos - c * tpc) * 256 + (lane & 15) * 16;
  const uint4* src = kv ? v_new : k_new;
  uint4* dst = reinterpret_cast<uint4*>(kv_va[b] + off);
  *dst = src[row * 16 + (lane & 15)];
}

}  // namespace

extern "C" int vt_kv_append(const vt_kv_geometry* g, int32_t layer_begin, int32_t n_layers,
                            const void* k_new, const void* v_new, const uint64_t* kv_va,
                            const int32_t* positions, int32_t batch, void* stream) {
  if (g->head_dim != 128) return cudaErrorInvalidValue;
  if (batch <= 0 || n_layers <= 0) return 0;
  const int64_t rows = static_cast<int64_t>(n_layers) * batch * g->kv_heads;
  const int threads = 256;
  const int64_t blocks = (rows * 32 + threads - 1) / threads;
  kv_append_kernel<<<static_cast<unsigned>(blocks), threads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(k_new), static_cast<const uint4*>(v_new), kv_va, positions, batch,
      g->kv_heads, layer_begin, n_layers, g->tokens_per_chunk, g->chunk_bytes);
  return cudaGetLastError();
}
