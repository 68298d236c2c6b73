// Host-side TMA descriptor encoding for the vTensor KV layout.
//
// A request's KV cache is one contiguous VA reserved for max_seq_len; chunk c
// holds tokens [c*tpc, (c+1)*tpc) of every layer, and inside a chunk block
// (layer, K|V, kv_head) is a dense [tpc][head_dim] bf16 tile (kv_layout.py).
// The 4-D tensor map (d, token-in-chunk, block, chunk) therefore addresses any
// 128-token x 64-dim tile of any (layer, K|V, head) with one TMA instruction,
// and only its chunk extent changes as the request grows: it is set to the
// number of chunks known to be mapped, so the TMA can never touch unmapped VA
// (out-of-range boxes are zero-filled by the hardware).

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/vt_attention.h"
#include "vt_tc_common.cuh"

namespace vt {

namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}
}  // namespace

int encode_tensor_map_bf16(CUtensorMap* m, void* base, int rank, const cuuint64_t* dims,
                           const cuuint64_t* strides, const cuuint32_t* box) {
  EncodeFn fn = encoder();
  if (!fn) return cudaErrorNotSupported;
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : cudaErrorInvalidValue;
}

}  // namespace vt

extern "C" int vt_kv_tensor_maps(const vt_kv_geometry* g, const uint64_t* va_host,
                                 const int32_t* n_tokens_host, int32_t batch, void* maps_host) {
  constexpr int kTile = 128;
  if (g->head_dim != 128) return cudaErrorInvalidValue;
  const int tpc = g->tokens_per_chunk;
  if (!((tpc < kTile && kTile % tpc == 0) || (tpc >= kTile && tpc % kTile == 0)))
    return cudaErrorInvalidValue;
  auto* maps = static_cast<CUtensorMap*>(maps_host);
  for (int b = 0; b < batch; ++b) {
    const cuuint64_t n_chunks = static_cast<cuuint64_t>((n_tokens_host[b] + tpc - 1) / tpc);
    const cuuint64_t dims[4] = {128, static_cast<cuuint64_t>(tpc),
                                static_cast<cuuint64_t>(2 * g->layers * g->kv_heads),
                                n_chunks > 0 ? n_chunks : 1};
    const cuuint64_t strides[3] = {256, static_cast<cuuint64_t>(tpc) * 256,
                                   static_cast<cuuint64_t>(g->chunk_bytes)};
    const cuuint32_t box[4] = {64, static_cast<cuuint32_t>(tpc < kTile ? tpc : kTile), 1,
                               static_cast<cuuint32_t>(tpc < kTile ? kTile / tpc : 1)};
    const int rc = vt::encode_tensor_map_bf16(&maps[b], reinterpret_cast<void*>(va_host[b]), 4,
                                              dims, strides, box);
    if (rc) return rc;
  }
  return 0;
}
