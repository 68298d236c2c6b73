// Temporary: the tcgen05 prefill lands in vt_prefill.cu.
#include <cuda_runtime.h>
#include "../../include/vt_attention.h"
extern "C" int vt_prefill_attention(const vt_kv_geometry*, int32_t, const void*, const uint64_t*,
                                    const int32_t*, int32_t, int32_t, float, void*, void*) {
  return cudaErrorNotSupported;
}
