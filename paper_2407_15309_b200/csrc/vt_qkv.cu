// Fused QKV projection + KV append into the vTensor cache (SURVEY.md §8(f)
// row 2) — tcgen05 + TMEM + TMA, split-K with an arrival-counter reduction, sm_100a.
//
//   qkv[t, f] = sum_k x[t, k] * W[f, k]          (bf16 in, fp32 accumulate)
//   f <  Hq*d           -> q_out[t, f]                         (bf16)
//   f in the K / V part -> straight into request tok_req[t]'s VA at position
//                          tok_pos[t] of `layer` (the vt_kv_append layout), so
//                          the new token's K/V never round-trip through a
//                          staging buffer (the progress contract of
//                          kvsim/scheduler.py:189-205: the page holding
//                          tok_pos[t] is mapped before this launch).
//
// D^T = W x^T: the weight tile is the M=128 operand (output features), the
// tokens are N (NT = 64/128/256 per tile), K = hidden in 64-element SW128
// blocks. Decode (T = batch) streams the 50 MB Llama-3-8B QKV weight once
// per layer — HBM-bound — so the K dimension is split into KS slices
// (n_feature_tiles x KS ~ 148 SMs, one wave): each CTA accumulates its slice
// in TMEM, writes the fp32 partial to an L2-resident workspace and the last
// slice to arrive reduces and stores (a self-resetting arrival counter per
// tile). A thread-block-cluster/DSMEM reduction was measured first: clusters
// of 3 do not all co-schedule on the GPCs (48 x 3 CTAs ran in two waves).
//
// Grid: (feature tile, K slice, token tile); one output tile per CTA.
//
// Warp roles (192 threads): warp 0 TMA producer (W and x tiles, 192 KiB
// ring: 8 stages at NT=64), warp 1 MMA issuer (one elected lane), warps 2-5
// epilogue (thread = TMEM lane = output feature; 16-byte row stores after a
// transpose through shared memory).

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/vt_attention.h"
#include "vt_tc_common.cuh"

namespace vt {
namespace qkv {

constexpr int BM = 128;  // output features per tile
constexpr int BK = 64;   // hidden elements per k-block (one 128-byte SW128 row)
constexpr int kThreads = 192;
constexpr int kRingBytes = 192 * 1024;

template <int NT>
struct Cfg {
  static constexpr int kStageBytes = BM * BK * 2 + NT * BK * 2;
  static constexpr int kStages = kRingBytes / kStageBytes;
  static_assert(kStages >= 2, "ring too small");
};

struct Args {
  __nv_bfloat16* q_out;       // [T, Hq, d]
  const uint64_t* kv_va;      // [n_req]
  const int32_t* tok_req;     // [T]
  const int32_t* tok_pos;     // [T]
  int32_t n_tokens, hidden, hq, hkv, tpc, layer, ks, kblocks;
  int64_t chunk_bytes;
  float* ws;                  // [mtiles][ks][NT][BM] fp32 split-K partials
  int* counters;              // [mtiles] arrival counters (zero between launches)
};

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) { tc::ld16(taddr, r); }

template <int NT>
__global__ void __launch_bounds__(kThreads, 1)
    qkv_append_kernel(const __grid_constant__ CUtensorMap w_map,
                      const __grid_constant__ CUtensorMap x_map, const Args a) {
  using C = Cfg<NT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  __shared__ uint64_t full[C::kStages], empty[C::kStages], acc_full;
  __shared__ uint64_t row_dst[NT];  // destination of each token's 256-byte head row
  __shared__ int last_flag;
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int mtile = blockIdx.x;
  const int slice = blockIdx.y;  // K slice of this CTA
  const int kb0 = slice * a.kblocks / a.ks;
  const int kb1 = (slice + 1) * a.kblocks / a.ks;
  const int tt = blockIdx.z;  // token tile
  const int tile_id = mtile * gridDim.z + tt;  // split-K reduction group

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&acc_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) tc::alloc(&tmem_base, NT);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  tc::grid_launch_dependents();  // the next launch may start its own prologue

  int it = 0;  // ring position
  {
    if (warp == 0) {
      if (lane == 0) {
        const uint64_t once = l2_evict_first_policy();  // W is read once per token tile
        const uint64_t keep = l2_evict_last_policy();   // x is re-read by every feature tile
        // Programmatic dependent launch: the weights do not depend on the
        // previous kernel, so the first ring's worth of W streams in while
        // that kernel drains; x (its output in a real layer stack) is read
        // only after griddepcontrol.wait.
        const int pre = min(kb1 - kb0, C::kStages);
        for (int i = 0; i < pre; ++i) {
          mbar_arrive_expect_tx(&full[i], C::kStageBytes);
          tc::tma_load_2d(ring + i * C::kStageBytes, &w_map, &full[i], (kb0 + i) * BK, mtile * BM,
                          once);
        }
        tc::grid_dependency_wait();
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int st = it % C::kStages;
          uint8_t* sw = ring + st * C::kStageBytes;
          if (it >= pre) {
            mbar_wait(&empty[st], ((it / C::kStages) & 1) ^ 1);
            mbar_arrive_expect_tx(&full[st], C::kStageBytes);
            tc::tma_load_2d(sw, &w_map, &full[st], kb * BK, mtile * BM, once);
          }
          tc::tma_load_2d(sw + BM * BK * 2, &x_map, &full[st], kb * BK, tt * NT, keep);
        }
      }
      __syncwarp();
    } else if (warp == 1) {
      constexpr uint32_t id = tc::idesc_bf16(BM, NT, false, false);
      constexpr uint32_t hi = tc::sdesc_hi(1024);
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        const int st = it % C::kStages;
        mbar_wait(&full[st], (it / C::kStages) & 1);
        tc::fence_after();
        const uint32_t base = smem_u32(ring + st * C::kStageBytes);
        const uint32_t la = tc::sdesc_lo(base, 16);
        const uint32_t lb = tc::sdesc_lo(base + BM * BK * 2, 16);
        if (tc::elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            tc::mma_ss(tmem, la + 2 * kk, hi, lb + 2 * kk, hi, id, (kb > kb0 || kk > 0) ? 1u : 0u);
          tc::commit(&empty[st]);
          if (kb == kb1 - 1) tc::commit(&acc_full);
        }
        __syncwarp();
      }
    } else {
      it += kb1 - kb0;
    }

    // ------------------------------ epilogue ---------------------------------
    // The feature tile is exactly one head of q, K or V (feature boundaries
    // are multiples of 128), so for every token its 128 outputs form one
    // contiguous 256-byte row at the destination. While the MMAs run, the
    // epilogue warps tabulate those row addresses. Split-K: every K slice
    // writes its fp32 partial tile to the workspace and bumps the tile's
    // arrival counter; the slice that arrives last sums the others into its
    // own accumulator, resets the counter, transposes the bf16 tile through
    // shared memory and stores 16-byte vectors (16 lanes per 256-byte row).
    if (warp >= 2) {
      tc::grid_dependency_wait();  // token tables, q_out and the cache belong to the previous kernel until now
      const int quarter = warp & 3;
      const int row = quarter * 32 + lane;  // this thread's output feature within the tile
      const int ep = threadIdx.x - 64;      // 0..127
      {
        const int hq = a.hq, hkv = a.hkv;
        const int kind = mtile < hq ? 0 : (mtile < hq + hkv ? 1 : 2);  // q | K | V
        const int head = kind == 0 ? mtile : (kind == 1 ? mtile - hq : mtile - hq - hkv);
        for (int i = ep; i < NT; i += 128) {
          const int t = tt * NT + i;
          uint64_t dst = 0;
          if (t < a.n_tokens) {
            if (kind == 0) {
              dst = reinterpret_cast<uint64_t>(a.q_out) + (static_cast<uint64_t>(t) * hq + head) * 256;
            } else {
              const int pos = a.tok_pos[t];
              const int chunk = pos / a.tpc;
              dst = a.kv_va[a.tok_req[t]] + static_cast<uint64_t>(chunk) * a.chunk_bytes +
                    (static_cast<uint64_t>(a.layer * 2 + kind - 1) * hkv + head) * a.tpc * 256 +
                    static_cast<uint64_t>(pos - chunk * a.tpc) * 256;
            }
          }
          row_dst[i] = dst;
        }
      }
      mbar_wait(&acc_full, 0);
      tc::fence_after();
      const uint32_t lane_addr = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
      bool last = true;
      if (a.ks > 1) {
        // partial [NT][BM] fp32 (coalesced across the warp's 32 features)
        float* mine = a.ws + (static_cast<size_t>(tile_id) * a.ks + slice) * NT * BM;
#pragma unroll 1
        for (int c = 0; c < NT; c += 16) {
          uint32_t r[16];
          tmem_ld16(lane_addr + c, r);
          tc::wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) __stcg(mine + (c + i) * BM + row, __uint_as_float(r[i]));
        }
        __threadfence();
        named_bar_sync(1, 128);
        if (ep == 0) {
          const int old = atomicAdd(a.counters + tile_id, 1);
          last_flag = old == a.ks - 1;
          if (last_flag) a.counters[tile_id] = 0;  // self-resetting for the next launch
        }
        named_bar_sync(1, 128);
        last = last_flag;
        if (last) __threadfence();
      }
      if (last) {
        __nv_bfloat16* tile_t = reinterpret_cast<__nv_bfloat16*>(ring);  // [NT][BM] bf16
#pragma unroll 1
        for (int c = 0; c < NT; c += 16) {
          uint32_t r[16];
          tmem_ld16(lane_addr + c, r);
          tc::wait_ld();
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
          for (int p = 0; p < a.ks; ++p) {
            if (p == slice) continue;
            const float* src = a.ws + (static_cast<size_t>(tile_id) * a.ks + p) * NT * BM;
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] += __ldcg(src + (c + i) * BM + row);
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) tile_t[(c + i) * BM + row] = __float2bfloat16_rn(v[i]);
        }
        named_bar_sync(1, 128);
        const int sub = ep & 15;
#pragma unroll 4
        for (int i = ep >> 4; i < NT; i += 8) {
          const uint64_t dst = row_dst[i];
          if (dst)
            *reinterpret_cast<uint4*>(dst + sub * 16) =
                *reinterpret_cast<const uint4*>(tile_t + i * BM + sub * 8);
        }
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 1) tc::dealloc(tmem, NT);
}

template <int NT>
int launch(const CUtensorMap& wm, const CUtensorMap& xm, const Args& a, int mtiles,
           cudaStream_t stream) {
  const size_t smem = kRingBytes + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(qkv_append_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    attr = true;
  }
  const int ttiles = (a.n_tokens + NT - 1) / NT;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(mtiles, a.ks, ttiles);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, qkv_append_kernel<NT>, wm, xm, a);
}

// Split-K workspace: grown on demand, counters zeroed once (the kernel resets
// each counter after use). One per process; calls are stream-ordered.
struct Workspace {
  float* partials = nullptr;
  size_t partial_bytes = 0;
  int* counters = nullptr;
  int n_counters = 0;
};
int workspace(size_t partial_bytes, int n_counters, Workspace** out) {
  static Workspace w;
  if (partial_bytes > w.partial_bytes) {
    if (w.partials) cudaFree(w.partials);
    if (cudaMalloc(&w.partials, partial_bytes) != cudaSuccess) return cudaErrorMemoryAllocation;
    w.partial_bytes = partial_bytes;
  }
  if (n_counters > w.n_counters) {
    if (w.counters) cudaFree(w.counters);
    if (cudaMalloc(&w.counters, n_counters * sizeof(int)) != cudaSuccess)
      return cudaErrorMemoryAllocation;
    cudaMemset(w.counters, 0, n_counters * sizeof(int));
    w.n_counters = n_counters;
  }
  *out = &w;
  return 0;
}

}  // namespace qkv
}  // namespace vt

using namespace vt::qkv;

extern "C" int vt_qkv_append(const vt_kv_geometry* g, int32_t layer, const void* x, const void* w,
                             int32_t hidden, int32_t n_tokens, const int32_t* tok_req,
                             const int32_t* tok_pos, const uint64_t* kv_va, void* q_out,
                             int32_t split_k, void* stream) {
  if (g->head_dim != 128 || hidden <= 0 || hidden % BK) return cudaErrorInvalidValue;
  if (n_tokens <= 0) return 0;
  const int feats = (g->q_heads + 2 * g->kv_heads) * 128;
  const int mtiles = feats / BM;
  const int kblocks = hidden / BK;
  const int nt = n_tokens <= 64 ? 64 : (n_tokens <= 128 ? 128 : 256);
  const int ttiles = (n_tokens + nt - 1) / nt;
  int ks = split_k;
  if (ks <= 0) {  // fill the SMs: feature tiles x token tiles x K slices ~ one wave
    static int n_sm = 0;
    if (!n_sm) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    }
    // Measured (Llama-3-8B, T=64): ks 1/2/3 = 18.2/16.0/16.9 us — past two
    // slices the extra reduction outweighs the added SMs (the stream itself
    // is ~8 us; launch, pipeline fill and the reduction chain are the rest).
    ks = n_sm / (mtiles * ttiles);
    if (ks > 2) ks = 2;
  }
  ks = ks < 1 ? 1 : (ks > 8 ? 8 : ks);
  if (ks > kblocks) ks = kblocks;
  Workspace* wsp = nullptr;
  if (ks > 1) {
    const int groups = mtiles * ttiles;
    int rc = workspace(static_cast<size_t>(groups) * ks * nt * BM * 4, groups, &wsp);
    if (rc) return rc;
  }

  CUtensorMap wm, xm;
  {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(hidden), static_cast<cuuint64_t>(feats)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(hidden) * 2};
    const cuuint32_t box[2] = {BK, BM};
    int rc = vt::encode_tensor_map_bf16(&wm, const_cast<void*>(w), 2, dims, strides, box);
    if (rc) return rc;
  }
  {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(hidden), static_cast<cuuint64_t>(n_tokens)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(hidden) * 2};
    const cuuint32_t box[2] = {BK, static_cast<cuuint32_t>(nt)};
    int rc = vt::encode_tensor_map_bf16(&xm, const_cast<void*>(x), 2, dims, strides, box);
    if (rc) return rc;
  }
  Args a{};
  a.q_out = static_cast<__nv_bfloat16*>(q_out);
  a.kv_va = kv_va;
  a.tok_req = tok_req;
  a.tok_pos = tok_pos;
  a.n_tokens = n_tokens;
  a.hidden = hidden;
  a.hq = g->q_heads;
  a.hkv = g->kv_heads;
  a.tpc = g->tokens_per_chunk;
  a.layer = layer;
  a.ks = ks;
  a.kblocks = kblocks;
  a.chunk_bytes = g->chunk_bytes;
  a.ws = wsp ? wsp->partials : nullptr;
  a.counters = wsp ? wsp->counters : nullptr;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int rc;
  if (nt == 64)
    rc = launch<64>(wm, xm, a, mtiles, s);
  else if (nt == 128)
    rc = launch<128>(wm, xm, a, mtiles, s);
  else
    rc = launch<256>(wm, xm, a, mtiles, s);
  if (rc) return rc;
  return cudaGetLastError();
}
