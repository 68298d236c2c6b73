// Prefill / prefix-prefill attention over a vTensor KV cache — tcgen05 + TMEM +
// TMA, sm_100a (row a28).
//
// CTA = (request b, q head h, tile of 128 new query tokens). The new tokens sit
// at absolute positions [start_b, start_b + n_new) and attend causally to the
// cache [0, pos]; the first start_b keys are the rTree-shared prefix chunks,
// which are mapped into the request's own VA (hard links), so the kernel reads
// them in place through the same TMA descriptor — no gather, no block table.
//
// Warp roles (192 threads):
//   warp 0    TMA producer: Q tile once; K and V tiles of 128 keys into a
//             2-stage ring (cp.async.bulk.tensor, SWIZZLE_128B). K/V come from
//             a per-request 4-D tensor map over the request VA
//             (d, token-in-chunk, (layer,K|V,head) block, chunk) whose chunk
//             extent is ceil(kv_len/tpc): the TMA never touches unmapped VA.
//   warp 1    MMA issuer (one thread): S_j = Q K_j^T into a double-buffered
//             TMEM tile (tcgen05.mma kind::f16, M=128 N=128, K-major A and B),
//             then O += P_j V_j (A = P from smem K-major, B = V MN-major) into a
//             TMEM accumulator. S_{j+1} is issued before PV_j so the tensor
//             core works while softmax_j runs. Completion via tcgen05.commit.
//   warps 2-5 softmax / correction / epilogue, thread <-> TMEM lane <-> query
//             row: tcgen05.ld of S, causal + length mask, online softmax in
//             the exp2 domain, O rescale in TMEM (tcgen05.ld/st, skipped when
//             no row of the warp moved its max), P -> smem as bf16 in the
//             SW128 K-major layout, final O / l -> bf16 -> global.

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/vt_attention.h"
#include "vt_tc_common.cuh"

namespace vt {
namespace pf {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int D = 128;
constexpr int kStages = 2;
constexpr int kThreads = 192;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kOCol = 256;  // S double buffer at columns 0 and 128

struct __align__(1024) Smem {
  __nv_bfloat16 q[2][BM * 64];            // SW128 K-major: d 0-63 | d 64-127
  __nv_bfloat16 k[kStages][2][BN * 64];   // SW128 K-major (keys x d)
  __nv_bfloat16 v[kStages][2][BN * 64];   // SW128, read as MN-major B (d x keys)
  __nv_bfloat16 p[2][BM * 64];            // SW128 K-major: keys 0-63 | 64-127
  uint64_t q_full;
  uint64_t k_full[kStages], k_empty[kStages];
  uint64_t v_full[kStages], v_empty[kStages];
  uint64_t s_full[2];
  uint64_t p_full;
  uint64_t pv_done;
  uint32_t tmem_base;
};

// UMMA shared-memory descriptor, SWIZZLE_128B, sm_100 version bits.
__device__ __forceinline__ uint64_t sdesc(const void* p, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  const uint64_t a = smem_u32(p);
  return ((a >> 4) & 0x3FFFull) | (static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}

// Instruction descriptor: bf16 x bf16 -> f32, M=128, N=128, A K-major.
__host__ __device__ constexpr uint32_t idesc(bool b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) |
         (static_cast<uint32_t>(BN >> 3) << 17) | (static_cast<uint32_t>(BM >> 4) << 24);
}

__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t id,
                                     uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

#define VT_R32(x)                                                                              \
  "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]),          \
      "=r"(x[7]), "=r"(x[8]), "=r"(x[9]), "=r"(x[10]), "=r"(x[11]), "=r"(x[12]), "=r"(x[13]),  \
      "=r"(x[14]), "=r"(x[15]), "=r"(x[16]), "=r"(x[17]), "=r"(x[18]), "=r"(x[19]),            \
      "=r"(x[20]), "=r"(x[21]), "=r"(x[22]), "=r"(x[23]), "=r"(x[24]), "=r"(x[25]),            \
      "=r"(x[26]), "=r"(x[27]), "=r"(x[28]), "=r"(x[29]), "=r"(x[30]), "=r"(x[31])
#define VT_W32(x)                                                                              \
  "r"(x[0]), "r"(x[1]), "r"(x[2]), "r"(x[3]), "r"(x[4]), "r"(x[5]), "r"(x[6]), "r"(x[7]),      \
      "r"(x[8]), "r"(x[9]), "r"(x[10]), "r"(x[11]), "r"(x[12]), "r"(x[13]), "r"(x[14]),        \
      "r"(x[15]), "r"(x[16]), "r"(x[17]), "r"(x[18]), "r"(x[19]), "r"(x[20]), "r"(x[21]),      \
      "r"(x[22]), "r"(x[23]), "r"(x[24]), "r"(x[25]), "r"(x[26]), "r"(x[27]), "r"(x[28]),      \
      "r"(x[29]), "r"(x[30]), "r"(x[31])

// 32 consecutive fp32 columns of this thread's TMEM lane.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : VT_R32(r)
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(
          taddr),
      VT_W32(r)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

struct Args {
  __nv_bfloat16* out;       // [B, n_new, Hq, D]
  const CUtensorMap* kv;    // [B] per-request maps
  const int32_t* start;     // [B]
  int32_t n_new, hq, hkv, tpc, layer;
  float scale_log2;
};

__global__ void __launch_bounds__(kThreads, 1)
    prefill_kernel(const __grid_constant__ CUtensorMap q_map, const Args a) {
  extern __shared__ uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                      ~static_cast<uintptr_t>(1023));
  const int n_qtiles = gridDim.x;
  const int t = n_qtiles - 1 - static_cast<int>(blockIdx.x);  // longest tiles first
  const int h = blockIdx.y;
  const int b = blockIdx.z;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int start = a.start[b];
  const int kv_len = start + a.n_new;
  const int q_last = min(a.n_new, (t + 1) * BM);  // exclusive, relative to start
  const int n_kv = (start + q_last + BN - 1) / BN;
  const int hk = h / (a.hq / a.hkv);
  const int blk_k = (a.layer * 2 + 0) * a.hkv + hk;
  const int blk_v = (a.layer * 2 + 1) * a.hkv + hk;
  const CUtensorMap* kvmap = a.kv + b;

  if (warp == 0 && lane == 0) {
    mbar_init(&sm.q_full, 1);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&sm.k_full[i], 1);
      mbar_init(&sm.k_empty[i], 1);
      mbar_init(&sm.v_full[i], 1);
      mbar_init(&sm.v_empty[i], 1);
    }
    mbar_init(&sm.s_full[0], 1);
    mbar_init(&sm.s_full[1], 1);
    mbar_init(&sm.p_full, 128);
    mbar_init(&sm.pv_done, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm.tmem_base)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    // ------------------------------ TMA producer ------------------------------
    if (lane == 0) {
      tma_prefetch_desc(&q_map);
      tma_prefetch_desc(kvmap);
      const uint64_t keep = l2_evict_last_policy();   // K/V re-read by the group's heads
      const uint64_t once = l2_evict_first_policy();
      mbar_arrive_expect_tx(&sm.q_full, 2 * BM * 64 * 2);
      tma_load_4d(sm.q[0], &q_map, &sm.q_full, 0, h, t * BM, b, once);
      tma_load_4d(sm.q[1], &q_map, &sm.q_full, 64, h, t * BM, b, once);
      for (int j = 0; j < n_kv; ++j) {
        const int s = j % kStages;
        const uint32_t ph = (j / kStages) & 1;
        const int tok0 = j * BN;
        const int c1 = tok0 % a.tpc;
        const int c3 = tok0 / a.tpc;
        if (j >= kStages) mbar_wait(&sm.k_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&sm.k_full[s], 2 * BN * 64 * 2);
        tma_load_4d(sm.k[s][0], kvmap, &sm.k_full[s], 0, c1, blk_k, c3, keep);
        tma_load_4d(sm.k[s][1], kvmap, &sm.k_full[s], 64, c1, blk_k, c3, keep);
        if (j >= kStages) mbar_wait(&sm.v_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&sm.v_full[s], 2 * BN * 64 * 2);
        tma_load_4d(sm.v[s][0], kvmap, &sm.v_full[s], 0, c1, blk_v, c3, keep);
        tma_load_4d(sm.v[s][1], kvmap, &sm.v_full[s], 64, c1, blk_v, c3, keep);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------- MMA issuer -------------------------------
    if (lane == 0) {
      constexpr uint32_t id_s = idesc(false);
      constexpr uint32_t id_pv = idesc(true);
      mbar_wait(&sm.q_full, 0);
      auto issue_pv = [&](int i) {
        mbar_wait(&sm.p_full, i & 1);
        mbar_wait(&sm.v_full[i % kStages], (i / kStages) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
          const uint64_t ad = sdesc(reinterpret_cast<const uint8_t*>(sm.p[kk >> 2]) + 32 * (kk & 3),
                                    16, 1024);
          const uint64_t bd = sdesc(reinterpret_cast<const uint8_t*>(sm.v[i % kStages][0]) +
                                        kk * 16 * 128,
                                    BN * 128, 1024);
          umma(tmem + kOCol, ad, bd, id_pv, (i > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(&sm.pv_done);
        umma_commit(&sm.v_empty[i % kStages]);
      };
      for (int j = 0; j < n_kv; ++j) {
        const int s = j % kStages;
        mbar_wait(&sm.k_full[s], (j / kStages) & 1);
        tc_fence_after();
        const uint32_t sc = static_cast<uint32_t>((j & 1) * BN);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t ad = sdesc(reinterpret_cast<const uint8_t*>(sm.q[kk >> 2]) + 32 * (kk & 3),
                                    16, 1024);
          const uint64_t bd = sdesc(reinterpret_cast<const uint8_t*>(sm.k[s][kk >> 2]) + 32 * (kk & 3),
                                    16, 1024);
          umma(tmem + sc, ad, bd, id_s, kk > 0 ? 1u : 0u);
        }
        umma_commit(&sm.s_full[j & 1]);
        umma_commit(&sm.k_empty[s]);
        if (j >= 1) issue_pv(j - 1);
      }
      issue_pv(n_kv - 1);
    }
    __syncwarp();
  } else {
    // ------------------------ softmax / correction / out ----------------------
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_addr = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    const int qpos = start + t * BM + row;  // absolute position of this query row
    float m_run = -INFINITY, l_run = 0.f;
    const float sl2 = a.scale_log2;
    for (int j = 0; j < n_kv; ++j) {
      const int kpos0 = j * BN;
      mbar_wait(&sm.s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      float s[BN];
      {
        uint32_t r[32];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          tmem_ld32(lane_addr + (j & 1) * BN + 32 * c, r);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) s[32 * c + i] = __uint_as_float(r[i]);
        }
      }
      const bool edge = kpos0 + BN - 1 > start + t * BM || kpos0 + BN > kv_len;
      if (edge) {
#pragma unroll
        for (int i = 0; i < BN; ++i) {
          const int kp = kpos0 + i;
          if (kp > qpos || kp >= kv_len) s[i] = -INFINITY;
        }
      }
      float mx = s[0];
#pragma unroll
      for (int i = 1; i < BN; ++i) mx = fmaxf(mx, s[i]);
      const float m_new = fmaxf(m_run, mx * sl2);
      const float alpha = ex2(m_run - m_new);
      float sum = 0.f;
#pragma unroll
      for (int i = 0; i < BN; ++i) {
        s[i] = ex2(fmaf(s[i], sl2, -m_new));
        sum += s[i];
      }
      l_run = l_run * alpha + sum;
      m_run = m_new;

      if (j >= 1) {
        mbar_wait(&sm.pv_done, (j - 1) & 1);  // PV_{j-1} done: P free, O stable
        tc_fence_after();
        if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t r[32];
            tmem_ld32(lane_addr + kOCol + 32 * c, r);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
            tmem_st32(lane_addr + kOCol + 32 * c, r);
          }
          tmem_wait_st();
        }
      }
      if (j == n_kv - 1 && kpos0 + BN > kv_len) {
        // Rows past kv_len may hold stale/uninitialised bytes of the last
        // mapped chunk: zero them so 0 * NaN cannot reach the accumulator.
        const int s = j % kStages;
        mbar_wait(&sm.v_full[s], (j / kStages) & 1);
        if (kpos0 + row >= kv_len) {
          uint4 z = make_uint4(0, 0, 0, 0);
          uint4* r0 = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(sm.v[s][0]) + row * 128);
          uint4* r1 = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(sm.v[s][1]) + row * 128);
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            r0[c] = z;
            r1[c] = z;
          }
        }
      }
      // P row -> smem, bf16, SW128 K-major: 16-byte chunk c of the 128-byte
      // row r lives at position c ^ (r % 8).
#pragma unroll
      for (int ci = 0; ci < BN / 8; ++ci) {
        const int kb = ci >> 3;
        const int c = ci & 7;
        uint4 w;
        w.x = pack_bf16(s[8 * ci + 0], s[8 * ci + 1]);
        w.y = pack_bf16(s[8 * ci + 2], s[8 * ci + 3]);
        w.z = pack_bf16(s[8 * ci + 4], s[8 * ci + 5]);
        w.w = pack_bf16(s[8 * ci + 6], s[8 * ci + 7]);
        *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(sm.p[kb]) + row * 128 +
                                  ((c ^ (row & 7)) << 4)) = w;
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&sm.p_full);
    }
    // epilogue
    mbar_wait(&sm.pv_done, (n_kv - 1) & 1);
    tc_fence_after();
    const int tok = t * BM + row;
    const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
    __nv_bfloat16* dst = a.out + ((static_cast<int64_t>(b) * a.n_new + tok) * a.hq + h) * D;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t r[32];
      tmem_ld32(lane_addr + kOCol + 32 * c, r);
      tmem_wait_ld();
      if (tok < a.n_new) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(r[i + 0]) * inv, __uint_as_float(r[i + 1]) * inv);
          w.y = pack_bf16(__uint_as_float(r[i + 2]) * inv, __uint_as_float(r[i + 3]) * inv);
          w.z = pack_bf16(__uint_as_float(r[i + 4]) * inv, __uint_as_float(r[i + 5]) * inv);
          w.w = pack_bf16(__uint_as_float(r[i + 6]) * inv, __uint_as_float(r[i + 7]) * inv);
          *reinterpret_cast<uint4*>(dst + 32 * c + i) = w;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(kTmemCols));
  }
}

}  // namespace pf
}  // namespace vt

using namespace vt::pf;

extern "C" int vt_prefill_attention(const vt_kv_geometry* g, int32_t layer, const void* q,
                                    const void* kv_maps, const int32_t* start, int32_t batch,
                                    int32_t n_new, float scale, void* out, void* stream) {
  if (g->head_dim != D || g->q_heads % g->kv_heads) return cudaErrorInvalidValue;
  if (batch <= 0 || n_new <= 0) return 0;
  CUtensorMap qmap;
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(g->q_heads),
                              static_cast<cuuint64_t>(n_new), static_cast<cuuint64_t>(batch)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(D * 2),
                                 static_cast<cuuint64_t>(g->q_heads) * D * 2,
                                 static_cast<cuuint64_t>(n_new) * g->q_heads * D * 2};
  const cuuint32_t box[4] = {64, 1, static_cast<cuuint32_t>(BM), 1};
  int rc = vt::encode_tensor_map_bf16(&qmap, const_cast<void*>(q), 4, dims, strides, box);
  if (rc) return rc;
  Args a{};
  a.out = static_cast<__nv_bfloat16*>(out);
  a.kv = static_cast<const CUtensorMap*>(kv_maps);
  a.start = start;
  a.n_new = n_new;
  a.hq = g->q_heads;
  a.hkv = g->kv_heads;
  a.tpc = g->tokens_per_chunk;
  a.layer = layer;
  a.scale_log2 = scale * 1.4426950408889634f;
  const size_t smem = sizeof(Smem) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(prefill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    attr = true;
  }
  dim3 grid((n_new + BM - 1) / BM, g->q_heads, batch);
  prefill_kernel<<<grid, kThreads, smem, static_cast<cudaStream_t>(stream)>>>(qmap, a);
  return cudaGetLastError();
}
