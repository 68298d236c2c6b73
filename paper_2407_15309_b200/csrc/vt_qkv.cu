// Fused QKV projection + KV append into the vTensor cache (SURVEY.md §8(f)
// row 2) — tcgen05 + TMEM, K split across a 2-CTA cluster, sm_100a.
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
// D^T = W x^T: a 128-feature weight block is the M=128 operand, the tokens are
// N (NT = 64/128/256 per tile), K = hidden in 64-element blocks. In decode
// (T = batch) the layer streams its 50 MB Llama-3-8B weight once — HBM-bound —
// so the work is laid out for streaming:
//
// * Packed weight. vt_qkv_pack_weight rewrites W once (weights are static)
//   into [feature tile][k block] blocks of 128 x 64 bf16 = 16 KiB, each already
//   in the SWIZZLE_128B K-major layout the MMA descriptor reads, so a CTA's
//   share of the weight is ONE contiguous byte range pulled with 16 KiB bulk
//   copies (no tensor map, sequential DRAM pages).
// * K split over a CTA pair (thread-block cluster of 2). Each feature tile is
//   computed by two CTAs, one per half of `hidden`, and each CTA finalises half
//   of the token columns: once both CTAs' MMAs are done (their rings are idle)
//   each writes the fp32 partial of the OTHER half straight from TMEM into the
//   peer's ring with asynchronous remote stores (st.async over distributed
//   shared memory, completing bytes on the peer's mbarrier), then adds the
//   peer's partial of its own half and stores it — the hand-off and the
//   stores split evenly over the pair (one-directional, with the lower CTA
//   storing everything, the tail was 2.5 us). The reduction never touches
//   global memory. Measured alternatives (tools/trace_qkv.py
//   timelines): a global split-K reduction (fp32 partials in L2 + arrival
//   counter) with a stream-K split over every SM streamed the weight at
//   6.9 TB/s but its chain of L2 round trips (~1 us each under load) added a
//   5-6 us tail; synchronous per-thread DSMEM stores of the partial took
//   1.4 us (scalar, coalesced) / 2.3 us (16-byte, strided); staging it in the
//   upper CTA's own ring for one bulk copy took 1.5 us and ran the same as
//   st.async end to end (12.7 us/layer).
//   Clusters of 2 all co-schedule (74 at one CTA per SM; clusters of 3 do
//   not: 45 < 48 tiles).
// * Split 3 (decode default, <= 64 tokens): the pair alone streams on 96 SMs
//   at ~57 GB/s each, below HBM; a helper CTA per tile takes the first
//   quarter of K and hands its fp32 partial to the pair through L2 (a
//   per-stream workspace + a self-resetting flag), so 144 SMs stream.
//
// Warp roles (192 threads): warp 0 producer (packed W + x tiles, 192 KiB
// ring), warp 1 MMA issuer (one elected lane), warps 2-5 epilogue (thread =
// TMEM lane = output feature). Stores go through a per-warp staging tile as
// 16-byte vectors; the destination rows (for K/V one per request, in as many
// different 2 MiB pages) are tabulated and prefetched into L2 while the
// weight streams, so their address translation is off the critical path.

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "../../include/vt_attention.h"
#include "vt_tc_common.cuh"

namespace vt {
namespace qkv {

constexpr int BM = 128;  // output features per tile
constexpr int BK = 64;   // hidden elements per k block (one 128-byte SW128 row)
constexpr int kBlockBytes = BM * BK * 2;  // one packed weight block (16 KiB)
constexpr int kThreads = 192;
#ifndef VT_QKV_RING_KB
#define VT_QKV_RING_KB 192  // (timing experiments override it: ring-depth sensitivity)
#endif
constexpr int kRingBytes = VT_QKV_RING_KB * 1024;

template <int NT>
struct Cfg {
  static constexpr int kXBytes = NT * BK * 2;
  static constexpr int kStageBytes = kBlockBytes + kXBytes;
  static constexpr int kStages = kRingBytes / kStageBytes;
  static constexpr int kTmemCols = NT;
  // K-split pair: the peer's fp32 partial of this CTA's token half lands in a
  // buffer of its own (when it fits beside the ring), so it can be sent the
  // moment the peer's accumulator is ready, with no "ring free" handshake
  static constexpr int kPartialBytes = NT / 2 * 128 * 4;
  static constexpr bool kDedicated = kPartialBytes <= 16 * 1024;
  static constexpr size_t kDynSmem = kRingBytes + (kDedicated ? kPartialBytes : 0) + 1024;
  static_assert(kStages >= 2, "ring too small");
  static_assert(NT / 2 * BM * 4 <= kRingBytes, "the peer's half partial must fit the ring");
};

struct Args {
  const uint8_t* w_packed;    // [mtiles][kblocks][16 KiB]
  __nv_bfloat16* q_out;       // [T, Hq, d]
  const uint64_t* kv_va;      // [n_req]
  const int32_t* tok_req;     // [T]
  const int32_t* tok_pos;     // [T]
  int32_t n_tokens, hq, hkv, tpc, layer, kblocks;
  int64_t chunk_bytes;
  int32_t mtiles, helper_kb;  // KS == 3: feature tiles, k blocks of each tile's helper CTA
  float* helper_part;         // KS == 3 workspace: [mtiles][64 tokens][128] fp32
  int32_t* helper_flag;       //                    [mtiles], zero between launches
  int32_t l2_prefetch;        // k blocks past the first ring to pull into L2 at entry
  int32_t l2_prefetch_helper; // the same for KS == 3 helper CTAs
};

// KS == 3 (pair + helper): a third CTA per feature tile streams the first
// `helper_kb` k blocks and hands its fp32 partial [NT=64 tokens][128 features]
// to the tile's pair through L2 (each warp store one full 128-byte line); the
// pair reads it while its own DSMEM hand-off is in flight and adds it last. The helper has
// fewer blocks than the pair CTAs, so its partial is in L2 before the pair's
// stream ends. Flags count up (helper +1, each pair CTA +1 after reading) and
// the last reader resets them, inside one launch (the next launch's helper
// writes only after griddepcontrol.wait). The partials and flags live in a
// caller-provided workspace (vt_qkv_workspace_bytes), private to the stream.
constexpr int kHelperPartFloats = 64 * BM;

// ------------------------------------------------- cluster / DSMEM helpers --
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// Start-up form: the only cross-CTA state published before it is the
// mbarrier initialisation, which fence.mbarrier_init.release.cluster already
// orders, so the arrive can be relaxed (a release arrive also waits for this
// thread's just-issued weight copies to be translated: ~2 us at launch).
__device__ __forceinline__ void cluster_sync_init() {
#ifdef VT_QKV_RELEASE_ARRIVE
  cluster_sync();
#else
  __syncthreads();  // CTA-local: TMEM address and barriers (bar.sync orders shared memory)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
#endif
}
// Address of the same shared variable in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t peer_addr(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void arrive_peer(uint32_t bar_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_addr)
               : "memory");
}
#ifdef VT_QKV_TRACE
// Debug timeline (tools/gpu_trace_qkv.sh): per CTA, %globaltimer at
// 0 entry, 1 setup done, 2 first W copy issued, 3 first stage landed,
// 4 last stage landed, 5 last MMA committed, 6 accumulator ready,
// 7 peer handshake done, 8 partial received / sent, 9 epilogue done,
// 10 (split 3) helper: partial published / pair: helper flag seen,
// 11 first ring issued, 12 TMEM allocated, 13 cluster barrier passed,
// 14 griddepcontrol.wait returned (producer). Two launch slots (layer & 1),
// so back-to-back launches show on one clock.
__device__ long long g_qkv_trace[2][256][16];
__device__ __forceinline__ void trace(int i, int slot) {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (blockIdx.y == 0 && blockIdx.x < 256) g_qkv_trace[slot & 1][blockIdx.x][i] = t;
}
#define QKV_TRACE(i) trace(i, a.layer)
#else
#define QKV_TRACE(i)
#endif

// KS = CTAs per feature tile (1, or 2 = cluster pair). Grid: (mtiles * KS, token tiles).
template <int NT, int KS>
__global__ void __launch_bounds__(kThreads, 1)
    qkv_append_kernel(const __grid_constant__ CUtensorMap x_map, const Args a) {
  using C = Cfg<NT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  __shared__ uint64_t full[C::kStages], empty[C::kStages], acc_full;
  __shared__ uint64_t peer_ready;    // the peer CTA's ring is free (its MMAs are done)
  __shared__ uint64_t partial_full;  // the peer's partial of our token half has landed
  __shared__ uint64_t helper_ready;  // KS == 3: the helper's partial is in L2 (seen by warp 0)
  __shared__ uint64_t row_dst[NT];   // destination of each token's 256-byte head row
  __shared__ __align__(16) __nv_bfloat16 stage_out[4][16][32];  // per epilogue warp
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tt = blockIdx.y;                           // token tile
  const int KB = a.kblocks;
  // feature tile, K range, and (KS == 3) whether this CTA is a tile's helper
  int m, kb0, kb1;
  uint32_t half = 0;
  bool helper = false;
  if constexpr (KS == 3) {
    const int cl = blockIdx.x >> 1;
    const uint32_t r = cluster_rank();
    const int hcl = (a.mtiles + 1) >> 1;  // helper clusters first (dispatched before the pairs)
    if (cl < hcl) {
      helper = true;
      m = cl * 2 + static_cast<int>(r);
      kb0 = 0;
      kb1 = m < a.mtiles ? a.helper_kb : 0;  // odd tile count: one idle helper
    } else {
      m = cl - hcl;
      half = r;
      const int mid = a.helper_kb + (KB - a.helper_kb) / 2;
      kb0 = r == 0 ? a.helper_kb : mid;
      kb1 = r == 0 ? mid : KB;
    }
  } else {
    m = blockIdx.x / KS;
    half = KS == 2 ? cluster_rank() : 0;  // K half of this CTA
    const int mid = KS == 2 ? KB / 2 : KB;  // (finishing the lower half earlier was measured: no gain)
    kb0 = half == 0 ? 0 : mid;
    kb1 = half == 0 ? mid : KB;
  }
  const bool pair = KS == 2 || (KS == 3 && !helper);  // exchanges partials with a cluster peer
  if (threadIdx.x == 0) QKV_TRACE(0);

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&acc_full, 1);
    mbar_init(&peer_ready, 1);
    mbar_init(&partial_full, 1);  // armed with the partial's bytes; the peer's st.async completes it
    mbar_init(&helper_ready, 1);
    fence_mbar_init();
    // The weights do not depend on the previous kernel or on the peer: the
    // first ring's worth is issued before the cluster barrier, TMEM
    // allocation and PDL wait (only this CTA's own barriers are involved).
    const uint64_t once = l2_evict_first_policy();
    const int n = kb1 - kb0;
    const uint64_t wsrc = reinterpret_cast<uint64_t>(a.w_packed) +
                          (static_cast<uint64_t>(m) * KB + kb0) * kBlockBytes;
    for (int i = 0; i < min(n, C::kStages); ++i) {
      mbar_arrive_expect_tx(&full[i], C::kStageBytes);
      bulk_g2s(ring + i * C::kStageBytes, wsrc + static_cast<uint64_t>(i) * kBlockBytes,
               kBlockBytes, &full[i], once);
      if (i == 0) QKV_TRACE(2);
    }
    // The next blocks into L2 as well: this CTA becomes resident as the
    // previous launch's CTAs leave, so these reads fill the HBM gap of that
    // launch's tail and of the dependency wait (x, hence the MMAs, only
    // arrive after griddepcontrol.wait).
    const int pf = helper ? a.l2_prefetch_helper : a.l2_prefetch;
    for (int i = C::kStages; i < min(n, C::kStages + pf); ++i)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(wsrc + static_cast<uint64_t>(i) * kBlockBytes),
                   "r"(kBlockBytes)
                   : "memory");
    QKV_TRACE(11);
  }
  if (warp == 1) tc::alloc(&tmem_base, C::kTmemCols);
  if (threadIdx.x == 32) QKV_TRACE(12);
  tc::fence_before();
  if constexpr (KS >= 2) {
    cluster_sync_init();  // the peer's barriers are initialised before any remote arrive
  } else {
    __syncthreads();
  }
  if (threadIdx.x == 0) QKV_TRACE(13);
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  tc::grid_launch_dependents();  // the next launch may start its own prologue
  if (threadIdx.x == 0) QKV_TRACE(1);
  if constexpr (KS >= 2 && C::kDedicated) {
    // the peer's partial may land any time after its MMAs: armed up front
    if (pair && threadIdx.x == 64) mbar_arrive_expect_tx(&partial_full, C::kPartialBytes);
  }

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t once = l2_evict_first_policy();  // W is read once per token tile
      const uint64_t keep = l2_evict_last_policy();   // x is re-read by every feature tile
      const int n = kb1 - kb0;
      const uint64_t wsrc = reinterpret_cast<uint64_t>(a.w_packed) +
                            (static_cast<uint64_t>(m) * KB + kb0) * kBlockBytes;
      // Programmatic dependent launch: the weights do not depend on the
      // previous kernel, so the first ring's worth streams in while that
      // kernel drains; x (its output in a real layer stack) only after
      // griddepcontrol.wait.
      const int pre = min(n, C::kStages);  // issued at barrier init
      tc::grid_dependency_wait();
      QKV_TRACE(14);
      for (int i = 0; i < n; ++i) {
        const int st = i % C::kStages;
        uint8_t* sw = ring + st * C::kStageBytes;
        if (i >= pre) {
          mbar_wait(&empty[st], ((i / C::kStages) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[st], C::kStageBytes);
          bulk_g2s(sw, wsrc + static_cast<uint64_t>(i) * kBlockBytes, kBlockBytes, &full[st], once);
        }
        tc::tma_load_2d(sw + kBlockBytes, &x_map, &full[st], (kb0 + i) * BK, tt * NT, keep);
      }
      if constexpr (KS == 3) {
        // the producer is idle from here: it watches for the helper's partial
        // (an L2 round trip per poll) so the epilogue does not have to
        if (!helper) {
          int f;
          uint32_t spins = 0;
          do {
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(f) : "l"(a.helper_flag + m) : "memory");
            if (++spins == (1u << 28)) asm volatile("trap;");  // a lost helper: fail, never hang
          } while (f < 1);
          QKV_TRACE(10);
          mbar_arrive(&helper_ready);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    constexpr uint32_t id = tc::idesc_bf16(BM, NT, false, false);
    constexpr uint32_t hi = tc::sdesc_hi(1024);
    for (int i = 0; i < kb1 - kb0; ++i) {
      const int st = i % C::kStages;
      mbar_wait(&full[st], (i / C::kStages) & 1);
      tc::fence_after();
#ifdef VT_QKV_TRACE
      if (lane == 0 && i == 0) QKV_TRACE(3);
      if (lane == 0 && i == kb1 - kb0 - 1) QKV_TRACE(4);
#endif
      const uint32_t base = smem_u32(ring + st * C::kStageBytes);
      const uint32_t la = tc::sdesc_lo(base, 16);
      const uint32_t lb = tc::sdesc_lo(base + kBlockBytes, 16);
      if (tc::elect_one()) {
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk)
          tc::mma_ss(tmem, la + 2 * kk, hi, lb + 2 * kk, hi, id, (i > 0 || kk > 0) ? 1u : 0u);
        tc::commit(&empty[st]);
        if (i == kb1 - kb0 - 1) {
          tc::commit(&acc_full);
          QKV_TRACE(5);
        }
      }
      __syncwarp();
    }
  } else {
    // ------------------------------ epilogue ---------------------------------
    // A feature tile is exactly one head of q, K or V (feature boundaries are
    // multiples of 128), so for every token its 128 outputs form one
    // contiguous 256-byte row at the destination.
    tc::grid_dependency_wait();  // token tables, q_out and the cache belong to the previous kernel until now
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;  // this thread's output feature within the tile
    const int ep = threadIdx.x - 64;      // 0..127
    if constexpr (KS == 3) {
      if (helper) {
        // fp32 partial of all NT tokens -> L2, then publish
        if (kb1 > kb0) {
          mbar_wait(&acc_full, 0);
          tc::fence_after();
          const uint32_t lane_addr = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
          float* dstp = a.helper_part + static_cast<size_t>(m) * kHelperPartFloats + row;
#pragma unroll 1
          for (int c = 0; c < NT; c += 32) {
            uint32_t r0[16], r1[16];
            tc::ld16(lane_addr + c, r0);
            tc::ld16(lane_addr + c + 16, r1);
            tc::wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              __stcg(dstp + (c + i) * BM, __uint_as_float(r0[i]));
              __stcg(dstp + (c + 16 + i) * BM, __uint_as_float(r1[i]));
            }
          }
          // the CTA barrier orders every thread's stores before thread 0's
          // gpu-scope release (cumulativity), so one release publishes them all
          named_bar_sync(1, 128);
          if (ep == 0) {
            asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(a.helper_flag + m) : "memory");
            QKV_TRACE(10);
          }
        }
      }
    }
    if (!helper) {
    // With a CTA pair each CTA finalises half of the token columns: it sends
    // its partial of the OTHER half to the peer and adds the peer's partial of
    // its own half, so hand-off and stores are split evenly across the pair.
    constexpr int kHalfNT = KS >= 2 ? NT / 2 : NT;
    const int my_c0 = static_cast<int>(half) * kHalfNT;          // token columns finalised here
    const int peer_c0 = KS >= 2 ? (1 - static_cast<int>(half)) * kHalfNT : 0;
    // [kHalfNT][BM] fp32 partial from the peer: its own buffer, or our ring once idle
    float* peer_part = reinterpret_cast<float*>(C::kDedicated ? ring + kRingBytes : ring);
    {
      const int kind = m < a.hq ? 0 : (m < a.hq + a.hkv ? 1 : 2);  // q | K | V
      const int head = kind == 0 ? m : (kind == 1 ? m - a.hq : m - a.hq - a.hkv);
      for (int i = my_c0 + ep; i < my_c0 + kHalfNT; i += 128) {
        const int t = tt * NT + i;
        uint64_t dst = 0;
        if (t < a.n_tokens) {
          if (kind == 0) {
            dst = reinterpret_cast<uint64_t>(a.q_out) + (static_cast<uint64_t>(t) * a.hq + head) * 256;
          } else {
            const int pos = a.tok_pos[t];
            const int chunk = pos / a.tpc;
            dst = a.kv_va[a.tok_req[t]] + static_cast<uint64_t>(chunk) * a.chunk_bytes +
                  (static_cast<uint64_t>(a.layer * 2 + kind - 1) * a.hkv + head) * a.tpc * 256 +
                  static_cast<uint64_t>(pos - chunk * a.tpc) * 256;
          }
          asm volatile("prefetch.global.L2 [%0];" ::"l"(dst));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(dst + 128));
        }
        row_dst[i] = dst;
      }
      named_bar_sync(1, 128);
    }
    float hp[KS == 3 ? kHalfNT : 1];  // KS == 3: the helper's partial of our token half
    mbar_wait(&acc_full, 0);
    tc::fence_after();
    if (ep == 0) QKV_TRACE(6);
    const uint32_t lane_addr = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    if constexpr (KS >= 2) {
      // our MMAs are done, so our ring is free for the peer's partial; once
      // the peer's is free too, asynchronous remote stores of the peer's half
      // straight from the accumulator, completing bytes on its barrier
      if constexpr (!C::kDedicated) {
        if (ep == 0) {
          mbar_arrive_expect_tx(&partial_full, kHalfNT * BM * 4);
          arrive_peer(peer_addr(&peer_ready, 1 - half));
        }
        mbar_wait(&peer_ready, 0);
      }
      if (ep == 0) QKV_TRACE(7);
      const uint32_t dst = peer_addr(peer_part, 1 - half);
      const uint32_t bar = peer_addr(&partial_full, 1 - half);
#pragma unroll 1
      for (int c = 0; c < kHalfNT; c += 32) {
        uint32_t r0[16], r1[16];
        tc::ld16(lane_addr + peer_c0 + c, r0);
        tc::ld16(lane_addr + peer_c0 + c + 16, r1);
        tc::wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
                           dst + ((c + i) * BM + row) * 4),
                       "r"(r0[i]), "r"(bar)
                       : "memory");
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
                           dst + ((c + 16 + i) * BM + row) * 4),
                       "r"(r1[i]), "r"(bar)
                       : "memory");
        }
      }
      if constexpr (KS == 3) {
        // read from L2 while our st.async hand-off is in flight (the helper
        // normally published before this CTA's own stream ended)
        mbar_wait(&helper_ready, 0);
        const float* srcp = a.helper_part + static_cast<size_t>(m) * kHelperPartFloats + my_c0 * BM + row;
#pragma unroll
        for (int i = 0; i < kHalfNT; ++i) hp[i] = __ldcg(srcp + i * BM);
      }
      mbar_wait(&partial_full, 0);
      if (ep == 0) QKV_TRACE(8);
    }
#pragma unroll 1
    for (int c = 0; c < kHalfNT; c += 32) {
      uint32_t r0[16], r1[16];
      tc::ld16(lane_addr + my_c0 + c, r0);
      tc::ld16(lane_addr + my_c0 + c + 16, r1);
      tc::wait_ld();
      float v[32];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        v[i] = __uint_as_float(r0[i]);
        v[16 + i] = __uint_as_float(r1[i]);
      }
      if (KS >= 2) {  // two K halves: one fp32 add (commutative, so bit-reproducible)
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] += peer_part[(c + i) * BM + row];
      }
      if constexpr (KS == 3) {  // + the helper's k blocks, in a fixed order
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] += hp[c + i];
      }
      // transpose through this warp's staging tile (16 tokens x 32
      // features), then 16-byte stores (4 per 64-byte token row segment)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          stage_out[quarter][i][lane] = __float2bfloat16_rn(v[h * 16 + i]);
        __syncwarp();
#pragma unroll
        for (int j = lane; j < 64; j += 32) {
          const uint64_t dst = row_dst[my_c0 + c + h * 16 + (j >> 2)];
          if (dst)
            *reinterpret_cast<uint4*>(dst + quarter * 64 + (j & 3) * 16) =
                *reinterpret_cast<const uint4*>(&stage_out[quarter][j >> 2][(j & 3) * 8]);
        }
        __syncwarp();
      }
    }
    if (ep == 0) QKV_TRACE(9);
    if constexpr (KS == 3) {
      // both pair CTAs have read the helper's partial: the second resets the flag
      if (ep == 0 && atomicAdd(a.helper_flag + m, 1) == 2) atomicExch(a.helper_flag + m, 0);
    }
    }  // !helper
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 1) tc::dealloc(tmem, C::kTmemCols);
}

// W [feats, hidden] row-major -> [feats/128][hidden/64][128 x 64] blocks in the
// SWIZZLE_128B K-major layout (16-byte chunk c of row r stored at c ^ (r & 7)).
// One thread per 16-byte chunk of the output (coalesced stores).
__global__ void pack_weight_kernel(const uint4* __restrict__ w, int hidden, long long n_chunks,
                                   uint4* __restrict__ out) {
  const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n_chunks) return;
  const int kblocks = hidden / BK;
  const long long blk = idx >> 10;  // 1024 chunks per 16 KiB block
  const int within = static_cast<int>(idx & 1023);
  const int r = within >> 3;
  const int c = (within & 7) ^ (r & 7);
  const long long m = blk / kblocks;
  const int kb = static_cast<int>(blk - m * kblocks);
  out[idx] = w[((m * BM + r) * hidden + kb * BK + c * 8) >> 3];
}

template <int NT, int KS>
int launch(const CUtensorMap& xm, const Args& a, int mtiles, int ttiles, cudaStream_t stream) {
  const size_t smem = KS >= 2 ? Cfg<NT>::kDynSmem : kRingBytes + 1024;
  static std::atomic<uint64_t> attr_devices{0};
  set_smem_limit_once(qkv_append_kernel<NT, KS>, smem, attr_devices);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(KS == 3 ? ((mtiles + 1) / 2 + mtiles) * 2 : mtiles * KS, ttiles, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = KS == 3 ? 2 : KS;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, qkv_append_kernel<NT, KS>, xm, a);
}

}  // namespace qkv
}  // namespace vt

using namespace vt::qkv;

#ifdef VT_QKV_TRACE
extern "C" int vt_qkv_trace(long long* host) {
  return cudaMemcpyFromSymbol(host, g_qkv_trace, sizeof(g_qkv_trace));
}
#endif

extern "C" int vt_qkv_pack_weight(const void* w, int32_t feats, int32_t hidden, void* w_packed,
                                  void* stream) {
  if (feats <= 0 || hidden <= 0 || feats % BM || hidden % BK) return cudaErrorInvalidValue;
  if ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(w_packed)) & 15)
    return cudaErrorInvalidValue;
  const long long n_chunks = static_cast<long long>(feats) * hidden / 8;
  const int threads = 256;
  pack_weight_kernel<<<static_cast<unsigned>((n_chunks + threads - 1) / threads), threads, 0,
                       static_cast<cudaStream_t>(stream)>>>(static_cast<const uint4*>(w), hidden,
                                                            n_chunks, static_cast<uint4*>(w_packed));
  return cudaGetLastError();
}

static size_t qkv_flags_bytes(int mtiles) {
  return (static_cast<size_t>(mtiles) * sizeof(int32_t) + 255) & ~static_cast<size_t>(255);
}

extern "C" size_t vt_qkv_workspace_bytes(const vt_kv_geometry* g) {
  const int mtiles = g->q_heads + 2 * g->kv_heads;  // one tile per head (head_dim 128)
  return qkv_flags_bytes(mtiles) + static_cast<size_t>(mtiles) * kHelperPartFloats * sizeof(float);
}

extern "C" int vt_qkv_append(const vt_kv_geometry* g, int32_t layer, const void* x,
                             const void* w_packed, int32_t hidden, int32_t n_tokens,
                             const int32_t* tok_req, const int32_t* tok_pos, const uint64_t* kv_va,
                             void* q_out, int32_t split_k, void* stream) {
  return vt_qkv_append_ws(g, layer, x, w_packed, hidden, n_tokens, tok_req, tok_pos, kv_va, q_out,
                          split_k, nullptr, stream);
}

extern "C" int vt_qkv_append_ws(const vt_kv_geometry* g, int32_t layer, const void* x,
                                const void* w_packed, int32_t hidden, int32_t n_tokens,
                                const int32_t* tok_req, const int32_t* tok_pos,
                                const uint64_t* kv_va, void* q_out, int32_t split_k,
                                void* workspace, void* stream) {
  if (g->head_dim != 128 || hidden <= 0 || hidden % BK) return cudaErrorInvalidValue;
  if (reinterpret_cast<uintptr_t>(w_packed) & 15) return cudaErrorInvalidValue;
  if (split_k > 3) return cudaErrorInvalidValue;
  if (n_tokens <= 0) return 0;
  const int feats = (g->q_heads + 2 * g->kv_heads) * 128;
  const int mtiles = feats / BM;
  const int kblocks = hidden / BK;
  const int nt = n_tokens <= 64 ? 64 : (n_tokens <= 128 ? 128 : 256);
  const int ttiles = (n_tokens + nt - 1) / nt;
  // Auto: with a workspace and one tile of <= 64 tokens (decode), three CTAs
  // per feature tile (a cluster pair + a helper through L2: 1.5x the SMs
  // streaming); else two (the K halves on a cluster pair) unless the tile
  // grid alone already covers the SMs several times over.
  const bool three_ok = workspace && nt == 64 && ttiles == 1 && kblocks >= 16;
  const int ks = split_k > 0 ? split_k
                             : (three_ok ? 3 : (kblocks >= 2 && mtiles * ttiles < 296 ? 2 : 1));
  if (ks == 2 && kblocks < 2) return cudaErrorInvalidValue;
  // split 3 needs the workspace, one 64-token tile and k blocks for three CTAs
  if (ks == 3 && (!workspace || nt != 64 || ttiles != 1 || kblocks < 4)) return cudaErrorInvalidValue;
  if (ks == 3 && (reinterpret_cast<uintptr_t>(workspace) & 255)) return cudaErrorInvalidValue;

  CUtensorMap xm;
  {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(hidden), static_cast<cuuint64_t>(n_tokens)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(hidden) * 2};
    const cuuint32_t box[2] = {BK, static_cast<cuuint32_t>(nt)};
    int rc = vt::encode_tensor_map_bf16(&xm, const_cast<void*>(x), 2, dims, strides, box);
    if (rc) return rc;
  }
  Args a{};
  a.w_packed = static_cast<const uint8_t*>(w_packed);
  a.q_out = static_cast<__nv_bfloat16*>(q_out);
  a.kv_va = kv_va;
  a.tok_req = tok_req;
  a.tok_pos = tok_pos;
  a.n_tokens = n_tokens;
  a.hq = g->q_heads;
  a.hkv = g->kv_heads;
  a.tpc = g->tokens_per_chunk;
  a.layer = layer;
  a.kblocks = kblocks;
  a.chunk_bytes = g->chunk_bytes;
  a.mtiles = mtiles;
  if (workspace) {
    a.helper_flag = static_cast<int32_t*>(workspace);
    a.helper_part = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + qkv_flags_bytes(mtiles));
  }
  {
    static const int helper_q8 = [] {  // helper share of K in 64ths (experiment knob)
      const char* e = std::getenv("VT_QKV_HELPER_Q64");
      return e ? std::atoi(e) : 16;
    }();
    a.helper_kb = std::max(1, std::min(kblocks - 2, kblocks * helper_q8 / 64));
    static const int l2_pf = [] {  // k blocks past the ring prefetched into L2 (A/B knob)
      const char* e = std::getenv("VT_QKV_L2_PREFETCH");
      return e ? std::atoi(e) : 4;  // r2as sweep at B=64: 0/4/8/16/64 -> 10.60/10.34/10.40/10.77/10.77 us
    }();
    static const int l2_pf_helper = [] {
      const char* e = std::getenv("VT_QKV_L2_PREFETCH_HELPER");
      return e ? std::atoi(e) : -1;
    }();
    a.l2_prefetch = ttiles == 1 ? l2_pf : 0;  // several token tiles re-read W from L2 anyway
    a.l2_prefetch_helper = l2_pf_helper >= 0 && ttiles == 1 ? l2_pf_helper : a.l2_prefetch;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int rc;
  if (ks == 3) {
    rc = launch<64, 3>(xm, a, mtiles, ttiles, s);
  } else if (ks == 2) {
    rc = nt == 64    ? launch<64, 2>(xm, a, mtiles, ttiles, s)
         : nt == 128 ? launch<128, 2>(xm, a, mtiles, ttiles, s)
                     : launch<256, 2>(xm, a, mtiles, ttiles, s);
  } else {
    rc = nt == 64    ? launch<64, 1>(xm, a, mtiles, ttiles, s)
         : nt == 128 ? launch<128, 1>(xm, a, mtiles, ttiles, s)
                     : launch<256, 1>(xm, a, mtiles, ttiles, s);
  }
  if (rc) return rc;
  return cudaGetLastError();
}
