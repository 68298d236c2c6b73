// Prefill / prefix-prefill attention over a vTensor KV cache — tcgen05 + TMEM +
// TMA, sm_100a (row a28).
//
// CTA = (request b, q-head pair {h0, h0+1} of one GQA group, tile of 128 new
// query tokens). The new tokens sit at absolute positions
// [start_b, start_b + n_new) and attend causally to the cache [0, pos]; the
// first start_b keys are the rTree-shared prefix chunks, mapped into the
// request's own VA (hard links), so the kernel reads them in place through the
// request's TMA descriptor — no gather, no block table.
//
// The two heads of a pair ("slots") share every K/V tile and have identical
// masks, so one TMA stream feeds two independent softmax pipelines and the
// tensor core alternates between them: while softmax warpgroup 0 turns S0(j)
// into P0(j), the tensor core runs slot 1's {PV1(j-1), S1(j)} and vice versa.
// (For odd GQA groups, e.g. MHA, a CTA runs one slot.) Every MMA is
// M128 x N128 x K16: on sm_100a switching between N=64 and N=128 shapes drains
// the tensor pipe (tools/mma_probe.cu: an 8 x N64 + 4 x N128 mix runs at 53% of
// the rate of either shape alone), so scores are computed in 128-key blocks.
//
// Warp roles (384 threads; registers moved to the softmax warpgroups with
// setmaxnreg):
//   warp 8     TMA producer: both slots' Q tiles once; K and V tiles of 128
//              keys into 2-stage rings (cp.async.bulk.tensor, SWIZZLE_128B).
//              K/V come from a per-request 4-D tensor map over the request VA
//              (d, token-in-chunk, (layer,K|V,head) block, chunk) whose chunk
//              extent is ceil(kv_len/tpc): the TMA never touches unmapped VA.
//   warp 9     MMA issuer. Per slot s: S_s(0), then per key block j one group
//                O_s  += P_s(j) V_j        (TS: P read from TMEM, V MN-major)
//                S_s(j+1) = Q_s K_{j+1}^T  (SS)
//              S_s(j+1) overwrites the columns of P_s(j) right after the PV
//              that consumes it (tcgen05.mma executes in issue order). The
//              whole warp walks the schedule (descriptors stay in uniform
//              registers); one elected lane issues.
//   warps 0-3  softmax slot 0;  warps 4-7  softmax slot 1. Thread <-> TMEM
//              lane <-> query row: tcgen05.ld of S, causal + length mask, online
//              softmax in the exp2 domain with a lazy running max (O and l are
//              rescaled only when a row's max grows by more than 2^8, which is
//              exact because numerator and denominator share the stale max),
//              packed fp32x2 arithmetic, 3/8 of the exponentials on the
//              FMA pipe (polynomial) to offload MUFU, P -> TMEM as packed bf16
//              over the first 64 S columns, final O / l -> bf16 -> global.
//
// TMEM (512 columns): slot s has S/P at [128 s, 128 s + 128) and O at
// [256 + 128 s, 384 + 128 s).

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include "../../include/vt_attention.h"
#include "vt_pf_common.cuh"

namespace vt {
namespace pf {

constexpr int BM = 128;  // query rows per slot
constexpr int BN = 128;  // keys per K/V tile and per score block
constexpr int D = 128;
constexpr int kStages = 2;
constexpr int kSlots = 2;
constexpr int kThreads = kSlots * 128 + 128;  // softmax WGs, then TMA/MMA WG
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kOCol = 256;
constexpr float kRescaleLog2 = 8.0f;  // lazy max: rescale only when it grows by > 2^8
#ifndef VT_PF_POLY_MASK
#define VT_PF_POLY_MASK 0x92
#endif
// Pair k of a row's scores takes exp2 on the FMA pipe (polynomial) when bit
// (k % 8) of this mask is set (3 of 8 measured best on config 3: 1117 vs 1092
// TFLOP/s for 2 of 8, 1015 for 4 of 8); the rest use MUFU.EX2.
constexpr uint32_t kPolyMask = VT_PF_POLY_MASK;

struct __align__(1024) Smem {
  __nv_bfloat16 q[kSlots][2][BM * 64];    // SW128 K-major: d 0-63 | d 64-127
  __nv_bfloat16 k[kStages][2][BN * 64];   // SW128 K-major (keys x d)
  __nv_bfloat16 v[kStages][2][BN * 64];   // SW128, read as MN-major B (d x keys)
  uint64_t q_full, q_empty;
  uint64_t k_full[kStages], k_empty[kStages];
  uint64_t v_full[kStages], v_empty[kStages];
  uint64_t s_full[kSlots];
  uint64_t p_full[kSlots][2];  // P of keys 0-63 / 64-127 of the block is in TMEM
  uint64_t o_done[kSlots];
  uint32_t tmem_base;
};

#ifdef VT_PF_TRACE
// Debug timeline of CTA 0 (clock64), per global key block g < 256:
// [0]/[2] slot 0/1 S ready (after s_full), [1]/[3] slot 0/1 P arrived,
// [4]/[5] MMA group {PV_s(g), S_s(g+1)} issued for slot 0/1,
// [6]/[7] slot 0 epilogue start / end (at the item's last g).
__device__ long long g_pf_trace[256][8];
__device__ long long g_pf_sub[256][4];  // slot 0 row 0: ld done, max done, exp done, st done
#define VT_SUB(cond, g, k) \
  if ((cond) && blockIdx.x == 0 && (g) < 256) g_pf_sub[(g)][(k)] = clock64();
#define VT_TRACE(cond, g, k) \
  if ((cond) && blockIdx.x == 0 && (g) < 256) g_pf_trace[(g)][(k)] = clock64();
#else
#define VT_TRACE(cond, g, k)
#define VT_SUB(cond, g, k)
#endif

struct Args {
  __nv_bfloat16* out;       // [total, Hq, D]: request b's rows at [q_off[b], q_off[b+1])
  const CUtensorMap* kv;    // [B] per-request maps
  const int32_t* start;     // [B]
  const int32_t* q_off;     // [B+1] token offsets (varlen), or null: uniform n_new
  int32_t n_new, hq, hkv, tpc, layer, slots;  // n_new: max new tokens of any request
  int32_t batch, pairs, n_qtiles, n_items;
  float scale_log2;
};

// Work item w -> (q tile, head pair, request). Longest q tiles first (a
// tile's key count grows with t), pairs of one kv head adjacent so concurrent
// CTAs share K/V tiles in L2; CTAs take items w = blockIdx.x + k * gridDim.x.
// With variable-length requests the tile grid is sized by the longest one;
// tiles past a shorter request's n_b are empty items every role skips.
struct Item {
  int t, h0, b, start, kv_len, n_kv, blk_k, blk_v, q0, n_b;
  bool valid;
};
__device__ __forceinline__ Item item_of(int w, const Args& a) {
  Item it;
  const int per_t = a.pairs * a.batch;
  it.t = a.n_qtiles - 1 - w / per_t;
  const int r = w % per_t;
  it.h0 = (r % a.pairs) * a.slots;
  it.b = r / a.pairs;
  it.start = a.start[it.b];
  if (a.q_off) {
    it.q0 = a.q_off[it.b];
    it.n_b = a.q_off[it.b + 1] - it.q0;
  } else {
    it.q0 = it.b * a.n_new;
    it.n_b = a.n_new;
  }
  it.valid = it.t * BM < it.n_b;
  it.kv_len = it.start + it.n_b;
  const int q_last = min(it.n_b, (it.t + 1) * BM);  // exclusive, relative to start
  it.n_kv = (it.start + q_last + BN - 1) / BN;
  const int hk = it.h0 / (a.hq / a.hkv);
  it.blk_k = (a.layer * 2 + 0) * a.hkv + hk;
  it.blk_v = (a.layer * 2 + 1) * a.hkv + hk;
  return it;
}

// Persistent: one CTA per SM walks its work items; barrier phases and the K/V
// ring run on per-CTA global counters (g = key blocks processed so far), so
// the next item's Q and first K/V tiles load while the current item drains.
__global__ void __launch_bounds__(kThreads, 1)
    prefill_kernel(const __grid_constant__ CUtensorMap q_map, const Args a) {
  extern __shared__ uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                      ~static_cast<uintptr_t>(1023));
  const int nslots = a.slots;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  constexpr int kTmaWarp = kSlots * 4, kMmaWarp = kSlots * 4 + 1;

  if (warp == kTmaWarp && lane == 0) {
    mbar_init(&sm.q_full, 1);
    mbar_init(&sm.q_empty, 1);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&sm.k_full[i], 1);
      mbar_init(&sm.k_empty[i], 1);
      mbar_init(&sm.v_full[i], 1);
      mbar_init(&sm.v_empty[i], 1);
    }
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&sm.s_full[s], 1);
      mbar_init(&sm.p_full[s][0], 128);
      mbar_init(&sm.p_full[s][1], 128);
      mbar_init(&sm.o_done[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == kMmaWarp) tc::alloc(&sm.tmem_base, kTmemCols);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp >= kSlots * 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");
    if (warp == kTmaWarp) {
      // ------------------------------ TMA producer ------------------------------
      if (lane == 0) {
        tma_prefetch_desc(&q_map);
        const uint64_t keep = l2_evict_last_policy();   // K/V re-read by the group's heads
        const uint64_t once = l2_evict_first_policy();
        int g = 0;  // K/V tiles loaded so far
        int n = 0;  // items so far
        for (int w = blockIdx.x; w < a.n_items; w += gridDim.x) {
          const Item it = item_of(w, a);
          if (!it.valid) continue;
          const CUtensorMap* kvmap = a.kv + it.b;
          if (n >= 1) mbar_wait(&sm.q_empty, (n - 1) & 1);  // last S of the previous item done
          mbar_arrive_expect_tx(&sm.q_full, nslots * 2 * BM * 64 * 2);
          for (int s = 0; s < nslots; ++s) {
            tma_load_4d(sm.q[s][0], &q_map, &sm.q_full, 0, it.h0 + s, it.q0 + it.t * BM, 0, once);
            tma_load_4d(sm.q[s][1], &q_map, &sm.q_full, 64, it.h0 + s, it.q0 + it.t * BM, 0, once);
          }
          // The next item's Q and first K/V tiles cannot enter shared memory
          // until this item's last tiles leave it; warm L2 with them now so
          // those loads are L2 hits at the item boundary instead of HBM trips
          // (measured: the tensor pipe idled ~6000 clk per item boundary).
          const Item nx = w + static_cast<int>(gridDim.x) < a.n_items ? item_of(w + gridDim.x, a)
                                                                     : Item{};
          if (nx.valid) {
            for (int s = 0; s < nslots; ++s) {  // its Q tiles too (loaded only after
              // this item's last S, otherwise straight from HBM at the boundary)
              tma_prefetch_l2_4d(&q_map, 0, nx.h0 + s, nx.q0 + nx.t * BM, 0);
              tma_prefetch_l2_4d(&q_map, 64, nx.h0 + s, nx.q0 + nx.t * BM, 0);
            }
            const CUtensorMap* nmap = a.kv + nx.b;
            for (int j = 0; j < min(nx.n_kv, kStages); ++j) {
              const int tok0 = j * BN;
              tma_prefetch_l2_4d(nmap, 0, tok0 % a.tpc, nx.blk_k, tok0 / a.tpc);
              tma_prefetch_l2_4d(nmap, 64, tok0 % a.tpc, nx.blk_k, tok0 / a.tpc);
              tma_prefetch_l2_4d(nmap, 0, tok0 % a.tpc, nx.blk_v, tok0 / a.tpc);
              tma_prefetch_l2_4d(nmap, 64, tok0 % a.tpc, nx.blk_v, tok0 / a.tpc);
            }
          }
          for (int j = 0; j < it.n_kv; ++j, ++g) {
            const int st = g % kStages;
            const uint32_t ph = (g / kStages) & 1;
            const int tok0 = j * BN;
            const int c1 = tok0 % a.tpc;
            const int c3 = tok0 / a.tpc;
            if (g >= kStages) mbar_wait(&sm.k_empty[st], ph ^ 1);
            mbar_arrive_expect_tx(&sm.k_full[st], 2 * BN * 64 * 2);
            tma_load_4d(sm.k[st][0], kvmap, &sm.k_full[st], 0, c1, it.blk_k, c3, keep);
            tma_load_4d(sm.k[st][1], kvmap, &sm.k_full[st], 64, c1, it.blk_k, c3, keep);
            if (g >= kStages) mbar_wait(&sm.v_empty[st], ph ^ 1);
            mbar_arrive_expect_tx(&sm.v_full[st], 2 * BN * 64 * 2);
            tma_load_4d(sm.v[st][0], kvmap, &sm.v_full[st], 0, c1, it.blk_v, c3, keep);
            tma_load_4d(sm.v[st][1], kvmap, &sm.v_full[st], 64, c1, it.blk_v, c3, keep);
          }
          ++n;
        }
      }
      __syncwarp();
    } else if (warp == kMmaWarp) {
      // ------------------------------- MMA issuer -------------------------------
      constexpr uint32_t id_s = tc::idesc_bf16(BM, BN, false, false);
      constexpr uint32_t id_pv = tc::idesc_bf16(BM, D, false, true);
      constexpr uint32_t hi = tc::sdesc_hi(1024);  // SW128: 8-row groups 1 KiB apart
      // Descriptor address fields count 16 B units: a [.][64] bf16 tile half
      // is 16 KiB = 1024 units, one 16-element K step inside a SW128 row = 2,
      // 16 keys of V = 128.
      const uint32_t lq = tc::sdesc_lo(smem_u32(sm.q[0][0]), 16);
      const uint32_t lk = tc::sdesc_lo(smem_u32(sm.k[0][0]), 16);
      const uint32_t lv = tc::sdesc_lo(smem_u32(sm.v[0][0]), BN * 128);
      auto wait_fence = [&](uint64_t* bar, uint32_t parity) {
        mbar_wait(bar, parity);
        tc::fence_after();
      };
      auto mma_s = [&](int s, int g) {  // elected lane only; g = global tile index
        const uint32_t b0 = lk + static_cast<uint32_t>((g % kStages) * 2048);
        const uint32_t a0 = lq + static_cast<uint32_t>(s * 2048);
        const uint32_t d = tmem + static_cast<uint32_t>(s * BN);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = static_cast<uint32_t>((kk >> 2) * 1024 + 2 * (kk & 3));
          tc::mma_ss(d, a0 + off, hi, b0 + off, hi, id_s, kk > 0 ? 1u : 0u);
        }
        tc::commit(&sm.s_full[s]);
      };
      // O += P V over keys [64 hf, 64 hf + 64) of the block (4 MMAs of K16):
      // the softmax hands P over in two halves so the first half's MMAs run
      // while it still exponentiates the second.
      auto mma_pv_half = [&](int s, int g, int hf, bool first) {  // elected lane only
        const uint32_t b0 = lv + static_cast<uint32_t>((g % kStages) * 2048);
        const uint32_t d = tmem + kOCol + static_cast<uint32_t>(s * D);
        const uint32_t p = tmem + static_cast<uint32_t>(s * BN);
#pragma unroll
        for (int k4 = 0; k4 < BN / 32; ++k4) {
          const int kk = hf * (BN / 32) + k4;
          tc::mma_ts(d, p + 8 * kk, b0 + static_cast<uint32_t>(kk * 128), hi, id_pv,
                     (!first || kk > 0) ? 1u : 0u);
        }
        if (hf == 1) tc::commit(&sm.o_done[s]);
      };
      int g = 0, n = 0;
      for (int w = blockIdx.x; w < a.n_items; w += gridDim.x) {
        const Item it = item_of(w, a);
        if (!it.valid) continue;
        const int n_kv = it.n_kv;
        // S(0) of every slot; its S buffer was last read by the previous
        // item's final PV, issued before (in-order).
        wait_fence(&sm.q_full, n & 1);
        wait_fence(&sm.k_full[g % kStages], (g / kStages) & 1);
        if (tc::elect_one()) {
#pragma unroll
          for (int s = 0; s < kSlots; ++s)
            if (s < nslots) mma_s(s, g);
          tc::commit(&sm.k_empty[g % kStages]);
          if (n_kv == 1) tc::commit(&sm.q_empty);
        }
        __syncwarp();
        for (int j = 0; j < n_kv; ++j, ++g) {
          const bool more = j + 1 < n_kv;
          mbar_wait(&sm.v_full[g % kStages], (g / kStages) & 1);
          if (more) mbar_wait(&sm.k_full[(g + 1) % kStages], ((g + 1) / kStages) & 1);
#pragma unroll
          for (int s = 0; s < kSlots; ++s) {
            if (s < nslots) {
              const bool last_slot = s == nslots - 1;
              wait_fence(&sm.p_full[s][0], g & 1);
              if (tc::elect_one()) mma_pv_half(s, g, 0, j == 0);
              __syncwarp();
              wait_fence(&sm.p_full[s][1], g & 1);
              VT_TRACE(lane == 0, g, 4 + s);
              if (tc::elect_one()) {
                mma_pv_half(s, g, 1, j == 0);
                if (last_slot) tc::commit(&sm.v_empty[g % kStages]);
                if (more) {
                  mma_s(s, g + 1);
                  if (last_slot) {
                    tc::commit(&sm.k_empty[(g + 1) % kStages]);
                    if (j + 2 == n_kv) tc::commit(&sm.q_empty);  // the item's last S
                  }
                }
              }
              __syncwarp();
            }
          }
        }
        ++n;
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 216;");
    if (warp / 4 < nslots) {
      // ------------------------------ softmax slot s ------------------------------
      const int s = warp / 4;
      const int quarter = warp & 3;  // TMEM lane quarter this warp may access
      const int row = quarter * 32 + lane;
      const uint32_t lane_addr = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
      const uint32_t s_addr = lane_addr + static_cast<uint32_t>(s * BN);
      const uint32_t o_addr = lane_addr + kOCol + static_cast<uint32_t>(s * D);
      const float sl2 = a.scale_log2;
      int g = 0;  // key blocks processed so far (barrier phases)
      for (int w = blockIdx.x; w < a.n_items; w += gridDim.x) {
        const Item it = item_of(w, a);
        if (!it.valid) continue;
        const int qpos = it.start + it.t * BM + row;  // absolute position of this query row
        const int qmin = it.start + it.t * BM;        // smallest query position of the tile
        float m_run = -INFINITY, l_run = 0.f;
        for (int j = 0; j < it.n_kv; ++j, ++g) {
          const int kpos0 = j * BN;
          mbar_wait(&sm.s_full[s], g & 1);
          tc::fence_after();
          VT_TRACE(row == 0, g, 2 * s);
          float x[BN];
          {
            uint32_t r[BN];
#pragma unroll
            for (int c = 0; c < BN / 32; ++c) tmem_ld32(s_addr + 32 * c, r + 32 * c);
            tc::wait_ld();
#pragma unroll
            for (int k = 0; k < BN; ++k) x[k] = __uint_as_float(r[k]);
          }
          VT_SUB(row == 0 && s == 0, g, 0);
          if (kpos0 + BN - 1 > qmin || kpos0 + BN > it.kv_len) {
            const int lim = min(qpos + 1, it.kv_len) - kpos0;  // keys [0, lim) are visible
#pragma unroll
            for (int k = 0; k < BN; ++k)
              if (k >= lim) x[k] = -INFINITY;
          }
          float mx;
          {
            float m8[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) m8[k] = fmaxf(x[k], x[k + 8]);
#pragma unroll
            for (int k = 16; k < BN; k += 16)
#pragma unroll
              for (int u = 0; u < 8; ++u) m8[u] = fmaxf(m8[u], fmaxf(x[k + u], x[k + 8 + u]));
            mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                       fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
          }
          VT_SUB(row == 0 && s == 0 && mx > -1e30f, g, 1);
          const float mx_s = mx * sl2;
          const bool grow = mx_s > m_run + kRescaleLog2;  // false while both are -inf
          const float m_new = grow ? mx_s : m_run;
          const float alpha = grow ? tc::ex2(m_run - m_new) : 1.f;
          const float m_use = m_new == -INFINITY ? 0.f : m_new;
          const float2 sl2v = make_float2(sl2, sl2);
          const float2 negm = make_float2(-m_use, -m_use);
          if (j >= 1 && __any_sync(0xffffffffu, grow)) {
            // Lazy rescale of O before any of this block's PV: PV(j-1) is
            // complete (S(j), issued after it, has completed).
            mbar_wait(&sm.o_done[s], (g - 1) & 1);
            tc::fence_after();
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              uint32_t r[32];
              tmem_ld32(o_addr + 32 * c, r);
              tc::wait_ld();
#pragma unroll
              for (int k = 0; k < 32; ++k) r[k] = __float_as_uint(__uint_as_float(r[k]) * alpha);
              tmem_st32(o_addr + 32 * c, r);
            }
          }
          bool zeroed = false;
          if (s == 0 && j == it.n_kv - 1 && kpos0 + BN > it.kv_len) {
            // Rows past kv_len may hold stale/uninitialised bytes of the last
            // mapped chunk: zero them so 0 * NaN cannot reach the accumulator.
            // (Slot 1's PV of this tile is issued after slot 0's P arrives.)
            const int st = g % kStages;
            mbar_wait(&sm.v_full[st], (g / kStages) & 1);
            if (kpos0 + row >= it.kv_len) {
              const uint4 z = make_uint4(0, 0, 0, 0);
              uint4* r0 = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(sm.v[st][0]) + row * 128);
              uint4* r1 = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(sm.v[st][1]) + row * 128);
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                r0[c] = z;
                r1[c] = z;
              }
            }
            zeroed = true;
          }
          float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                           make_float2(0.f, 0.f)};
          // Two halves of 64 keys: P of keys 0-63 goes to TMEM columns 0-31 and
          // is handed to the MMA warp (its PV half runs) while the second half
          // is exponentiated. Column c = keys (2c, 2c+1) as bf16x2.
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            uint32_t pr[BN / 4];
#pragma unroll
            for (int k2 = 0; k2 < BN / 4; ++k2) {
              const int k = hf * (BN / 4) + k2;
              float2 e = __ffma2_rn(make_float2(x[2 * k], x[2 * k + 1]), sl2v, negm);
              if ((kPolyMask >> (k & 7)) & 1u) {
                e = ex2_poly2(e);
              } else {
                e.x = tc::ex2(e.x);
                e.y = tc::ex2(e.y);
              }
              acc[k & 3] = __fadd2_rn(acc[k & 3], e);
              pr[k2] = pack_bf16(e.x, e.y);
            }
            tmem_st32(s_addr + 32 * hf, pr);
            tc::wait_st();
            if (hf == 0 && zeroed) fence_proxy_async_smem();
            tc::fence_before();
            mbar_arrive(&sm.p_full[s][hf]);
          }
          const float2 a01 = __fadd2_rn(__fadd2_rn(acc[0], acc[1]), __fadd2_rn(acc[2], acc[3]));
          l_run = fmaf(l_run, alpha, a01.x + a01.y);
          m_run = m_new;
          VT_SUB(row == 0 && s == 0, g, 3);
          VT_TRACE(row == 0, g, 2 * s + 1);
        }
        // epilogue: PV(n_kv-2) completed before S(n_kv-1); wait for the last PV.
        VT_TRACE(row == 0 && s == 0, g - 1, 6);
        mbar_wait(&sm.o_done[s], (g - 1) & 1);
        tc::fence_after();
        const int tok = it.t * BM + row;
        const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
        __nv_bfloat16* dst =
            a.out + ((static_cast<int64_t>(it.q0) + tok) * a.hq + (it.h0 + s)) * D;
        uint32_t r[D];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(o_addr + 32 * c, r + 32 * c);
        tc::wait_ld();
        if (tok < it.n_b) {
          // 32-byte stores (st.global.v8): a thread writes its 256-byte row
          // in 8 instructions instead of 16 — the row-per-thread pattern
          // makes every instruction touch 32 rows 8 KiB apart (epilogue
          // 4700 -> 2760 clk per slot, measured with the trace).
#pragma unroll
          for (int k = 0; k < D; k += 16) {
            uint32_t w8[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
              w8[u] = pack_bf16(__uint_as_float(r[k + 2 * u]) * inv, __uint_as_float(r[k + 2 * u + 1]) * inv);
            asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + k),
                         "r"(w8[0]), "r"(w8[1]), "r"(w8[2]), "r"(w8[3]), "r"(w8[4]), "r"(w8[5]),
                         "r"(w8[6]), "r"(w8[7])
                         : "memory");
          }

        }
        // O is read: the next item's PV(0) (acc = 0) may overwrite it. That
        // PV waits for this warpgroup's next P, which comes after this point.
        tc::fence_before();
        VT_TRACE(row == 0 && s == 0, g - 1, 7);
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == kMmaWarp) tc::dealloc(tmem, kTmemCols);
}

}  // namespace pf
}  // namespace vt

using namespace vt::pf;

#ifdef VT_PF_TRACE
extern "C" int vt_prefill_trace(long long* out) {  // 256 x 8 + 256 x 4 values
  cudaMemcpyFromSymbol(out + 256 * 8, g_pf_sub, sizeof(g_pf_sub));
  return cudaMemcpyFromSymbol(out, g_pf_trace, sizeof(g_pf_trace));
}
#endif

namespace vt {
int launch_prefill_pair(const vt_kv_geometry* g, int32_t layer, const void* q, const void* kv_maps,
                        const int32_t* start, const int32_t* q_off, int32_t batch,
                        int32_t max_n_new, int64_t total, float scale, void* out, void* stream);
}

namespace {

int launch_prefill(const vt_kv_geometry* g, int32_t layer, const void* q, const void* kv_maps,
                   const int32_t* start, const int32_t* q_off, int32_t batch, int32_t max_n_new,
                   int64_t total, float scale, void* out, void* stream) {
  static const bool pair = [] {
    const char* e = std::getenv("VT_PREFILL_PAIR");
    return e && std::atoi(e) != 0;
  }();
  if (pair)
    return vt::launch_prefill_pair(g, layer, q, kv_maps, start, q_off, batch, max_n_new, total,
                                   scale, out, stream);
  if (g->head_dim != D || g->q_heads % g->kv_heads) return cudaErrorInvalidValue;
  if (batch <= 0 || max_n_new <= 0 || total <= 0) return 0;
  // Q as one packed [total tokens][Hq][D] tensor (a 4-D map with a unit outer
  // dim): request b's tile t starts at row q_off[b] + 128 t. A tile running
  // past its request's rows loads the next request's (or zero-filled OOB)
  // rows, which are masked like any row past n_b and never stored.
  CUtensorMap qmap;
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(g->q_heads),
                              static_cast<cuuint64_t>(total), 1};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(D * 2),
                                 static_cast<cuuint64_t>(g->q_heads) * D * 2,
                                 static_cast<cuuint64_t>(total) * g->q_heads * D * 2};
  const cuuint32_t box[4] = {64, 1, static_cast<cuuint32_t>(BM), 1};
  int rc = vt::encode_tensor_map_bf16(&qmap, const_cast<void*>(q), 4, dims, strides, box);
  if (rc) return rc;
  const int group = g->q_heads / g->kv_heads;
  Args a{};
  a.out = static_cast<__nv_bfloat16*>(out);
  a.kv = static_cast<const CUtensorMap*>(kv_maps);
  a.start = start;
  a.q_off = q_off;
  a.n_new = max_n_new;
  a.hq = g->q_heads;
  a.hkv = g->kv_heads;
  a.tpc = g->tokens_per_chunk;
  a.layer = layer;
  a.slots = group % kSlots == 0 ? kSlots : 1;  // a pair never straddles two kv heads
  a.batch = batch;
  a.pairs = g->q_heads / a.slots;
  a.n_qtiles = (max_n_new + BM - 1) / BM;
  a.n_items = a.n_qtiles * a.pairs * batch;
  a.scale_log2 = scale * 1.4426950408889634f;
  const size_t smem = sizeof(Smem) + 1024;
  static std::atomic<uint64_t> attr_devices{0};
  vt::set_smem_limit_once(prefill_kernel, smem, attr_devices);
  static int n_sm = 0;
  if (!n_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  }
  const int grid = a.n_items < n_sm ? a.n_items : n_sm;  // persistent: one CTA per SM
  prefill_kernel<<<grid, kThreads, smem, static_cast<cudaStream_t>(stream)>>>(qmap, a);
  return cudaGetLastError();
}

}  // namespace

extern "C" int vt_prefill_attention(const vt_kv_geometry* g, int32_t layer, const void* q,
                                    const void* kv_maps, const int32_t* start, int32_t batch,
                                    int32_t n_new, float scale, void* out, void* stream) {
  return launch_prefill(g, layer, q, kv_maps, start, nullptr, batch, n_new,
                        static_cast<int64_t>(batch) * n_new, scale, out, stream);
}

extern "C" int vt_prefill_attention_varlen(const vt_kv_geometry* g, int32_t layer, const void* q,
                                           const void* kv_maps, const int32_t* start,
                                           const int32_t* q_offsets, int32_t batch,
                                           int32_t max_n_new, int64_t total_tokens, float scale,
                                           void* out, void* stream) {
  if (!q_offsets) return cudaErrorInvalidValue;
  return launch_prefill(g, layer, q, kv_maps, start, q_offsets, batch, max_n_new, total_tokens,
                        scale, out, stream);
}
