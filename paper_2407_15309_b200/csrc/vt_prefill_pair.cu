// Prefill / prefix-prefill attention on a CTA PAIR (tcgen05 cta_group::2,
// sm_100a) — the same contract as vt_prefill.cu (row a28), built so the
// tensor pipe never waits for the softmax.
//
// Why a pair. One CTA computing S = Q K^T for two q heads (vt_prefill.cu)
// serialises, per head, softmax(j) -> PV(j) -> S(j+1), because S(j+1) must
// overwrite the TMEM columns P(j) is read from; its key-block period is ~3000
// clk for 2060 clk of MMA. And SS MMAs read both operands through the SM's
// 128 B/clk shared-memory port (measured: SS 128x128 = 8 KiB / 64 clk, SS
// 128x64 = 6 KiB / 48 clk), so one CTA has no bandwidth left for moving P
// through shared memory. On a pair, `tcgen05.mma.cta_group::2` computes
// M = 256 rows (128 per CTA, each CTA's own A operand) with the B operand
// split by N across the two CTAs, so each CTA streams half the K/V bytes per
// FLOP and TMEM has room for S, P and O side by side:
//
//   TMEM (per CTA, 512 columns): S [0,256) fp32 scores of one 256-key block
//   (two 128-column halves), P [256,384) bf16 probabilities of that block
//   (natural key order, 2 keys per column), O [384,512) fp32 accumulator.
//
// A pair item = 128 query rows per CTA attending to one kv head: the two q
// heads {2p, 2p+1} of a GQA group for the same 128-token tile (group size
// even), or the same head for q tiles {2t', 2t'+1} (odd groups, e.g. MHA).
// Keys advance in blocks of 256 = two 128-key tiles: CTA r loads tile 2j+r of
// K (all 128 dims) and the d-half r of both V tiles. With the B operand split
// by N, an N = 128 MMA over this layout yields S columns [0,64) = keys 0-63 of
// tile 2j and [64,128) = keys 0-63 of tile 2j+1 ("half A"; "half B" = keys
// 64-127 of both), so the softmax works on 128-column halves and writes P in
// natural key order, which the PV MMAs (K = keys) read against V.
//
// Schedule per block j (leader CTA's MMA warp, in issue order):
//   S_A(j+1) once both softmaxes hold S_A(j) in registers (s_free[0]),
//   PV_A(j)  once P_A(j) is in TMEM (p_full[0]; implies both V halves landed),
//   S_B(j+1) once both softmaxes hold S_B(j),
//   PV_B(j)  once P_B(j) is in TMEM.
// The softmax of block j+1 therefore finds S(j+1) computed while it worked
// on block j: the tensor pipe has 2048 clk of work per block and the softmax
// (~2 x 950 clk) overlaps it instead of alternating with it.
//
// Warps (192 threads per CTA): 0-3 softmax (thread = TMEM lane = query row;
// lazy running max, 3/8 of the exponentials on the FMA pipe, as vt_prefill.cu),
// 4 TMA producer, 5 MMA issuer (leader CTA; in the peer it only co-allocates
// TMEM). Barrier placement: Q / K loads are 2-CTA TMA completing on the
// leader's q_full / k_full; each CTA's V half completes on its own v_full,
// which its softmax waits for (and, in an item's last block, zeroes the V rows
// past kv_len) before handing P over, so p_full at the leader implies both V
// halves are in place. MMA completions are multicast commits to both CTAs.

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/vt_attention.h"
#include "vt_pf_common.cuh"

namespace vt {
namespace pf2 {

using pf::ex2_poly2;
using pf::pack_bf16;
using pf::tmem_ld32;
using pf::tmem_st32;

constexpr int BM = 128;   // query rows per CTA
constexpr int BT = 128;   // keys per K/V tile (one TMA box)
constexpr int D = 128;
constexpr int kKStages = 3;
constexpr int kVStages = 2;
constexpr int kThreads = 192;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kPCol = 256;
constexpr uint32_t kOCol = 384;
constexpr float kRescaleLog2 = 8.0f;
#ifndef VT_PF_POLY_MASK
#define VT_PF_POLY_MASK 0x92
#endif
constexpr uint32_t kPolyMask = VT_PF_POLY_MASK;

struct __align__(1024) Smem {
  __nv_bfloat16 q[2][2][BM * 64];         // per item parity: d 0-63 | d 64-127 (SW128 K-major)
  __nv_bfloat16 k[kKStages][2][BT * 64];  // tile 2j+r: d 0-63 | d 64-127 (SW128 K-major)
  __nv_bfloat16 v[kVStages][2][BT * 64];  // d-half r of tile 2j | of tile 2j+1 (SW128, MN-major B)
  // leader-side (waited by the MMA warp)
  uint64_t q_full[2], k_full[kKStages];
  uint64_t s_free[2], p_full[2], o_free;
  // both CTAs (multicast commits / own TMA)
  uint64_t q_empty[2], k_empty[kKStages], v_full[kVStages], v_empty[kVStages];
  uint64_t s_full[2], pv_done[2], o_full;
  uint64_t drain;  // the leader's last commit: no arrive is still in flight at exit
  uint32_t tmem_base;
};

// ----------------------------------------------------------- pair plumbing --
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// shared::cluster address of `p` in the leader CTA (rank 0).
__device__ __forceinline__ uint32_t leader_addr(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}
// Arrive on the leader's barrier. Default (.release.cta) semantics: the data
// handed over lives in TMEM / is read by the tensor core, ordered by
// tcgen05.wait + tcgen05.fence::before_thread_sync ahead of this arrive; a
// .release.cluster arrive compiles to MEMBAR.ALL.GPU and was 23% of the
// kernel's stall samples (ncu, profiles/r02).
__device__ __forceinline__ void arrive_leader(const uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(leader_addr(bar)) : "memory");
}
// 2-CTA TMA: lands in this CTA's shared memory, completes bytes on the
// LEADER's mbarrier.
__device__ __forceinline__ void tma_load_4d_pair(void* dst, const void* tmap, const uint64_t* bar,
                                                 int c0, int c1, int c2, int c3, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(leader_addr(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void mma2_ss(uint32_t d, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo,
                                        uint32_t b_hi, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 da, db;\n\t"
      "setp.ne.b32 p, %6, 0;\n\tmov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, p;\n\t}" ::"r"(d),
      "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a_tmem, uint32_t b_lo, uint32_t b_hi,
                                        uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 db;\n\t"
      "setp.ne.b32 p, %5, 0;\n\tmov.b64 db, {%2, %3};\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], db, %4, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "r"(b_lo), "r"(b_hi), "r"(id), "r"(acc));
}
// Completion of the leader's MMAs so far, arrived on `bar` in BOTH CTAs.
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}
__device__ __forceinline__ void tmem_alloc2(uint32_t* dst, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)),
               "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}

#ifdef VT_PF2_TRACE
// Debug timeline of pair 0 (clock64 of the leader CTA), per global block g <
// 256: [0]/[2] half A/B S ready at softmax row 0, [1]/[3] P_A/P_B arrived,
// [4] S_A(g+1), [5] PV_A(g), [6] S_B(g+1), [7] PV_B(g) issued.
__device__ long long g_pf2_trace[256][8];
#define PF2_TRACE(cond, g, k) \
  if ((cond) && blockIdx.x == 0 && (g) < 256) g_pf2_trace[(g)][(k)] = clock64();
#else
#define PF2_TRACE(cond, g, k)
#endif

struct Args {
  __nv_bfloat16* out;       // [total, Hq, D]
  const CUtensorMap* kv;    // [B] per-request maps (128-token boxes)
  const int32_t* start;     // [B]
  const int32_t* q_off;     // [B+1] or null (uniform n_new)
  int32_t n_new, hq, hkv, tpc, layer;
  int32_t batch, head_pairs;  // head_pairs: 1 -> the pair is two q heads of one tile
  int32_t n_units, n_items;   // units per (request, q tile | tile pair); items = units x batch
  float scale_log2;
};

// Pair item w: request b, this CTA's q head h and q tile t, and the pair's
// key range (keys needed by the later of the two tiles). Longest first.
struct Item {
  int b, h, t, q0, n_b, start, kv_len, n_blk, blk_k, blk_v, qmin;
  bool valid;
};
__device__ __forceinline__ Item item_of(int w, const Args& a, int r) {
  Item it;
  const int per_t = a.n_units * a.batch;   // items per (tile | tile pair) row
  const int n_rows = a.n_items / per_t;
  const int tt = n_rows - 1 - w / per_t;  // tile (head pairs) or tile pair index
  const int rem = w % per_t;
  const int u = rem % a.n_units;
  it.b = rem / a.n_units;
  int t_hi;
  if (a.head_pairs) {
    it.h = 2 * u + r;
    it.t = tt;
    t_hi = tt;
  } else {
    it.h = u;
    it.t = 2 * tt + r;
    t_hi = 2 * tt + 1;
  }
  it.start = a.start[it.b];
  if (a.q_off) {
    it.q0 = a.q_off[it.b];
    it.n_b = a.q_off[it.b + 1] - it.q0;
  } else {
    it.q0 = it.b * a.n_new;
    it.n_b = a.n_new;
  }
  const int t_lo = a.head_pairs ? tt : 2 * tt;
  it.valid = t_lo * BM < it.n_b;  // the pair has work if its first tile does
  it.kv_len = it.start + it.n_b;
  const int q_last = min(it.n_b, (t_hi + 1) * BM);
  const int n_keys = it.start + q_last;
  it.n_blk = (n_keys + 2 * BT - 1) / (2 * BT);
  const int hk = it.h / (a.hq / a.hkv);
  it.blk_k = (a.layer * 2 + 0) * a.hkv + hk;
  it.blk_v = (a.layer * 2 + 1) * a.hkv + hk;
  it.qmin = it.start + it.t * BM;
  return it;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    prefill_pair_kernel(const __grid_constant__ CUtensorMap q_map, const Args a) {
  extern __shared__ uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                      ~static_cast<uintptr_t>(1023));
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int r = static_cast<int>(cta_rank());
  const bool leader = r == 0;
  const int pair = blockIdx.x >> 1;
  const int n_pairs = gridDim.x >> 1;
  constexpr int kTmaWarp = 4, kMmaWarp = 5;

  if (warp == kTmaWarp && lane == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.q_full[i], 1);
      mbar_init(&sm.q_empty[i], 1);
      mbar_init(&sm.s_free[i], 8);  // lane 0 of the 4 softmax warps of both CTAs
      mbar_init(&sm.p_full[i], 8);
      mbar_init(&sm.s_full[i], 1);
      mbar_init(&sm.pv_done[i], 1);
    }
    for (int i = 0; i < kKStages; ++i) {
      mbar_init(&sm.k_full[i], 1);
      mbar_init(&sm.k_empty[i], 1);
    }
    for (int i = 0; i < kVStages; ++i) {
      mbar_init(&sm.v_full[i], 1);
      mbar_init(&sm.v_empty[i], 1);
    }
    mbar_init(&sm.o_free, 8);
    mbar_init(&sm.o_full, 1);
    mbar_init(&sm.drain, 1);
    fence_mbar_init();
  }
  if (warp == kMmaWarp) tmem_alloc2(&sm.tmem_base, kTmemCols);
  tc::fence_before();
  cluster_sync();  // barriers and TMEM of both CTAs exist before any cross-CTA use
  tc::fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == kTmaWarp) {
    // ------------------------------ TMA producer ------------------------------
    if (lane == 0) {
      tma_prefetch_desc(&q_map);
      const uint64_t keep = l2_evict_last_policy();
      const uint64_t once = l2_evict_first_policy();
      int n = 0, u = 0;  // items, key blocks
      for (int w = pair; w < a.n_items; w += n_pairs) {
        const Item it = item_of(w, a, r);
        if (!it.valid) continue;
        const CUtensorMap* kvmap = a.kv + it.b;
        const int qb = n & 1;
        if (n >= 2) mbar_wait(&sm.q_empty[qb], ((n >> 1) - 1) & 1);
        if (leader) mbar_arrive_expect_tx(&sm.q_full[qb], 2 * 2 * BM * 64 * 2);
        tma_load_4d_pair(sm.q[qb][0], &q_map, &sm.q_full[qb], 0, it.h, it.q0 + it.t * BM, 0, once);
        tma_load_4d_pair(sm.q[qb][1], &q_map, &sm.q_full[qb], 64, it.h, it.q0 + it.t * BM, 0, once);
        for (int j = 0; j < it.n_blk; ++j, ++u) {
          const int ks = u % kKStages, vs = u % kVStages;
          const int tk = (2 * j + r) * BT;  // this CTA's K tile
          if (u >= kKStages) mbar_wait(&sm.k_empty[ks], ((u / kKStages) & 1) ^ 1);
          if (leader) mbar_arrive_expect_tx(&sm.k_full[ks], 2 * 2 * BT * 64 * 2);
          tma_load_4d_pair(sm.k[ks][0], kvmap, &sm.k_full[ks], 0, tk % a.tpc, it.blk_k, tk / a.tpc, keep);
          tma_load_4d_pair(sm.k[ks][1], kvmap, &sm.k_full[ks], 64, tk % a.tpc, it.blk_k, tk / a.tpc, keep);
          if (u >= kVStages) mbar_wait(&sm.v_empty[vs], ((u / kVStages) & 1) ^ 1);
          mbar_arrive_expect_tx(&sm.v_full[vs], 2 * BT * 64 * 2);
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            const int tv = (2 * j + s) * BT;
            tma_load_4d(sm.v[vs][s], kvmap, &sm.v_full[vs], 64 * r, tv % a.tpc, it.blk_v, tv / a.tpc,
                        keep);
          }
        }
        ++n;
      }
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    // ------------------------------- MMA issuer -------------------------------
    if (leader) {
      // M = 256 (128 rows per CTA), N = 128: S halves (B = 64 keys of each
      // CTA's K tile) and PV (B = each CTA's 64-dim half of V).
      constexpr uint32_t id_s = tc::idesc_bf16(2 * BM, 128, false, false);
      constexpr uint32_t id_pv = tc::idesc_bf16(2 * BM, D, false, true);
      constexpr uint32_t hi = tc::sdesc_hi(1024);
      const uint32_t lq = tc::sdesc_lo(smem_u32(sm.q[0][0]), 16);
      const uint32_t lk = tc::sdesc_lo(smem_u32(sm.k[0][0]), 16);
      const uint32_t lv = tc::sdesc_lo(smem_u32(sm.v[0][0]), BT * 128);
      auto wait_fence = [&](uint64_t* bar, uint32_t parity) {
        mbar_wait(bar, parity);
        tc::fence_after();
      };
      // S half hf of global block g (item ordinal n, block j of it).
      auto issue_s = [&](int g, int n, int j, int hf, bool item_last) {
        const int ks = g % kKStages;
        if (hf == 0) {
          if (j == 0) wait_fence(&sm.q_full[n & 1], (n >> 1) & 1);
          wait_fence(&sm.k_full[ks], (g / kKStages) & 1);
        }
        if (tc::elect_one()) {
          const uint32_t a0 = lq + static_cast<uint32_t>((n & 1) * 2048);
          const uint32_t b0 = lk + static_cast<uint32_t>(ks * 2048 + hf * 512);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = static_cast<uint32_t>((kk >> 2) * 1024 + 2 * (kk & 3));
            mma2_ss(tmem + 128 * hf, a0 + off, hi, b0 + off, hi, id_s, kk > 0 ? 1u : 0u);
          }
          commit2(&sm.s_full[hf]);
          if (hf == 1) {
            commit2(&sm.k_empty[ks]);
            if (item_last) commit2(&sm.q_empty[n & 1]);
          }
        }
        __syncwarp();
      };
      // PV half hf of block g: K steps over the keys of that half, in
      // natural order: tile 2j keys [64 hf, 64 hf + 64), then tile 2j+1's.
      auto issue_pv = [&](int g, int j, int hf, bool item_last) {
        const int vs = g % kVStages;
        if (tc::elect_one()) {
          const uint32_t b0 = lv + static_cast<uint32_t>(vs * 2048);
#pragma unroll
          for (int s = 0; s < 2; ++s) {
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4) {
              const int kk = s * 8 + hf * 4 + k4;  // 16-key step in the 256-key block
              mma2_ts(tmem + kOCol, tmem + kPCol + 8 * kk, b0 + static_cast<uint32_t>(kk * 128), hi,
                      id_pv, (j > 0 || hf > 0 || s > 0 || k4 > 0) ? 1u : 0u);
            }
          }
          commit2(&sm.pv_done[hf]);
          if (hf == 1) {
            commit2(&sm.v_empty[vs]);
            if (item_last) commit2(&sm.o_full);
          }
        }
        __syncwarp();
      };
      // Walk the pair's block stream with the S cursor one block ahead.
      int w = pair, n = 0, j = 0;
      Item it{};
      auto next_valid = [&](int from) {
        int x = from;
        while (x < a.n_items && !item_of(x, a, 0).valid) x += n_pairs;
        return x;
      };
      w = next_valid(w);
      if (w < a.n_items) {
        it = item_of(w, a, 0);
        // S cursor = (ws, ns, js)
        int ws = w, ns = 0, js = 0;
        Item its = it;
        issue_s(0, 0, 0, 0, its.n_blk == 1);
        issue_s(0, 0, 0, 1, its.n_blk == 1);
        // advance S cursor
        auto adv_s = [&]() {
          if (++js == its.n_blk) {
            ws = next_valid(ws + n_pairs);
            js = 0;
            ++ns;
            if (ws < a.n_items) its = item_of(ws, a, 0);
          }
        };
        adv_s();
        for (int g = 0;; ++g) {
          const bool s_more = ws < a.n_items;
          const bool last_of_item = j == it.n_blk - 1;
          // S_A(g+1) once both softmaxes hold S_A(g)
          if (s_more) {
            wait_fence(&sm.s_free[0], g & 1);
            PF2_TRACE(lane == 0, g, 4);
            issue_s(g + 1, ns, js, 0, js == its.n_blk - 1);
          }
          // PV_A(g)
          if (j == 0 && n >= 1) wait_fence(&sm.o_free, (n - 1) & 1);  // epilogue read O
          wait_fence(&sm.p_full[0], g & 1);
          PF2_TRACE(lane == 0, g, 5);
          issue_pv(g, j, 0, last_of_item);
          if (s_more) {
            wait_fence(&sm.s_free[1], g & 1);
            PF2_TRACE(lane == 0, g, 6);
            issue_s(g + 1, ns, js, 1, js == its.n_blk - 1);
            adv_s();
          }
          wait_fence(&sm.p_full[1], g & 1);
          PF2_TRACE(lane == 0, g, 7);
          issue_pv(g, j, 1, last_of_item);
          if (++j == it.n_blk) {
            w = next_valid(w + n_pairs);
            if (w >= a.n_items) break;
            it = item_of(w, a, 0);
            j = 0;
            ++n;
          }
        }
      }
      // commits complete in order: once this lands in both CTAs, so have all
      if (tc::elect_one()) commit2(&sm.drain);
      __syncwarp();
    }
    mbar_wait(&sm.drain, 0);
    __syncwarp();
  } else {
    // ------------------------------- softmax -------------------------------
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_addr = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    const float sl2 = a.scale_log2;
    int g = 0, n = 0;
    for (int w = pair; w < a.n_items; w += n_pairs) {
      const Item it = item_of(w, a, r);
      if (!it.valid) continue;
      const int qpos = it.qmin + row;
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < it.n_blk; ++j, ++g) {
        const int key0 = 2 * j * BT;  // first key of the 256-key block
        const bool last = j == it.n_blk - 1;
#pragma unroll 1
        for (int hf = 0; hf < 2; ++hf) {
          mbar_wait(&sm.s_full[hf], g & 1);
          tc::fence_after();
          PF2_TRACE(r == 0 && row == 0, g, 2 * hf);
          float x[128];
          {
            uint32_t rr[128];
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_ld32(lane_addr + 128 * hf + 32 * c, rr + 32 * c);
            tc::wait_ld();
#pragma unroll
            for (int k = 0; k < 128; ++k) x[k] = __uint_as_float(rr[k]);
          }
          tc::fence_before();
          __syncwarp();
          if (lane == 0) arrive_leader(&sm.s_free[hf]);  // S_hf(g+1) may overwrite
          // column c: tile 2j + (c >> 6), key (c & 63) + 64 hf of that tile
          if (key0 + 2 * BT - 1 > it.qmin || key0 + 2 * BT > it.kv_len) {
            const int lim = min(qpos + 1, it.kv_len);
#pragma unroll
            for (int c = 0; c < 128; ++c) {
              const int kpos = key0 + (c >> 6) * BT + (c & 63) + 64 * hf;
              if (kpos >= lim) x[c] = -INFINITY;
            }
          }
          float mx;
          {
            float m8[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) m8[k] = fmaxf(x[k], x[k + 8]);
#pragma unroll
            for (int k = 16; k < 128; k += 16)
#pragma unroll
              for (int u8 = 0; u8 < 8; ++u8) m8[u8] = fmaxf(m8[u8], fmaxf(x[k + u8], x[k + 8 + u8]));
            mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                       fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
          }
          const float mx_s = mx * sl2;
          const bool grow = mx_s > m_run + kRescaleLog2;
          const float m_new = grow ? mx_s : m_run;
          const float alpha = grow ? tc::ex2(m_run - m_new) : 1.f;
          const float m_use = m_new == -INFINITY ? 0.f : m_new;
          const float2 sl2v = make_float2(sl2, sl2);
          const float2 negm = make_float2(-m_use, -m_use);
          const bool first_half = j == 0 && hf == 0;
          if (!first_half && __any_sync(0xffffffffu, grow)) {
            // every PV issued so far must have landed in O: the previous half's
            mbar_wait(&sm.pv_done[hf ^ 1], (hf == 0 ? g - 1 : g) & 1);
            tc::fence_after();
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
              uint32_t rr[32];
              tmem_ld32(lane_addr + kOCol + 32 * c, rr);
              tc::wait_ld();
#pragma unroll
              for (int k = 0; k < 32; ++k) rr[k] = __float_as_uint(__uint_as_float(rr[k]) * alpha);
              tmem_st32(lane_addr + kOCol + 32 * c, rr);
            }
            tc::wait_st();
          }
          float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                           make_float2(0.f, 0.f)};
          uint32_t pr[64];
#pragma unroll
          for (int k = 0; k < 64; ++k) {
            float2 e = __ffma2_rn(make_float2(x[2 * k], x[2 * k + 1]), sl2v, negm);
            if ((kPolyMask >> (k & 7)) & 1u) {
              e = ex2_poly2(e);
            } else {
              e.x = tc::ex2(e.x);
              e.y = tc::ex2(e.y);
            }
            acc[k & 3] = __fadd2_rn(acc[k & 3], e);
            pr[k] = pack_bf16(e.x, e.y);
          }
          if (hf == 0) {
            // This CTA's V half of the block has landed (the leader's PV waits
            // for this warp's P, so p_full implies both halves are in place).
            const int vs = g % kVStages;
            mbar_wait(&sm.v_full[vs], (g / kVStages) & 1);
            if (last && key0 + 2 * BT > it.kv_len) {
              // rows past kv_len may hold stale / uninitialised bytes: zero
              // them so 0 * NaN never reaches the accumulator
#pragma unroll
              for (int s = 0; s < 2; ++s) {
                if (key0 + s * BT + row >= it.kv_len) {
                  uint4* p = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(sm.v[vs][s]) + row * 128);
                  const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
                  for (int c = 0; c < 8; ++c) p[c] = z;
                }
              }
              fence_proxy_async_smem();
            }
          }
          // P of this half replaces the previous block's: its PV must be done
          if (g >= 1) mbar_wait(&sm.pv_done[hf], (g - 1) & 1);
          // natural key order: tile 2j keys 64hf.. -> P cols 32hf..; tile 2j+1 -> 64 + 32hf
          tmem_st32(lane_addr + kPCol + 32 * hf, pr);
          tmem_st32(lane_addr + kPCol + 64 + 32 * hf, pr + 32);
          tc::wait_st();
          tc::fence_before();
          __syncwarp();
          if (lane == 0) arrive_leader(&sm.p_full[hf]);
          PF2_TRACE(r == 0 && row == 0, g, 2 * hf + 1);
          const float2 a01 = __fadd2_rn(__fadd2_rn(acc[0], acc[1]), __fadd2_rn(acc[2], acc[3]));
          l_run = fmaf(l_run, alpha, a01.x + a01.y);
          m_run = m_new;
        }
      }
      // epilogue: the item's last PV has landed in O
      mbar_wait(&sm.o_full, n & 1);
      tc::fence_after();
      uint32_t o[D];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(lane_addr + kOCol + 32 * c, o + 32 * c);
      tc::wait_ld();
      tc::fence_before();
      __syncwarp();
      if (lane == 0) arrive_leader(&sm.o_free);  // the next item's PV may overwrite O
      const int tok = it.t * BM + row;
      if (tok < it.n_b) {
        const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
        __nv_bfloat16* dst = a.out + ((static_cast<int64_t>(it.q0) + tok) * a.hq + it.h) * D;
#pragma unroll
        for (int k = 0; k < D; k += 16) {
          uint32_t w8[8];
#pragma unroll
          for (int u8 = 0; u8 < 8; ++u8)
            w8[u8] = pack_bf16(__uint_as_float(o[k + 2 * u8]) * inv, __uint_as_float(o[k + 2 * u8 + 1]) * inv);
          asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + k),
                       "r"(w8[0]), "r"(w8[1]), "r"(w8[2]), "r"(w8[3]), "r"(w8[4]), "r"(w8[5]),
                       "r"(w8[6]), "r"(w8[7])
                       : "memory");
        }
      }
      ++n;
    }
  }
  tc::fence_before();
  cluster_sync();  // both CTAs done with TMEM and with each other's barriers
  tc::fence_after();
  if (warp == kMmaWarp) tmem_dealloc2(tmem, kTmemCols);
}

}  // namespace pf2

#ifdef VT_PF2_TRACE
extern "C" int vt_prefill_pair_trace(long long* out) {  // 256 x 8 values
  return cudaMemcpyFromSymbol(out, pf2::g_pf2_trace, sizeof(pf2::g_pf2_trace));
}
#endif

// Host launcher (called by vt_prefill.cu's entry points when the pair kernel
// applies): same arguments as launch_prefill.
int launch_prefill_pair(const vt_kv_geometry* g, int32_t layer, const void* q, const void* kv_maps,
                        const int32_t* start, const int32_t* q_off, int32_t batch,
                        int32_t max_n_new, int64_t total, float scale, void* out, void* stream) {
  using namespace pf2;
  if (g->head_dim != D || g->q_heads % g->kv_heads) return cudaErrorInvalidValue;
  const int tpc = g->tokens_per_chunk;
  if (!((tpc < BT && BT % tpc == 0) || (tpc >= BT && tpc % BT == 0))) return cudaErrorInvalidValue;
  if (batch <= 0 || max_n_new <= 0 || total <= 0) return 0;
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
  const int n_qtiles = (max_n_new + BM - 1) / BM;
  Args a{};
  a.out = static_cast<__nv_bfloat16*>(out);
  a.kv = static_cast<const CUtensorMap*>(kv_maps);
  a.start = start;
  a.q_off = q_off;
  a.n_new = max_n_new;
  a.hq = g->q_heads;
  a.hkv = g->kv_heads;
  a.tpc = tpc;
  a.layer = layer;
  a.batch = batch;
  a.head_pairs = group % 2 == 0 ? 1 : 0;
  if (a.head_pairs) {
    a.n_units = g->q_heads / 2;
    a.n_items = a.n_units * batch * n_qtiles;
  } else {
    a.n_units = g->q_heads;
    a.n_items = a.n_units * batch * ((n_qtiles + 1) / 2);
  }
  a.scale_log2 = scale * 1.4426950408889634f;
  const size_t smem = sizeof(Smem) + 1024;
  static std::atomic<uint64_t> attr_devices{0};
  vt::set_smem_limit_once(prefill_pair_kernel, smem, attr_devices);
  static int n_sm = 0;
  if (!n_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  }
  const int pairs = a.n_items < n_sm / 2 ? a.n_items : n_sm / 2;  // persistent: one pair per 2 SMs
  prefill_pair_kernel<<<2 * pairs, kThreads, smem, static_cast<cudaStream_t>(stream)>>>(qmap, a);
  return cudaGetLastError();
}

}  // namespace vt
