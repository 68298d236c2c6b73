// Decode attention on the 5th-gen tensor cores — sm_100a (row a27, the
// headline kernel).
//
// Decode is HBM-bound (G FLOP per KV byte), so the goal is to keep the TMA
// engine streaming K/V at full bandwidth while spending as few SM issue slots
// per byte as possible. The dot products therefore go to tcgen05 with the KV
// tile as the M=128 operand and the G = q_heads/kv_heads query heads of the
// group as N=16 (padded) columns:
//
//   S^T[128 tok, 16]  = K[128 tok, 128 d]   . Q^T[128 d, 16]    (A K-major, B K-major)
//   O^T[128 d, 16]   += V^T[128 d, 128 tok] . P^T[128 tok, 16]  (A MN-major, B K-major)
//
// Accumulators live in TMEM (S^T double-buffered, O^T per work unit).
//
// Persistent CTAs (one per SM), statically strided over work units
// (request b, kv head h, split s). Warp roles (192 threads):
//   warp 0    TMA producer. Q (16 rows x 128 d) per unit and 128-token K / V
//             tiles through 3-deep rings, via the request's 4-D tensor map over
//             its vTensor VA — the map's chunk extent is the mapped prefix, so
//             no load can fault; it streams across unit boundaries without
//             draining.
//   warp 1    MMA issuer (one elected thread), S^T_{j+1} before PV_j.
//   warps 2-5 one thread per TMEM lane: per tile it reads its token's G scores
//             (tcgen05.ld), masks tokens >= seq_len, joins a warp-shuffle +
//             smem column max across the 128 tokens, writes P^T (bf16) to
//             smem, and rescales O^T rows in TMEM when a head's max moved. The
//             softmax denominator is accumulated per thread and reduced once
//             per unit. Epilogue: thread d writes o[qh][d] (coalesced).
// Splits of one request are merged by decode_combine_kernel (vt_decode.cu).

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/vt_attention.h"
#include "vt_tc_common.cuh"

namespace vt {
namespace dtc {

#ifdef VT_DTC_HANG_DEBUG
// Debug build (tools/hang_probe_decode.py): an mbarrier wait that has not
// completed after 2 s records (source line, CTA, thread, parity, raw barrier
// word) into host-mapped memory once, then keeps waiting, so a hung process
// can say which wait it is stuck in.
__device__ unsigned long long* g_dbg;
__device__ void dbg_wait(uint64_t* bar, uint32_t parity, int line) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  bool recorded = false;
  while (!mbar_try_wait(bar, parity)) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (!recorded && t - t0 > 2000000000ull && g_dbg) {
      recorded = true;
      const unsigned long long i = atomicAdd(g_dbg, 1ull);
      if (i < 256) {
        unsigned long long raw;
        asm volatile("ld.shared.b64 %0, [%1];" : "=l"(raw) : "r"(smem_u32(bar)));
        volatile unsigned long long* r = g_dbg + 1 + i * 6;
        r[0] = line;
        r[1] = blockIdx.x;
        r[2] = threadIdx.x;
        r[3] = parity;
        r[4] = raw;
        r[5] = smem_u32(bar);
        __threadfence_system();
      }
    }
  }
}
#define mbar_wait(b, p) dbg_wait((b), (p), __LINE__)
#endif

constexpr int TILE = 128;   // tokens per KV tile (MMA M)
constexpr int D = 128;
constexpr int NQ = 16;      // padded q-head columns (MMA N)
constexpr int KSTAGES = 3;
constexpr int VSTAGES = 3;
constexpr int kThreads = 224;  // + warp 6: epilogue
constexpr int MAXG = 8;        // q heads per kv head handled by this kernel
constexpr uint32_t kTmemCols = 64;
constexpr uint32_t kSCol = 0;   // S^T buffers at columns 0 and 16
constexpr uint32_t kOCol = 32;  // per-tile O^T buffers at columns 32 and 48

constexpr int kLensSmem = 1024;

struct __align__(1024) Smem {
  __nv_bfloat16 k[KSTAGES][2][TILE * 64];  // SW128 K-major (tok x d)
  __nv_bfloat16 v[VSTAGES][2][TILE * 64];  // SW128, read as MN-major A (d x tok)
  __nv_bfloat16 q[2][2][NQ * 64];          // [unit buf][d half] SW128 K-major (16 x 64)
  __nv_bfloat16 p[2][2][NQ * 64];          // [tile parity] P^T [16 x 128 tok], tok halves
  float red[2][4][NQ];                     // per-warp column maxima (tile parity)
  struct Epi {                             // softmax -> epilogue hand-off, per unit
    float o[MAXG][D];
    float lpart[4][MAXG];
    float m[MAXG];
  } epi[2];
  int32_t lens[kLensSmem];                 // seq_lens of the first kLensSmem requests, staged once
  uint64_t k_full[KSTAGES], k_empty[KSTAGES];
  uint64_t v_full[VSTAGES], v_empty[VSTAGES];
  uint64_t q_full[2], q_empty[2];
  uint64_t s_full[2];
  // By tile parity: a waiter can never fall two phases behind. (A single
  // p_full let the softmax arrive P(g) — S(g) is issued before the MMA warp
  // waits for P(g-1) — before the MMA warp had observed P(g-1)'s phase; the
  // barrier then read as pending again and the two roles deadlocked. Seen
  // only when a time-sliced second process delayed the MMA warp, r02:
  // tools/hang_probe_decode.py, profiles/r02/timeslice/.)
  uint64_t p_full[2];
  uint64_t pv_done[2];
  uint64_t epi_full[2], epi_empty[2];
  uint32_t tmem_base;
};

struct Args {
  const CUtensorMap* kv;    // [B] per-request maps over the vTensor VAs
  const int32_t* seq_lens;  // [B]
  __nv_bfloat16* out;       // [B, Hq, D]
  float* part_o;            // [B, Hkv, S, G, D]
  float* part_ml;           // [B, Hkv, S, G, 2]
  int32_t* arrivals;        // [B, Hkv] split arrival counters (self-resetting)
  int32_t batch, hq, hkv, group, n_splits, split_tok, tpc, layer;
  float scale_log2;
};

struct Unit {
  int b, h, s, t0, t1, splits_b;
};

// Split-major unit order: the CTA striding u, u+grid, ... gets a mix of long
// (first) and short (last) splits of a request instead of always the same split.
__device__ __forceinline__ bool unit_of(const Args& a, const int32_t* lens, int u, Unit& w) {
  const int nbh = a.batch * a.hkv;
  w.s = u / nbh;
  const int bh = u % nbh;
  w.h = bh % a.hkv;
  w.b = bh / a.hkv;
  const int len = w.b < kLensSmem ? lens[w.b] : __ldg(a.seq_lens + w.b);  // larger batches: L1/L2
  w.t0 = w.s * a.split_tok;
  w.t1 = min(len, w.t0 + a.split_tok);
  w.splits_b = (len + a.split_tok - 1) / a.split_tok;
  return w.t0 < w.t1;
}

// Column max of G scores across the 32 lanes of a warp by exchange-halving:
// each step trades half of the remaining columns with the partner lane, so
// G=8 costs 9 shuffles instead of 40. Returns the max of column `col`.
template <int G>
__device__ __forceinline__ float warp_colmax(float (&v)[G], int lane, int& col) {
  int n = G;
  int own = 0;
#pragma unroll
  for (int bit = 4; bit >= 0; --bit) {
    const int m = 1 << bit;
    if (n > 1) {
      const int half = n >> 1;
      const bool up = (lane >> bit) & 1;
#pragma unroll
      for (int i = 0; i < G / 2; ++i) {
        if (i < half) {
          const float send = up ? v[i] : v[i + half];
          const float keep = up ? v[i + half] : v[i];
          v[i] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, m));
        }
      }
      own += up ? half : 0;
      n = half;
    } else {
      v[0] = fmaxf(v[0], __shfl_xor_sync(0xffffffffu, v[0], m));
    }
  }
  col = own;
  return v[0];
}

template <int G>
__global__ void __launch_bounds__(kThreads, 1)
    decode_tc_kernel(const __grid_constant__ CUtensorMap q_map, const Args a) {
  extern __shared__ uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                      ~static_cast<uintptr_t>(1023));
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_units = a.batch * a.hkv * a.n_splits;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < KSTAGES; ++i) {
      mbar_init(&sm.k_full[i], 1);
      mbar_init(&sm.k_empty[i], 1);
    }
    for (int i = 0; i < VSTAGES; ++i) {
      mbar_init(&sm.v_full[i], 1);
      mbar_init(&sm.v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.q_full[i], 1);
      mbar_init(&sm.q_empty[i], 1);
      mbar_init(&sm.s_full[i], 1);
    }
    mbar_init(&sm.p_full[0], 128);
    mbar_init(&sm.p_full[1], 128);
    mbar_init(&sm.pv_done[0], 1);
    mbar_init(&sm.pv_done[1], 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.epi_full[i], 128);
      mbar_init(&sm.epi_empty[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tc::alloc(&sm.tmem_base, kTmemCols);
  for (int i = threadIdx.x; i < min(a.batch, kLensSmem); i += kThreads) sm.lens[i] = a.seq_lens[i];
  // P^T rows G..15 are never written: zero the whole buffer once.
  for (int i = threadIdx.x; i < 4 * NQ * 64 / 8; i += kThreads)
    reinterpret_cast<uint4*>(&sm.p[0][0][0])[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = sm.tmem_base;
  tc::grid_launch_dependents();  // the next layer's CTAs may take SMs this grid frees

  if (warp == 0) {
    // -------------------------------- producer --------------------------------
    if (lane == 0) {
      tma_prefetch_desc(&q_map);
      const uint64_t once = l2_evict_first_policy();
      int kc = 0, vc = 0, qc = 0;
      bool dep_waited = false;
      auto issue_kv = [&](const CUtensorMap* kvmap, int blk_k, int blk_v, int tok0) {
        const int c1 = tok0 % a.tpc;
        const int c3 = tok0 / a.tpc;
        const int ks = kc % KSTAGES;
        if (kc >= KSTAGES) mbar_wait(&sm.k_empty[ks], ((kc / KSTAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&sm.k_full[ks], 2 * TILE * 64 * 2);
        tma_load_4d(sm.k[ks][0], kvmap, &sm.k_full[ks], 0, c1, blk_k, c3, once);
        tma_load_4d(sm.k[ks][1], kvmap, &sm.k_full[ks], 64, c1, blk_k, c3, once);
        ++kc;
        const int vs = vc % VSTAGES;
        if (vc >= VSTAGES) mbar_wait(&sm.v_empty[vs], ((vc / VSTAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&sm.v_full[vs], 2 * TILE * 64 * 2);
        tma_load_4d(sm.v[vs][0], kvmap, &sm.v_full[vs], 0, c1, blk_v, c3, once);
        tma_load_4d(sm.v[vs][1], kvmap, &sm.v_full[vs], 64, c1, blk_v, c3, once);
        ++vc;
      };
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        Unit w;
        if (!unit_of(a, sm.lens, u, w)) continue;
        const CUtensorMap* kvmap = a.kv + w.b;
        if (u + static_cast<int>(gridDim.x) < n_units)  // warm the next unit's descriptor
          tma_prefetch_desc(a.kv + ((u + gridDim.x) % (a.batch * a.hkv)) / a.hkv);
        const int blk_k = (a.layer * 2 + 0) * a.hkv + w.h;
        const int blk_v = (a.layer * 2 + 1) * a.hkv + w.h;
        int tok0 = w.t0;
        if (!dep_waited) {
          // Programmatic dependent launch: this layer's K/V do not depend on
          // the previous kernel (in a layer stack, q does), so the first
          // ring's worth of K/V streams while that kernel drains.
          for (int j = 0; j < KSTAGES && j < VSTAGES && tok0 < w.t1; ++j, tok0 += TILE)
            issue_kv(kvmap, blk_k, blk_v, tok0);
          tc::grid_dependency_wait();
          dep_waited = true;
        }
        const int qb = qc & 1;
        if (qc >= 2) mbar_wait(&sm.q_empty[qb], ((qc >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&sm.q_full[qb], 2 * NQ * 64 * 2);
        const int qrow = w.b * a.hq + w.h * G;
        tc::tma_load_2d(sm.q[qb][0], &q_map, &sm.q_full[qb], 0, qrow, once);
        tc::tma_load_2d(sm.q[qb][1], &q_map, &sm.q_full[qb], 64, qrow, once);
        ++qc;
        for (; tok0 < w.t1; tok0 += TILE) issue_kv(kvmap, blk_k, blk_v, tok0);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------- MMA issuer -------------------------------
    if (lane == 0) {
      constexpr uint32_t id_s = tc::idesc_bf16(TILE, NQ, false, false);
      constexpr uint32_t id_o = tc::idesc_bf16(D, NQ, true, false);
      int g = 0;   // global tile counter (S/P/PV phases)
      int qc = 0;
      auto issue_pv = [&](int gt) {
        mbar_wait(&sm.p_full[gt & 1], (gt >> 1) & 1);
        const int vs = gt % VSTAGES;
        mbar_wait(&sm.v_full[vs], (gt / VSTAGES) & 1);
        tc::fence_after();
        const uint8_t* pb = reinterpret_cast<const uint8_t*>(sm.p[gt & 1][0]);
#pragma unroll
        for (int kk = 0; kk < TILE / 16; ++kk) {
          const uint64_t ad = tc::sdesc(reinterpret_cast<const uint8_t*>(sm.v[vs][0]) + kk * 2048,
                                        TILE * 128, 1024);
          const uint64_t bd = tc::sdesc(pb + (kk >> 2) * (NQ * 128) + 32 * (kk & 3), 16, 1024);
          tc::mma(tmem + kOCol + (gt & 1) * NQ, ad, bd, id_o, kk > 0 ? 1u : 0u);
        }
        tc::commit(&sm.pv_done[gt & 1]);
        tc::commit(&sm.v_empty[vs]);
      };
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        Unit w;
        if (!unit_of(a, sm.lens, u, w)) continue;
        const int qb = qc & 1;
        mbar_wait(&sm.q_full[qb], (qc >> 1) & 1);
        int pending = -1;  // tile of this unit whose PV is not yet issued
        for (int tok0 = w.t0; tok0 < w.t1; tok0 += TILE, ++g) {
          const int ks = g % KSTAGES;
          mbar_wait(&sm.k_full[ks], (g / KSTAGES) & 1);
          tc::fence_after();
          const uint32_t sc = kSCol + static_cast<uint32_t>((g & 1) * NQ);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint64_t ad = tc::sdesc(reinterpret_cast<const uint8_t*>(sm.k[ks][kk >> 2]) +
                                              32 * (kk & 3),
                                          16, 1024);
            const uint64_t bd = tc::sdesc(reinterpret_cast<const uint8_t*>(sm.q[qb][kk >> 2]) +
                                              32 * (kk & 3),
                                          16, 1024);
            tc::mma(tmem + sc, ad, bd, id_s, kk > 0 ? 1u : 0u);
          }
          tc::commit(&sm.s_full[g & 1]);
          tc::commit(&sm.k_empty[ks]);
          if (pending >= 0) issue_pv(pending);  // S_{j+1} overlaps softmax_j
          pending = g;
        }
        tc::commit(&sm.q_empty[qb]);
        ++qc;
        issue_pv(pending);  // close the unit now: its epilogue must not wait on the next unit
      }
    }
    __syncwarp();
  } else if (warp == 6) {
    // -------------------------------- epilogue --------------------------------
    // Global writes, the split-arrival atomic and the log-sum-exp merge of a
    // request's splits happen here, off the softmax critical path.
    tc::grid_dependency_wait();  // outputs and the split workspace: previous kernel's until now
    int uc = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      Unit w;
      if (!unit_of(a, sm.lens, u, w)) continue;
      const int eb = uc & 1;
      mbar_wait(&sm.epi_full[eb], (uc >> 1) & 1);
      const auto& e = sm.epi[eb];
      const int64_t bh = static_cast<int64_t>(w.b) * a.hkv + w.h;
      const int64_t unit = bh * a.n_splits + w.s;
      __nv_bfloat16* dst = a.out + (static_cast<int64_t>(w.b) * a.hq + w.h * G) * D;
      if (w.splits_b == 1) {
        for (int i = lane; i < G * D; i += 32) {
          const int c = i / D;
          const float l = e.lpart[0][c] + e.lpart[1][c] + e.lpart[2][c] + e.lpart[3][c];
          dst[i] = __float2bfloat16(l > 0.f ? e.o[c][i % D] / l : 0.f);
        }
      } else {
        for (int i = lane; i < G * D; i += 32) a.part_o[unit * G * D + i] = e.o[i / D][i % D];
        if (lane < G) {
          a.part_ml[(unit * G + lane) * 2 + 0] = e.m[lane];
          a.part_ml[(unit * G + lane) * 2 + 1] =
              e.lpart[0][lane] + e.lpart[1][lane] + e.lpart[2][lane] + e.lpart[3][lane];
        }
        __syncwarp();  // orders the warp's partial writes before lane 0's release
        int last = 0;
        if (lane == 0) {
          int prev;
          asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;"
                       : "=r"(prev)
                       : "l"(&a.arrivals[bh])
                       : "memory");
          last = prev == w.splits_b - 1;
          if (last) a.arrivals[bh] = 0;  // self-reset for the next launch
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
          // Log-sum-exp merge of the request's splits, all G heads at once:
          // lane l owns head l % G for the (split, head) pairs p = l, l+32, ...
          // (G divides 32), so each phase is one round of independent loads
          // plus a shuffle reduction — not G rounds of dependent ones (the
          // per-head loop made the epilogue warp the bottleneck at G = 8).
          const int64_t u0 = bh * a.n_splits;
          const int S = w.splits_b;
          const float* ml = a.part_ml + u0 * G * 2;  // [split][head][m, l]
          float mloc = -INFINITY;
          for (int p = lane; p < S * G; p += 32) mloc = fmaxf(mloc, __ldcg(ml + p * 2));
#pragma unroll
          for (int m = 16; m >= G; m >>= 1) mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, m));
          float dloc = 0.f;
          for (int p = lane; p < S * G; p += 32)
            dloc += tc::ex2(__ldcg(ml + p * 2) - mloc) * __ldcg(ml + p * 2 + 1);
#pragma unroll
          for (int m = 16; m >= G; m >>= 1) dloc += __shfl_xor_sync(0xffffffffu, dloc, m);
          const float inv = dloc > 0.f ? 1.f / dloc : 0.f;
          float mx_c[G], inv_c[G], acc[G][D / 32];
#pragma unroll
          for (int c = 0; c < G; ++c) {
            mx_c[c] = __shfl_sync(0xffffffffu, mloc, c);
            inv_c[c] = __shfl_sync(0xffffffffu, inv, c);
#pragma unroll
            for (int j = 0; j < D / 32; ++j) acc[c][j] = 0.f;
          }
          for (int k = 0; k < S; ++k) {
            const float* po = a.part_o + (u0 + k) * G * D + lane;
#pragma unroll
            for (int c = 0; c < G; ++c) {
              const float wgt = tc::ex2(__ldcg(ml + (k * G + c) * 2) - mx_c[c]);
#pragma unroll
              for (int j = 0; j < D / 32; ++j)
                acc[c][j] = fmaf(wgt, __ldcg(po + c * D + 32 * j), acc[c][j]);
            }
          }
#pragma unroll
          for (int c = 0; c < G; ++c)
#pragma unroll
            for (int j = 0; j < D / 32; ++j)
              dst[c * D + lane + 32 * j] = __float2bfloat16(acc[c][j] * inv_c[c]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.epi_empty[eb]);
      ++uc;
    }
  } else {
    // ------------------------ softmax / correction / out ----------------------
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;  // token in tile (S^T) / d (O^T)
    const uint32_t lane_addr = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    const float sl2 = a.scale_log2;
    const int tid = threadIdx.x - 64;  // 0..127
    tc::grid_dependency_wait();  // (zero outputs of empty requests below)
    int g = 0;
    int uc = 0;  // units handed to the epilogue warp
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      Unit w;
      if (!unit_of(a, sm.lens, u, w)) {
        if (w.s == 0 && w.t1 <= 0) {  // empty request: defined output is zero
          for (int c = 0; c < G; ++c)
            a.out[(static_cast<int64_t>(w.b) * a.hq + w.h * G + c) * D + row] = __float2bfloat16(0.f);
        }
        continue;
      }
      float m_run[G], l_thr[G], o_acc[G], alpha_prev[G];
#pragma unroll
      for (int c = 0; c < G; ++c) {
        m_run[c] = -INFINITY;
        l_thr[c] = 0.f;
        o_acc[c] = 0.f;
        alpha_prev[c] = 1.f;
      }
      // Fold tile gt's O^T (in TMEM) into the register accumulator:
      // o = o * alpha_gt + O_gt. Runs one tile late, so the PV latency is off
      // the softmax critical path.
      auto fold = [&](int gt) {
        mbar_wait(&sm.pv_done[gt & 1], (gt >> 1) & 1);
        tc::fence_after();
        uint32_t o[NQ];
        tc::ld16(lane_addr + kOCol + (gt & 1) * NQ, o);
        tc::wait_ld();
#pragma unroll
        for (int c = 0; c < G; ++c) o_acc[c] = fmaf(o_acc[c], alpha_prev[c], __uint_as_float(o[c]));
      };
      const int g_first = g;
      for (int tok0 = w.t0; tok0 < w.t1; tok0 += TILE, ++g) {
        mbar_wait(&sm.s_full[g & 1], (g >> 1) & 1);
        tc::fence_after();
        uint32_t r[NQ];
        tc::ld16(lane_addr + kSCol + (g & 1) * NQ, r);
        tc::wait_ld();
        const bool valid = tok0 + row < w.t1;
        float x[G];
        float mx[G];
#pragma unroll
        for (int c = 0; c < G; ++c) {
          x[c] = valid ? __uint_as_float(r[c]) * sl2 : -INFINITY;
          mx[c] = x[c];
        }
        {
          int col;
          const float cm = warp_colmax<G>(mx, lane, col);
          if ((lane & ((32 / G) - 1)) == 0) sm.red[g & 1][quarter][col] = cm;
        }
        named_bar_sync(1, 128);
        float alpha[G];
#pragma unroll
        for (int c = 0; c < G; ++c) {
          const float(*rd)[NQ] = sm.red[g & 1];
          const float tmax = fmaxf(fmaxf(rd[0][c], rd[1][c]), fmaxf(rd[2][c], rd[3][c]));
          const float m_new = fmaxf(m_run[c], tmax);
          alpha[c] = tc::ex2(m_run[c] - m_new);
          m_run[c] = m_new;
          const float p = tc::ex2(x[c] - m_new);
          x[c] = p;
          l_thr[c] = l_thr[c] * alpha[c] + p;
        }
        if (tok0 + TILE > w.t1) {
          // tail tile: rows >= t1 may be stale bytes of the last mapped chunk
          const int vs = g % VSTAGES;
          mbar_wait(&sm.v_full[vs], (g / VSTAGES) & 1);
          if (!valid) {
            uint4 z = make_uint4(0, 0, 0, 0);
            uint4* r0 = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(sm.v[vs][0]) + row * 128);
            uint4* r1 = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(sm.v[vs][1]) + row * 128);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              r0[c] = z;
              r1[c] = z;
            }
          }
        }
        // P^T[c][row] (bf16), SW128 K-major, buffer g&1 (PV_{g-2} finished:
        // it was folded during the previous tile)
        {
          uint8_t* blk = reinterpret_cast<uint8_t*>(sm.p[g & 1][row >> 6]);
          const int tk = row & 63;
#pragma unroll
          for (int c = 0; c < G; ++c) {
            const int chunk = (tk >> 3) ^ (c & 7);
            *reinterpret_cast<__nv_bfloat16*>(blk + c * 128 + (chunk << 4) + (tk & 7) * 2) =
                __float2bfloat16(x[c]);
          }
        }
        fence_proxy_async_smem();
        tc::fence_before();
        mbar_arrive(&sm.p_full[g & 1]);
        if (g > g_first) fold(g - 1);
#pragma unroll
        for (int c = 0; c < G; ++c) alpha_prev[c] = alpha[c];
      }
      // ----- unit epilogue: hand (o, m, l) to the epilogue warp -----
      fold(g - 1);
      const int eb = uc & 1;
      if (uc >= 2) mbar_wait(&sm.epi_empty[eb], ((uc >> 1) & 1) ^ 1);
#pragma unroll
      for (int c = 0; c < G; ++c) {
        const float lw = warp_sum(l_thr[c]);
        sm.epi[eb].o[c][row] = o_acc[c];
        if (lane == 0) sm.epi[eb].lpart[quarter][c] = lw;
        if (tid == 0) sm.epi[eb].m[c] = m_run[c];
      }
      mbar_arrive(&sm.epi_full[eb]);
      ++uc;
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 1) tc::dealloc(tmem, kTmemCols);
}

}  // namespace dtc
}  // namespace vt

using namespace vt::dtc;

#ifdef VT_DTC_HANG_DEBUG
extern "C" int vt_dtc_debug_set(unsigned long long* host_mapped) {
  return cudaMemcpyToSymbol(g_dbg, &host_mapped, sizeof(host_mapped));
}
#endif

// Called from vt_decode.cu's dispatcher (same workspace layout as the CUDA-core
// path, so the combine kernel is shared).
int vt_launch_decode_tc(const vt_kv_geometry* g, int32_t layer, const void* q,
                        const void* kv_maps, const int32_t* seq_lens, int32_t batch,
                        int32_t n_splits, int32_t split, float scale, void* out, float* part_o,
                        float* part_ml, int32_t* arrivals, int32_t n_sms, bool pdl,
                        cudaStream_t stream) {
  const int G = g->q_heads / g->kv_heads;
  if (G > MAXG || split % TILE) return cudaErrorInvalidValue;
  static_assert(sizeof(Smem) + 1024 <= 232448, "shared memory budget");
  CUtensorMap qmap;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(D),
                              static_cast<cuuint64_t>(batch) * g->q_heads};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(D * 2)};
  const cuuint32_t box[2] = {64, NQ};
  int rc = vt::encode_tensor_map_bf16(&qmap, const_cast<void*>(q), 2, dims, strides, box);
  if (rc) return rc;
  Args a{};
  a.kv = static_cast<const CUtensorMap*>(kv_maps);
  a.seq_lens = seq_lens;
  a.out = static_cast<__nv_bfloat16*>(out);
  a.part_o = part_o;
  a.part_ml = part_ml;
  a.arrivals = arrivals;
  a.batch = batch;
  a.hq = g->q_heads;
  a.hkv = g->kv_heads;
  a.group = G;
  a.n_splits = n_splits;
  a.split_tok = split;
  a.tpc = g->tokens_per_chunk;
  a.layer = layer;
  a.scale_log2 = scale * 1.4426950408889634f;
  const size_t smem = sizeof(Smem) + 1024;
  const int units = batch * g->kv_heads * n_splits;
  const int grid = units < n_sms ? units : n_sms;
  auto launch = [&](auto kernel) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    // Chained launches (a decode layer right after another decode layer)
    // use programmatic dependent launch: this grid's CTAs start streaming
    // their first ring of K/V while the previous layer drains; q, outputs and
    // the split workspace are touched only after griddepcontrol.wait. The
    // first decode after the step's KV append is a plain launch (it reads the
    // K/V that kernel writes). Measured (bench, config 2): 6392 -> 6632 GB/s
    // per step. Cost: with boundaries only once per step the driver applies
    // the worker's concurrent cuMemMap / cuMemSetAccess at the next plain
    // kernel boundary (SetAccess 0.7 -> 2.7 ms at 8B, ~17 ms at 32k), which
    // the map-ahead extends absorb (0 host waits, 0 stalled steps).
    if (pdl) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid, 1, 1);
      cfg.blockDim = dim3(kThreads, 1, 1);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, kernel, qmap, a);
    } else {
      kernel<<<grid, kThreads, smem, stream>>>(qmap, a);
    }
  };
  switch (G) {
    case 1: launch(decode_tc_kernel<1>); break;
    case 2: launch(decode_tc_kernel<2>); break;
    case 4: launch(decode_tc_kernel<4>); break;
    case 8: launch(decode_tc_kernel<8>); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}
