// Decode attention over a vTensor KV cache — sm_100a (row a27).
//
// Work unit = (request b, kv head h, split s): KV tokens [s*split, (s+1)*split)
// of one request's VA, clipped to seq_len. One CTA per unit:
//   warp 4      : producer. Streams the unit's K and V rows in 64-token stages
//                 into a 2-deep shared-memory ring with cp.async.bulk
//                 (UBLKCP) + mbarrier complete_tx. A stage that crosses chunk
//                 boundaries is one bulk copy per chunk run; with tpc = 16
//                 that is 4 KiB contiguous per copy. No block table: the
//                 address is va + chunk*chunk_bytes + block offset.
//   warps 0..3  : consumers, for the G = q_heads/kv_heads query heads that
//                 share kv head h (GQA grouping: K/V are read once per group).
//                 Scores: 8 lanes per token, each holding a 16-element slice
//                 of d (two 16 B smem vectors, conflict-free), packed FFMA2
//                 (fma.rn.f32x2) dot products, then an exchange-halving warp
//                 shuffle reduction (G=4: 4 SHFL instead of 12).
//                 Online softmax per stage with warp-shuffle max/sum (exp2
//                 domain, scale folded into q). PV: each thread owns 8 d
//                 columns x G heads in packed fp32 accumulators.
// Partial (o, m, l) per unit go to a workspace and a combine kernel merges the
// splits (log-sum-exp); a request with a single split writes its output
// directly.
//
// Memory safety: only chunks holding tokens < seq_len are ever touched, so a
// unit never reads unmapped VA. Stale rows of a partial
// stage are masked to -inf in the scores and skipped in PV.

#include <algorithm>

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/vt_attention.h"
#include "vt_common.cuh"

namespace vt {

constexpr int kD = 128;
constexpr int kStageTok = 64;
constexpr int kConsumerWarps = 4;
constexpr int kThreads = (kConsumerWarps + 1) * 32;

// Per-group-size tuning: G=8 needs 2x the q/acc registers, so it runs one CTA
// per SM with a deeper ring to keep the same bytes in flight per SM.
template <int G>
struct DecodeCfg {
  static constexpr int kStages = G >= 8 ? 5 : 2;
  static constexpr int kMinBlocks = G >= 8 ? 1 : 3;
};

struct DecodeArgs {
  const __nv_bfloat16* q;
  const uint64_t* kv_va;
  const int32_t* seq_lens;
  __nv_bfloat16* out;
  float* part_o;   // [B, Hkv, S, G, D]
  float* part_ml;  // [B, Hkv, S, G, 2]
  int32_t batch, hkv, n_splits, split_tok, tpc;
  int64_t chunk_bytes;
  int64_t k_off, v_off;   // byte offset of (layer, K|V, head 0) inside a chunk
  int64_t head_bytes;     // tpc * D * 2
  float scale_log2;
  // Paged baseline (vt_decode_attention_paged): chunk c of request b lives at
  // pool_base + block_table[b * max_blocks + c] * chunk_bytes instead of at
  // kv_va[b] + c * chunk_bytes — one dependent table load per block.
  const int32_t* block_table;
  int32_t max_blocks;
  uint64_t pool_base;
};

template <int G>
struct DecodeSmem {
  static constexpr int kStages = DecodeCfg<G>::kStages;
  __nv_bfloat16 k[kStages][kStageTok * kD];
  __nv_bfloat16 v[kStages][kStageTok * kD];
  float s[G][kStageTok];     // scores (log2 domain)
  float p[kStageTok][G];     // probabilities
  float alpha[G];
  float ml[G][2];
  uint64_t full[kStages];
  uint64_t empty[kStages];
};

__device__ __forceinline__ void bf16x8_to_f2(const uint4& w, float2 (&f)[4]) {
  const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[i].x = __uint_as_float(u[i] << 16);
    f[i].y = __uint_as_float(u[i] & 0xffff0000u);
  }
}

template <int G>
__global__ void __launch_bounds__(kThreads, DecodeCfg<G>::kMinBlocks)
    decode_splitkv_kernel(const DecodeArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  auto& sm = *reinterpret_cast<DecodeSmem<G>*>(smem_raw);
  constexpr int kStages = DecodeCfg<G>::kStages;

  const int s = blockIdx.x;
  const int h = blockIdx.y;
  const int b = blockIdx.z;
  const int len = a.seq_lens[b];
  const int t_begin = s * a.split_tok;
  if (t_begin >= len) {  // whole CTA exits before any barrier use
    if (s == 0 && len == 0)  // empty request: defined output is zero
      for (int i = threadIdx.x; i < G * kD; i += blockDim.x)
        a.out[(static_cast<int64_t>(b) * a.hkv + h) * G * kD + i] = __float2bfloat16(0.f);
    return;
  }
  const int t_end = min(len, t_begin + a.split_tok);
  const int n_stage = (t_end - t_begin + kStageTok - 1) / kStageTok;
  const int splits_b = (len + a.split_tok - 1) / a.split_tok;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ------------------------------ producer ------------------------------
    const uint64_t va = a.block_table == nullptr ? a.kv_va[b] : 0;
    const uint64_t policy = l2_evict_first_policy();
    for (int st = 0; st < n_stage; ++st) {
      const int slot = st % kStages;
      if (st >= kStages) mbar_wait(&sm.empty[slot], ((st / kStages) & 1) ^ 1);
      const int tok0 = t_begin + st * kStageTok;
      const int ntok = min(kStageTok, t_end - tok0);
      if (lane == 0) mbar_arrive_expect_tx(&sm.full[slot], 2u * ntok * kD * 2);
      __syncwarp();
      const int c0 = tok0 / a.tpc;
      const int c1 = (tok0 + ntok - 1) / a.tpc;
      for (int c = c0 + lane; c <= c1; c += 32) {
        const int p0 = max(tok0, c * a.tpc);
        const int p1 = min(tok0 + ntok, (c + 1) * a.tpc);
        const uint32_t bytes = static_cast<uint32_t>(p1 - p0) * kD * 2;
        const uint64_t chunk_base =
            a.block_table == nullptr
                ? va + static_cast<uint64_t>(c) * a.chunk_bytes
                : a.pool_base + static_cast<uint64_t>(
                                    __ldg(&a.block_table[static_cast<int64_t>(b) * a.max_blocks + c])) *
                                    a.chunk_bytes;
        const uint64_t src = chunk_base + static_cast<uint64_t>(h) * a.head_bytes +
                             static_cast<uint64_t>(p0 - c * a.tpc) * kD * 2;
        const int row = p0 - tok0;
        bulk_g2s(&sm.k[slot][row * kD], src + a.k_off, bytes, &sm.full[slot], policy);
        bulk_g2s(&sm.v[slot][row * kD], src + a.v_off, bytes, &sm.full[slot], policy);
      }
    }
    return;
  }

  // ------------------------------- consumers -------------------------------
  const int g = lane >> 3;  // token slot within a pass
  const int r = lane & 7;   // d-slice owner: elements [8r,8r+8) and [64+8r,64+8r+8)
  // q slice for the G heads of this group, pre-scaled by scale*log2(e).
  float2 qf[G][8];
  {
    const __nv_bfloat16* qb = a.q + (static_cast<int64_t>(b) * a.hkv + h) * G * kD;
#pragma unroll
    for (int qh = 0; qh < G; ++qh) {
      const uint4 lo = *reinterpret_cast<const uint4*>(qb + qh * kD + 8 * r);
      const uint4 hi = *reinterpret_cast<const uint4*>(qb + qh * kD + 64 + 8 * r);
      float2 f[4];
      bf16x8_to_f2(lo, f);
#pragma unroll
      for (int i = 0; i < 4; ++i) qf[qh][i] = make_float2(f[i].x * a.scale_log2, f[i].y * a.scale_log2);
      bf16x8_to_f2(hi, f);
#pragma unroll
      for (int i = 0; i < 4; ++i) qf[qh][4 + i] = make_float2(f[i].x * a.scale_log2, f[i].y * a.scale_log2);
    }
  }
  constexpr int kOwn = (G + kConsumerWarps - 1) / kConsumerWarps;
  float m_run[kOwn], l_run[kOwn];
#pragma unroll
  for (int i = 0; i < kOwn; ++i) {
    m_run[i] = -INFINITY;
    l_run[i] = 0.f;
  }
  const int tid = threadIdx.x;  // 0..127
  const int tg = tid >> 4;      // PV token group 0..7
  const int dc = tid & 15;      // PV d chunk: columns [8dc, 8dc+8)
  float2 acc[G][4];
#pragma unroll
  for (int qh = 0; qh < G; ++qh)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[qh][i] = make_float2(0.f, 0.f);

  for (int st = 0; st < n_stage; ++st) {
    const int slot = st % kStages;
    const int tok0 = t_begin + st * kStageTok;
    const int ntok = min(kStageTok, t_end - tok0);
    mbar_wait(&sm.full[slot], (st / kStages) & 1);

    // ---- phase A: scores for 64 tokens (warp w: tokens 16w..16w+15) ----
    const __nv_bfloat16* kbase = sm.k[slot];
#pragma unroll
    for (int pass = 0; pass < 4; ++pass) {
      const int t = warp * 16 + pass * 4 + g;
      const uint4 lo = *reinterpret_cast<const uint4*>(kbase + t * kD + 8 * r);
      const uint4 hi = *reinterpret_cast<const uint4*>(kbase + t * kD + 64 + 8 * r);
      float2 kf[8];
      {
        float2 f[4];
        bf16x8_to_f2(lo, f);
#pragma unroll
        for (int i = 0; i < 4; ++i) kf[i] = f[i];
        bf16x8_to_f2(hi, f);
#pragma unroll
        for (int i = 0; i < 4; ++i) kf[4 + i] = f[i];
      }
      float v[G];
#pragma unroll
      for (int qh = 0; qh < G; ++qh) {
        float2 d2 = __fmul2_rn(qf[qh][0], kf[0]);
#pragma unroll
        for (int i = 1; i < 8; ++i) d2 = __ffma2_rn(qf[qh][i], kf[i], d2);
        v[qh] = d2.x + d2.y;
      }
      // Exchange-halving reduction over the 8 lanes of this token.
      int own = 0;
      int n = G;
#pragma unroll
      for (int bit = 2; bit >= 0; --bit) {
        const int mask = 1 << bit;
        if (n > 1) {
          const int half = n >> 1;
          const bool up = (r >> bit) & 1;
#pragma unroll
          for (int i = 0; i < half; ++i) {
            const float send = up ? v[i] : v[i + half];
            const float keep = up ? v[i + half] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, mask);
          }
          own += up ? half : 0;
          n = half;
        } else {
          v[0] += __shfl_xor_sync(0xffffffffu, v[0], mask);
        }
      }
      const bool valid = tok0 + t < t_end;
      sm.s[own][t] = valid ? v[0] : -INFINITY;
    }
    named_bar_sync(1, kConsumerWarps * 32);

    // ---- phase B: online softmax for the heads this warp owns ----
#pragma unroll
    for (int i = 0; i < kOwn; ++i) {
      const int qh = warp + i * kConsumerWarps;
      if (qh < G) {
        const float x0 = sm.s[qh][lane];
        const float x1 = sm.s[qh][lane + 32];
        const float mt = warp_max(fmaxf(x0, x1));
        const float m_new = fmaxf(m_run[i], mt);
        const float alpha = exp2f(m_run[i] - m_new);
        const float p0 = exp2f(x0 - m_new);
        const float p1 = exp2f(x1 - m_new);
        const float sum = warp_sum(p0 + p1);
        l_run[i] = l_run[i] * alpha + sum;
        m_run[i] = m_new;
        sm.p[lane][qh] = p0;
        sm.p[lane + 32][qh] = p1;
        if (lane == 0) sm.alpha[qh] = alpha;
      }
    }
    named_bar_sync(1, kConsumerWarps * 32);

    // ---- phase C: acc = alpha * acc + P V ----
#pragma unroll
    for (int qh = 0; qh < G; ++qh) {
      const float al = sm.alpha[qh];
      const float2 al2 = make_float2(al, al);
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[qh][i] = __fmul2_rn(acc[qh][i], al2);
    }
    const __nv_bfloat16* vbase = sm.v[slot];
    for (int t = tg; t < ntok; t += 8) {
      const uint4 w = *reinterpret_cast<const uint4*>(vbase + t * kD + 8 * dc);
      float2 vf[4];
      bf16x8_to_f2(w, vf);
      float pr[G];
      if constexpr (G % 4 == 0) {
#pragma unroll
        for (int j = 0; j < G; j += 4) {
          const float4 p4 = *reinterpret_cast<const float4*>(&sm.p[t][j]);
          pr[j] = p4.x;
          pr[j + 1] = p4.y;
          pr[j + 2] = p4.z;
          pr[j + 3] = p4.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < G; ++j) pr[j] = sm.p[t][j];
      }
#pragma unroll
      for (int qh = 0; qh < G; ++qh) {
        const float2 p2 = make_float2(pr[qh], pr[qh]);
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[qh][i] = __ffma2_rn(p2, vf[i], acc[qh][i]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[slot]);
  }

  // ---- epilogue: reduce the 8 token groups, then write partial or final ----
#pragma unroll
  for (int i = 0; i < kOwn; ++i) {
    const int qh = warp + i * kConsumerWarps;
    if (qh < G && lane == 0) {
      sm.ml[qh][0] = m_run[i];
      sm.ml[qh][1] = l_run[i];
    }
  }
  named_bar_sync(1, kConsumerWarps * 32);  // ring is free now: reuse it
  float* red = reinterpret_cast<float*>(&sm.k[0][0]);  // [8][G][D]
#pragma unroll
  for (int qh = 0; qh < G; ++qh) {
    float4* dst = reinterpret_cast<float4*>(red + (tg * G + qh) * kD + 8 * dc);
    dst[0] = make_float4(acc[qh][0].x, acc[qh][0].y, acc[qh][1].x, acc[qh][1].y);
    dst[1] = make_float4(acc[qh][2].x, acc[qh][2].y, acc[qh][3].x, acc[qh][3].y);
  }
  named_bar_sync(1, kConsumerWarps * 32);
  const int64_t unit = (static_cast<int64_t>(b) * a.hkv + h) * a.n_splits + s;
  for (int idx = tid; idx < G * kD; idx += kConsumerWarps * 32) {
    float o = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) o += red[k * G * kD + idx];
    const int qh = idx / kD;
    if (splits_b == 1) {
      const float l = sm.ml[qh][1];
      const float inv = l > 0.f ? 1.f / l : 0.f;
      a.out[(static_cast<int64_t>(b) * a.hkv + h) * G * kD + idx] = __float2bfloat16(o * inv);
    } else {
      a.part_o[unit * G * kD + idx] = o;
    }
  }
  if (splits_b > 1 && tid < G) {
    a.part_ml[(unit * G + tid) * 2 + 0] = sm.ml[tid][0];
    a.part_ml[(unit * G + tid) * 2 + 1] = sm.ml[tid][1];
  }
}

// Merge split partials: one CTA per (request, q head), thread per d element.
__global__ void __launch_bounds__(kD) decode_combine_kernel(const DecodeArgs a, int G) {
  const int b = blockIdx.y;
  const int hq = blockIdx.x;
  const int len = a.seq_lens[b];
  const int splits_b = (len + a.split_tok - 1) / a.split_tok;
  if (splits_b <= 1) return;  // written directly by the decode CTA
  const int h = hq / G;
  const int qh = hq % G;
  const int64_t unit0 = (static_cast<int64_t>(b) * a.hkv + h) * a.n_splits;
  float mx = -INFINITY;
  for (int s = 0; s < splits_b; ++s) mx = fmaxf(mx, a.part_ml[((unit0 + s) * G + qh) * 2]);
  float den = 0.f, num = 0.f;
  for (int s = 0; s < splits_b; ++s) {
    const float m = a.part_ml[((unit0 + s) * G + qh) * 2];
    const float l = a.part_ml[((unit0 + s) * G + qh) * 2 + 1];
    const float w = exp2f(m - mx);
    den += w * l;
    num += w * a.part_o[((unit0 + s) * G + qh) * kD + threadIdx.x];
  }
  a.out[(static_cast<int64_t>(b) * a.hkv * G + hq) * kD + threadIdx.x] =
      __float2bfloat16(den > 0.f ? num / den : 0.f);
}

template <int G>
cudaError_t launch_decode(const DecodeArgs& args, dim3 grid, cudaStream_t stream) {
  const size_t smem = sizeof(DecodeSmem<G>);
  static std::atomic<uint64_t> attr_devices{0};
  set_smem_limit_once(decode_splitkv_kernel<G>, smem, attr_devices);
  decode_splitkv_kernel<G><<<grid, kThreads, smem, stream>>>(args);
  return cudaGetLastError();
}

}  // namespace vt

using namespace vt;

static thread_local int32_t g_last_launches = 0;

extern "C" int32_t vt_attn_last_launches(void) { return g_last_launches; }

// Persistent tcgen05 kernel: pick the split count that minimises the makespan
// in 128-token tiles, ceil(units / SMs) * (tiles per unit + 1 unit overhead),
// then spread max_seq_len evenly over that many splits (multiple of 128).
static int tc_split(int32_t batch, int32_t hkv, int32_t max_seq_len, int n_sms) {
  int best = 1;
  long best_cost = -1;
  for (int ns = 1; ns <= 16; ++ns) {
    const long units = static_cast<long>(batch) * hkv * ns;
    const long per_sm = (units + n_sms - 1) / n_sms;
    const long tiles = (((max_seq_len + ns - 1) / ns) + 127) / 128;
    const long cost = per_sm * (tiles + 1);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = ns;
    }
  }
  return (((max_seq_len + best - 1) / best) + 127) / 128 * 128;
}

static int default_split(int32_t max_seq_len, bool tcgen05) {
  // tcgen05 (persistent): long units amortise the per-unit prologue; >= 2
  // splits per (request, kv head) keep ~7 units per SM at batch 64.
  // CUDA-core (one CTA per unit): ~4 units per (request, kv head) at 4k.
  if (tcgen05) return max_seq_len >= 8192 ? 4096 : max_seq_len >= 4096 ? 2048 : 512;
  return max_seq_len >= 4096 ? 1024 : 512;
}

static size_t counters_bytes(int32_t batch, int32_t hkv) {
  return (static_cast<size_t>(batch) * hkv * sizeof(int32_t) + 255) & ~static_cast<size_t>(255);
}

extern "C" size_t vt_decode_workspace_bytes(const vt_kv_geometry* g, int32_t batch,
                                            int32_t max_seq_len, int32_t split_tokens) {
  // sized for the smallest split either path may pick (tc_split >= 128 tokens per
  // split only when it needs <= 16 splits; CUDA-core default >= 512)
  if (max_seq_len < 1) max_seq_len = 1;  // all-empty batches still get a valid size
  const int split = split_tokens > 0 ? split_tokens : std::min(default_split(max_seq_len, false),
                                                               (max_seq_len + 15) / 16);
  const int64_t n_splits = (max_seq_len + split - 1) / split;
  const int64_t units = static_cast<int64_t>(batch) * g->kv_heads * n_splits;
  const int64_t G = g->q_heads / g->kv_heads;
  // [arrival counters, one per (request, kv head), 256-B padded][partial o][m, l]
  return counters_bytes(batch, g->kv_heads) + static_cast<size_t>(units * G * (kD + 2) * sizeof(float));
}

int vt_launch_decode_tc(const vt_kv_geometry* g, int32_t layer, const void* q,
                        const void* kv_maps, const int32_t* seq_lens, int32_t batch,
                        int32_t n_splits, int32_t split, float scale, void* out, float* part_o,
                        float* part_ml, int32_t* arrivals, int32_t n_sms, bool pdl,
                        cudaStream_t stream);

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

static int decode_impl(const vt_kv_geometry* g, int32_t layer, const void* q,
                       const uint64_t* kv_va, const void* kv_maps, const int32_t* block_table,
                       int32_t max_blocks, uint64_t pool_base, const int32_t* seq_lens,
                       int32_t batch, int32_t max_seq_len, float scale, void* out,
                       void* workspace, size_t workspace_bytes, int32_t split_tokens,
                       bool chained, void* stream) {
  g_last_launches = 0;
  if (g->head_dim != kD || g->q_heads % g->kv_heads) return cudaErrorInvalidValue;
  const int G = g->q_heads / g->kv_heads;
  const bool tc = kv_maps != nullptr;  // any batch (no silent switch of kernel family)
  const int split = split_tokens > 0 ? split_tokens
                    : tc             ? tc_split(batch, g->kv_heads, max_seq_len, num_sms())
                                     : default_split(max_seq_len, false);
  if (split % kStageTok) return cudaErrorInvalidValue;
  if (batch <= 0) return 0;
  if (max_seq_len <= 0)  // every request is empty: softmax over nothing is defined as zeros
    return cudaMemsetAsync(out, 0, static_cast<size_t>(batch) * g->q_heads * kD * 2,
                           static_cast<cudaStream_t>(stream));
  const int n_splits = (max_seq_len + split - 1) / split;
  if (workspace_bytes < vt_decode_workspace_bytes(g, batch, max_seq_len, split))
    return cudaErrorInvalidValue;
  DecodeArgs a{};
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.kv_va = kv_va;
  a.seq_lens = seq_lens;
  a.out = static_cast<__nv_bfloat16*>(out);
  const int64_t units = static_cast<int64_t>(batch) * g->kv_heads * n_splits;
  int32_t* arrivals = static_cast<int32_t*>(workspace);
  a.part_o = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) +
                                      counters_bytes(batch, g->kv_heads));
  a.part_ml = a.part_o + units * G * kD;
  a.batch = batch;
  a.hkv = g->kv_heads;
  a.n_splits = n_splits;
  a.split_tok = split;
  a.tpc = g->tokens_per_chunk;
  a.chunk_bytes = g->chunk_bytes;
  a.head_bytes = static_cast<int64_t>(g->tokens_per_chunk) * kD * 2;
  a.k_off = static_cast<int64_t>(layer * 2 + 0) * g->kv_heads * a.head_bytes;
  a.v_off = static_cast<int64_t>(layer * 2 + 1) * g->kv_heads * a.head_bytes;
  a.scale_log2 = scale * 1.4426950408889634f;
  a.block_table = block_table;
  a.max_blocks = max_blocks;
  a.pool_base = pool_base;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  dim3 grid(n_splits, g->kv_heads, batch);
  cudaError_t e;
  if (tc) {  // tcgen05 path (TMA maps over the request VAs)
    int rc = vt_launch_decode_tc(g, layer, q, kv_maps, seq_lens, batch, n_splits, split, scale,
                                 out, a.part_o, a.part_ml, arrivals, num_sms(), chained, st);
    g_last_launches = 1;
    return rc;
  } else switch (G) {
    case 1: e = launch_decode<1>(a, grid, st); break;
    case 2: e = launch_decode<2>(a, grid, st); break;
    case 4: e = launch_decode<4>(a, grid, st); break;
    case 8: e = launch_decode<8>(a, grid, st); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  g_last_launches = 1;
  if (n_splits > 1) {
    decode_combine_kernel<<<dim3(g->q_heads, batch), kD, 0, st>>>(a, G);
    e = cudaGetLastError();
    g_last_launches = 2;
  }
  return e;
}

extern "C" int vt_decode_attention(const vt_kv_geometry* g, int32_t layer, const void* q,
                                   const uint64_t* kv_va, const void* kv_maps,
                                   const int32_t* seq_lens, int32_t batch, int32_t max_seq_len,
                                   float scale, void* out, void* workspace, size_t workspace_bytes,
                                   int32_t split_tokens, void* stream) {
  return decode_impl(g, layer, q, kv_va, kv_maps, nullptr, 0, 0, seq_lens, batch, max_seq_len,
                     scale, out, workspace, workspace_bytes, split_tokens, false, stream);
}

extern "C" int vt_decode_attention_chained(const vt_kv_geometry* g, int32_t layer, const void* q,
                                           const uint64_t* kv_va, const void* kv_maps,
                                           const int32_t* seq_lens, int32_t batch,
                                           int32_t max_seq_len, float scale, void* out,
                                           void* workspace, size_t workspace_bytes,
                                           int32_t split_tokens, void* stream) {
  return decode_impl(g, layer, q, kv_va, kv_maps, nullptr, 0, 0, seq_lens, batch, max_seq_len,
                     scale, out, workspace, workspace_bytes, split_tokens, true, stream);
}

extern "C" int vt_decode_attention_paged(const vt_kv_geometry* g, int32_t layer, const void* q,
                                         const void* pool_base, const int32_t* block_table,
                                         int32_t max_blocks, const int32_t* seq_lens,
                                         int32_t batch, int32_t max_seq_len, float scale,
                                         void* out, void* workspace, size_t workspace_bytes,
                                         int32_t split_tokens, void* stream) {
  if (block_table == nullptr || pool_base == nullptr) return cudaErrorInvalidValue;
  return decode_impl(g, layer, q, nullptr, nullptr, block_table, max_blocks,
                     reinterpret_cast<uint64_t>(pool_base), seq_lens, batch, max_seq_len, scale,
                     out, workspace, workspace_bytes, split_tokens, false, stream);
}
