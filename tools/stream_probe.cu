// How fast can CTAs stream a weight with 16 KiB cp.async.bulk copies through
// an mbarrier ring (the fused QKV kernel's pattern, no MMA)? DESIGN §3.5.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/stream_probe tools/stream_probe.cu
//   ./tools/stream_probe CTAS KIB_PER_CTA CHUNK_KIB STAGES
//
// Streams CTAS x KIB_PER_CTA of a 4-way rotated 4 x (CTAS x KIB) buffer set
// (never L2-resident), 200 launches, prints GB/s per launch (events).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../paper_2407_15309_b200/csrc/vt_common.cuh"

using namespace vt;

__global__ void __launch_bounds__(32, 1) stream(const uint8_t* src, int per_cta, int chunk, int stages,
                                                 unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ uint64_t full[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  const uint64_t base = reinterpret_cast<uint64_t>(src) + static_cast<uint64_t>(blockIdx.x) * per_cta;
  const int n = per_cta / chunk;
  const uint64_t once = l2_evict_first_policy();
  unsigned long long acc = 0;
  for (int i = 0; i < n + stages; ++i) {
    if (i >= stages) {  // consume chunk i - stages
      const int j = i - stages;
      mbar_wait(&full[j % stages], (j / stages) & 1);
      acc += ring[(j % stages) * chunk];
    }
    if (i < n) {
      const int st = i % stages;
      mbar_arrive_expect_tx(&full[st], chunk);
      bulk_g2s(ring + st * chunk, base + static_cast<uint64_t>(i) * chunk, chunk, &full[st], once);
    }
  }
  if (acc == 0x7fffffffffffffffull) *sink = acc;
}

int main(int argc, char** argv) {
  const int ctas = argc > 1 ? atoi(argv[1]) : 144;
  const int kib = argc > 2 ? atoi(argv[2]) : 352;
  const int chunk = (argc > 3 ? atoi(argv[3]) : 16) * 1024;
  const int stages = argc > 4 ? atoi(argv[4]) : 8;
  const size_t per = static_cast<size_t>(ctas) * kib * 1024;
  uint8_t* buf = nullptr;
  unsigned long long* sink = nullptr;
  cudaMalloc(&buf, 4 * per);
  cudaMalloc(&sink, 8);
  cudaMemset(buf, 1, 4 * per);
  const int smem = stages * chunk;
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int i = 0; i < 8; ++i) stream<<<ctas, 32, smem>>>(buf + (i & 3) * per, kib * 1024, chunk, stages, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 200;
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) stream<<<ctas, 32, smem>>>(buf + (i & 3) * per, kib * 1024, chunk, stages, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  const double us = 1000.0 * ms / reps;
  printf("{\"ctas\": %d, \"kib_per_cta\": %d, \"chunk_kib\": %d, \"stages\": %d, \"MB\": %.1f, \"us\": %.2f, \"GBps\": %.0f, \"err\": \"%s\"}\n",
         ctas, kib, chunk / 1024, stages, per / 1e6, us, per / (us * 1e-6) / 1e9, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
