// How fast can CTAs stream a weight with 16 KiB cp.async.bulk copies through
// an mbarrier ring (the fused QKV kernel's pattern, no MMA)? DESIGN §3.5.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/stream_probe tools/stream_probe.cu
//   ./tools/stream_probe CTAS KIB_PER_CTA CHUNK_KIB STAGES [PDL]
// PDL=1: launches carry programmatic stream serialization and each kernel
// triggers its dependents at entry and waits (griddepcontrol.wait) before its
// first copy, like a layer whose input is the previous layer's output; PDL=2:
// the same without the wait (no dependency: the overlap's upper bound);
// PDL=3: the first ring is issued at entry and the rest after the wait (the
// fused QKV kernel's order).
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
                                                 unsigned long long* sink, int pdl) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ uint64_t full[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) mbar_init(&full[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x != 0) return;
  if (pdl == 1) asm volatile("griddepcontrol.wait;" ::: "memory");
  // PDL=3 (the QKV kernel's order): the first ring is issued at entry, the
  // rest only after griddepcontrol.wait
  bool waited = pdl != 3;
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
    if (!waited && i == stages) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      waited = true;
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
  const int pdl = argc > 5 ? atoi(argv[5]) : 0;
  const size_t per = static_cast<size_t>(ctas) * kib * 1024;
  uint8_t* buf = nullptr;
  unsigned long long* sink = nullptr;
  cudaMalloc(&buf, 4 * per);
  cudaMalloc(&sink, 8);
  cudaMemset(buf, 1, 4 * per);
  const int smem = stages * chunk;
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  auto launch = [&](int i) {
    cudaLaunchKernelEx(&cfg, stream, static_cast<const uint8_t*>(buf + (i & 3) * per), kib * 1024, chunk, stages,
                       sink, pdl);
  };
  for (int i = 0; i < 8; ++i) launch(i);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 200;
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) launch(i);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  const double us = 1000.0 * ms / reps;
  printf("{\"pdl\": %d, \"ctas\": %d, \"kib_per_cta\": %d, \"chunk_kib\": %d, \"stages\": %d, \"MB\": %.1f, \"us\": %.2f, \"GBps\": %.0f, \"err\": \"%s\"}\n",
         pdl, ctas, kib, chunk / 1024, stages, per / 1e6, us, per / (us * 1e-6) / 1e9, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
