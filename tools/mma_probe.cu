// tcgen05.mma issue/throughput probe (sm_100a): cycles per MMA instruction for
// the shapes the prefill kernel uses, alone and with concurrent TMEM loads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_probe tools/mma_probe.cu
// Operand contents are irrelevant (throughput only).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2407_15309_b200/csrc/vt_tc_common.cuh"

using namespace vt;

constexpr int kIters = 528;  // multiple of 12, 16 and 3

// mode: 0 SS 128x64, 1 SS 128x128, 2 TS 128x128 (A in TMEM), 3 SS 128x256,
//       4 SS 128x64 + TS 128x128 alternating (prefill mix: 2 S + 1 PV)
template <int kMode, bool kLoad>
__global__ void __launch_bounds__(128, 1) probe(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ int stop;
  const int warp = threadIdx.x >> 5;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    stop = 0;
  }
  if (warp == 0) tc::alloc(&tbase, 512);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tbase;
  const uint32_t lo_a = tc::sdesc_lo(smem_u32(base), 16);
  const uint32_t lo_b = tc::sdesc_lo(smem_u32(base + 65536), 16);
  constexpr uint32_t hi = tc::sdesc_hi(1024);
  if (warp == 0) {
    long long t0 = clock64();
    if (tc::elect_one()) {
      for (int it = 0; it < kIters; ++it) {
        if (kMode == 0) tc::mma_ss(tmem, lo_a, hi, lo_b, hi, tc::idesc_bf16(128, 64, false, false), 1);
        if (kMode == 1) tc::mma_ss(tmem, lo_a, hi, lo_b, hi, tc::idesc_bf16(128, 128, false, false), 1);
        if (kMode == 2) tc::mma_ts(tmem + 256, tmem, lo_b, hi, tc::idesc_bf16(128, 128, false, true), 1);
        if (kMode == 3) tc::mma_ss(tmem, lo_a, hi, lo_b, hi, tc::idesc_bf16(128, 256, false, false), 1);
        if (kMode == 4) {
          if (it % 3 != 2)
            tc::mma_ss(tmem + 64 * (it % 3), lo_a, hi, lo_b, hi, tc::idesc_bf16(128, 64, false, false), 1);
          else
            tc::mma_ts(tmem + 256, tmem + 128, lo_b, hi, tc::idesc_bf16(128, 128, false, true), 1);
        }
        if (kMode == 7)  // SS 128x128 with MN-major B (the V operand)
          tc::mma_ss(tmem + 256, lo_a, hi, tc::sdesc_lo(smem_u32(base + 131072), 128 * 128) + (it & 3) * 128, hi,
                     tc::idesc_bf16(128, 128, false, true), 1);
        if (kMode == 8) {  // 8 SS64 (K-major) then 4 SS128 K-major B
          const int k = it % 12;
          if (k < 8)
            tc::mma_ss(tmem + 64 * ((it / 12) & 1), lo_a + 2 * (k & 3), hi, lo_b + 2 * (k & 3), hi,
                       tc::idesc_bf16(128, 64, false, false), 1);
          else
            tc::mma_ss(tmem + 256, lo_a + 2 * (k & 3), hi, lo_b + 2 * (k & 3), hi,
                       tc::idesc_bf16(128, 128, false, false), 1);
        }
        if (kMode == 9) {  // 8 SS64 then 4 TS128 whose A columns the SS do not write
          const int k = it % 12;
          if (k < 8)
            tc::mma_ss(tmem + 64 * ((it / 12) & 1), lo_a + 2 * (k & 3), hi, lo_b + 2 * (k & 3), hi,
                       tc::idesc_bf16(128, 64, false, false), 1);
          else
            tc::mma_ts(tmem + 256, tmem + 384 + 8 * (k - 8), lo_b, hi, tc::idesc_bf16(128, 128, false, false), 1);
        }
        if (kMode == 10) {  // 8 SS64 then 4 TS128 (K-major B), TS reads the SS output columns
          const int k = it % 12;
          if (k < 8)
            tc::mma_ss(tmem + 64 * ((it / 12) & 1), lo_a + 2 * (k & 3), hi, lo_b + 2 * (k & 3), hi,
                       tc::idesc_bf16(128, 64, false, false), 1);
          else
            tc::mma_ts(tmem + 256, tmem + 64 * ((it / 12) & 1) + 8 * (k - 8), lo_b, hi,
                       tc::idesc_bf16(128, 128, false, false), 1);
        }
        if (kMode == 11) {  // 8 SS128 then 8 TS128 (A = other slot's S region)
          const int k = it % 16, g = it / 16;
          if (k < 8)
            tc::mma_ss(tmem + 128 * (g & 1), lo_a + 2 * (k & 3), hi, lo_b + 2 * (k & 3), hi,
                       tc::idesc_bf16(128, 128, false, false), 1);
          else
            tc::mma_ts(tmem + 256 + 128 * (g & 1), tmem + 128 * ((g + 1) & 1) + 8 * (k - 8), lo_b, hi,
                       tc::idesc_bf16(128, 128, false, true), 1);
        }
        if (kMode == 12) {  // 8 SS64 then 8 TS64 (all N = 64)
          const int k = it % 16, g = it / 16;
          if (k < 8)
            tc::mma_ss(tmem + 64 * (g & 1), lo_a + 2 * (k & 3), hi, lo_b + 2 * (k & 3), hi,
                       tc::idesc_bf16(128, 64, false, false), 1);
          else
            tc::mma_ts(tmem + 256 + 64 * (k & 1), tmem + 128 + 8 * ((k - 8) >> 1), lo_b, hi,
                       tc::idesc_bf16(128, 64, false, true), 1);
        }
        if (kMode == 13)
          tc::mma_ts(tmem + 256, tmem + 8 * (it & 7), lo_b, hi, tc::idesc_bf16(128, 64, false, true), 1);
        if (kMode == 5 || kMode == 6) {
          // the prefill group: 8 SS 128x64 over K=128 (Q / K tiles with the
          // kernel's kk offsets), then 4 TS 128x128 with MN-major V.
          const int g = it / 12, k = it % 12;
          const uint32_t lv = tc::sdesc_lo(smem_u32(base + 131072), 128 * 128);
          if (k < 8) {
            const uint32_t off = (k >> 2) * 1024 + 2 * (k & 3);
            tc::mma_ss(tmem + 64 * (g & 1), lo_a + off, hi, lo_b + (g & 3) * 512 + off, hi,
                       tc::idesc_bf16(128, 64, false, false), k > 0);
          } else if (kMode == 5) {
            tc::mma_ts(tmem + 256, tmem + 64 * (g & 1) + 8 * (k - 8), lv + (g & 1) * 512 + (k - 8) * 128, hi,
                       tc::idesc_bf16(128, 128, false, true), 1);
          } else {
            tc::mma_ss(tmem + 256, lo_a + 2 * (k - 8), hi, lv + (g & 1) * 512 + (k - 8) * 128, hi,
                       tc::idesc_bf16(128, 128, false, true), 1);
          }
        }
      }
      tc::commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) {
      out[blockIdx.x] = t1 - t0;
      stop = 1;
    }
  } else if (kLoad) {
    // Concurrent TMEM reads of the S region (like the softmax warps).
    const uint32_t addr = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + 384;
    uint32_t r[32];
    float acc = 0.f;
    while (!*(volatile int*)&stop) {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
          "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
            "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
            "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
            "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(addr));
      tc::wait_ld();
      acc += __uint_as_float(r[0]) + __uint_as_float(r[31]);
    }
    if (acc == 12345.f) out[1000] = 1;
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::dealloc(tmem, 512);
}

template <int M, bool L>
void run(const char* name, long long* d, int flops_per) {
  cudaFuncSetAttribute(probe<M, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  probe<M, L><<<148, 128, 200 * 1024>>>(d);
  probe<M, L><<<148, 128, 200 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  s /= 148;
  printf("%-34s %s cycles/MMA %.1f  flop/clk/SM %.0f\n", name, e ? cudaGetErrorString(e) : "",
         s / kIters, flops_per / (s / kIters));
}

int main() {
  long long* d;
  cudaMalloc(&d, 2048 * sizeof(long long));
  run<0, false>("SS 128x64x16", d, 2 * 128 * 64 * 16);
  run<1, false>("SS 128x128x16", d, 2 * 128 * 128 * 16);
  run<2, false>("TS 128x128x16 (A in TMEM)", d, 2 * 128 * 128 * 16);
  run<3, false>("SS 128x256x16", d, 2 * 128 * 256 * 16);
  run<4, false>("mix 2xSS64 + 1xTS128", d, (2 * 2 * 128 * 64 * 16 + 2 * 128 * 128 * 16) / 3);
  run<5, false>("prefill group (8 SS64 + 4 TS128)", d, (8 * 2 * 128 * 64 * 16 + 4 * 2 * 128 * 128 * 16) / 12);
  run<6, false>("prefill group, PV as SS (P in smem)", d, (8 * 2 * 128 * 64 * 16 + 4 * 2 * 128 * 128 * 16) / 12);
  run<7, false>("SS 128x128 MN-major B", d, 2 * 128 * 128 * 16);
  run<8, false>("8 SS64 + 4 SS128 (K-major)", d, (8 * 2 * 128 * 64 * 16 + 4 * 2 * 128 * 128 * 16) / 12);
  run<9, false>("8 SS64 + 4 TS128, disjoint A cols", d, (8 * 2 * 128 * 64 * 16 + 4 * 2 * 128 * 128 * 16) / 12);
  run<10, false>("8 SS64 + 4 TS128, A = SS output", d, (8 * 2 * 128 * 64 * 16 + 4 * 2 * 128 * 128 * 16) / 12);
  run<11, false>("8 SS128 + 8 TS128", d, 2 * 128 * 128 * 16);
  run<12, false>("8 SS64 + 8 TS64", d, 2 * 128 * 64 * 16);
  run<13, false>("TS 128x64", d, 2 * 128 * 64 * 16);
  run<4, false>("mix 2xSS64 + 1xTS128 (again)", d, (2 * 2 * 128 * 64 * 16 + 2 * 128 * 128 * 16) / 3);
  run<5, true>("prefill group + TMEM loads", d, (8 * 2 * 128 * 64 * 16 + 4 * 2 * 128 * 128 * 16) / 12);
  run<0, true>("SS 128x64x16 + TMEM loads", d, 2 * 128 * 64 * 16);
  run<1, true>("SS 128x128x16 + TMEM loads", d, 2 * 128 * 128 * 16);
  run<2, true>("TS 128x128x16 + TMEM loads", d, 2 * 128 * 128 * 16);
  run<4, true>("mix + TMEM loads", d, (2 * 2 * 128 * 64 * 16 + 2 * 128 * 128 * 16) / 3);
  return 0;
}
