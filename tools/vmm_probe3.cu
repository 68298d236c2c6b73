// vmm_probe3 — which process state makes cuMemSetAccess / cuMemCreate slow?
// (vmm_probe2: 155 us per 2 MiB SetAccess in a pure-driver process; vmm_probe:
// 550-750 us once the runtime has allocated memory and launched kernels.)
// Measures 64 x (create, map, SetAccess, unmap) after each process-state step.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//        -o tools/vmm_probe3 tools/vmm_probe3.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <unistd.h>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    CUresult r_ = (x);                                                         \
    if (r_ != CUDA_SUCCESS) {                                                  \
      const char* s_ = nullptr;                                                \
      cuGetErrorString(r_, &s_);                                               \
      std::fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x, s_);    \
      std::exit(1);                                                            \
    }                                                                          \
  } while (0)

static double wall_us() {
  return std::chrono::duration<double, std::micro>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
static double med(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v.empty() ? 0 : v[v.size() / 2];
}

__global__ void tiny(float* p) {
  if (p && threadIdx.x == 1234567) p[0] = 1.f;
}
__global__ void touch(const float4* __restrict__ s, size_t n, float* sink) {
  float a = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    a += s[i].x;
  if (a == 1234.5f) sink[0] = a;
}

static const size_t CH = 2ull << 20;
static CUmemAllocationProp ap{};
static CUmemAccessDesc ad{};

static void measure(const char* stage, int n = 64, bool fresh_va = false) {
  static CUdeviceptr va = 0;
  if (!va || fresh_va) CK(cuMemAddressReserve(&va, 256 * CH, CH, 0, 0));
  std::vector<CUmemGenericAllocationHandle> h(n);
  std::vector<double> cw, aw, uw, rw, a2;
  for (auto& x : h) {
    double t = wall_us();
    CK(cuMemCreate(&x, CH, &ap, 0));
    cw.push_back(wall_us() - t);
  }
  for (int k = 0; k < n; ++k) {
    CK(cuMemMap(va + k * CH, CH, 0, h[k], 0));
    double t = wall_us();
    CK(cuMemSetAccess(va + k * CH, CH, &ad, 1));
    aw.push_back(wall_us() - t);
  }
  for (int k = 0; k < n; ++k) {
    double t = wall_us();
    CK(cuMemUnmap(va + k * CH, CH));
    uw.push_back(wall_us() - t);
  }
  // second pass with the same (already once-mapped) handles
  for (int k = 0; k < n; ++k) {
    CK(cuMemMap(va + k * CH, CH, 0, h[k], 0));
    double t = wall_us();
    CK(cuMemSetAccess(va + k * CH, CH, &ad, 1));
    a2.push_back(wall_us() - t);
  }
  for (int k = 0; k < n; ++k) CK(cuMemUnmap(va + k * CH, CH));
  for (auto& x : h) {
    double t = wall_us();
    CK(cuMemRelease(x));
    rw.push_back(wall_us() - t);
  }
  std::printf(
      "{\"stage\":\"%s\",\"create_us\":%.1f,\"access_us\":%.1f,\"access_again_us\":%.1f,"
      "\"unmap_us\":%.1f,\"release_us\":%.1f}\n",
      stage, med(cw), med(aw), med(a2), med(uw), med(rw));
  std::fflush(stdout);
}

static void setup_driver() {
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUcontext ctx;
  CK(cuDevicePrimaryCtxRetain(&ctx, dev));
  CK(cuCtxSetCurrent(ctx));
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ad.location = ap.location;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
}

// argv[1] = mode: "stages" (default), "timeline", "spin", "blocking", "yield"
int main(int argc, char** argv) {
  const char* mode = argc > 1 ? argv[1] : "stages";
  if (strcmp(mode, "stages") != 0) {
    unsigned flags = 0;
    if (!strcmp(mode, "spin")) flags = cudaDeviceScheduleSpin;
    if (!strcmp(mode, "blocking")) flags = cudaDeviceScheduleBlockingSync;
    if (!strcmp(mode, "yield")) flags = cudaDeviceScheduleYield;
    if (flags) cudaSetDeviceFlags(flags);
    cudaSetDevice(0);
    cudaFree(0);
    setup_driver();
    double t0 = wall_us();
    for (int i = 0; i < 12; ++i) {
      char nm[64];
      snprintf(nm, sizeof nm, "%s_t%.1fs", mode, (wall_us() - t0) / 1e6);
      measure(nm, 32);
      usleep(400000);
    }
    return 0;
  }
  setup_driver();

  measure("pure_driver_first");
  measure("pure_driver_second");
  cudaSetDevice(0);
  cudaFree(0);
  measure("runtime_initialised");
  tiny<<<1, 32>>>(nullptr);
  cudaDeviceSynchronize();
  measure("after_one_tiny_kernel");
  float* small = nullptr;
  cudaMalloc(&small, 64 << 20);
  measure("after_cudaMalloc_64MiB");
  float4* big = nullptr;
  cudaMalloc(&big, 8ull << 30);
  measure("after_cudaMalloc_8GiB");
  cudaMemset(big, 0, 8ull << 30);
  cudaDeviceSynchronize();
  measure("after_memset_8GiB");
  for (int i = 0; i < 50; ++i) touch<<<148 * 4, 512>>>(big, (8ull << 30) / 16, small);
  cudaDeviceSynchronize();
  measure("after_50_streaming_kernels");
  measure("after_50_streaming_kernels_fresh_va", 64, true);
  cudaFree(big);
  measure("after_cudaFree_8GiB");
  // many live VMM chunks (like the bench: thousands of mapped 2 MiB chunks)
  {
    CUdeviceptr bva;
    const int NB = 4096;
    CK(cuMemAddressReserve(&bva, NB * CH, CH, 0, 0));
    std::vector<CUmemGenericAllocationHandle> hb(NB);
    double t = wall_us();
    for (int k = 0; k < NB; ++k) {
      CK(cuMemCreate(&hb[k], CH, &ap, 0));
      CK(cuMemMap(bva + k * CH, CH, 0, hb[k], 0));
    }
    double t2 = wall_us();
    CK(cuMemSetAccess(bva, NB * CH, &ad, 1));
    std::printf("{\"stage\":\"bulk_4096\",\"create_map_us_per\":%.1f,\"one_access_8GiB_us\":%.1f}\n",
                (t2 - t) / NB, wall_us() - t2);
    measure("with_4096_live_chunks");
    for (int k = 0; k < NB; ++k) CK(cuMemUnmap(bva + k * CH, CH));
    for (auto& x : hb) CK(cuMemRelease(x));
    measure("after_freeing_4096");
  }
  return 0;
}
