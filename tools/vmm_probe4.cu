// vmm_probe4 — what does the per-chunk cost of cuMemMap + cuMemSetAccess (and
// cuMemCreate) scale with? (under the HBM-saturating decode with
// ~16k chunks mapped, SetAccess costs 2-3 ms per call and cuMemCreate ~4.7 ms,
// vs 155 us / 73 us in a fresh process.)
//
// For an increasing number M of live mapped chunks (each its own 2 MiB
// allocation, or slab allocations of S chunks mapped by offset), measure the
// median latency of 64 (create), (map + SetAccess) of fresh chunks, with the
// GPU idle and with an HBM-streaming kernel flood running. One JSON line per
// case.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//        -o tools/vmm_probe4 tools/vmm_probe4.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#define CK(x)                                                               \
  do {                                                                      \
    CUresult r_ = (x);                                                      \
    if (r_ != CUDA_SUCCESS) {                                               \
      const char* s_ = nullptr;                                             \
      cuGetErrorString(r_, &s_);                                            \
      std::fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x, s_); \
      std::exit(1);                                                         \
    }                                                                       \
  } while (0)
#define RK(x)                                                               \
  do {                                                                      \
    cudaError_t e_ = (x);                                                   \
    if (e_ != cudaSuccess) {                                                \
      std::fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x,      \
                   cudaGetErrorString(e_));                                 \
      std::exit(1);                                                         \
    }                                                                       \
  } while (0)

static double now_us() {
  return std::chrono::duration<double, std::micro>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
static double med(std::vector<double> v) {
  if (v.empty()) return 0;
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

__global__ void stream_kernel(const float4* __restrict__ src, size_t n, float* sink) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    float4 v = __ldcs(src + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 1234.5f) sink[0] = acc;
}

int main(int argc, char** argv) {
  const size_t CH = 2ull << 20;
  const int slab = argc > 1 ? atoi(argv[1]) : 1;  // chunks per physical allocation
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUcontext ctx;
  CK(cuDevicePrimaryCtxRetain(&ctx, dev));
  CK(cuCtxSetCurrent(ctx));
  RK(cudaSetDevice(0));
  int sms = 0;
  RK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t buf_bytes = 4ull << 30;
  float4* buf;
  float* sink;
  RK(cudaMalloc(&buf, buf_bytes));
  RK(cudaMemset(buf, 0, buf_bytes));
  RK(cudaMalloc(&sink, 64));
  cudaStream_t s;
  RK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));

  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  CUmemAccessDesc ad{};
  ad.location = ap.location;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;

  const int kMaxLive = 24576;  // 48 GiB of live mappings at most
  CUdeviceptr live_va;
  CK(cuMemAddressReserve(&live_va, CH * kMaxLive, CH, 0, 0));
  std::vector<CUmemGenericAllocationHandle> live_h;
  int live = 0;
  auto grow_to = [&](int m) {  // map m live chunks (slab allocations of `slab` chunks)
    while (live < m) {
      CUmemGenericAllocationHandle h;
      CK(cuMemCreate(&h, CH * slab, &ap, 0));
      live_h.push_back(h);
      for (int k = 0; k < slab && live < m; ++k, ++live) {
        CK(cuMemMap(live_va + CH * live, CH, CH * k, h, 0));
        CK(cuMemSetAccess(live_va + CH * live, CH, &ad, 1));
      }
    }
  };

  const int kProbe = 64;
  CUdeviceptr probe_va;
  CK(cuMemAddressReserve(&probe_va, CH * kProbe, CH, 0, 0));
  std::atomic<bool> stop{false};
  auto measure = [&](int m, bool load) {
    std::thread launcher;
    if (load) {
      stop = false;
      launcher = std::thread([&] {
        CK(cuCtxSetCurrent(ctx));
        cudaEvent_t e;
        RK(cudaEventCreate(&e));
        while (!stop.load()) {  // ~32 x 0.6 ms kernels in flight, like a decode step
          for (int i = 0; i < 32; ++i)
            stream_kernel<<<sms * 4, 512, 0, s>>>(buf, buf_bytes / 16, sink);
          RK(cudaEventRecord(e, s));
          RK(cudaEventSynchronize(e));
        }
      });
      std::this_thread::sleep_for(std::chrono::milliseconds(200));
    }
    std::vector<double> create_us, map_us, access_us, unmap_us;
    std::vector<CUmemGenericAllocationHandle> hs(kProbe);
    for (int i = 0; i < kProbe; ++i) {
      double t0 = now_us();
      CK(cuMemCreate(&hs[i], CH, &ap, 0));
      create_us.push_back(now_us() - t0);
    }
    for (int i = 0; i < kProbe; ++i) {
      double t0 = now_us();
      CK(cuMemMap(probe_va + CH * i, CH, 0, hs[i], 0));
      double t1 = now_us();
      CK(cuMemSetAccess(probe_va + CH * i, CH, &ad, 1));
      map_us.push_back(t1 - t0);
      access_us.push_back(now_us() - t1);
    }
    // one SetAccess over a run of 16 freshly mapped chunks
    for (int i = 0; i < kProbe; ++i) {
      double t0 = now_us();
      CK(cuMemUnmap(probe_va + CH * i, CH));
      unmap_us.push_back(now_us() - t0);
    }
    double run16 = 0;
    {
      for (int i = 0; i < 16; ++i) CK(cuMemMap(probe_va + CH * i, CH, 0, hs[i], 0));
      double t0 = now_us();
      CK(cuMemSetAccess(probe_va, CH * 16, &ad, 1));
      run16 = now_us() - t0;
      for (int i = 0; i < 16; ++i) CK(cuMemUnmap(probe_va + CH * i, CH));
    }
    for (auto h : hs) CK(cuMemRelease(h));
    // slab creates: one allocation of `slab` chunks, cost per 2 MiB chunk
    double slab_us = 0;
    if (slab > 1) {
      std::vector<double> v;
      for (int i = 0; i < 8; ++i) {
        CUmemGenericAllocationHandle h;
        double t0 = now_us();
        CK(cuMemCreate(&h, CH * slab, &ap, 0));
        v.push_back((now_us() - t0) / slab);
        CK(cuMemRelease(h));
      }
      slab_us = med(v);
    }
    if (load) {
      stop = true;
      launcher.join();
    }
    std::printf(
        "{\"slab\":%d,\"live_chunks\":%d,\"live_allocations\":%zu,\"load\":\"%s\",\"create_us\":%.1f,"
        "\"map_us\":%.1f,\"setaccess_us\":%.1f,\"unmap_us\":%.1f,\"setaccess_run16_us\":%.1f,"
        "\"slab_create_us_per_chunk\":%.1f}\n",
        slab, m, live_h.size(), load ? "hbm_stream" : "idle", med(create_us), med(map_us),
        med(access_us), med(unmap_us), run16, slab_us);
    std::fflush(stdout);
  };
  for (int m : {0, 512, 2048, 8192, 16384, 24576}) {
    grow_to(m);
    measure(m, false);
    measure(m, true);
  }
  return 0;
}
