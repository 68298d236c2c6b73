// vmm_probe7 — is cuMemSetAccess slow because the driver is still busy with
// earlier bulk allocation / release work (e.g. scrubbing physical memory)?
// Time series of the latency of one map + SetAccess + unmap of a probe chunk,
// sampled every ~2 ms, across phases: process start (the previous process on
// this GPU freed its memory at exit), after creating + mapping 32 GiB of 2 MiB
// chunks (as the bench's setup), after releasing them, and the same under an
// HBM-streaming kernel flood. One JSON line per 100 ms window.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//        -o tools/vmm_probe7 tools/vmm_probe7.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
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
static double pct(std::vector<double> v, double p) {
  if (v.empty()) return 0;
  std::sort(v.begin(), v.end());
  return v[std::min(v.size() - 1, (size_t)(p * v.size()))];
}

__global__ void stream_kernel(const float4* __restrict__ src, size_t n, float* sink, int pdl) {
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  float acc = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    float4 v = __ldcs(src + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 1234.5f) sink[0] = acc;
}
__global__ void touch(unsigned* p, size_t words, unsigned* bad) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < words;
       i += (size_t)gridDim.x * blockDim.x)
    p[i] = (unsigned)i;
  __threadfence();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < words;
       i += (size_t)gridDim.x * blockDim.x)
    if (p[i] != (unsigned)i) atomicAdd(bad, 1u);
}


int main(int argc, char** argv) {
  const int n_bulk = argc > 1 ? atoi(argv[1]) : 16384;  // 2 MiB chunks (32 GiB)
  const size_t CH = 2ull << 20;
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUcontext prim;
  CK(cuDevicePrimaryCtxRetain(&prim, dev));
  CK(cuCtxSetCurrent(prim));
  RK(cudaSetDevice(0));
  int sms = 0;
  RK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  CUmemAccessDesc ad{};
  ad.location = ap.location;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUmemGenericAllocationHandle probe_h;
  CK(cuMemCreate(&probe_h, CH, &ap, 0));
  CUdeviceptr probe_va;
  CK(cuMemAddressReserve(&probe_va, CH, CH, 0, 0));
  const double t_start = now_us();
  auto sample = [&](const char* phase, double seconds) {
    double t_end = now_us() + seconds * 1e6;
    std::vector<double> win;
    double w0 = now_us();
    while (now_us() < t_end) {
      CK(cuMemMap(probe_va, CH, 0, probe_h, 0));
      double t0 = now_us();
      CK(cuMemSetAccess(probe_va, CH, &ad, 1));
      win.push_back(now_us() - t0);
      CK(cuMemUnmap(probe_va, CH));
      std::this_thread::sleep_for(std::chrono::microseconds(2000));
      if (now_us() - w0 > 1e5) {
        std::printf("{\"phase\":\"%s\",\"t_ms\":%.0f,\"n\":%zu,\"p50_us\":%.1f,\"max_us\":%.1f}\n", phase,
                    (w0 - t_start) / 1e3, win.size(), pct(win, 0.5), pct(win, 1.0));
        std::fflush(stdout);
        win.clear();
        w0 = now_us();
      }
    }
  };
  sample("process_start", 3.0);
  // bulk: create + map + SetAccess n_bulk chunks (one range, as the bench's live KV)
  CUdeviceptr bulk_va;
  CK(cuMemAddressReserve(&bulk_va, CH * n_bulk, CH, 0, 0));
  std::vector<CUmemGenericAllocationHandle> hs(n_bulk);
  double t0 = now_us();
  for (int i = 0; i < n_bulk; ++i) {
    CK(cuMemCreate(&hs[i], CH, &ap, 0));
    CK(cuMemMap(bulk_va + CH * i, CH, 0, hs[i], 0));
    CK(cuMemSetAccess(bulk_va + CH * i, CH, &ad, 1));
  }
  std::printf("{\"phase\":\"bulk_create_map\",\"chunks\":%d,\"ms\":%.0f}\n", n_bulk, (now_us() - t0) / 1e3);
  sample("after_bulk_create", 6.0);
  t0 = now_us();
  for (int i = 0; i < n_bulk; ++i) {
    CK(cuMemUnmap(bulk_va + CH * i, CH));
    CK(cuMemRelease(hs[i]));
  }
  std::printf("{\"phase\":\"bulk_release\",\"ms\":%.0f}\n", (now_us() - t0) / 1e3);
  sample("after_bulk_release", 6.0);
  // the same again with the GPU streaming HBM (kernels of ~160 us, plain launches)
  const size_t buf_bytes = 1ull << 30;
  float4* buf;
  float* sink;
  RK(cudaMalloc(&buf, buf_bytes));
  RK(cudaMemset(buf, 0, buf_bytes));
  RK(cudaMalloc(&sink, 64));
  cudaStream_t s;
  RK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  RK(cudaDeviceSynchronize());
  std::atomic<bool> stop{false};
  std::thread launcher([&] {
    CK(cuCtxSetCurrent(prim));
    cudaEvent_t ev[2];
    RK(cudaEventCreate(&ev[0]));
    RK(cudaEventCreate(&ev[1]));
    for (long step = 0; !stop.load(); ++step) {
      if (step >= 2) RK(cudaEventSynchronize(ev[step & 1]));
      for (int i = 0; i < 32; ++i)
        stream_kernel<<<sms * 2, 512, 0, s>>>((const float4*)buf, buf_bytes / 16, sink, 0);
      RK(cudaEventRecord(ev[step & 1], s));
    }
    RK(cudaStreamSynchronize(s));
  });
  sample("stream_only", 2.0);
  t0 = now_us();
  for (int i = 0; i < n_bulk; ++i) {
    CK(cuMemCreate(&hs[i], CH, &ap, 0));
    CK(cuMemMap(bulk_va + CH * i, CH, 0, hs[i], 0));
    CK(cuMemSetAccess(bulk_va + CH * i, CH, &ad, 1));
  }
  std::printf("{\"phase\":\"bulk_create_map_under_stream\",\"ms\":%.0f}\n", (now_us() - t0) / 1e3);
  sample("stream_after_bulk_create", 6.0);
  stop = true;
  launcher.join();
  return 0;
}
