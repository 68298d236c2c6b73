// vmm_probe6 — what sets the cost of cuMemSetAccess under decode-like load?
// A launcher thread streams HBM with ~160 us kernels in "steps" of 32 (the
// bench's decode layer count), host bounded to 2 steps ahead; the kernels of
// a step are chained with programmatic dependent launch except every
// `plain_every`-th (0 = only the first of the step). Meanwhile the calling
// thread maps + SetAccesses fresh 2 MiB chunks one at a time. Swept: chaining,
// plain boundaries per step, and how many other physical allocations exist
// (mapped elsewhere) — the bench holds ~16-24k.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//        -o tools/vmm_probe6 tools/vmm_probe6.cu -lcuda
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


int main() {
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
  const size_t buf_bytes = 1ull << 30;  // ~160 us per streaming kernel
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
  const int N = 256;  // measured maps per configuration
  std::vector<CUmemGenericAllocationHandle> hs(N);
  for (auto& h : hs) CK(cuMemCreate(&h, CH, &ap, 0));
  CUdeviceptr va;
  CK(cuMemAddressReserve(&va, CH * N, CH, 0, 0));
  // background population: mapped + accessible elsewhere, as the bench's live KV
  const int kMaxBg = 24576;
  CUdeviceptr bg_va;
  CK(cuMemAddressReserve(&bg_va, CH * kMaxBg, CH, 0, 0));
  std::vector<CUmemGenericAllocationHandle> bg;
  auto grow_bg = [&](int target) {
    while ((int)bg.size() < target) {
      CUmemGenericAllocationHandle h;
      CK(cuMemCreate(&h, CH, &ap, 0));
      CK(cuMemMap(bg_va + CH * bg.size(), CH, 0, h, 0));
      CK(cuMemSetAccess(bg_va + CH * bg.size(), CH, &ad, 1));
      bg.push_back(h);
    }
  };
  struct Cfg { int bg, chain, plain_every; };
  std::vector<Cfg> cfgs = {
      {0, 0, 0}, {0, 1, 0}, {0, 1, 4},
      {8192, 0, 0}, {8192, 1, 0}, {8192, 1, 4},
      {20000, 0, 0}, {20000, 1, 0}, {20000, 1, 4}, {20000, 1, 1}};
  for (const Cfg& c : cfgs) {
    grow_bg(c.bg);
    RK(cudaDeviceSynchronize());
    for (int load : {0, 1}) {
      std::atomic<bool> stop{false};
      std::thread launcher;
      if (load) {
        launcher = std::thread([&] {
          CK(cuCtxSetCurrent(prim));
          cudaEvent_t ev[2];
          RK(cudaEventCreate(&ev[0]));
          RK(cudaEventCreate(&ev[1]));
          cudaLaunchConfig_t cfg{};
          cfg.gridDim = dim3(sms * 2);
          cfg.blockDim = dim3(512);
          cfg.stream = s;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = at;
          for (long step = 0; !stop.load(); ++step) {
            if (step >= 2) RK(cudaEventSynchronize(ev[step & 1]));  // 2 steps ahead at most
            for (int i = 0; i < 32; ++i) {
              const bool chained = c.chain && i > 0 && !(c.plain_every && i % c.plain_every == 0);
              cfg.numAttrs = chained ? 1 : 0;
              RK(cudaLaunchKernelEx(&cfg, stream_kernel, (const float4*)buf, buf_bytes / 16, sink,
                                    chained ? 1 : 0));
            }
            RK(cudaEventRecord(ev[step & 1], s));
          }
          RK(cudaStreamSynchronize(s));
        });
        std::this_thread::sleep_for(std::chrono::milliseconds(100));
      }
      std::vector<double> acc_us;
      double t_all = now_us();
      for (int i = 0; i < N; ++i) {
        CK(cuMemMap(va + CH * i, CH, 0, hs[i], 0));
        double t1 = now_us();
        CK(cuMemSetAccess(va + CH * i, CH, &ad, 1));
        acc_us.push_back(now_us() - t1);
      }
      t_all = now_us() - t_all;
      if (load) {
        stop = true;
        launcher.join();
      }
      std::printf("{\"bg_allocs\":%d,\"chain\":%d,\"plain_every\":%d,\"load\":\"%s\","
                  "\"setaccess_us_p50\":%.1f,\"p90\":%.1f,\"p99\":%.1f,\"max\":%.1f,"
                  "\"chunks_per_ms\":%.3f}\n",
                  (int)bg.size(), c.chain, c.plain_every, load ? "stream" : "idle",
                  pct(acc_us, 0.5), pct(acc_us, 0.9), pct(acc_us, 0.99), pct(acc_us, 1.0),
                  N / (t_all / 1e3));
      std::fflush(stdout);
      for (int i = 0; i < N; ++i) CK(cuMemUnmap(va + CH * i, CH));
    }
  }
  return 0;
}
