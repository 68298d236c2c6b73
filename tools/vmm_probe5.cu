// vmm_probe5 — does a VMM call wait on the kernels queued in the calling
// context? cuMemMap + cuMemSetAccess latency under an HBM-streaming kernel
// flood (launched in the primary context), issued (a) from the primary
// context, (b) from a second context created on the same device
// (cuCtxCreate). After (b), a kernel in the primary context writes and reads
// every freshly mapped chunk, so the mapping is proven usable there.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//        -o tools/vmm_probe5 tools/vmm_probe5.cu -lcuda
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
  CUcontext prim, side;
  CK(cuDevicePrimaryCtxRetain(&prim, dev));
  CK(cuCtxSetCurrent(prim));
  RK(cudaSetDevice(0));
  int sms = 0;
  RK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t buf_bytes = 4ull << 30;
  float4* buf;
  float* sink;
  unsigned* bad;
  RK(cudaMalloc(&buf, buf_bytes));
  RK(cudaMemset(buf, 0, buf_bytes));
  RK(cudaMalloc(&sink, 64));
  RK(cudaMalloc(&bad, 4));
  cudaStream_t s;
  RK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cuCtxCreate(&side, 0, dev));
  CK(cuCtxSetCurrent(prim));

  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  CUmemAccessDesc ad{};
  ad.location = ap.location;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  const int N = 64;
  std::vector<CUmemGenericAllocationHandle> hs(N);
  for (auto& h : hs) CK(cuMemCreate(&h, CH, &ap, 0));
  CUdeviceptr va;
  CK(cuMemAddressReserve(&va, CH * N, CH, 0, 0));

  for (int pdl : {0, 1}) {
    for (int use_side : {0, 1}) {
      for (int load : {0, 1}) {
        std::atomic<bool> stop{false};
        std::thread launcher;
        if (load) {
          launcher = std::thread([&] {
            CK(cuCtxSetCurrent(prim));
            cudaEvent_t e;
            RK(cudaEventCreate(&e));
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(sms * 4);
            cfg.blockDim = dim3(512);
            cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            while (!stop.load()) {  // 32 x ~0.6 ms streaming kernels per "step"
              for (int i = 0; i < 32; ++i) {
                cfg.numAttrs = (pdl && i > 0) ? 1 : 0;
                RK(cudaLaunchKernelEx(&cfg, stream_kernel, (const float4*)buf, buf_bytes / 16, sink,
                                      (pdl && i > 0) ? 1 : 0));
              }
              RK(cudaEventRecord(e, s));
              RK(cudaEventSynchronize(e));
            }
          });
          std::this_thread::sleep_for(std::chrono::milliseconds(200));
        }
        CK(cuCtxSetCurrent(use_side ? side : prim));
        std::vector<double> map_us, acc_us;
        double t_all = now_us();
        for (int i = 0; i < N; ++i) {
          double t0 = now_us();
          CK(cuMemMap(va + CH * i, CH, 0, hs[i], 0));
          double t1 = now_us();
          CK(cuMemSetAccess(va + CH * i, CH, &ad, 1));
          map_us.push_back(t1 - t0);
          acc_us.push_back(now_us() - t1);
        }
        t_all = now_us() - t_all;
        if (load) {
          stop = true;
          launcher.join();
        }
        CK(cuCtxSetCurrent(prim));
        RK(cudaMemset(bad, 0, 4));
        touch<<<sms * 4, 512, 0, s>>>(reinterpret_cast<unsigned*>(va), CH * N / 4, bad);
        unsigned h_bad = 0;
        RK(cudaMemcpyAsync(&h_bad, bad, 4, cudaMemcpyDeviceToHost, s));
        RK(cudaStreamSynchronize(s));
        std::printf("{\"pdl_chain\":%d,\"vmm_ctx\":\"%s\",\"load\":\"%s\",\"map_us_p50\":%.1f,"
                    "\"setaccess_us_p50\":%.1f,\"setaccess_us_p90\":%.1f,\"chunks_per_ms\":%.3f,"
                    "\"usable_from_primary\":%s}\n",
                    pdl, use_side ? "second_context" : "primary", load ? "hbm_stream" : "idle",
                    pct(map_us, 0.5), pct(acc_us, 0.5), pct(acc_us, 0.9), N / (t_all / 1e3),
                    h_bad == 0 ? "true" : "false");
        std::fflush(stdout);
        CK(cuCtxSetCurrent(use_side ? side : prim));
        for (int i = 0; i < N; ++i) CK(cuMemUnmap(va + CH * i, CH));
        CK(cuCtxSetCurrent(prim));
      }
    }
  }
  return 0;
}
