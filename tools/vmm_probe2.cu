// vmm_probe2 — idle-GPU cost structure of the VMM calls on this driver:
// per-call cost vs mapping size, vs number of live mappings, slab offsets,
// and host CPU time vs wall time inside each call (is the driver computing,
// or waiting on the GPU / its firmware?). One JSON line per case.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//        -o tools/vmm_probe2 tools/vmm_probe2.cu -lcuda
#include <cuda.h>
#include <time.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
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
static double cpu_us() {
  timespec t;
  clock_gettime(CLOCK_THREAD_CPUTIME_ID, &t);
  return t.tv_sec * 1e6 + t.tv_nsec / 1e3;
}

struct T {
  double w0, c0;
  T() : w0(wall_us()), c0(cpu_us()) {}
  double wall() const { return wall_us() - w0; }
  double cpu() const { return cpu_us() - c0; }
};

static const size_t CH = 2ull << 20;
static CUmemAllocationProp ap{};
static CUmemAccessDesc ad{};

static double med(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v.empty() ? 0 : v[v.size() / 2];
}

int main() {
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
  size_t gmin = 0, grec = 0;
  CK(cuMemGetAllocationGranularity(&gmin, &ap, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
  CK(cuMemGetAllocationGranularity(&grec, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  int drv = 0;
  cuDriverGetVersion(&drv);
  std::printf("{\"case\":\"granularity\",\"min\":%zu,\"recommended\":%zu,\"driver\":%d}\n", gmin,
              grec, drv);

  // 1) create / map / setaccess / unmap / release per size (one handle each)
  for (size_t mib : {2, 32, 512}) {
    size_t sz = mib << 20;
    std::vector<double> cw, cc, mw, aw, ac, uw, rw;
    int reps = mib == 512 ? 4 : 16;
    for (int i = 0; i < reps; ++i) {
      CUmemGenericAllocationHandle h;
      CUdeviceptr va;
      CK(cuMemAddressReserve(&va, sz, CH, 0, 0));
      T t1;
      CK(cuMemCreate(&h, sz, &ap, 0));
      cw.push_back(t1.wall());
      cc.push_back(t1.cpu());
      T t2;
      CK(cuMemMap(va, sz, 0, h, 0));
      mw.push_back(t2.wall());
      T t3;
      CK(cuMemSetAccess(va, sz, &ad, 1));
      aw.push_back(t3.wall());
      ac.push_back(t3.cpu());
      T t4;
      CK(cuMemUnmap(va, sz));
      uw.push_back(t4.wall());
      T t5;
      CK(cuMemRelease(h));
      rw.push_back(t5.wall());
      CK(cuMemAddressFree(va, sz));
    }
    std::printf(
        "{\"case\":\"single_handle\",\"mib\":%zu,\"create_us\":%.1f,\"create_cpu_us\":%.1f,"
        "\"map_us\":%.1f,\"access_us\":%.1f,\"access_cpu_us\":%.1f,\"unmap_us\":%.1f,"
        "\"release_us\":%.1f}\n",
        mib, med(cw), med(cc), med(mw), med(aw), med(ac), med(uw), med(rw));
    std::fflush(stdout);
  }

  // 2) slab: one 64 MiB handle, 2 MiB sub-ranges mapped at nonzero offsets
  {
    const size_t SL = 64ull << 20;
    CUmemGenericAllocationHandle h;
    CK(cuMemCreate(&h, SL, &ap, 0));
    CUdeviceptr va;
    CK(cuMemAddressReserve(&va, SL, CH, 0, 0));
    std::vector<double> mw, aw;
    bool ok = true;
    for (size_t off = 0; off < SL; off += CH) {
      // map slab piece k at VA slot (31 - k): scattered, non-identity placement
      size_t slot = (SL - CH) - off;
      T t2;
      CUresult r = cuMemMap(va + slot, CH, off, h, 0);
      if (r != CUDA_SUCCESS) {
        const char* s = nullptr;
        cuGetErrorString(r, &s);
        std::printf("{\"case\":\"slab_offset_map\",\"ok\":false,\"err\":\"%s\",\"offset\":%zu}\n",
                    s, off);
        ok = false;
        break;
      }
      mw.push_back(t2.wall());
      T t3;
      CK(cuMemSetAccess(va + slot, CH, &ad, 1));
      aw.push_back(t3.wall());
    }
    if (ok)
      std::printf("{\"case\":\"slab_offset_map\",\"ok\":true,\"map_us\":%.1f,\"access_us\":%.1f}\n",
                  med(mw), med(aw));
    if (ok) {
      // unmap + remap all pieces into one contiguous run, single setaccess
      for (size_t off = 0; off < SL; off += CH) CK(cuMemUnmap(va + off, CH));
      T t;
      for (size_t off = 0; off < SL; off += CH) CK(cuMemMap(va + off, CH, off, h, 0));
      double m = t.wall();
      T t2;
      CK(cuMemSetAccess(va, SL, &ad, 1));
      std::printf("{\"case\":\"slab_32_pieces_one_access\",\"map_us_total\":%.1f,\"access_us\":%.1f}\n",
                  m, t2.wall());
      T t3;
      for (size_t off = 0; off < SL; off += CH) CK(cuMemUnmap(va + off, CH));
      std::printf("{\"case\":\"slab_unmap_32\",\"us_total\":%.1f}\n", t3.wall());
      // whole slab mapped as one mapping
      T t4;
      CK(cuMemMap(va, SL, 0, h, 0));
      double m4 = t4.wall();
      T t5;
      CK(cuMemSetAccess(va, SL, &ad, 1));
      std::printf("{\"case\":\"slab_whole_one_mapping\",\"map_us\":%.1f,\"access_us\":%.1f}\n", m4,
                  t5.wall());
      CK(cuMemUnmap(va, SL));
    }
    std::fflush(stdout);
  }

  // 3) setaccess cost vs number of live mappings elsewhere in the process
  {
    std::vector<CUmemGenericAllocationHandle> bg;
    std::vector<CUdeviceptr> bgva;
    CUdeviceptr probe_va;
    CK(cuMemAddressReserve(&probe_va, 64 * CH, CH, 0, 0));
    std::vector<CUmemGenericAllocationHandle> ph(64);
    for (auto& x : ph) CK(cuMemCreate(&x, CH, &ap, 0));
    size_t live = 0;
    for (size_t target : {0, 512, 2048, 8192}) {
      while (live < target) {
        // background mappings: 256-chunk spaces, each fully mapped + accessed
        CUdeviceptr va;
        CK(cuMemAddressReserve(&va, 256 * CH, CH, 0, 0));
        for (int k = 0; k < 256; ++k) {
          CUmemGenericAllocationHandle h;
          CK(cuMemCreate(&h, CH, &ap, 0));
          CK(cuMemMap(va + k * CH, CH, 0, h, 0));
          bg.push_back(h);
        }
        CK(cuMemSetAccess(va, 256 * CH, &ad, 1));
        bgva.push_back(va);
        live += 256;
      }
      std::vector<double> aw, ac, uw;
      for (int k = 0; k < 64; ++k) {
        CK(cuMemMap(probe_va + k * CH, CH, 0, ph[k], 0));
        T t;
        CK(cuMemSetAccess(probe_va + k * CH, CH, &ad, 1));
        aw.push_back(t.wall());
        ac.push_back(t.cpu());
      }
      for (int k = 0; k < 64; ++k) {
        T t;
        CK(cuMemUnmap(probe_va + k * CH, CH));
        uw.push_back(t.wall());
      }
      std::printf(
          "{\"case\":\"access_vs_live_mappings\",\"live\":%zu,\"access_us\":%.1f,"
          "\"access_cpu_us\":%.1f,\"unmap_us\":%.1f}\n",
          live, med(aw), med(ac), med(uw));
      std::fflush(stdout);
    }
    // 4) remap of the same handle into the same slot it just left
    std::vector<double> rw;
    for (int k = 0; k < 32; ++k) {
      CK(cuMemMap(probe_va, CH, 0, ph[0], 0));
      T t;
      CK(cuMemSetAccess(probe_va, CH, &ad, 1));
      rw.push_back(t.wall());
      CK(cuMemUnmap(probe_va, CH));
    }
    std::printf("{\"case\":\"same_slot_remap\",\"access_us\":%.1f}\n", med(rw));
  }
  return 0;
}
