// libvtensor.so — the vTensor device shim (C ABI in include/vtensor.h).
//
// Two layers in one object:
//   1. A bookkeeping state machine that is bit-exact with the reference's
//      simulated device (kvsim/device.py:118-295): monotone never-reused
//      ordinals for range bases (device.py:199-201) and handle ids
//      (device.py:212-213), byte accounting (device.py:141-182), the
//      instrumented call log (device.py:184-187) and the nine error classes.
//      Ordering decisions never depend on real CUdeviceptr or CUDA handle
//      values, so manager state stays identical to the oracle.
//   2. On a GPU, a CUDA-driver VMM backend. reserve runs inline (the VA must
//      be known immediately); create/map/unmap/destroy/release are queued in
//      issue order to a per-device worker thread so chunk mapping overlaps the
//      decode kernels (north_star item 1). OOM is decided by the configured
//      byte budget (device.py:153-160, 208-211), never by the driver.
//
// The driver is loaded with dlopen at first use: the CPU CI container has no
// libcuda.so.1, and the simulated backend must work there.

#include "../../include/vtensor.h"

#include <cuda.h>
#include <dlfcn.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

namespace {

int64_t now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// ---------------------------------------------------------------------------
// Driver entry points (resolved once with dlopen/dlsym).
// ---------------------------------------------------------------------------
struct Driver {
  bool loaded = false;
  std::string error;
  CUresult (*Init)(unsigned int);
  CUresult (*DeviceGet)(CUdevice*, int);
  CUresult (*PrimaryCtxRetain)(CUcontext*, CUdevice);
  CUresult (*PrimaryCtxRelease)(CUdevice);
  CUresult (*CtxSetCurrent)(CUcontext);
  CUresult (*CtxGetCurrent)(CUcontext*);
  CUresult (*CtxCreate)(CUcontext*, unsigned int, CUdevice);
  CUresult (*CtxDestroy)(CUcontext);
  CUresult (*CtxPopCurrent)(CUcontext*);
  CUresult (*AddrReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
  CUresult (*AddrFree)(CUdeviceptr, size_t);
  CUresult (*MemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                        unsigned long long);
  CUresult (*MemRelease)(CUmemGenericAllocationHandle);
  CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle,
                     unsigned long long);
  CUresult (*MemUnmap)(CUdeviceptr, size_t);
  CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
  CUresult (*Granularity)(size_t*, const CUmemAllocationProp*,
                          CUmemAllocationGranularity_flags);
  CUresult (*EventCreate)(CUevent*, unsigned int);
  CUresult (*EventRecord)(CUevent, CUstream);
  CUresult (*EventSynchronize)(CUevent);
  CUresult (*EventDestroy)(CUevent);
  CUresult (*StreamCreate)(CUstream*, unsigned int);
  CUresult (*StreamDestroy)(CUstream);
  CUresult (*StreamWaitEvent)(CUstream, CUevent, unsigned int);
  CUresult (*GetErrorString)(CUresult, const char**);
  // Optional (cross-device chunk sharing): nullptr if the driver lacks them.
  CUresult (*ExportShareable)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                              unsigned long long);
  CUresult (*ImportShareable)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType);
  CUresult (*TensorMapEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);
};

Driver& driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libcuda.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      d.error = std::string("cannot dlopen libcuda.so.1: ") + dlerror();
      return;
    }
    bool ok = true;
    auto sym = [&](const char* name) -> void* {
      void* p = dlsym(h, name);
      if (!p) {
        ok = false;
        d.error += std::string("missing driver symbol ") + name + "; ";
      }
      return p;
    };
#define VT_SYM(field, name) d.field = reinterpret_cast<decltype(d.field)>(sym(name))
    VT_SYM(Init, "cuInit");
    VT_SYM(DeviceGet, "cuDeviceGet");
    VT_SYM(PrimaryCtxRetain, "cuDevicePrimaryCtxRetain");
    VT_SYM(PrimaryCtxRelease, "cuDevicePrimaryCtxRelease_v2");
    VT_SYM(CtxSetCurrent, "cuCtxSetCurrent");
    VT_SYM(CtxGetCurrent, "cuCtxGetCurrent");
    VT_SYM(CtxCreate, "cuCtxCreate_v2");
    VT_SYM(CtxDestroy, "cuCtxDestroy_v2");
    VT_SYM(CtxPopCurrent, "cuCtxPopCurrent_v2");
    VT_SYM(AddrReserve, "cuMemAddressReserve");
    VT_SYM(AddrFree, "cuMemAddressFree");
    VT_SYM(MemCreate, "cuMemCreate");
    VT_SYM(MemRelease, "cuMemRelease");
    VT_SYM(MemMap, "cuMemMap");
    VT_SYM(MemUnmap, "cuMemUnmap");
    VT_SYM(MemSetAccess, "cuMemSetAccess");
    VT_SYM(Granularity, "cuMemGetAllocationGranularity");
    VT_SYM(EventCreate, "cuEventCreate");
    VT_SYM(EventRecord, "cuEventRecord");
    VT_SYM(EventSynchronize, "cuEventSynchronize");
    VT_SYM(EventDestroy, "cuEventDestroy_v2");
    VT_SYM(StreamCreate, "cuStreamCreate");
    VT_SYM(StreamDestroy, "cuStreamDestroy_v2");
    VT_SYM(StreamWaitEvent, "cuStreamWaitEvent");
    VT_SYM(GetErrorString, "cuGetErrorString");
    VT_SYM(TensorMapEncodeTiled, "cuTensorMapEncodeTiled");
#undef VT_SYM
    d.ExportShareable = reinterpret_cast<decltype(d.ExportShareable)>(
        dlsym(h, "cuMemExportToShareableHandle"));
    d.ImportShareable = reinterpret_cast<decltype(d.ImportShareable)>(
        dlsym(h, "cuMemImportFromShareableHandle"));
    if (ok && d.Init(0) != CUDA_SUCCESS) {
      ok = false;
      d.error += "cuInit failed; ";
    }
    d.loaded = ok;
  });
  return d;
}

std::string cu_err(CUresult r) {
  const char* s = nullptr;
  if (driver().GetErrorString) driver().GetErrorString(r, &s);
  return s ? std::string(s) : ("CUresult " + std::to_string(static_cast<int>(r)));
}

// ---------------------------------------------------------------------------
// Worker-side driver ops.
// ---------------------------------------------------------------------------
enum class DrvKind : uint8_t { kCreate, kMap, kUnmap, kDestroy, kRelease, kExport, kImport, kFill };

struct DrvOp {
  DrvKind kind;
  int64_t handle_id;     // create / map / destroy
  CUdeviceptr addr;      // map / unmap / release
  size_t size;           // release
  uint64_t fence_epoch;  // teardown ops wait for this stream event
  uint64_t ticket;
  int64_t submit_ns;
  int fd;                // import: the shareable handle (consumed)
  int* fd_out;           // export: where the new shareable handle goes
  bool imported;         // destroy: the chunk belongs to another pool
};

constexpr int kFenceRing = 64;

}  // namespace

// One reserved range: its page -> handle-id table (-1 = unmapped).
struct RangeState {
  int64_t pages = 0;
  int64_t mapped = 0;
  std::vector<int64_t> slot;
  CUdeviceptr va = 0;
};

struct vt_device {
  vt_config cfg{};
  int ordinal = -1;  // <0: simulated
  std::string last_error;

  // --- bookkeeping state machine (device.py:127-137) ---
  std::map<int64_t, RangeState> ranges;               // ordered: live_ranges() sorted
  std::map<int64_t, int64_t> handles;                 // id -> map_count, ordered
  std::set<int64_t> imported;                         // ids of chunks owned by another device
  int64_t next_base = 0;
  int64_t next_handle = 0;
  int64_t mapped_pages = 0;
  int64_t active_requests = 0;
  int64_t reserved_bytes = 0;
  std::vector<vt_call> log;

  // --- CUDA backend ---
  CUcontext ctx = nullptr;
  // Context the driver worker (and pool) issue the VMM calls from: the
  // primary context, or with VT_WORKER_CTX=1 a private one on the same
  // device (mappings are per device, so kernels in the primary context see
  // them; tools/vmm_probe5.cu measured the calls there under chained launches).
  CUcontext work_ctx = nullptr;
  bool own_work_ctx = false;
  CUdevice cu_dev = 0;
  CUmemAllocationProp prop{};
  CUmemAccessDesc access{};
  bool async = true;  // guarded by mu (the worker reads it in its wait predicate)
  std::thread worker;
  std::mutex mu;
  std::condition_variable cv_work, cv_done;
  std::deque<DrvOp> queue;
  bool stopping = false;
  uint64_t next_ticket = 0;                 // submitted
  std::atomic<uint64_t> done_ticket{0};     // completed
  std::string drv_error;                    // sticky worker error
  std::atomic<bool> drv_failed{false};
  // Fences: vt_fence(stream) makes a private in-order fence stream wait on
  // the caller's stream and records epoch e there, so epoch e completing
  // implies every earlier fence (whatever stream it named) has completed.
  CUstream fence_stream = nullptr;
  CUevent fence_src = nullptr;              // scratch: marks the caller's stream
  CUevent fence_events[kFenceRing] = {};
  uint64_t fence_epoch = 0;                 // recorded by the caller
  uint64_t synced_epoch = 0;                // waited by the worker
  std::mutex phys_mu;  // phys + reserve (pool threads)
  std::unordered_map<int64_t, CUmemGenericAllocationHandle> phys;
  std::vector<CUmemGenericAllocationHandle> reserve;  // pre-created, not yet a logical chunk
  int64_t reserve_target = 0;
  std::mutex stat_mu;
  vt_driver_stats dstats{};
  // driver pool (parallel_for); the worker thread is member 0
  std::vector<std::thread> pool;
  std::mutex pool_mu;
  std::condition_variable pool_cv, pool_done_cv;
  const std::function<void(size_t)>* job_fn = nullptr;
  size_t job_n = 0;
  uint64_t job_gen = 0;
  bool pool_stop = false;
  int job_active = 0;  // pool threads inside the current job (guarded by pool_mu)
  std::atomic<size_t> job_next{0}, job_left{0};
  int driver_threads = 1;
  bool setaccess_runs = false;  // one cuMemSetAccess per contiguous run of maps (VT_SETACCESS_RUNS=1)
  std::mutex lat_mu;
  // [0,6): per vt_op, submit -> completed (ns); 6 / 7: duration of each raw
  // cuMemMap / cuMemSetAccess driver call (ns)
  std::vector<int64_t> lat[8];

  bool is_cuda() const { return ordinal >= 0; }

  void note_latency(const DrvOp& op, int64_t done_ns) {
    if (op.kind >= DrvKind::kExport) return;  // not one of the reference's device ops
    static const int kOp[] = {VT_OP_CREATE_CHUNK, VT_OP_MAP_PAGE, VT_OP_UNMAP_PAGE,
                              VT_OP_DESTROY_CHUNK, VT_OP_RELEASE_ADDRESS, VT_OP_CREATE_CHUNK,
                              VT_OP_CREATE_CHUNK, VT_OP_CREATE_CHUNK};
    std::lock_guard<std::mutex> lk(lat_mu);
    auto& v = lat[kOp[static_cast<int>(op.kind)]];
    if (v.size() < (1u << 20)) v.push_back(done_ns - op.submit_ns);
  }
  void note_call(int ring, int64_t ns) {
    std::lock_guard<std::mutex> lk(lat_mu);
    auto& v = lat[ring];
    if (v.size() < (1u << 20)) v.push_back(ns);
  }
  // Imported chunks live in another device's pool and budget.
  int64_t created_bytes() const {
    return static_cast<int64_t>(handles.size() - imported.size()) * cfg.chunk_bytes;
  }
  int64_t activation_bytes() const {
    return active_requests * cfg.activation_bytes_per_request;
  }
  int64_t free_bytes() const {
    return cfg.capacity_bytes - cfg.weights_bytes - activation_bytes() - created_bytes();
  }

  int fail(int code, std::string msg) {
    last_error = std::move(msg);
    return code;
  }

  void log_call(vt_op op, int64_t base, int64_t page, int64_t handle, int64_t pages) {
    vt_call c{};
    c.seq = static_cast<int64_t>(log.size());
    c.op = op;
    c.base = base;
    c.page = page;
    c.handle = handle;
    c.pages = pages;
    c.created_bytes_after = created_bytes();
    log.push_back(c);
  }

  // ---- worker plumbing ----
  bool ensure_ctx() {
    CUcontext cur = nullptr;
    driver().CtxGetCurrent(&cur);
    if (cur != ctx) return driver().CtxSetCurrent(ctx) == CUDA_SUCCESS;
    return true;
  }

  // Ops are queued in issue order; kick() hands everything queued so far to
  // the worker (async) or executes it inline as one batch (sync), so a batched
  // map of consecutive pages always costs a single cuMemSetAccess.
  void enqueue(DrvOp op) {
    op.submit_ns = now_ns();
    op.fence_epoch = fence_epoch;
    std::lock_guard<std::mutex> lk(mu);
    op.ticket = ++next_ticket;
    queue.push_back(op);
  }

  void kick() {
    if (!is_cuda()) return;
    if (async) {
      cv_work.notify_one();
      return;
    }
    // Sync mode: the worker is parked (its wait predicate requires `async`),
    // so the queue is drained here, on the caller's thread, before returning.
    std::vector<DrvOp> batch;
    {
      std::lock_guard<std::mutex> lk(mu);
      batch.assign(queue.begin(), queue.end());
      queue.clear();
    }
    if (batch.empty()) return;
    execute_run(batch.data(), batch.size());
  }

  // done_ticket is published under `mu` so a waiter that has checked its
  // predicate (under `mu`) is already blocked before the notify can happen.
  void publish_done(uint64_t ticket) {
    {
      std::lock_guard<std::mutex> lk(mu);
      done_ticket.store(ticket);
    }
    cv_done.notify_all();
  }

  void record_error(const std::string& what) {
    {
      std::lock_guard<std::mutex> lk(mu);
      if (drv_error.empty()) drv_error = what;
      drv_failed.store(true);
    }
    cv_done.notify_all();
  }

  void wait_fence(uint64_t epoch) {
    if (epoch == 0 || epoch <= synced_epoch) return;
    int64_t t0 = now_ns();
    CUevent ev = fence_events[epoch % kFenceRing];
    CUresult r = driver().EventSynchronize(ev);
    if (r != CUDA_SUCCESS) record_error("cuEventSynchronize: " + cu_err(r));
    synced_epoch = epoch;
    std::lock_guard<std::mutex> lk(stat_mu);
    dstats.fence_waits++;
    dstats.fence_wait_ns_total += now_ns() - t0;
  }

  // ---- physical handle table + reserve (shared by the pool threads) ----
  CUmemGenericAllocationHandle phys_get(int64_t id, bool* found) {
    std::lock_guard<std::mutex> lk(phys_mu);
    auto it = phys.find(id);
    *found = it != phys.end();
    return *found ? it->second : 0;
  }
  void phys_put(int64_t id, CUmemGenericAllocationHandle h) {
    std::lock_guard<std::mutex> lk(phys_mu);
    phys[id] = h;
  }
  bool phys_take(int64_t id, CUmemGenericAllocationHandle* h) {
    std::lock_guard<std::mutex> lk(phys_mu);
    auto it = phys.find(id);
    if (it == phys.end()) return false;
    *h = it->second;
    phys.erase(it);
    return true;
  }
  // A pre-created handle from the reserve, if any (cuMemCreate off the path).
  bool reserve_pop(CUmemGenericAllocationHandle* h) {
    std::lock_guard<std::mutex> lk(phys_mu);
    if (reserve.empty()) return false;
    *h = reserve.back();
    reserve.pop_back();
    return true;
  }
  // A destroyed chunk's memory goes back to the reserve while it is short.
  bool reserve_push(CUmemGenericAllocationHandle h) {
    std::lock_guard<std::mutex> lk(phys_mu);
    if (static_cast<int64_t>(reserve.size()) >= reserve_target) return false;
    reserve.push_back(h);
    return true;
  }
  int64_t reserve_deficit() {
    std::lock_guard<std::mutex> lk(phys_mu);
    return reserve_target - static_cast<int64_t>(reserve.size());
  }

  void stat_add(int64_t vt_driver_stats::*calls, int64_t vt_driver_stats::*ns, int64_t dt) {
    std::lock_guard<std::mutex> lk(stat_mu);
    dstats.*calls += 1;
    dstats.*ns += dt;
  }

  // ---- driver thread pool: parallel_for over independent driver ops ----
  // On an idle GPU (tools/vmm_probe.cu "alternate") one thread completes
  // 0.5-1.6 map+SetAccess per ms and four threads 2-6 per ms; under the decode
  // stream concurrent calls serialise in the driver and block kernel launches,
  // so the default is one thread (see vt_dev_open).
  // A job is closed only when every item ran AND every pool thread that
  // joined it has left it (job_fn is cleared first, so no thread can join
  // late): a thread still inside run_job_items must never claim an item of
  // the next job with this job's (by then destroyed) function.
  void parallel_for(size_t n, const std::function<void(size_t)>& fn) {
    if (n == 0) return;
    if (n == 1 || pool.empty()) {
      for (size_t k = 0; k < n; ++k) fn(k);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(pool_mu);
      job_fn = &fn;
      job_n = n;
      job_next.store(0);
      job_left.store(n);
      ++job_gen;
    }
    pool_cv.notify_all();
    run_job_items(fn, n);
    std::unique_lock<std::mutex> lk(pool_mu);
    pool_done_cv.wait(lk, [&] { return job_left.load() == 0; });
    job_fn = nullptr;
    pool_done_cv.wait(lk, [&] { return job_active == 0; });
  }
  void run_job_items(const std::function<void(size_t)>& fn, size_t n) {
    for (;;) {
      size_t k = job_next.fetch_add(1);
      if (k >= n) return;
      fn(k);
      if (job_left.fetch_sub(1) == 1) {
        std::lock_guard<std::mutex> lk(pool_mu);
        pool_done_cv.notify_all();
      }
    }
  }
  void pool_main() {
    driver().CtxSetCurrent(work_ctx);
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(size_t)>* fn;
      size_t n;
      {
        std::unique_lock<std::mutex> lk(pool_mu);
        pool_cv.wait(lk, [&] { return pool_stop || (job_gen != seen && job_fn); });
        if (pool_stop) return;
        seen = job_gen;
        fn = job_fn;
        n = job_n;
        ++job_active;
      }
      run_job_items(*fn, n);
      {
        std::lock_guard<std::mutex> lk(pool_mu);
        --job_active;
      }
      pool_done_cv.notify_all();
    }
  }
  void start_pool(int threads) {
    for (int t = 1; t < threads; ++t) pool.emplace_back([this] { pool_main(); });
  }
  void stop_pool() {
    {
      std::lock_guard<std::mutex> lk(pool_mu);
      pool_stop = true;
    }
    pool_cv.notify_all();
    for (auto& t : pool) t.join();
    pool.clear();
    pool_stop = false;
  }

  void do_create(const DrvOp& op) {
    int64_t t0 = now_ns();
    CUmemGenericAllocationHandle h = 0;
    if (reserve_pop(&h)) {
      phys_put(op.handle_id, h);
      std::lock_guard<std::mutex> lk(stat_mu);
      dstats.reserve_hits++;
      return;
    }
    CUresult r = driver().MemCreate(&h, static_cast<size_t>(cfg.chunk_bytes), &prop, 0);
    if (r != CUDA_SUCCESS)
      record_error("cuMemCreate: " + cu_err(r));
    else
      phys_put(op.handle_id, h);
    stat_add(&vt_driver_stats::create_calls, &vt_driver_stats::create_ns_total, now_ns() - t0);
  }
  void do_map_one(const DrvOp& op) {
    Driver& d = driver();
    int64_t t0 = now_ns();
    bool found = false;
    CUmemGenericAllocationHandle h = phys_get(op.handle_id, &found);
    if (!found) {
      record_error("map of a chunk the driver never created (id " +
                   std::to_string(op.handle_id) + ")");
      return;
    }
    const size_t len = static_cast<size_t>(cfg.chunk_bytes);
    CUresult r = d.MemMap(op.addr, len, 0, h, 0);
    if (r != CUDA_SUCCESS) record_error("cuMemMap: " + cu_err(r));
    int64_t ta = now_ns();
    r = d.MemSetAccess(op.addr, len, &access, 1);
    if (r != CUDA_SUCCESS) record_error("cuMemSetAccess: " + cu_err(r));
    int64_t t1 = now_ns();
    note_call(6, ta - t0);
    note_call(7, t1 - ta);
    std::lock_guard<std::mutex> lk(stat_mu);
    dstats.map_calls++;
    dstats.access_calls++;
    dstats.access_ns_total += t1 - ta;
    dstats.map_ns_total += t1 - t0;
  }
  // A run of maps onto consecutive pages: one cuMemMap per chunk (every chunk
  // is its own allocation), then ONE cuMemSetAccess over the whole run.
  void do_map_run(const DrvOp* ops, size_t n) {
    Driver& d = driver();
    const size_t len = static_cast<size_t>(cfg.chunk_bytes);
    int64_t t0 = now_ns();
    size_t mapped = 0;
    for (; mapped < n; ++mapped) {
      bool found = false;
      CUmemGenericAllocationHandle h = phys_get(ops[mapped].handle_id, &found);
      if (!found) {
        record_error("map of a chunk the driver never created (id " +
                     std::to_string(ops[mapped].handle_id) + ")");
        break;
      }
      const int64_t tm = now_ns();
      CUresult r = d.MemMap(ops[mapped].addr, len, 0, h, 0);
      note_call(6, now_ns() - tm);
      if (r != CUDA_SUCCESS) {
        record_error("cuMemMap: " + cu_err(r));
        break;
      }
    }
    int64_t ta = now_ns();
    if (mapped) {
      CUresult r = d.MemSetAccess(ops[0].addr, len * mapped, &access, 1);
      if (r != CUDA_SUCCESS) record_error("cuMemSetAccess: " + cu_err(r));
    }
    int64_t t1 = now_ns();
    if (mapped) note_call(7, t1 - ta);
    std::lock_guard<std::mutex> lk(stat_mu);
    dstats.map_calls += static_cast<int64_t>(mapped);
    dstats.access_calls++;
    dstats.access_ns_total += t1 - ta;
    dstats.map_ns_total += t1 - t0;
  }
  void do_unmap(const DrvOp& op) {
    int64_t t0 = now_ns();
    CUresult r = driver().MemUnmap(op.addr, static_cast<size_t>(cfg.chunk_bytes));
    if (r != CUDA_SUCCESS) record_error("cuMemUnmap: " + cu_err(r));
    stat_add(&vt_driver_stats::unmap_calls, &vt_driver_stats::unmap_ns_total, now_ns() - t0);
  }
  void do_destroy(const DrvOp& op) {
    int64_t t0 = now_ns();
    CUmemGenericAllocationHandle h;
    if (phys_take(op.handle_id, &h)) {
      // Imported chunks belong to another pool: always drop the reference.
      if (!op.imported && reserve_push(h)) return;
      CUresult r = driver().MemRelease(h);
      if (r != CUDA_SUCCESS) record_error("cuMemRelease: " + cu_err(r));
    }
    stat_add(&vt_driver_stats::destroy_calls, &vt_driver_stats::destroy_ns_total, now_ns() - t0);
  }
  void fill_reserve() {
    int64_t n = reserve_deficit();
    if (n <= 0) return;
    parallel_for(static_cast<size_t>(n), [&](size_t) {
      CUmemGenericAllocationHandle h = 0;
      int64_t t0 = now_ns();
      CUresult r = driver().MemCreate(&h, static_cast<size_t>(cfg.chunk_bytes), &prop, 0);
      if (r != CUDA_SUCCESS) {
        record_error("cuMemCreate (reserve): " + cu_err(r));
        return;
      }
      if (!reserve_push(h)) driver().MemRelease(h);
      stat_add(&vt_driver_stats::create_calls, &vt_driver_stats::create_ns_total, now_ns() - t0);
    });
  }
  void drain_reserve() {
    std::vector<CUmemGenericAllocationHandle> hs;
    {
      std::lock_guard<std::mutex> lk(phys_mu);
      hs.swap(reserve);
    }
    for (auto h : hs) driver().MemRelease(h);
  }

  // Executes ops[0..n), in issue order, as maximal segments of one kind. Ops
  // inside a segment are independent — creates of distinct ids, maps into
  // distinct free slots of handles created in an earlier segment, unmaps of
  // distinct mapped slots, releases of handles whose unmaps came earlier — so
  // each segment runs on the driver pool in parallel; the segment boundary
  // keeps every cross-kind dependency (create -> map -> unmap -> destroy). A
  // teardown segment first waits for the newest fence any of its ops names
  // (epochs are monotone in issue order and the fence stream is in order).
  // done_ticket advances after every segment, so maps are ready before a
  // later fenced unmap in the same batch has waited for its kernels.
  void execute_run(DrvOp* ops, size_t n) {
    Driver& d = driver();
    size_t i = 0;
    while (i < n) {
      const DrvKind kind = ops[i].kind;
      size_t j = i + 1;
      const bool parallel = kind == DrvKind::kCreate || kind == DrvKind::kMap ||
                            kind == DrvKind::kUnmap || kind == DrvKind::kDestroy;
      if (parallel)
        while (j < n && ops[j].kind == kind) ++j;
      DrvOp* seg = ops + i;
      const size_t m = j - i;
      if (kind == DrvKind::kUnmap || kind == DrvKind::kDestroy || kind == DrvKind::kRelease)
        wait_fence(seg[m - 1].fence_epoch);
      switch (kind) {
        case DrvKind::kCreate:
          parallel_for(m, [&](size_t k) { do_create(seg[k]); });
          break;
        case DrvKind::kMap:
          if (setaccess_runs) {
            // contiguous runs (an extend maps consecutive pages of one space)
            std::vector<std::pair<size_t, size_t>> runs;
            for (size_t k = 0; k < m; ++k) {
              if (!runs.empty() && seg[k].addr == seg[k - 1].addr + static_cast<CUdeviceptr>(cfg.chunk_bytes))
                runs.back().second++;
              else
                runs.push_back({k, 1});
            }
            parallel_for(runs.size(), [&](size_t r) { do_map_run(seg + runs[r].first, runs[r].second); });
          } else {
            parallel_for(m, [&](size_t k) { do_map_one(seg[k]); });
          }
          break;
        case DrvKind::kUnmap:
          parallel_for(m, [&](size_t k) { do_unmap(seg[k]); });
          break;
        case DrvKind::kDestroy:
          parallel_for(m, [&](size_t k) { do_destroy(seg[k]); });
          break;
        case DrvKind::kRelease: {
          CUresult r = d.AddrFree(seg[0].addr, seg[0].size);
          if (r != CUDA_SUCCESS) record_error("cuMemAddressFree: " + cu_err(r));
          break;
        }
        case DrvKind::kExport: {
          bool found = false;
          CUmemGenericAllocationHandle h = phys_get(seg[0].handle_id, &found);
          if (!found) {
            record_error("export of a chunk the driver never created (id " +
                         std::to_string(seg[0].handle_id) + ")");
          } else {
            CUresult r = d.ExportShareable(seg[0].fd_out, h,
                                           CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
            if (r != CUDA_SUCCESS) record_error("cuMemExportToShareableHandle: " + cu_err(r));
          }
          break;
        }
        case DrvKind::kImport: {
          CUmemGenericAllocationHandle h = 0;
          CUresult r = d.ImportShareable(
              &h, reinterpret_cast<void*>(static_cast<intptr_t>(seg[0].fd)),
              CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
          if (r != CUDA_SUCCESS)
            record_error("cuMemImportFromShareableHandle: " + cu_err(r));
          else
            phys_put(seg[0].handle_id, h);
          ::close(seg[0].fd);
          break;
        }
        case DrvKind::kFill:
          fill_reserve();
          break;
      }
      const int64_t done = now_ns();
      for (size_t k = 0; k < m; ++k) note_latency(seg[k], done);
      {
        std::lock_guard<std::mutex> lk(stat_mu);
        dstats.max_op_ns = std::max<int64_t>(dstats.max_op_ns, done - seg[m - 1].submit_ns);
        dstats.ops_completed += static_cast<int64_t>(m);
      }
      publish_done(seg[m - 1].ticket);
      i = j;
    }
  }

  void worker_main() {
    driver().CtxSetCurrent(work_ctx);
    std::vector<DrvOp> batch;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu);
        cv_work.wait(lk, [&] { return stopping || (async && !queue.empty()); });
        if (stopping && (queue.empty() || !async)) return;
        batch.assign(queue.begin(), queue.end());
        queue.clear();
      }
      execute_run(batch.data(), batch.size());
    }
  }
};

namespace {

// Makes the device's context current on the calling thread for one call and
// restores whatever was current before (the caller's CUDA runtime state, e.g.
// torch on another GPU of the same process, must not see a foreign context).
struct CtxScope {
  CUcontext prev = nullptr;
  bool swapped = false;
  explicit CtxScope(vt_device* d) {
    Driver& drv = driver();
    drv.CtxGetCurrent(&prev);
    if (prev != d->ctx) swapped = drv.CtxSetCurrent(d->ctx) == CUDA_SUCCESS;
  }
  ~CtxScope() {
    if (swapped) driver().CtxSetCurrent(prev);
  }
};

int check_map_args(vt_device* d, int64_t base, int64_t page, int64_t id, RangeState** out) {
  auto it = d->ranges.find(base);
  if (it == d->ranges.end())
    return d->fail(VT_E_UNKNOWN_RANGE, "range base " + std::to_string(base) + " is not reserved");
  RangeState& rs = it->second;
  if (page < 0 || page >= rs.pages)
    return d->fail(VT_E_INDEX_OUT_OF_RANGE, "page " + std::to_string(page) + " outside range of " +
                                                std::to_string(rs.pages) + " pages");
  if (d->handles.find(id) == d->handles.end())
    return d->fail(VT_E_STALE_HANDLE,
                   "handle " + std::to_string(id) + " was destroyed or never created");
  if (rs.slot[static_cast<size_t>(page)] >= 0)
    return d->fail(VT_E_PAGE_ALREADY_MAPPED,
                   "page " + std::to_string(page) + " of base " + std::to_string(base) + " is mapped");
  *out = &rs;
  return VT_OK;
}

int do_map(vt_device* d, int64_t base, int64_t page, int64_t id) {
  RangeState* rs = nullptr;
  int rc = check_map_args(d, base, page, id, &rs);
  if (rc) return rc;
  rs->slot[static_cast<size_t>(page)] = id;
  rs->mapped++;
  d->handles[id] += 1;
  d->mapped_pages++;
  d->log_call(VT_OP_MAP_PAGE, base, page, id, 0);
  if (d->is_cuda()) {
    DrvOp op{};
    op.kind = DrvKind::kMap;
    op.handle_id = id;
    op.addr = rs->va + static_cast<CUdeviceptr>(page) * static_cast<CUdeviceptr>(d->cfg.chunk_bytes);
    d->enqueue(op);
  }
  return VT_OK;
}

int do_unmap(vt_device* d, int64_t base, int64_t page, int64_t* id_out) {
  auto it = d->ranges.find(base);
  if (it == d->ranges.end())
    return d->fail(VT_E_UNKNOWN_RANGE, "range base " + std::to_string(base) + " is not reserved");
  RangeState& rs = it->second;
  if (page < 0 || page >= rs.pages || rs.slot[static_cast<size_t>(page)] < 0)
    return d->fail(VT_E_PAGE_NOT_MAPPED, "page " + std::to_string(page) + " of base " +
                                             std::to_string(base) + " is not mapped");
  int64_t id = rs.slot[static_cast<size_t>(page)];
  rs.slot[static_cast<size_t>(page)] = -1;
  rs.mapped--;
  d->handles[id] -= 1;
  d->mapped_pages--;
  d->log_call(VT_OP_UNMAP_PAGE, base, page, id, 0);
  if (d->is_cuda()) {
    DrvOp op{};
    op.kind = DrvKind::kUnmap;
    op.addr = rs.va + static_cast<CUdeviceptr>(page) * static_cast<CUdeviceptr>(d->cfg.chunk_bytes);
    d->enqueue(op);
  }
  if (id_out) *id_out = id;
  return VT_OK;
}

}  // namespace

extern "C" {

int vt_dev_open(const vt_config* cfg, int cuda_ordinal, vt_device** out) {
  if (!cfg || !out) return VT_E_ARG;
  *out = nullptr;
  if (cfg->capacity_bytes <= 0 || cfg->chunk_bytes <= 0) return VT_E_ARG;
  if (cfg->weights_bytes < 0 || cfg->weights_bytes > cfg->capacity_bytes) return VT_E_ARG;
  vt_device* d = new vt_device();
  d->cfg = *cfg;
  d->ordinal = cuda_ordinal;
  if (cuda_ordinal >= 0) {
    Driver& drv = driver();
    if (!drv.loaded) {
      d->last_error = "CUDA driver unavailable: " + drv.error;
      static thread_local std::string err;
      err = d->last_error;
      std::fprintf(stderr, "vtensor: %s\n", err.c_str());
      delete d;
      return VT_E_CUDA;
    }
    CUdevice dev;
    CUresult r = drv.DeviceGet(&dev, cuda_ordinal);
    if (r == CUDA_SUCCESS) r = drv.PrimaryCtxRetain(&d->ctx, dev);
    if (r != CUDA_SUCCESS) {
      std::fprintf(stderr, "vtensor: device %d: %s\n", cuda_ordinal, cu_err(r).c_str());
      delete d;
      return VT_E_CUDA;
    }
    d->cu_dev = dev;
    auto fail_open = [&](int code) {
      for (auto& ev : d->fence_events)
        if (ev) drv.EventDestroy(ev);
      if (d->fence_src) drv.EventDestroy(d->fence_src);
      if (d->fence_stream) drv.StreamDestroy(d->fence_stream);
      drv.PrimaryCtxRelease(dev);
      delete d;
      return code;
    };
    CtxScope scope(d);
    d->prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    d->prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    d->prop.location.id = cuda_ordinal;
    size_t gran = 0;
    r = drv.Granularity(&gran, &d->prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM);
    if (r != CUDA_SUCCESS || gran == 0 || cfg->chunk_bytes % static_cast<int64_t>(gran) != 0) {
      std::fprintf(stderr, "vtensor: chunk %lld is not a multiple of VMM granularity %zu\n",
                   static_cast<long long>(cfg->chunk_bytes), gran);
      return fail_open(VT_E_ARG);
    }
    d->access.location = d->prop.location;
    d->access.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    for (auto& ev : d->fence_events) {
      r = drv.EventCreate(&ev, CU_EVENT_DISABLE_TIMING);
      if (r != CUDA_SUCCESS) return fail_open(VT_E_CUDA);
    }
    if (drv.EventCreate(&d->fence_src, CU_EVENT_DISABLE_TIMING) != CUDA_SUCCESS ||
        drv.StreamCreate(&d->fence_stream, CU_STREAM_NON_BLOCKING) != CUDA_SUCCESS)
      return fail_open(VT_E_CUDA);
    // One driver thread by default. Measured in the config-2 bench (300 steps,
    // 1200 chunks mapped under the decode stream, profiles/r02/bench/
    // cfg2_300_*.json): with 4 threads issuing map + SetAccess concurrently the
    // calls serialise inside the driver and keep the lock the launching thread
    // needs (GPU idle 1477 ms, 145 host waits, 3537 GB/s); one thread: 0 host
    // waits, 6669 GB/s. More threads only pay off for bulk work on an idle GPU.
    int threads = 1;
    if (const char* e = std::getenv("VT_DRIVER_THREADS")) threads = std::atoi(e);
    d->driver_threads = std::max(1, std::min(threads, 16));
    if (const char* e = std::getenv("VT_SETACCESS_RUNS")) d->setaccess_runs = std::atoi(e) != 0;
    d->work_ctx = d->ctx;
    if (const char* e = std::getenv("VT_WORKER_CTX")) {
      if (std::atoi(e) != 0) {
        CUcontext c = nullptr, popped = nullptr;
        if (drv.CtxCreate(&c, 0, dev) == CUDA_SUCCESS) {
          drv.CtxPopCurrent(&popped);  // cuCtxCreate pushed it on this thread
          d->work_ctx = c;
          d->own_work_ctx = true;
        }
      }
    }
    d->start_pool(d->driver_threads);
    d->worker = std::thread([d] { d->worker_main(); });
  }
  *out = d;
  return VT_OK;
}

int vt_dev_close(vt_device* d) {
  if (!d) return VT_OK;
  if (d->is_cuda()) {
    {
      std::lock_guard<std::mutex> lk(d->mu);
      d->stopping = true;
    }
    d->cv_work.notify_all();
    if (d->worker.joinable()) d->worker.join();
    d->stop_pool();
    Driver& drv = driver();
    CtxScope scope(d);
    d->drain_reserve();
    // Tear down whatever the manager left behind (caller is responsible for
    // having synchronised the streams that read these pages).
    for (auto& kv : d->ranges) {
      RangeState& rs = kv.second;
      for (int64_t p = 0; p < rs.pages; ++p)
        if (rs.slot[static_cast<size_t>(p)] >= 0)
          drv.MemUnmap(rs.va + static_cast<CUdeviceptr>(p) * d->cfg.chunk_bytes,
                       static_cast<size_t>(d->cfg.chunk_bytes));
      drv.AddrFree(rs.va, static_cast<size_t>(rs.pages * d->cfg.chunk_bytes));
    }
    for (auto& kv : d->phys) drv.MemRelease(kv.second);
    for (auto& ev : d->fence_events)
      if (ev) drv.EventDestroy(ev);
    if (d->fence_src) drv.EventDestroy(d->fence_src);
    if (d->fence_stream) drv.StreamDestroy(d->fence_stream);
    if (d->own_work_ctx) drv.CtxDestroy(d->work_ctx);
    drv.PrimaryCtxRelease(d->cu_dev);
  }
  delete d;
  return VT_OK;
}

int vt_dev_is_cuda(const vt_device* d) { return d && d->is_cuda() ? 1 : 0; }

const char* vt_last_error(const vt_device* d) {
  if (!d) return "null device";
  return d->last_error.c_str();
}

// device.py:191-204
int vt_reserve(vt_device* d, int64_t size, int64_t* base, int64_t* pages) {
  const int64_t page = d->cfg.chunk_bytes;
  if (size <= 0 || size % page != 0)
    return d->fail(VT_E_INVALID_SIZE, "reserve size must be a positive multiple of " +
                                          std::to_string(page) + ", got " + std::to_string(size));
  const int64_t n = size / page;
  RangeState rs;
  rs.pages = n;
  rs.slot.assign(static_cast<size_t>(n), -1);
  if (d->is_cuda()) {
    CtxScope scope(d);
    CUdeviceptr va = 0;
    CUresult r = driver().AddrReserve(&va, static_cast<size_t>(size),
                                      static_cast<size_t>(page), 0, 0);
    if (r != CUDA_SUCCESS) return d->fail(VT_E_CUDA, "cuMemAddressReserve: " + cu_err(r));
    rs.va = va;
  }
  const int64_t b = d->next_base;
  d->next_base += n;  // disjoint ordinal intervals, never reused
  d->ranges.emplace(b, std::move(rs));
  d->reserved_bytes += size;
  d->log_call(VT_OP_RESERVE_ADDRESS, b, 0, 0, n);
  *base = b;
  *pages = n;
  return VT_OK;
}

// device.py:206-216
int vt_create_chunk(vt_device* d, int64_t* id) {
  if (d->free_bytes() < d->cfg.chunk_bytes)
    return d->fail(VT_E_OUT_OF_MEMORY, "need " + std::to_string(d->cfg.chunk_bytes) + " bytes, " +
                                           std::to_string(d->free_bytes()) + " free");
  const int64_t h = d->next_handle++;
  d->handles.emplace(h, 0);
  d->log_call(VT_OP_CREATE_CHUNK, 0, 0, h, 0);
  if (d->is_cuda()) {
    DrvOp op{};
    op.kind = DrvKind::kCreate;
    op.handle_id = h;
    d->enqueue(op);
    d->kick();
  }
  *id = h;
  return VT_OK;
}

// device.py:218-233
int vt_map_page(vt_device* d, int64_t base, int64_t page, int64_t id) {
  int rc = do_map(d, base, page, id);
  d->kick();
  return rc;
}

int vt_map_pages(vt_device* d, int64_t base, int64_t first_page, const int64_t* ids, int64_t n,
                 int64_t* n_done) {
  int64_t k = 0;
  int rc = VT_OK;
  for (; k < n; ++k) {
    rc = do_map(d, base, first_page + k, ids[k]);
    if (rc) break;
  }
  if (n_done) *n_done = k;
  d->kick();
  return rc;
}

// One scheduler extend (scheduler.py:166-180 = ops.py:83-112 p_alloc followed by
// ops.py:133-146 map_chunks) in one crossing: n_create chunks created, then the
// n_reuse parked handles and the created ones mapped at consecutive pages from
// first_page. The call log equals create_chunk x n_create, then map_page per
// page, and the driver work is queued with one wake-up. All-or-nothing: every
// precondition (budget, range, free slots, live reused handles) is checked
// before any state changes; on failure nothing happened and the caller takes
// the per-op path, which reproduces the reference's partial behaviour.
int vt_extend(vt_device* d, int64_t base, int64_t first_page, const int64_t* reuse_ids,
              int64_t n_reuse, int64_t n_create, int64_t* created_ids) {
  if (n_reuse < 0 || n_create < 0)
    return d->fail(VT_E_INDEX_OUT_OF_RANGE, "negative chunk count");
  if (n_create > 0 && d->free_bytes() < n_create * d->cfg.chunk_bytes)
    return d->fail(VT_E_OUT_OF_MEMORY,
                   "need " + std::to_string(n_create * d->cfg.chunk_bytes) + " bytes, " +
                       std::to_string(d->free_bytes()) + " free");
  auto it = d->ranges.find(base);
  if (it == d->ranges.end())
    return d->fail(VT_E_UNKNOWN_RANGE, "range base " + std::to_string(base) + " is not reserved");
  RangeState& rs = it->second;
  const int64_t n = n_reuse + n_create;
  if (first_page < 0 || first_page + n > rs.pages)
    return d->fail(VT_E_INDEX_OUT_OF_RANGE, "pages " + std::to_string(first_page) + ".." +
                                                std::to_string(first_page + n - 1) +
                                                " outside range of " + std::to_string(rs.pages) +
                                                " pages");
  for (int64_t k = 0; k < n; ++k)
    if (rs.slot[static_cast<size_t>(first_page + k)] >= 0)
      return d->fail(VT_E_PAGE_ALREADY_MAPPED, "page " + std::to_string(first_page + k) +
                                                   " of base " + std::to_string(base) +
                                                   " is mapped");
  for (int64_t k = 0; k < n_reuse; ++k)
    if (d->handles.find(reuse_ids[k]) == d->handles.end())
      return d->fail(VT_E_STALE_HANDLE, "handle " + std::to_string(reuse_ids[k]) +
                                            " was destroyed or never created");
  for (int64_t k = 0; k < n_create; ++k) {
    const int64_t h = d->next_handle++;
    d->handles.emplace(h, 0);
    d->log_call(VT_OP_CREATE_CHUNK, 0, 0, h, 0);
    if (d->is_cuda()) {
      DrvOp op{};
      op.kind = DrvKind::kCreate;
      op.handle_id = h;
      d->enqueue(op);
    }
    created_ids[k] = h;
  }
  int rc = VT_OK;
  for (int64_t k = 0; k < n && rc == VT_OK; ++k)
    rc = do_map(d, base, first_page + k, k < n_reuse ? reuse_ids[k] : created_ids[k - n_reuse]);
  d->kick();
  return rc;  // VT_OK: the checks above leave do_map nothing to reject
}

// device.py:235-245
int vt_unmap_page(vt_device* d, int64_t base, int64_t page, int64_t* id) {
  int rc = do_unmap(d, base, page, id);
  d->kick();
  return rc;
}

int vt_unmap_tail(vt_device* d, int64_t base, int64_t from_page, int64_t down_to, int64_t* ids,
                  int64_t* n_done) {
  int64_t k = 0;
  int rc = VT_OK;
  for (int64_t p = from_page; p >= down_to; --p, ++k) {
    rc = do_unmap(d, base, p, ids ? &ids[k] : nullptr);
    if (rc) break;
  }
  if (n_done) *n_done = k;
  d->kick();
  return rc;
}

// device.py:247-257
int vt_release(vt_device* d, int64_t base) {
  auto it = d->ranges.find(base);
  if (it == d->ranges.end())
    return d->fail(VT_E_UNKNOWN_RANGE, "range base " + std::to_string(base) + " is not reserved");
  if (it->second.mapped)
    return d->fail(VT_E_RANGE_STILL_MAPPED, "range base " + std::to_string(base) + " still has " +
                                               std::to_string(it->second.mapped) + " mapped pages");
  if (d->is_cuda()) {
    DrvOp op{};
    op.kind = DrvKind::kRelease;
    op.addr = it->second.va;
    op.size = static_cast<size_t>(it->second.pages * d->cfg.chunk_bytes);
    d->enqueue(op);
    d->kick();
  }
  d->reserved_bytes -= it->second.pages * d->cfg.chunk_bytes;
  d->ranges.erase(it);
  d->log_call(VT_OP_RELEASE_ADDRESS, base, 0, 0, 0);
  return VT_OK;
}

// device.py:259-268
int vt_destroy_chunk(vt_device* d, int64_t id) {
  auto it = d->handles.find(id);
  if (it == d->handles.end())
    return d->fail(VT_E_STALE_HANDLE,
                   "handle " + std::to_string(id) + " was destroyed or never created");
  if (it->second != 0)
    return d->fail(VT_E_CHUNK_STILL_MAPPED, "handle " + std::to_string(id) + " still mapped " +
                                                std::to_string(it->second) + " times");
  d->handles.erase(it);
  // An imported chunk's release drops this device's reference only; it is not
  // one of the reference's device ops, so it stays out of the call log.
  const bool imported = d->imported.erase(id) != 0;
  if (!imported) d->log_call(VT_OP_DESTROY_CHUNK, 0, 0, id, 0);
  if (d->is_cuda()) {
    DrvOp op{};
    op.kind = DrvKind::kDestroy;
    op.handle_id = id;
    op.imported = imported;
    d->enqueue(op);
    d->kick();
  }
  return VT_OK;
}

int vt_dev_set_shareable(vt_device* d, int enabled) {
  if (!d->is_cuda()) return enabled ? d->fail(VT_E_ARG, "a simulated device has no shareable chunks")
                                    : VT_OK;
  if (enabled && !driver().ExportShareable)
    return d->fail(VT_E_CUDA, "driver lacks cuMemExportToShareableHandle");
  // Applies to chunks created from now on (the worker reads prop when it
  // executes a create; ops already queued keep the old setting only if they
  // ran before this call, so drain first).
  vt_wait(d, vt_ticket(d));
  d->drain_reserve();  // pre-created handles carry the old allocation properties
  d->prop.requestedHandleTypes =
      enabled ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR : CU_MEM_HANDLE_TYPE_NONE;
  return VT_OK;
}

int vt_export_chunk(vt_device* d, int64_t id, int* fd_out) {
  if (!d->is_cuda()) return d->fail(VT_E_ARG, "a simulated device has no shareable chunks");
  if (!driver().ExportShareable) return d->fail(VT_E_CUDA, "driver lacks cuMemExportToShareableHandle");
  if (d->handles.find(id) == d->handles.end())
    return d->fail(VT_E_STALE_HANDLE,
                   "handle " + std::to_string(id) + " was destroyed or never created");
  *fd_out = -1;
  DrvOp op{};
  op.kind = DrvKind::kExport;
  op.handle_id = id;
  op.fd_out = fd_out;
  d->enqueue(op);
  d->kick();
  const int rc = vt_wait(d, vt_ticket(d));  // the fd is needed now
  if (rc) return rc;
  return *fd_out >= 0 ? VT_OK : d->fail(VT_E_CUDA, "export produced no handle");
}

int vt_import_chunk(vt_device* d, int fd, int64_t* id_out) {
  if (!d->is_cuda()) return d->fail(VT_E_ARG, "a simulated device cannot import chunks");
  if (!driver().ImportShareable)
    return d->fail(VT_E_CUDA, "driver lacks cuMemImportFromShareableHandle");
  if (fd < 0) return d->fail(VT_E_ARG, "invalid shareable handle");
  const int64_t h = d->next_handle++;
  d->handles.emplace(h, 0);
  d->imported.insert(h);
  DrvOp op{};
  op.kind = DrvKind::kImport;
  op.handle_id = h;
  op.fd = fd;
  d->enqueue(op);
  d->kick();
  *id_out = h;
  return VT_OK;
}

int vt_chunk_is_imported(const vt_device* d, int64_t id) {
  return d->imported.count(id) ? 1 : 0;
}

// device.py:166-174
int vt_set_active_requests(vt_device* d, int64_t n) {
  if (n < 0) return d->fail(VT_E_ARG, "active request count cannot be negative");
  const int64_t delta = (n - d->active_requests) * d->cfg.activation_bytes_per_request;
  if (delta > d->free_bytes())
    return d->fail(VT_E_OUT_OF_MEMORY,
                   "activation scratch for " + std::to_string(n) + " requests exceeds free memory");
  d->active_requests = n;
  return VT_OK;
}

int vt_get_stats(const vt_device* d, vt_stats* s) {
  s->created_bytes = d->created_bytes();
  s->reserved_virtual_bytes = d->reserved_bytes;
  s->mapped_page_count = d->mapped_pages;
  s->free_bytes = d->free_bytes();
  s->activation_bytes = d->activation_bytes();
  s->active_requests = d->active_requests;
  s->live_handles = static_cast<int64_t>(d->handles.size());
  s->live_ranges = static_cast<int64_t>(d->ranges.size());
  return VT_OK;
}

// device.py:272-283
int vt_resolve(const vt_device* d, int64_t base, int64_t page, int64_t* id) {
  auto* md = const_cast<vt_device*>(d);
  auto it = d->ranges.find(base);
  if (it == d->ranges.end())
    return md->fail(VT_E_UNKNOWN_RANGE, "range base " + std::to_string(base) + " is not reserved");
  const RangeState& rs = it->second;
  if (page < 0 || page >= rs.pages)
    return md->fail(VT_E_INDEX_OUT_OF_RANGE, "page " + std::to_string(page) +
                                                 " outside range of " + std::to_string(rs.pages) +
                                                 " pages");
  if (rs.slot[static_cast<size_t>(page)] < 0)
    return md->fail(VT_E_PAGE_NOT_MAPPED, "page " + std::to_string(page) + " of base " +
                                              std::to_string(base) + " is not mapped");
  *id = rs.slot[static_cast<size_t>(page)];
  return VT_OK;
}

int vt_handle_alive(const vt_device* d, int64_t id, int64_t* map_count) {
  auto it = d->handles.find(id);
  if (it == d->handles.end()) return VT_E_STALE_HANDLE;
  if (map_count) *map_count = it->second;
  return VT_OK;
}

int vt_live_handles(const vt_device* d, int64_t* ids, int64_t cap, int64_t* n) {
  int64_t k = 0;
  for (const auto& kv : d->handles) {
    if (k < cap) ids[k] = kv.first;
    ++k;
  }
  *n = k;
  return k <= cap ? VT_OK : VT_E_ARG;
}

int vt_live_ranges(const vt_device* d, int64_t* bases, int64_t* pages, int64_t cap, int64_t* n) {
  int64_t k = 0;
  for (const auto& kv : d->ranges) {
    if (k < cap) {
      bases[k] = kv.first;
      pages[k] = kv.second.pages;
    }
    ++k;
  }
  *n = k;
  return k <= cap ? VT_OK : VT_E_ARG;
}

// device.py:291-295
int vt_range_mappings(const vt_device* d, int64_t base, int64_t* pages_out, int64_t* ids_out,
                      int64_t cap, int64_t* n) {
  auto* md = const_cast<vt_device*>(d);
  auto it = d->ranges.find(base);
  if (it == d->ranges.end())
    return md->fail(VT_E_UNKNOWN_RANGE, "range base " + std::to_string(base) + " is not reserved");
  int64_t k = 0;
  const RangeState& rs = it->second;
  for (int64_t p = 0; p < rs.pages; ++p) {
    if (rs.slot[static_cast<size_t>(p)] < 0) continue;
    if (k < cap) {
      pages_out[k] = p;
      ids_out[k] = rs.slot[static_cast<size_t>(p)];
    }
    ++k;
  }
  *n = k;
  return k <= cap ? VT_OK : VT_E_ARG;
}

int64_t vt_call_log_len(const vt_device* d) { return static_cast<int64_t>(d->log.size()); }

int vt_call_log_read(const vt_device* d, int64_t from, vt_call* buf, int64_t cap, int64_t* n) {
  const int64_t total = static_cast<int64_t>(d->log.size());
  if (from < 0) from = 0;
  int64_t k = std::max<int64_t>(0, std::min<int64_t>(cap, total - from));
  if (k) std::memcpy(buf, d->log.data() + from, static_cast<size_t>(k) * sizeof(vt_call));
  *n = k;
  return VT_OK;
}

uint64_t vt_ticket(const vt_device* d) {
  auto* md = const_cast<vt_device*>(d);
  std::lock_guard<std::mutex> lk(md->mu);
  return d->next_ticket;
}

int vt_wait(vt_device* d, uint64_t ticket) {
  if (!d->is_cuda()) return VT_OK;
  if (d->done_ticket.load() < ticket) {
    std::unique_lock<std::mutex> lk(d->mu);
    d->cv_done.wait(lk, [&] { return d->done_ticket.load() >= ticket || d->drv_failed.load(); });
  }
  if (d->drv_failed.load()) {
    std::lock_guard<std::mutex> lk(d->mu);
    return d->fail(VT_E_CUDA, d->drv_error);
  }
  return VT_OK;
}

int vt_poll(const vt_device* d, uint64_t ticket, int* done) {
  *done = (!d->is_cuda() || d->done_ticket.load() >= ticket) ? 1 : 0;
  return d->drv_failed.load() ? VT_E_CUDA : VT_OK;
}

int vt_fence(vt_device* d, void* stream) {
  if (!d->is_cuda()) return VT_OK;
  CtxScope scope(d);
  Driver& drv = driver();
  // Route every fence through the one in-order fence stream: epoch e then
  // completes only after all earlier fences, whichever streams they named, so
  // a teardown op that waits for its own epoch also waits for every kernel
  // fenced before it. The worker may still wait on the ring slot being
  // re-recorded; that is safe because the later record completes no earlier.
  CUresult r = drv.EventRecord(d->fence_src, reinterpret_cast<CUstream>(stream));
  if (r == CUDA_SUCCESS) r = drv.StreamWaitEvent(d->fence_stream, d->fence_src, 0);
  if (r != CUDA_SUCCESS) return d->fail(VT_E_CUDA, "fence: " + cu_err(r));
  uint64_t e = d->fence_epoch + 1;
  r = drv.EventRecord(d->fence_events[e % kFenceRing], d->fence_stream);
  if (r != CUDA_SUCCESS) return d->fail(VT_E_CUDA, "cuEventRecord: " + cu_err(r));
  std::lock_guard<std::mutex> lk(d->mu);
  d->fence_epoch = e;
  return VT_OK;
}

int vt_set_async(vt_device* d, int enabled) {
  if (!d->is_cuda()) return VT_OK;
  if (!enabled) vt_wait(d, vt_ticket(d));  // drain before switching to inline
  {
    std::lock_guard<std::mutex> lk(d->mu);
    d->async = enabled != 0;
  }
  d->cv_work.notify_one();
  return VT_OK;
}

int vt_driver_stats_get(const vt_device* d, vt_driver_stats* out) {
  auto* md = const_cast<vt_device*>(d);
  {
    std::lock_guard<std::mutex> lk(md->stat_mu);
    *out = d->dstats;
  }
  std::lock_guard<std::mutex> lk(md->phys_mu);
  out->reserve_chunks = static_cast<int64_t>(d->reserve.size());
  out->driver_threads = d->driver_threads;
  return VT_OK;
}

int vt_set_driver_threads(vt_device* d, int threads) {
  if (threads < 1 || threads > 16) return d->fail(VT_E_ARG, "driver threads must be in 1..16");
  if (!d->is_cuda()) return VT_OK;
  vt_wait(d, vt_ticket(d));  // the pool is idle between batches once drained
  std::lock_guard<std::mutex> lk(d->mu);  // keeps the worker from starting a batch
  d->stop_pool();
  d->driver_threads = threads;
  d->start_pool(threads);
  return VT_OK;
}

int vt_set_phys_reserve(vt_device* d, int64_t chunks) {
  if (chunks < 0) return d->fail(VT_E_ARG, "reserve size cannot be negative");
  if (!d->is_cuda()) return VT_OK;
  {
    std::lock_guard<std::mutex> lk(d->phys_mu);
    d->reserve_target = chunks;
    while (static_cast<int64_t>(d->reserve.size()) > chunks) {
      driver().MemRelease(d->reserve.back());
      d->reserve.pop_back();
    }
  }
  DrvOp op{};
  op.kind = DrvKind::kFill;
  d->enqueue(op);
  d->kick();
  return VT_OK;
}

int vt_driver_latencies(vt_device* d, int32_t op, int64_t* ns_out, int64_t cap, int64_t* n,
                        int reset) {
  if (op < 0 || op > 7) return VT_E_ARG;
  std::lock_guard<std::mutex> lk(d->lat_mu);
  auto& v = d->lat[op];
  *n = static_cast<int64_t>(v.size());
  const int64_t k = std::min<int64_t>(cap, *n);
  if (k > 0 && ns_out) std::memcpy(ns_out, v.data(), static_cast<size_t>(k) * sizeof(int64_t));
  if (reset) v.clear();
  return VT_OK;
}

int vt_va(const vt_device* d, int64_t base, uint64_t* devptr) {
  auto it = d->ranges.find(base);
  if (it == d->ranges.end()) {
    auto* md = const_cast<vt_device*>(d);
    return md->fail(VT_E_UNKNOWN_RANGE, "range base " + std::to_string(base) + " is not reserved");
  }
  *devptr = static_cast<uint64_t>(it->second.va);
  return VT_OK;
}

int vt_encode_tensor_map(const vt_device* d, uint64_t global_addr, int rank, const uint64_t* dims,
                         const uint64_t* strides_bytes, const uint32_t* box, int swizzle_128b,
                         void* out128) {
  (void)d;
  Driver& drv = driver();
  if (!drv.loaded) return VT_E_CUDA;
  cuuint32_t estride[5] = {1, 1, 1, 1, 1};
  CUresult r = drv.TensorMapEncodeTiled(
      reinterpret_cast<CUtensorMap*>(out128), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
      static_cast<cuuint32_t>(rank), reinterpret_cast<void*>(global_addr),
      reinterpret_cast<const cuuint64_t*>(dims), reinterpret_cast<const cuuint64_t*>(strides_bytes),
      reinterpret_cast<const cuuint32_t*>(box), estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
      swizzle_128b ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? VT_OK : VT_E_CUDA;
}

}  // extern "C"
