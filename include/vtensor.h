/*
 * vtensor.h — C ABI of libvtensor.so, the vTensor device shim.
 *
 * This is the drop-in boundary for layer L0 of the reference (kvsim): every
 * entry point below replaces one method of
 * `kvsim.device.VirtualMemoryDevice` (/root/reference/pkg/src/kvsim/device.py).
 * The state machine (ordinals, accounting, call log, error classes) is
 * bit-exact with the reference; on a GPU the same calls additionally drive the
 * CUDA driver VMM API (cuMemAddressReserve / cuMemCreate / cuMemMap /
 * cuMemSetAccess / cuMemUnmap / cuMemRelease / cuMemAddressFree) on a
 * per-device worker thread, so chunk mapping overlaps running kernels.
 *
 * Conventions: plain C types only, every function returns a vt_status, nothing
 * throws across the ABI, one writer thread per device.
 */
#ifndef VTENSOR_H_
#define VTENSOR_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes: 1:1 with the DeviceError subclasses of device.py:18-55. */
typedef enum vt_status {
  VT_OK = 0,
  VT_E_INVALID_SIZE = 1,        /* InvalidSize          device.py:22 */
  VT_E_OUT_OF_MEMORY = 2,       /* DeviceOutOfMemory    device.py:26 */
  VT_E_PAGE_ALREADY_MAPPED = 3, /* PageAlreadyMapped    device.py:30 */
  VT_E_PAGE_NOT_MAPPED = 4,     /* PageNotMapped        device.py:34 */
  VT_E_STALE_HANDLE = 5,        /* StaleHandle          device.py:38 */
  VT_E_INDEX_OUT_OF_RANGE = 6,  /* IndexOutOfRange      device.py:42 */
  VT_E_RANGE_STILL_MAPPED = 7,  /* RangeStillMapped     device.py:46 */
  VT_E_UNKNOWN_RANGE = 8,       /* UnknownRange         device.py:50 */
  VT_E_CHUNK_STILL_MAPPED = 9,  /* ChunkStillMapped     device.py:54 */
  VT_E_CUDA = 10,               /* driver failure after the budget check: fatal */
  VT_E_ARG = 11,                /* contract misuse (ValueError in Python)       */
} vt_status;

/* Call-log op codes (device.py:184-187 op strings). */
typedef enum vt_op {
  VT_OP_RESERVE_ADDRESS = 0,
  VT_OP_CREATE_CHUNK = 1,
  VT_OP_MAP_PAGE = 2,
  VT_OP_UNMAP_PAGE = 3,
  VT_OP_RELEASE_ADDRESS = 4,
  VT_OP_DESTROY_CHUNK = 5,
} vt_op;

typedef struct vt_device vt_device;

/* DeviceConfig, device.py:93-109 (page size == chunk size). */
typedef struct vt_config {
  int64_t capacity_bytes;
  int64_t chunk_bytes;
  int64_t weights_bytes;
  int64_t activation_bytes_per_request;
} vt_config;

/* DeviceStats, device.py:75-80, plus the other accounting properties. */
typedef struct vt_stats {
  int64_t created_bytes;          /* device.py:141-143 */
  int64_t reserved_virtual_bytes; /* device.py:145-147 (kept incrementally) */
  int64_t mapped_page_count;
  int64_t free_bytes;             /* device.py:153-160 */
  int64_t activation_bytes;       /* device.py:149-151 */
  int64_t active_requests;
  int64_t live_handles;
  int64_t live_ranges;
} vt_stats;

/* DeviceCall, device.py:83-90, in structured form (detail is formatted by the
 * caller from base/page/handle/pages exactly as device.py:203,215,233,244,257,268). */
typedef struct vt_call {
  int64_t seq;
  int32_t op; /* vt_op */
  int32_t _pad;
  int64_t base;
  int64_t page;
  int64_t handle;
  int64_t pages;
  int64_t created_bytes_after;
} vt_call;

/* Driver-side latency accounting (submit -> completed on the worker). */
typedef struct vt_driver_stats {
  int64_t ops_completed;
  int64_t map_calls, unmap_calls, create_calls, destroy_calls, access_calls;
  int64_t map_ns_total, unmap_ns_total, create_ns_total, destroy_ns_total;
  int64_t access_ns_total; /* cuMemSetAccess share of map_ns_total */
  int64_t fence_waits, fence_wait_ns_total;
  int64_t max_op_ns;
  int64_t reserve_hits;   /* creates served from the pre-created reserve */
  int64_t reserve_chunks; /* handles in the reserve now */
  int64_t driver_threads; /* threads executing driver ops in parallel */
} vt_driver_stats;

/* ---- lifetime ------------------------------------------------------------
 * cuda_ordinal < 0  : simulated backend (the reference's in-process device).
 * cuda_ordinal >= 0 : CUDA driver VMM backend on that device; chunk_bytes must
 *                     be a multiple of the allocation granularity (2 MiB). */
int vt_dev_open(const vt_config* cfg, int cuda_ordinal, vt_device** out);
int vt_dev_close(vt_device* dev);
int vt_dev_is_cuda(const vt_device* dev);
const char* vt_last_error(const vt_device* dev);

/* ---- primitives (device.py:191-268) -------------------------------------- */
int vt_reserve(vt_device* dev, int64_t size_bytes, int64_t* base, int64_t* pages);
int vt_create_chunk(vt_device* dev, int64_t* handle_id);
int vt_map_page(vt_device* dev, int64_t base, int64_t page, int64_t handle_id);
int vt_unmap_page(vt_device* dev, int64_t base, int64_t page, int64_t* handle_id);
int vt_release(vt_device* dev, int64_t base);
int vt_destroy_chunk(vt_device* dev, int64_t handle_id);

/* Cross-device chunk sharing (extends the rTree hard
 * link of kvsim/scheduler.py:128-130 across pools — no reference counterpart).
 * vt_dev_set_shareable: opt in (off by default: shareable allocations cost
 *   more per cuMemCreate) — chunks created afterwards can be exported.
 * vt_export_chunk: a POSIX file descriptor for a live chunk of a CUDA device
 *   (cuMemExportToShareableHandle); blocks until the chunk exists. The caller
 *   owns the fd (send it to another process with SCM_RIGHTS, or import it).
 * vt_import_chunk: takes ownership of fd (closed after the import) and
 *   returns a new handle ordinal of this device naming the same physical
 *   memory (cuMemImportFromShareableHandle). It maps like a local chunk — on
 *   another GPU the mapping's cuMemSetAccess grants this device peer access
 *   over NVLink — but it is not counted in created_bytes / the budget, and
 *   neither the import nor its destroy (= dropping this reference) enters the
 *   call log. Simulated devices return VT_E_ARG. */
int vt_dev_set_shareable(vt_device* dev, int enabled); /* chunks created afterwards are exportable */
int vt_export_chunk(vt_device* dev, int64_t handle_id, int* fd_out);
int vt_import_chunk(vt_device* dev, int fd, int64_t* handle_id_out);
int vt_chunk_is_imported(const vt_device* dev, int64_t handle_id);

/* Batched forms used by VTO map_chunks / _unmap_tail (ops.py:133-146,171-178):
 * identical call-log entries to the per-page loop; stop at the first error and
 * report how many pages were processed in *n_done. */
int vt_map_pages(vt_device* dev, int64_t base, int64_t first_page,
                 const int64_t* handle_ids, int64_t n, int64_t* n_done);
int vt_unmap_tail(vt_device* dev, int64_t base, int64_t from_page_inclusive,
                  int64_t down_to_inclusive, int64_t* handle_ids_out, int64_t* n_done);

/* One scheduler extend in one call (scheduler.py:166-180: ops.py:83-112 p_alloc
 * then ops.py:133-146 map_chunks): creates n_create chunks (ids written to
 * created_ids), then maps the n_reuse parked handles followed by the created
 * ones at pages first_page.. of the range. Call log = create_chunk x n_create,
 * then map_page per page, exactly as the two-op sequence; the driver work is
 * queued with one worker wake-up. All-or-nothing: on any error nothing
 * changed (the caller then runs the per-op sequence, which reproduces the
 * reference's partial-failure behaviour). */
int vt_extend(vt_device* dev, int64_t base, int64_t first_page, const int64_t* reuse_ids,
              int64_t n_reuse, int64_t n_create, int64_t* created_ids);

/* ---- accounting / inspection (device.py:141-187, 272-295) ---------------- */
int vt_set_active_requests(vt_device* dev, int64_t n);
int vt_get_stats(const vt_device* dev, vt_stats* out);
int vt_resolve(const vt_device* dev, int64_t base, int64_t page, int64_t* handle_id);
int vt_handle_alive(const vt_device* dev, int64_t handle_id, int64_t* map_count);
int vt_live_handles(const vt_device* dev, int64_t* ids, int64_t cap, int64_t* n);
int vt_live_ranges(const vt_device* dev, int64_t* bases, int64_t* pages, int64_t cap, int64_t* n);
int vt_range_mappings(const vt_device* dev, int64_t base, int64_t* pages_out,
                      int64_t* ids_out, int64_t cap, int64_t* n);
int64_t vt_call_log_len(const vt_device* dev);
int vt_call_log_read(const vt_device* dev, int64_t from, vt_call* buf, int64_t cap, int64_t* n);

/* ---- async driver execution (SPEC.md:303-304 completion-token contract) ---
 * Every driver op is queued in issue order; vt_ticket() is the ticket of the
 * latest one. vt_wait() blocks (GIL released by the caller) until the worker
 * has executed everything up to the ticket. vt_fence() records an event on a
 * CUDA stream; unmap/destroy/release ops submitted afterwards wait for it, so
 * pages are never torn down under a kernel that still reads them. */
uint64_t vt_ticket(const vt_device* dev);
int vt_wait(vt_device* dev, uint64_t ticket);
int vt_poll(const vt_device* dev, uint64_t ticket, int* done);
int vt_fence(vt_device* dev, void* cuda_stream);
int vt_set_async(vt_device* dev, int enabled);
int vt_driver_stats_get(const vt_device* dev, vt_driver_stats* out);
/* Driver-op parallelism (no reference counterpart: the reference's device is
 * in-process and instantaneous, device.py:118-295). Each queued batch runs
 * as maximal same-kind segments in issue order; the ops of one segment are
 * independent and run on `threads` threads (default 1, env VT_DRIVER_THREADS).
 * Several threads multiply the mapping rate on an idle GPU (tools/vmm_probe.cu)
 * but, under the decode stream, concurrent map/SetAccess calls serialise in
 * the driver and starve the launching thread, so serving runs
 * with one. Blocks until queued work has drained. */
int vt_set_driver_threads(vt_device* dev, int threads);
/* Physical-handle reserve: keep up to `chunks` cuMemCreate'd handles that are
 * not (yet) logical chunks. A logical create_chunk takes one from the reserve
 * instead of calling cuMemCreate on the extend path, and a destroyed chunk's
 * memory refills it while it is short. Purely physical: the call log, byte
 * accounting and every manager decision are unchanged (the reserve is HBM the
 * budget does not see — size it inside the headroom between the configured
 * capacity and the device). Queues a fill: vt_wait(vt_ticket()) returns once
 * it is full. 0 releases it. */
int vt_set_phys_reserve(vt_device* dev, int64_t chunks);
/* Submit -> completed latency (ns) of every driver op of kind `op` (a vt_op
 * code: create/map/unmap/destroy/release) completed since the last reset;
 * copies up to `cap` samples, *n = total available. reset != 0 clears. This
 * is the "vTensor extend latency" distribution (p50/p99) for maps. op 6 / 7:
 * the duration of each raw cuMemMap / cuMemSetAccess call the worker made. */
int vt_driver_latencies(vt_device* dev, int32_t op, int64_t* ns_out, int64_t cap, int64_t* n,
                        int reset);

/* Device virtual address of a reserved range (CUdeviceptr), valid while the
 * range is reserved; 0 on the simulated backend. */
int vt_va(const vt_device* dev, int64_t base, uint64_t* devptr);

/* TMA descriptor for a reserved range (cuTensorMapEncodeTiled, 128 bytes),
 * written to out128. Fixed for the range's life: the VA never moves. */
int vt_encode_tensor_map(const vt_device* dev, uint64_t global_addr, int rank,
                         const uint64_t* dims, const uint64_t* strides_bytes,
                         const uint32_t* box, int swizzle_128b, void* out128);

#ifdef __cplusplus
}
#endif
#endif /* VTENSOR_H_ */
