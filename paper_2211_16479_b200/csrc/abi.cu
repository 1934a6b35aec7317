// abi.cu -- the C ABI of include/msort.h: argument validation, dtype
// dispatch, workspace handling, error text and kernel accounting.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "msort_internal.h"
#include "plan.cuh"

namespace msort {

msort_status dist_nccl(const void* in_keys, const void* in_vals, void* keys, void* vals, size_t n,
                       msort_dtype kd, msort_dtype vd, msort_comm_s* comm, void* ws,
                       cudaStream_t s, int64_t* split_out);
msort_status tree_nccl(const void* in_keys, const void* in_vals, size_t n, msort_dtype kd,
                       msort_dtype vd, msort_comm_s* comm, void* root_k, void* root_v,
                       size_t root_cap, cudaStream_t s, int64_t* total_out);
msort_status dist_emulated(void* const* keys, void* const* vals, const size_t* n, int world,
                           msort_dtype kd, msort_dtype vd, void* const* ws, cudaStream_t s,
                           int64_t* split_out);
msort_status comm_unique_id(void* out);
msort_status comm_init(const void* idp, int rank, int world, msort_comm_s** out);
msort_status comm_destroy(msort_comm_s* c);
msort_status comm_wrap(void* nccl_comm, msort_comm_s** out);
msort_status comm_reserve(msort_comm_s* c, size_t n_max, msort_dtype kd, msort_dtype vd,
                          cudaStream_t s);
int comm_world(msort_comm_s* c);

// ---------------------------------------------------------------- errors
static thread_local std::string g_last_error;
void set_error(const std::string& s) { g_last_error = s; }
msort_status cuda_fail(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  if (e == cudaErrorMemoryAllocation) return MSORT_ERROR_OUT_OF_MEMORY;
  return MSORT_ERROR_CUDA;
}

// ------------------------------------------------------ kernel accounting
static std::atomic<int64_t> g_launches{0};
static std::atomic<int> g_profile{0};
struct EventRec {
  cudaEvent_t a, b;
  KernelClass kc;
};
static std::mutex g_prof_mu;
static std::vector<EventRec> g_pending;
static std::vector<cudaEvent_t> g_free_events;
static int64_t g_prof_launches[MSORT_PROFILE_CLASSES];
static double g_prof_ms[MSORT_PROFILE_CLASSES];

static cudaEvent_t get_event() {
  if (!g_free_events.empty()) {
    cudaEvent_t e = g_free_events.back();
    g_free_events.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

LaunchScope::LaunchScope(KernelClass k, cudaStream_t st) : kc(k), s(st), slot(-1) {
  if (k != KC_NCCL && k != KC_EXCHANGE) g_launches.fetch_add(1, std::memory_order_relaxed);
  if (g_profile.load(std::memory_order_relaxed)) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    EventRec r{get_event(), get_event(), kc};
    cudaEventRecord(r.a, s);
    g_pending.push_back(r);
    slot = (int)g_pending.size() - 1;
  }
}
LaunchScope::~LaunchScope() {
  if (slot >= 0) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEventRecord(g_pending[slot].b, s);
  }
}

// The library's own stream-ordered pool, one per device (created on first
// use).  Its release threshold is raised so freed blocks stay reserved for
// the next call; the device's default pool -- which torch and the host
// application may use -- is never touched.
static std::mutex g_pool_mu;
static cudaMemPool_t g_pool[64] = {};
static cudaError_t library_pool(int dev, cudaMemPool_t* out) {
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!g_pool[dev]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool;
    cudaError_t e = cudaMemPoolCreate(&pool, &props);
    if (e != cudaSuccess) return e;
    uint64_t keep = ~0ull;
    e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    if (e != cudaSuccess) {
      cudaMemPoolDestroy(pool);
      return e;
    }
    g_pool[dev] = pool;
  }
  *out = g_pool[dev];
  return cudaSuccess;
}

cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  cudaMemPool_t pool;
  e = library_pool(dev, &pool);
  if (e != cudaSuccess) return e;
  return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

// ------------------------------------------------------------- helpers
size_t dtype_size(msort_dtype d) {
  switch (d) {
    case MSORT_INT32:
    case MSORT_UINT32: return 4;
    case MSORT_INT64:
    case MSORT_UINT64: return 8;
    default: return 0;
  }
}

static size_t single_ws_bytes_w(size_t n, msort_dtype kd, msort_dtype vd);
size_t single_ws_bytes(size_t n, msort_dtype kd, msort_dtype vd) {
  if (dtype_size(kd) != 8) return single_ws_bytes_w(n, kd, vd);
  // 8-byte keys: room for the key-range narrowed sort too (sort_narrowed:
  // 32-bit keys + the 4-byte sort's workspace, overlapping the 8-byte sort's)
  // and the range itself in the last 256 bytes
  const size_t nar = align_up(n * 4, 256) + single_ws_bytes_w(n, MSORT_UINT32, vd);
  return std::max(single_ws_bytes_w(n, kd, vd), nar) + 256;
}
static size_t single_ws_bytes_w(size_t n, msort_dtype kd, msort_dtype vd) {
  const int T = tile_size_for(kd, vd);
  size_t b = align_up(n * dtype_size(kd), 256);
  if (vd != MSORT_NONE) b += align_up(n * 4, 256);
  // partitions: one per output tile (+ slack for the k-way merge's extra tiles)
  b += align_up((n / (size_t)T + 2 + 2 * 64) * sizeof(int64_t), 256);
  // 4-way pass segment boundaries (4 x int64 each)
  size_t q = align_up((2 * (n / (size_t)T) + 64) * 4 * sizeof(int64_t), 256);
  if (dtype_size(kd) == 4 && vd == MSORT_NONE) {
    // K6 partition (Kernels::k6_*): unit states (32 B) and tiles (72 B) per
    // unit, cut records (16 B) and piece tiles (72 B) per piece, a counter
    const size_t nu = n / 3998 + n / (4 * (size_t)T) + 2, ex = n / 4568 + nu + 1;
    q = std::max(q, align_up(32 * nu, 256) + align_up(72 * nu, 256) + align_up(16 * ex, 256) +
                        align_up(72 * ex, 256) + 256);
  }
  return b + q;
}

static msort_status check_device() {
  int major = 0, minor = 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  // cache per device id (small fixed table; one atomic word per device:
  // 0 = unknown, else 1 + major * 64 + minor -- calls may come from many threads)
  static std::atomic<int> cached[64];
  const int c = dev < 64 ? cached[dev].load(std::memory_order_acquire) : 0;
  if (c) {
    major = (c - 1) / 64;
    minor = (c - 1) % 64;
  } else {
    int ma = 0, mi = 0;
    e = cudaDeviceGetAttribute(&ma, cudaDevAttrComputeCapabilityMajor, dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&mi, cudaDevAttrComputeCapabilityMinor, dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    major = ma, minor = mi;
    if (dev < 64) cached[dev].store(1 + major * 64 + minor, std::memory_order_release);
  }
  if (major != 10 || minor != 0) {
    set_error("device is sm_" + std::to_string(major) + std::to_string(minor) +
              "; this library is built for sm_100a (B200) only");
    return MSORT_ERROR_NOT_SUPPORTED;
  }
  return MSORT_SUCCESS;
}

static bool overlaps(const void* a, size_t na, const void* b, size_t nb) {
  const char* x = (const char*)a;
  const char* y = (const char*)b;
  return x < y + nb && y < x + na;
}

static msort_status validate(void* keys, void* vals, size_t n, msort_dtype kd, msort_dtype vd,
                             bool allow_null_ok) {
  const size_t wk = dtype_size(kd);
  if (!wk) {
    set_error("unknown key dtype");
    return MSORT_ERROR_INVALID_VALUE;
  }
  if (vd != MSORT_NONE && vd != MSORT_UINT32 && vd != MSORT_INT32) {
    if (dtype_size(vd)) {
      set_error("only 4-byte payloads are built");
      return MSORT_ERROR_NOT_SUPPORTED;
    }
    set_error("unknown value dtype");
    return MSORT_ERROR_INVALID_VALUE;
  }
  if (n > (size_t(1) << 40)) {
    set_error("n > 2^40");
    return MSORT_ERROR_INVALID_VALUE;
  }
  if (n > 0 && !keys && !allow_null_ok) {
    set_error("keys is NULL");
    return MSORT_ERROR_INVALID_VALUE;
  }
  if (n > 0 && vd != MSORT_NONE && !vals) {
    set_error("vals is NULL");
    return MSORT_ERROR_INVALID_VALUE;
  }
  if (((uintptr_t)keys) % wk) {
    set_error("keys not aligned to its element size");
    return MSORT_ERROR_INVALID_VALUE;
  }
  if (vd != MSORT_NONE && ((uintptr_t)vals) % 4) {
    set_error("vals not aligned to 4 bytes");
    return MSORT_ERROR_INVALID_VALUE;
  }
  if (vd != MSORT_NONE && n > 0 && overlaps(keys, n * wk, vals, n * 4)) {
    set_error("keys and vals overlap");
    return MSORT_ERROR_INVALID_VALUE;
  }
  return MSORT_SUCCESS;
}

static msort_status validate_ws(void* keys, void* vals, size_t n, msort_dtype kd, msort_dtype vd,
                                void* ws, size_t ws_bytes, size_t need) {
  if (ws_bytes < need) {
    set_error("workspace too small: need " + std::to_string(need) + " bytes");
    return MSORT_ERROR_INVALID_VALUE;
  }
  if (!ws || ((uintptr_t)ws) % 256) {
    set_error("workspace NULL or not 256-byte aligned");
    return MSORT_ERROR_INVALID_VALUE;
  }
  if (overlaps(ws, ws_bytes, keys, n * dtype_size(kd)) ||
      (vd != MSORT_NONE && overlaps(ws, ws_bytes, vals, n * 4))) {
    set_error("workspace overlaps keys/vals");
    return MSORT_ERROR_INVALID_VALUE;
  }
  return MSORT_SUCCESS;
}

static msort_status sort_alloc(void* keys, void* vals, size_t n, msort_dtype kd, msort_dtype vd,
                               cudaStream_t s) {
  MSORT_TRY(validate(keys, vals, n, kd, vd, false));
  if (n < 2) return MSORT_SUCCESS;  // "less than two elements, return"
  MSORT_TRY(check_device());
  size_t need = single_ws_bytes(n, kd, vd);
  void* ws = nullptr;
  MSORT_CUDA_TRY(scratch_alloc(&ws, need, s));
  msort_status st = sort_single_dispatch(keys, vals, keys, vals, n, kd, vd, ws, need, s);
  cudaError_t e = cudaFreeAsync(ws, s);
  if (st != MSORT_SUCCESS) return st;
  if (e != cudaSuccess) return cuda_fail(e, "cudaFreeAsync");
  return MSORT_SUCCESS;
}

}  // namespace msort

using namespace msort;

extern "C" {

msort_status msort_sort(void* keys, size_t n, msort_dtype key_dtype, msort_stream_t stream) {
  return sort_alloc(keys, nullptr, n, key_dtype, MSORT_NONE, (cudaStream_t)stream);
}

msort_status msort_sort_pairs(void* keys, void* vals, size_t n, msort_dtype key_dtype,
                              msort_dtype val_dtype, msort_stream_t stream) {
  if (val_dtype == MSORT_NONE) {
    set_error("msort_sort_pairs needs a payload dtype");
    return MSORT_ERROR_INVALID_VALUE;
  }
  return sort_alloc(keys, vals, n, key_dtype, val_dtype, (cudaStream_t)stream);
}

msort_status msort_workspace_bytes(size_t n, msort_dtype key_dtype, msort_dtype val_dtype,
                                   int world, size_t* bytes) {
  if (!bytes || !dtype_size(key_dtype) ||
      (val_dtype != MSORT_NONE && val_dtype != MSORT_UINT32 && val_dtype != MSORT_INT32) ||
      world < 1) {
    set_error("bad argument to msort_workspace_bytes");
    return MSORT_ERROR_INVALID_VALUE;
  }
  *bytes = world <= 1 ? single_ws_bytes(n, key_dtype, val_dtype)
                      : dist_ws_bytes(n, key_dtype, val_dtype, world);
  return MSORT_SUCCESS;
}

static size_t seg_ws_bytes(size_t n, size_t nseg, msort_dtype kd, msort_dtype vd) {
  // Kernels::sort_segmented: ping-pong keys (+ vals) for the segments longer
  // than a tile T; the uploaded tables (<= 2 words per short segment, 2 per
  // K1 tile of a long one, 3.5 + 1 per long segment); the merge completion
  // counters (<= 48 levels x merge tiles, Tm >= T/2); the chunk counter.
  const size_t T = (size_t)tile_size_for(kd, vd);
  const size_t tiles = n / T + 1;
  size_t b = align_up(n * dtype_size(kd), 256);
  if (vd != MSORT_NONE) b += align_up(n * 4, 256);
  b += align_up(8 * (8 * nseg + 2 * tiles + 8), 256);  // host tables (mid bins included)
  b += align_up(8 * (nseg + 1), 256);  // a long host offsets table, uploaded
  // device-resident offsets: the classifier's lists (<= n / 257, n / 2177,
  // n / (T + 1) entries of 16 bytes) and counters
  b += align_up(16 * (n / 33 + 1), 256) + align_up(16 * (n / 257 + 1), 256) +
       align_up(16 * (n / 2177 + 1), 256) + align_up(16 * (n / (T + 1) + 1), 256) + 256;
  b += align_up(4 * 48 * (2 * tiles + nseg), 256);
  return b + 256 + 1024;
}

msort_status msort_segmented_workspace_bytes(size_t n, size_t nseg, msort_dtype key_dtype,
                                             msort_dtype val_dtype, size_t* bytes) {
  if (!bytes || !dtype_size(key_dtype) ||
      (val_dtype != MSORT_NONE && val_dtype != MSORT_UINT32 && val_dtype != MSORT_INT32)) {
    set_error("bad argument to msort_segmented_workspace_bytes");
    return MSORT_ERROR_INVALID_VALUE;
  }
  *bytes = seg_ws_bytes(n, nseg, key_dtype, val_dtype);
  return MSORT_SUCCESS;
}

msort_status msort_sort_segmented(void* keys, void* vals, size_t n, const int64_t* seg_offsets,
                                  size_t nseg, msort_dtype key_dtype, msort_dtype val_dtype,
                                  void* ws, size_t ws_bytes, msort_stream_t stream) {
  MSORT_TRY(validate(keys, vals, n, key_dtype, val_dtype, false));
  if (!seg_offsets) {
    set_error("seg_offsets is NULL");
    return MSORT_ERROR_INVALID_VALUE;
  }
  // where the table lives: device memory is classified (and checked) on the
  // device; anything else is read here
  bool dev_off = false;
  {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, seg_offsets) == cudaSuccess)
      dev_off = pa.type == cudaMemoryTypeDevice;
    (void)cudaGetLastError();
  }
  if (!dev_off) {
    if (seg_offsets[0] != 0 || seg_offsets[nseg] != (int64_t)n) {
      set_error("seg_offsets must start at 0 and end at n");
      return MSORT_ERROR_INVALID_VALUE;
    }
    for (size_t i = 0; i < nseg; ++i)
      if (seg_offsets[i + 1] < seg_offsets[i]) {
        set_error("seg_offsets decrease at segment " + std::to_string(i));
        return MSORT_ERROR_INVALID_VALUE;
      }
  }
  if (n < 2 || nseg == 0) return MSORT_SUCCESS;
  MSORT_TRY(check_device());
  MSORT_TRY(validate_ws(keys, vals, n, key_dtype, val_dtype, ws, ws_bytes,
                        seg_ws_bytes(n, nseg, key_dtype, val_dtype)));
  return sort_segmented_dispatch(keys, vals, seg_offsets, nseg, dev_off, n, key_dtype, val_dtype,
                                 ws, ws_bytes, (cudaStream_t)stream);
}

msort_status msort_sort_ws(void* keys, void* vals, size_t n, msort_dtype key_dtype,
                           msort_dtype val_dtype, void* ws, size_t ws_bytes,
                           msort_stream_t stream) {
  MSORT_TRY(validate(keys, vals, n, key_dtype, val_dtype, false));
  if (n < 2) return MSORT_SUCCESS;
  MSORT_TRY(check_device());
  MSORT_TRY(validate_ws(keys, vals, n, key_dtype, val_dtype, ws, ws_bytes,
                        single_ws_bytes(n, key_dtype, val_dtype)));
  return sort_single_dispatch(keys, vals, keys, vals, n, key_dtype, val_dtype, ws, ws_bytes,
                              (cudaStream_t)stream);
}

static msort_status validate_out(const void* ik, const void* iv, void* ok, void* ov, size_t n,
                                 msort_dtype kd, msort_dtype vd) {
  MSORT_TRY(validate(ok, ov, n, kd, vd, false));
  MSORT_TRY(validate(const_cast<void*>(ik), const_cast<void*>(iv), n, kd, vd, false));
  const size_t wk = dtype_size(kd);
  // the input may be the output (in place) but must not partially overlap it
  if (ik != ok && n > 0 && overlaps(ik, n * wk, ok, n * wk)) {
    set_error("input and output keys partially overlap");
    return MSORT_ERROR_INVALID_VALUE;
  }
  if (vd != MSORT_NONE && iv != ov && n > 0 && overlaps(iv, n * 4, ov, n * 4)) {
    set_error("input and output vals partially overlap");
    return MSORT_ERROR_INVALID_VALUE;
  }
  return MSORT_SUCCESS;
}

msort_status msort_sort_out_ws(const void* in_keys, const void* in_vals, void* keys_out,
                               void* vals_out, size_t n, msort_dtype key_dtype,
                               msort_dtype val_dtype, void* ws, size_t ws_bytes,
                               msort_stream_t stream) {
  MSORT_TRY(validate_out(in_keys, in_vals, keys_out, vals_out, n, key_dtype, val_dtype));
  if (n == 0) return MSORT_SUCCESS;
  MSORT_TRY(check_device());
  if (n >= 2)
    MSORT_TRY(validate_ws(keys_out, vals_out, n, key_dtype, val_dtype, ws, ws_bytes,
                          single_ws_bytes(n, key_dtype, val_dtype)));
  return sort_single_dispatch(in_keys, in_vals, keys_out, vals_out, n, key_dtype, val_dtype, ws,
                              ws_bytes, (cudaStream_t)stream);
}

msort_status msort_sort_host(const void* host_keys, const void* host_vals, void* host_keys_out,
                             void* host_vals_out, size_t n, msort_dtype key_dtype,
                             msort_dtype val_dtype, void* dev_keys, void* dev_vals, void* ws,
                             size_t ws_bytes, msort_stream_t stream) {
  if (n == 0) return MSORT_SUCCESS;
  const bool pairs = val_dtype != MSORT_NONE;
  if (!host_keys || !host_keys_out || (pairs && (!host_vals || !host_vals_out))) {
    set_error("msort_sort_host: NULL host pointer");
    return MSORT_ERROR_INVALID_VALUE;
  }
  MSORT_TRY(validate_out(dev_keys, pairs ? dev_vals : nullptr, dev_keys,
                         pairs ? dev_vals : nullptr, n, key_dtype, val_dtype));
  MSORT_TRY(check_device());
  if (n >= 2)
    MSORT_TRY(validate_ws(dev_keys, pairs ? dev_vals : nullptr, n, key_dtype, val_dtype, ws,
                          ws_bytes, single_ws_bytes(n, key_dtype, val_dtype)));
  cudaStream_t s = (cudaStream_t)stream;
  const size_t kb = n * dtype_size(key_dtype);
  MSORT_CUDA_TRY(cudaMemcpyAsync(dev_keys, host_keys, kb, cudaMemcpyHostToDevice, s));
  if (pairs) MSORT_CUDA_TRY(cudaMemcpyAsync(dev_vals, host_vals, n * 4, cudaMemcpyHostToDevice, s));
  MSORT_TRY(sort_single_dispatch(dev_keys, pairs ? dev_vals : nullptr, dev_keys,
                                 pairs ? dev_vals : nullptr, n, key_dtype, val_dtype, ws, ws_bytes,
                                 s));
  MSORT_CUDA_TRY(cudaMemcpyAsync(host_keys_out, dev_keys, kb, cudaMemcpyDeviceToHost, s));
  if (pairs)
    MSORT_CUDA_TRY(cudaMemcpyAsync(host_vals_out, dev_vals, n * 4, cudaMemcpyDeviceToHost, s));
  return MSORT_SUCCESS;
}

msort_status msort_merge_runs_workspace_bytes(size_t n, int p, msort_dtype key_dtype,
                                              msort_dtype val_dtype, size_t* bytes) {
  if (!bytes || !dtype_size(key_dtype) || p < 1 ||
      (val_dtype != MSORT_NONE && val_dtype != MSORT_UINT32 && val_dtype != MSORT_INT32)) {
    set_error("bad argument to msort_merge_runs_workspace_bytes");
    return MSORT_ERROR_INVALID_VALUE;
  }
  *bytes = merge_runs_ws_bytes(n, p, key_dtype, val_dtype);
  return MSORT_SUCCESS;
}

msort_status msort_merge_runs(const void* in_keys, const void* in_vals,
                              const int64_t* run_offsets, int p, void* keys_out, void* vals_out,
                              msort_dtype key_dtype, msort_dtype val_dtype, void* ws,
                              size_t ws_bytes, msort_stream_t stream) {
  if (!run_offsets || p < 1 || p > 128) {
    set_error("msort_merge_runs: run_offsets NULL or p outside [1, 128]");
    return MSORT_ERROR_INVALID_VALUE;
  }
  if (run_offsets[0] != 0) {
    set_error("msort_merge_runs: run_offsets[0] must be 0");
    return MSORT_ERROR_INVALID_VALUE;
  }
  for (int j = 0; j < p; ++j)
    if (run_offsets[j + 1] < run_offsets[j]) {
      set_error("msort_merge_runs: run_offsets decrease at run " + std::to_string(j));
      return MSORT_ERROR_INVALID_VALUE;
    }
  const size_t n = (size_t)run_offsets[p];
  MSORT_TRY(validate_out(in_keys, in_vals, keys_out, vals_out, n, key_dtype, val_dtype));
  const size_t wk = dtype_size(key_dtype);
  if (n > 0 && (overlaps(in_keys, n * wk, keys_out, n * wk) ||
                (val_dtype != MSORT_NONE && overlaps(in_vals, n * 4, vals_out, n * 4)))) {
    set_error("msort_merge_runs: input and output overlap (the merge is out of place)");
    return MSORT_ERROR_INVALID_VALUE;
  }
  if (n == 0) return MSORT_SUCCESS;
  MSORT_TRY(check_device());
  MSORT_TRY(validate_ws(keys_out, vals_out, n, key_dtype, val_dtype, ws, ws_bytes,
                        merge_runs_ws_bytes(n, p, key_dtype, val_dtype)));
  if (overlaps(ws, ws_bytes, in_keys, n * wk) ||
      (val_dtype != MSORT_NONE && overlaps(ws, ws_bytes, in_vals, n * 4))) {
    set_error("workspace overlaps the input");
    return MSORT_ERROR_INVALID_VALUE;
  }
  return merge_runs_dispatch(in_keys, in_vals, run_offsets, p, keys_out, vals_out, key_dtype,
                             val_dtype, ws, ws_bytes, (cudaStream_t)stream);
}

msort_status msort_comm_unique_id(void* id_out) {
  if (!id_out) {
    set_error("id_out is NULL");
    return MSORT_ERROR_INVALID_VALUE;
  }
  return comm_unique_id(id_out);
}

msort_status msort_comm_init(const void* id, int rank, int world, msort_comm_t* out) {
  if (!id || !out || world < 1 || rank < 0 || rank >= world) {
    set_error("bad argument to msort_comm_init");
    return MSORT_ERROR_INVALID_VALUE;
  }
  MSORT_TRY(check_device());
  return comm_init(id, rank, world, out);
}

msort_status msort_comm_wrap(void* nccl_comm, msort_comm_t* out) {
  if (!nccl_comm || !out) {
    set_error("bad argument to msort_comm_wrap");
    return MSORT_ERROR_INVALID_VALUE;
  }
  MSORT_TRY(check_device());
  return comm_wrap(nccl_comm, out);
}

msort_status msort_comm_destroy(msort_comm_t comm) { return comm_destroy(comm); }

msort_status msort_comm_reserve(msort_comm_t comm, size_t n_max, msort_dtype key_dtype,
                                msort_dtype val_dtype, msort_stream_t stream) {
  if (!comm || !dtype_size(key_dtype) ||
      (val_dtype != MSORT_NONE && val_dtype != MSORT_UINT32 && val_dtype != MSORT_INT32)) {
    set_error("bad argument to msort_comm_reserve");
    return MSORT_ERROR_INVALID_VALUE;
  }
  MSORT_TRY(check_device());
  return comm_reserve(comm, n_max, key_dtype, val_dtype, (cudaStream_t)stream);
}

msort_status msort_sort_distributed_ws(void* keys, void* vals, size_t n_local,
                                       msort_dtype key_dtype, msort_dtype val_dtype,
                                       msort_comm_t comm, void* ws, size_t ws_bytes,
                                       msort_stream_t stream, int64_t* split_matrix_out) {
  if (!comm) {
    set_error("comm is NULL");
    return MSORT_ERROR_INVALID_VALUE;
  }
  // n_local == 0 ranks still take part in the collectives
  MSORT_TRY(validate(keys, vals, n_local, key_dtype, val_dtype, false));
  MSORT_TRY(check_device());
  const int world = comm_world(comm);
  MSORT_TRY(validate_ws(keys, vals, n_local, key_dtype, val_dtype, ws, ws_bytes,
                        dist_ws_bytes(n_local, key_dtype, val_dtype, world)));
  return dist_nccl(keys, vals, keys, vals, n_local, key_dtype, val_dtype, comm, ws,
                   (cudaStream_t)stream, split_matrix_out);
}

msort_status msort_sort_distributed_out_ws(const void* in_keys, const void* in_vals,
                                           void* keys_out, void* vals_out, size_t n_local,
                                           msort_dtype key_dtype, msort_dtype val_dtype,
                                           msort_comm_t comm, void* ws, size_t ws_bytes,
                                           msort_stream_t stream, int64_t* split_matrix_out) {
  if (!comm) {
    set_error("comm is NULL");
    return MSORT_ERROR_INVALID_VALUE;
  }
  MSORT_TRY(validate_out(in_keys, in_vals, keys_out, vals_out, n_local, key_dtype, val_dtype));
  MSORT_TRY(check_device());
  const int world = comm_world(comm);
  MSORT_TRY(validate_ws(keys_out, vals_out, n_local, key_dtype, val_dtype, ws, ws_bytes,
                        dist_ws_bytes(n_local, key_dtype, val_dtype, world)));
  if (overlaps(ws, ws_bytes, in_keys, n_local * dtype_size(key_dtype))) {
    set_error("workspace overlaps the input");
    return MSORT_ERROR_INVALID_VALUE;
  }
  return dist_nccl(in_keys, in_vals, keys_out, vals_out, n_local, key_dtype, val_dtype, comm, ws,
                   (cudaStream_t)stream, split_matrix_out);
}

msort_status msort_sort_distributed_host(const void* host_keys, const void* host_vals,
                                         void* host_keys_out, void* host_vals_out,
                                         size_t n_local, msort_dtype key_dtype,
                                         msort_dtype val_dtype, msort_comm_t comm,
                                         void* dev_keys, void* dev_vals, void* ws,
                                         size_t ws_bytes, msort_stream_t stream) {
  if (!comm) {
    set_error("comm is NULL");
    return MSORT_ERROR_INVALID_VALUE;
  }
  const bool pairs = val_dtype != MSORT_NONE;
  if (n_local > 0 && (!host_keys || !host_keys_out || (pairs && (!host_vals || !host_vals_out)))) {
    set_error("msort_sort_distributed_host: NULL host pointer");
    return MSORT_ERROR_INVALID_VALUE;
  }
  MSORT_TRY(validate(dev_keys, pairs ? dev_vals : nullptr, n_local, key_dtype, val_dtype, false));
  MSORT_TRY(check_device());
  const int world = comm_world(comm);
  MSORT_TRY(validate_ws(dev_keys, pairs ? dev_vals : nullptr, n_local, key_dtype, val_dtype, ws,
                        ws_bytes, dist_ws_bytes(n_local, key_dtype, val_dtype, world)));
  cudaStream_t s = (cudaStream_t)stream;
  const size_t kb = n_local * dtype_size(key_dtype);
  if (n_local > 0) {
    MSORT_CUDA_TRY(cudaMemcpyAsync(dev_keys, host_keys, kb, cudaMemcpyHostToDevice, s));
    if (pairs)
      MSORT_CUDA_TRY(
          cudaMemcpyAsync(dev_vals, host_vals, n_local * 4, cudaMemcpyHostToDevice, s));
  }
  MSORT_TRY(dist_nccl(dev_keys, pairs ? dev_vals : nullptr, dev_keys, pairs ? dev_vals : nullptr,
                      n_local, key_dtype, val_dtype, comm, ws, s, nullptr));
  if (n_local > 0) {
    MSORT_CUDA_TRY(cudaMemcpyAsync(host_keys_out, dev_keys, kb, cudaMemcpyDeviceToHost, s));
    if (pairs)
      MSORT_CUDA_TRY(
          cudaMemcpyAsync(host_vals_out, dev_vals, n_local * 4, cudaMemcpyDeviceToHost, s));
  }
  return MSORT_SUCCESS;
}

msort_status msort_sort_distributed(void* keys, void* vals, size_t n_local,
                                    msort_dtype key_dtype, msort_dtype val_dtype,
                                    msort_comm_t comm, msort_stream_t stream,
                                    int64_t* split_matrix_out) {
  if (!comm) {
    set_error("comm is NULL");
    return MSORT_ERROR_INVALID_VALUE;
  }
  MSORT_TRY(validate(keys, vals, n_local, key_dtype, val_dtype, false));
  MSORT_TRY(check_device());
  cudaStream_t s = (cudaStream_t)stream;
  size_t need = dist_ws_bytes(n_local, key_dtype, val_dtype, comm_world(comm));
  void* ws = nullptr;
  MSORT_CUDA_TRY(scratch_alloc(&ws, need, s));
  msort_status st = dist_nccl(keys, vals, keys, vals, n_local, key_dtype, val_dtype, comm, ws, s,
                              split_matrix_out);
  cudaError_t e = cudaFreeAsync(ws, s);
  if (st != MSORT_SUCCESS) return st;
  if (e != cudaSuccess) return cuda_fail(e, "cudaFreeAsync");
  return MSORT_SUCCESS;
}

msort_status msort_sort_distributed_tree(const void* in_keys, const void* in_vals, size_t n_local,
                                         msort_dtype key_dtype, msort_dtype val_dtype,
                                         msort_comm_t comm, void* root_keys, void* root_vals,
                                         size_t root_capacity, msort_stream_t stream,
                                         int64_t* total_out) {
  if (!comm) {
    set_error("comm is NULL");
    return MSORT_ERROR_INVALID_VALUE;
  }
  if (val_dtype == MSORT_NONE) in_vals = nullptr, root_vals = nullptr;
  MSORT_TRY(validate(const_cast<void*>(in_keys), const_cast<void*>(in_vals), n_local, key_dtype,
                     val_dtype, false));
  MSORT_TRY(validate(root_keys, root_vals, root_capacity, key_dtype, val_dtype, false));
  MSORT_TRY(check_device());
  return tree_nccl(in_keys, in_vals, n_local, key_dtype, val_dtype, comm, root_keys, root_vals,
                   root_capacity, (cudaStream_t)stream, total_out);
}

msort_status msort_sort_distributed_tree_emulated(const void* const* keys,
                                                  const void* const* vals,
                                                  const size_t* n_local, int world,
                                                  msort_dtype key_dtype, msort_dtype val_dtype,
                                                  void* root_keys, void* root_vals,
                                                  msort_stream_t stream) {
  if (!keys || !n_local || world < 1 || world > 1024 || (val_dtype != MSORT_NONE && !vals)) {
    set_error("bad argument to msort_sort_distributed_tree_emulated");
    return MSORT_ERROR_INVALID_VALUE;
  }
  if (val_dtype == MSORT_NONE) vals = nullptr, root_vals = nullptr;
  size_t total = 0;
  for (int r = 0; r < world; ++r) {
    MSORT_TRY(validate(const_cast<void*>(keys[r]), vals ? const_cast<void*>(vals[r]) : nullptr,
                       n_local[r], key_dtype, val_dtype, false));
    total += n_local[r];
  }
  MSORT_TRY(validate(root_keys, root_vals, total, key_dtype, val_dtype, false));
  if (total == 0) return MSORT_SUCCESS;
  MSORT_TRY(check_device());
  return tree_emulated(keys, vals, n_local, world, key_dtype, val_dtype, root_keys, root_vals,
                       (cudaStream_t)stream);
}

msort_status msort_sort_distributed_emulated(void* const* keys, void* const* vals,
                                             const size_t* n_local, int world,
                                             msort_dtype key_dtype, msort_dtype val_dtype,
                                             void* const* ws, size_t ws_bytes,
                                             msort_stream_t stream,
                                             int64_t* split_matrix_out) {
  if (!keys || !n_local || !ws || world < 1 || (val_dtype != MSORT_NONE && !vals)) {
    set_error("bad argument to msort_sort_distributed_emulated");
    return MSORT_ERROR_INVALID_VALUE;
  }
  MSORT_TRY(check_device());
  for (int r = 0; r < world; ++r) {
    void* v = val_dtype == MSORT_NONE ? nullptr : vals[r];
    MSORT_TRY(validate(keys[r], v, n_local[r], key_dtype, val_dtype, false));
    MSORT_TRY(validate_ws(keys[r], v, n_local[r], key_dtype, val_dtype, ws[r], ws_bytes,
                          dist_ws_bytes(n_local[r], key_dtype, val_dtype, world)));
  }
  return dist_emulated(keys, vals, n_local, world, key_dtype, val_dtype, ws,
                       (cudaStream_t)stream, split_matrix_out);
}

// ------------------------------------------------------------ planning
int msort_plan_rounds(msort_dtype key_dtype) {
  size_t w = dtype_size(key_dtype);
  return w == 4 ? 4 : (w == 8 ? 8 : 0);
}

int msort_plan_candidates_per_round(void) { return kCandidates; }

msort_status msort_plan_init(msort_dtype key_dtype, int world, uint64_t* lohi) {
  size_t w = dtype_size(key_dtype);
  if (!w || world < 1 || !lohi) {
    set_error("bad argument to msort_plan_init");
    return MSORT_ERROR_INVALID_VALUE;
  }
  for (int r = 0; r + 1 < world; ++r) lohi[2 * r] = 0, lohi[2 * r + 1] = w == 4 ? 0xffffffffull : ~0ull;
  return MSORT_SUCCESS;
}

msort_status msort_plan_candidates(int world, const uint64_t* lohi, uint64_t* cand) {
  if (world < 1 || (world > 1 && (!lohi || !cand))) {
    set_error("bad argument to msort_plan_candidates");
    return MSORT_ERROR_INVALID_VALUE;
  }
  for (int r = 0; r + 1 < world; ++r)
    for (int b = 0; b < kCandidates; ++b)
      cand[(size_t)r * kCandidates + b] = plan::candidate(lohi[2 * r], lohi[2 * r + 1], b, kCandidates);
  return MSORT_SUCCESS;
}

msort_status msort_plan_narrow(int world, const uint64_t* K, const uint64_t* total,
                               uint64_t* lohi) {
  if (world < 1 || (world > 1 && (!K || !total || !lohi))) {
    set_error("bad argument to msort_plan_narrow");
    return MSORT_ERROR_INVALID_VALUE;
  }
  for (int r = 0; r + 1 < world; ++r)
    plan::narrow(lohi[2 * r], lohi[2 * r + 1], total + (size_t)r * kCandidates, kCandidates, K[r + 1]);
  return MSORT_SUCCESS;
}

msort_status msort_plan_fill(int world, const uint64_t* K, const uint64_t* lteq, int64_t* out) {
  if (world < 1 || !K || !out || (world > 1 && !lteq)) {
    set_error("bad argument to msort_plan_fill");
    return MSORT_ERROR_INVALID_VALUE;
  }
  for (int r = 0; r <= world; ++r)
    for (int j = 0; j < world; ++j) {
      int64_t v;
      if (r == 0) v = 0;
      else if (r == world) v = (int64_t)(K[j + 1] - K[j]);
      else v = plan::fill_one(K[r], lteq, world, r, j);
      out[(size_t)r * world + j] = v;
    }
  return MSORT_SUCCESS;
}

int msort_plan_tree_rounds(int world) { return world < 1 ? 0 : plan::tree_rounds(world); }

int msort_plan_tree_role(int world, int rank, int round, int* peer) {
  int q = -1;
  const int r = (world < 1 || rank < 0 || rank >= world || round < 0)
                    ? 0
                    : plan::tree_role(world, rank, round, &q);
  if (peer) *peer = q;
  return r;
}

// ------------------------------------------------------- status / timing
const char* msort_status_string(msort_status s) {
  switch (s) {
    case MSORT_SUCCESS: return "MSORT_SUCCESS";
    case MSORT_ERROR_INVALID_VALUE: return "MSORT_ERROR_INVALID_VALUE";
    case MSORT_ERROR_NOT_SUPPORTED: return "MSORT_ERROR_NOT_SUPPORTED";
    case MSORT_ERROR_OUT_OF_MEMORY: return "MSORT_ERROR_OUT_OF_MEMORY";
    case MSORT_ERROR_CUDA: return "MSORT_ERROR_CUDA";
    case MSORT_ERROR_NCCL: return "MSORT_ERROR_NCCL";
    default: return "MSORT_UNKNOWN_STATUS";
  }
}

const char* msort_last_error(void) { return g_last_error.c_str(); }

void msort_profile_enable(int on) { g_profile.store(on ? 1 : 0); }

void msort_profile_reset(void) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& r : g_pending) g_free_events.push_back(r.a), g_free_events.push_back(r.b);
  g_pending.clear();
  for (int i = 0; i < MSORT_PROFILE_CLASSES; ++i) g_prof_launches[i] = 0, g_prof_ms[i] = 0.0;
  g_launches.store(0);
}

msort_status msort_profile_read(int64_t* launches, double* ms) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& r : g_pending) {
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventSynchronize");
    float t = 0.f;
    e = cudaEventElapsedTime(&t, r.a, r.b);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventElapsedTime");
    g_prof_launches[r.kc] += 1;
    g_prof_ms[r.kc] += t;
    g_free_events.push_back(r.a), g_free_events.push_back(r.b);
  }
  g_pending.clear();
  for (int i = 0; i < MSORT_PROFILE_CLASSES; ++i) {
    if (launches) launches[i] = g_prof_launches[i];
    if (ms) ms[i] = g_prof_ms[i];
  }
  return MSORT_SUCCESS;
}

int64_t msort_launch_count(void) { return g_launches.load(); }

int msort_tile_size(msort_dtype key_dtype, msort_dtype val_dtype) {
  return tile_size_for(key_dtype, val_dtype);
}

}  // extern "C"
