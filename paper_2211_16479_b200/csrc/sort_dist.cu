// sort_dist.cu -- multi-GPU stable merge sort (one process per GPU, NCCL).
//
// The paper's MPI merge sort: scatter equal chunks from rank 0
// (P:412-434), sort each chunk locally (the "subsort"), then merge
// up a rank tree until rank 0 holds everything.  Re-designed for
// B200 + NVLink 5 / NVSwitch (every peer at full bandwidth):
//   D1  local sort of each rank's shard            (sort_single.cu, K1..K3)
//   D2  exact splitters by co-ranking the sorted shards: value-space
//       bucket search, 8 bits per round, one tiny ncclAllReduce per round,
//       then one ncclAllGather of (lt, eq) and a rank-order tie fill (K4)
//   D3  one variable all-to-all of the sorted segments (grouped
//       ncclSend/ncclRecv), the only bulk transfer
//   D4  local stable k-way merge of the received runs, lower rank first (K5)
// Output: rank r holds global stable positions [K_r, K_r + n_r) (DESIGN.md
// R10/R11), so the call is in place and balanced for any key distribution.
#include <nccl.h>

#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <chrono>
#include <atomic>
#include <map>
#include <string>
#include <vector>

#include "msort_device.cuh"
#include "msort_internal.h"
#include "plan.cuh"

struct msort_comm_s {
  ncclComm_t comm;
  int rank;
  int world;
  // pull exchange: peers' exchange buffers opened through CUDA IPC, cached by
  // (rank, handle) -- the workspace allocation is normally reused call to call
  std::map<std::pair<int, std::string>, void*> ipc_open;
  bool aborted = false;  // set when a failure aborted the NCCL communicator
  bool owned = true;     // false: wraps a caller's communicator (never destroyed / aborted here)
  int exchange = -1;     // exchange mode of this communicator (-1: the process default)
  // page-locked staging for the small host<->device copies of a call (split
  // matrix, sizes, IPC records): copies from/to pageable memory would block
  // the host inside cudaMemcpyAsync, out of reach of the failure detection
  unsigned char* pinned = nullptr;
  size_t pinned_bytes = 0;
  // small device scratch of the communicator's own collectives (sizes and
  // agreement flags of the rank-tree gather): 8 * (2 * world + 64) bytes
  uint64_t* dscratch = nullptr;
  // pull exchange: the sorted shard that the peers read in place lives in a
  // buffer the communicator owns, from cudaMalloc (IPC-exportable whatever
  // allocator the caller's workspace came from); grown on demand and reused
  // (its IPC handle, opened once by each peer, stays valid between calls)
  void* xbuf = nullptr;
  size_t xbuf_bytes = 0;
  // msort_comm_reserve: the exchange buffer holds up to reserved_n local keys
  // (+ payloads) on every rank, its IPC mappings are open, and dbases (device
  // table of the p ranks' shard pointers) lets the pull path plan K5 on the
  // device -- no host synchronisation per call
  size_t reserved_n = 0;
  size_t reserved_wk = 0;
  bool reserved_vals = false;
  const void** dbases = nullptr;
};

namespace msort {

constexpr int B = kCandidates;
constexpr int kMaxWorld = 128;

static msort_status nccl_fail(ncclResult_t r, const char* what) {
  set_error(std::string(what) + ": " + ncclGetErrorString(r));
  return MSORT_ERROR_NCCL;
}
#define MSORT_NCCL_TRY(expr)                                  \
  do {                                                        \
    ncclResult_t _r = (expr);                                 \
    if (_r != ncclSuccess) return ::msort::nccl_fail(_r, #expr); \
  } while (0)

// ncclGroupStart/End bracket that is closed on every path: an early error
// return between the two must not leave this thread's NCCL group open.
struct NcclGroup {
  bool open = false;
  ncclResult_t start() {
    ncclResult_t r = ncclGroupStart();
    open = r == ncclSuccess;
    return r;
  }
  ncclResult_t end() {
    open = false;
    return ncclGroupEnd();
  }
  ~NcclGroup() {
    if (open) ncclGroupEnd();
  }
};

// Host wait for the distributed call's stream with failure detection
// (SURVEY.md §5): instead of blocking in cudaStreamSynchronize -- which never
// returns if a peer died inside a collective -- poll the stream and the
// communicator's asynchronous error state; on an NCCL error, or after
// MSORT_NCCL_TIMEOUT_S seconds (environment, default 0 = no timeout), abort
// the communicator (it is unusable afterwards) and return MSORT_ERROR_NCCL.
static msort_status wait_stream_nccl(msort_comm_s* c, cudaStream_t s, const char* what) {
  static const double limit = [] {  // read once (thread-safe static initialisation)
    const char* e = getenv("MSORT_NCCL_TIMEOUT_S");
    return e ? atof(e) : 0.0;
  }();
  const auto t0 = std::chrono::steady_clock::now();
  for (unsigned spin = 0;; ++spin) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) return MSORT_SUCCESS;
    if (q != cudaErrorNotReady) return cuda_fail(q, what);
    ncclResult_t ae = ncclSuccess;
    if (ncclCommGetAsyncError(c->comm, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress) {
      if (c->owned) ncclCommAbort(c->comm);  // a borrowed communicator is its owner's to abort
      c->aborted = true;
      return nccl_fail(ae, what);
    }
    const double el =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (limit > 0 && el > limit) {
      if (c->owned) ncclCommAbort(c->comm);
      c->aborted = true;
      set_error(std::string(what) + ": timed out after " + std::to_string(el) +
                " s (MSORT_NCCL_TIMEOUT_S); communicator aborted");
      return MSORT_ERROR_NCCL;
    }
    if (spin > 256) std::this_thread::sleep_for(std::chrono::microseconds(5));  // keep the wait tight
  }
}

// ------------------------------------------------------------- K4 kernels
__global__ void k4_set_u64(uint64_t* p, uint64_t v) { *p = v; }

__global__ void k4_init(uint64_t* lohi, int nb, uint64_t umax) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < nb) lohi[2 * r] = 0, lohi[2 * r + 1] = umax;
}

// First index i of the sorted shard keys[0, n) with image(keys[i]) > c
// (UPPER: the count of keys <= c) or >= c (lower: the count of keys < c), by
// one warp: each round probes 32 evenly spaced candidates of [lo, hi) and
// keeps the bucket where the monotone predicate turns true -- log32(n)
// dependent rounds of global-memory probes instead of log2(n) (the splitter
// rounds are latency-bound; D2 is latency-bound).
template <class K, bool UPPER>
__device__ __forceinline__ int64_t warp_bound(const K* __restrict__ keys, int64_t n, uint64_t c,
                                              int lane) {
  int64_t lo = 0, hi = n;
  while (hi > lo) {
    const int64_t span = hi - lo;
    const int64_t step = (span + 31) >> 5;
    const int64_t off = step * (lane + 1);
    const int64_t p = lo + (off < span ? off : span) - 1;
    const uint64_t x = (uint64_t)KeyTraits<K>::image(__ldg(keys + p));
    const bool past = UPPER ? x > c : x >= c;
    const unsigned m = __ballot_sync(0xffffffffu, past);
    if (m == 0) {
      lo = hi;
    } else {
      const int f = __ffs(m) - 1;
      const int64_t pf = __shfl_sync(0xffffffffu, p, f);
      const int64_t pp = __shfl_sync(0xffffffffu, p, f > 0 ? f - 1 : 0);
      hi = pf;
      if (f > 0) lo = pp + 1;
    }
  }
  return lo;
}

// cnt[r*B + b] = #{x in local shard : image(x) <= candidate b of boundary r};
// one warp per (boundary, candidate)
template <class K>
__global__ void __launch_bounds__(256)
    k4_count(const K* __restrict__ keys, int64_t n, const uint64_t* __restrict__ lohi, int nb,
             uint64_t* __restrict__ cnt) {
  const int t = (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= nb * B) return;  // warp-uniform
  const int r = t / B, b = t % B;
  const uint64_t c = plan::candidate(lohi[2 * r], lohi[2 * r + 1], b, B);
  const int64_t lo = warp_bound<K, true>(keys, n, c, lane);
  if (lane == 0) cnt[t] = (uint64_t)lo;
}

// One thread per boundary r = 1..world-1: narrow [lo, hi] from the global counts.
__global__ void k4_narrow(uint64_t* lohi, const uint64_t* __restrict__ total,
                          const uint64_t* __restrict__ nsz, int world) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= world - 1) return;
  uint64_t K = 0;
  for (int j = 0; j <= r; ++j) K += nsz[j];  // K_{r+1}
  uint64_t lo = lohi[2 * r], hi = lohi[2 * r + 1];
  plan::narrow(lo, hi, total + (size_t)r * B, B, K);
  lohi[2 * r] = lo, lohi[2 * r + 1] = hi;
}

// (lt, eq) of the local shard at v*_r = lo_r (= hi_r after the last round);
// one warp per bound
template <class K>
__global__ void k4_lteq(const K* __restrict__ keys, int64_t n, const uint64_t* __restrict__ lohi,
                        int nb, uint64_t* __restrict__ lteq) {
  const int t = (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= 2 * nb) return;  // warp-uniform
  const int r = t / 2, upper = t % 2;
  const uint64_t v = lohi[2 * r];
  const int64_t lo = upper ? warp_bound<K, true>(keys, n, v, lane)
                           : warp_bound<K, false>(keys, n, v, lane);
  if (lane == 0) lteq[t] = (uint64_t)lo;  // t even: lower bound (lt); odd: upper bound (le)
}

// le -> eq in place after the gather would need a pass; instead convert locally
__global__ void k4_le_to_eq(uint64_t* lteq, int nb) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < nb) lteq[2 * r + 1] -= lteq[2 * r];
}

__global__ void k4_fill(const uint64_t* __restrict__ lteq_all, const uint64_t* __restrict__ nsz,
                        int world, int64_t* __restrict__ split) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (world + 1) * world) return;
  int r = t / world, j = t % world;
  int64_t v;
  if (r == 0) v = 0;
  else if (r == world) v = (int64_t)nsz[j];
  else {
    uint64_t K = 0;
    for (int q = 0; q < r; ++q) K += nsz[q];
    v = plan::fill_one(K, lteq_all, world, r, j);
  }
  split[t] = v;
}

// ------------------------------------------ emulation collectives (1 GPU)
struct PtrTable {
  uint64_t* p[kMaxWorld];
};
__global__ void k_emul_allreduce(PtrTable t, int world, int count) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  uint64_t s = 0;
  for (int r = 0; r < world; ++r) s += t.p[r][i];
  for (int r = 0; r < world; ++r) t.p[r][i] = s;
}
__global__ void k_emul_allgather(PtrTable src, PtrTable dst, int world, int count) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= world * count) return;
  int from = i / count, k = i % count;
  uint64_t v = src.p[from][k];
  for (int r = 0; r < world; ++r) dst.p[r][i] = v;
}

// -------------------------------------------------------- workspace carve
struct DistWs {
  char* sort_ws;
  size_t sort_ws_bytes;
  void* rk;  // receive keys
  void* rv;  // receive vals
  uint64_t *nsz_send, *nsz, *lohi, *cnt, *lteq, *lteq_all;
  int64_t* split;
  unsigned char *ipc_send, *ipc_all;  // pull exchange: (handle, offset) of the exchange buffers
};

// CUDA IPC record of one rank's exchange buffers (keys, vals).
struct IpcRec {
  cudaIpcMemHandle_t hk, hv;
  int64_t ok, ov;  // offsets of the buffers inside their allocations
};
constexpr size_t kIpcBytes = (sizeof(IpcRec) + 255) / 256 * 256;

static size_t d2_bytes(int world) {
  size_t nb = world > 1 ? world - 1 : 1;
  size_t b = 0;
  b += align_up(8, 256);                               // nsz_send
  b += align_up(8 * (size_t)world, 256);               // nsz
  b += align_up(16 * nb, 256);                         // lohi
  b += align_up(8 * nb * B, 256);                      // cnt
  b += align_up(16 * nb, 256);                         // lteq
  b += align_up(16 * nb * (size_t)world, 256);         // lteq_all
  b += align_up(8 * (size_t)(world + 1) * world, 256); // split
  b += kIpcBytes * (size_t)(world + 1);                // ipc_send, ipc_all
  return b;
}

static DistWs carve(void* ws, size_t n, msort_dtype kd, msort_dtype vd, int world) {
  DistWs d{};
  char* w = static_cast<char*>(ws);
  const size_t wk = dtype_size(kd);
  const bool pairs = vd != MSORT_NONE;
  d.sort_ws = w;
  d.sort_ws_bytes = single_ws_bytes(n, kd, vd);
  if (world <= 1) return d;  // one rank: the local sort is the whole job
  w += align_up(d.sort_ws_bytes, 256);
  d.rk = w;
  w += align_up(n * wk, 256);
  d.rv = pairs ? w : nullptr;
  if (pairs) w += align_up(n * 4, 256);
  size_t nb = world > 1 ? world - 1 : 1;
  d.nsz_send = (uint64_t*)w; w += align_up(8, 256);
  d.nsz = (uint64_t*)w; w += align_up(8 * (size_t)world, 256);
  d.lohi = (uint64_t*)w; w += align_up(16 * nb, 256);
  d.cnt = (uint64_t*)w; w += align_up(8 * nb * B, 256);
  d.lteq = (uint64_t*)w; w += align_up(16 * nb, 256);
  d.lteq_all = (uint64_t*)w; w += align_up(16 * nb * (size_t)world, 256);
  d.split = (int64_t*)w; w += align_up(8 * (size_t)(world + 1) * world, 256);
  d.ipc_send = (unsigned char*)w; w += kIpcBytes;
  d.ipc_all = (unsigned char*)w;
  return d;
}

size_t dist_ws_bytes(size_t n, msort_dtype kd, msort_dtype vd, int world) {
  if (world <= 1) return single_ws_bytes(n, kd, vd);
  size_t b = align_up(single_ws_bytes(n, kd, vd), 256);
  b += align_up(n * dtype_size(kd), 256);
  if (vd != MSORT_NONE) b += align_up(n * 4, 256);
  b += d2_bytes(world);
  return b;
}

// ------------------------------------------------------------ the driver
struct RankIO {
  const void* in_keys;  // input shard (== keys for the in-place call)
  const void* in_vals;
  void* keys;  // output shard
  void* vals;
  size_t n;
  DistWs ws;
  void* sk;  // where D1 leaves the sorted shard: keys, or (pull) the exchange buffer ws.rk
  void* sv;
};

static ncclDataType_t nccl_type(msort_dtype d) {
  switch (d) {
    case MSORT_INT32: return ncclInt32;
    case MSORT_UINT32: return ncclUint32;
    case MSORT_INT64: return ncclInt64;
    default: return ncclUint64;
  }
}

// Collectives over NCCL: one local rank.
struct NcclColl {
  msort_comm_s* c;
  cudaStream_t s;
  int world() const { return c->world; }
  msort_status allgather_u64(RankIO* io, uint64_t* DistWs::*src, uint64_t* DistWs::*dst,
                             size_t count) {
    LaunchScope ls(KC_NCCL, s);
    MSORT_NCCL_TRY(ncclAllGather(io[0].ws.*src, io[0].ws.*dst, count, ncclUint64, c->comm, s));
    return MSORT_SUCCESS;
  }
  msort_status allreduce_u64(RankIO* io, uint64_t* DistWs::*buf, size_t count) {
    LaunchScope ls(KC_NCCL, s);
    MSORT_NCCL_TRY(ncclAllReduce(io[0].ws.*buf, io[0].ws.*buf, count, ncclUint64, ncclSum,
                                 c->comm, s));
    return MSORT_SUCCESS;
  }
  // D3: rank me sends keys[s[r][me], s[r+1][me]) to every r; receives run j
  // (length s[me+1][j] - s[me][j]) into recv at offset sum_{j'<j} of those.
  msort_status exchange(RankIO* io, const std::vector<int64_t>& S, msort_dtype kd,
                        msort_dtype vd) {
    const int p = c->world, me = c->rank;
    const size_t wk = dtype_size(kd);
    RankIO& r0 = io[0];
    auto sp = [&](int r, int j) { return S[(size_t)r * p + j]; };
    LaunchScope ls(KC_EXCHANGE, s);
    // the self segment: a local device copy, enqueued outside the NCCL group
    {
      int64_t roff = 0;
      for (int j = 0; j < me; ++j) roff += sp(me + 1, j) - sp(me, j);
      const int64_t rc = sp(me + 1, me) - sp(me, me);
      if (rc > 0) {
        MSORT_CUDA_TRY(cudaMemcpyAsync((char*)r0.ws.rk + roff * wk,
                                       (char*)r0.keys + sp(me, me) * wk, rc * wk,
                                       cudaMemcpyDeviceToDevice, s));
        if (vd != MSORT_NONE)
          MSORT_CUDA_TRY(cudaMemcpyAsync((char*)r0.ws.rv + roff * 4,
                                         (char*)r0.vals + sp(me, me) * 4, rc * 4,
                                         cudaMemcpyDeviceToDevice, s));
      }
    }
    // every other segment: one grouped send/recv per peer; zero-length
    // segments are skipped on both sides (both hold the same split matrix)
    int64_t roff = 0;
    NcclGroup grp;
    MSORT_NCCL_TRY(grp.start());
    for (int j = 0; j < p; ++j) {
      const int64_t rc = sp(me + 1, j) - sp(me, j);  // run j, received from rank j
      const int64_t sc = sp(j + 1, me) - sp(j, me);  // what I send to rank j
      if (j != me) {
        if (sc > 0) {
          MSORT_NCCL_TRY(ncclSend((char*)r0.keys + sp(j, me) * wk, (size_t)sc, nccl_type(kd), j,
                                  c->comm, s));
          if (vd != MSORT_NONE)
            MSORT_NCCL_TRY(ncclSend((char*)r0.vals + sp(j, me) * 4, (size_t)sc, ncclUint32, j,
                                    c->comm, s));
        }
        if (rc > 0) {
          MSORT_NCCL_TRY(ncclRecv((char*)r0.ws.rk + roff * wk, (size_t)rc, nccl_type(kd), j,
                                  c->comm, s));
          if (vd != MSORT_NONE)
            MSORT_NCCL_TRY(ncclRecv((char*)r0.ws.rv + roff * 4, (size_t)rc, ncclUint32, j,
                                    c->comm, s));
        }
      }
      roff += rc;
    }
    MSORT_NCCL_TRY(grp.end());
    return MSORT_SUCCESS;
  }
  int rank_of(int local) const { return c->rank + local; }
  // Sync-free pull (after msort_comm_reserve): the device table of the
  // ranks' shard pointers, or nullptr when the communicator is not reserved
  // for this call's size (the host-planned pull path runs instead).
  const void* const* reserved_bases(RankIO* io, msort_dtype kd, bool pairs) {
    if (!c->dbases || pairs || io[0].n > c->reserved_n || dtype_size(kd) > c->reserved_wk)
      return nullptr;
    return c->dbases;
  }
  msort_status wait(const char* what) { return wait_stream_nccl(c, s, what); }
  // device -> host copy of `bytes` through the pinned staging, then the wait
  msort_status fetch(void* host, const void* dev, size_t bytes, const char* what) {
    if (bytes > c->pinned_bytes) {
      set_error(std::string(what) + ": staging too small");
      return MSORT_ERROR_NOT_SUPPORTED;
    }
    MSORT_CUDA_TRY(cudaMemcpyAsync(c->pinned, dev, bytes, cudaMemcpyDeviceToHost, s));
    MSORT_TRY(wait(what));
    memcpy(host, c->pinned, bytes);
    return MSORT_SUCCESS;
  }
  // pull exchange: after the peers' reads, nobody may reuse its buffer
  msort_status barrier(RankIO* io) {
    LaunchScope ls(KC_NCCL, s);
    MSORT_NCCL_TRY(ncclAllReduce(io[0].ws.nsz, io[0].ws.nsz, 1, ncclUint64, ncclMax, c->comm, s));
    return MSORT_SUCCESS;
  }
  // pull exchange, step 1 (enqueued before the host sync): publish the CUDA
  // IPC handles of this rank's exchange buffers and gather everyone's into
  // `host` (valid after the stream synchronises).
  msort_status ipc_publish(RankIO* io, unsigned char* host) {
    IpcRec me{};
    for (int which = 0; which < 2; ++which) {
      void* p = which == 0 ? io[0].sk : io[0].sv;
      if (!p) continue;
      // the driver's cuMemGetAddressRange through the runtime (no libcuda link)
      using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
      static GetRange get_range = nullptr;
      if (!get_range) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        MSORT_CUDA_TRY(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
        get_range = reinterpret_cast<GetRange>(fn);
      }
      CUdeviceptr base = 0;
      size_t size = 0;
      if (!get_range || get_range(&base, &size, (CUdeviceptr)p) != CUDA_SUCCESS) {
        set_error("pull exchange: cuMemGetAddressRange failed on the workspace");
        return MSORT_ERROR_NOT_SUPPORTED;
      }
      cudaIpcMemHandle_t h;
      MSORT_CUDA_TRY(cudaIpcGetMemHandle(&h, (void*)base));
      (which == 0 ? me.hk : me.hv) = h;
      (which == 0 ? me.ok : me.ov) = (int64_t)((CUdeviceptr)p - base);
    }
    memcpy(c->pinned, &me, sizeof(me));
    MSORT_CUDA_TRY(
        cudaMemcpyAsync(io[0].ws.ipc_send, c->pinned, sizeof(me), cudaMemcpyHostToDevice, s));
    {
      LaunchScope ls(KC_NCCL, s);
      MSORT_NCCL_TRY(ncclAllGather(io[0].ws.ipc_send, io[0].ws.ipc_all, kIpcBytes, ncclUint8,
                                   c->comm, s));
    }
    // (the pinned record must outlive the async upload: fetch waits for both)
    MSORT_TRY(fetch(host, io[0].ws.ipc_all, kIpcBytes * c->world, "ipc handle gather"));
    return MSORT_SUCCESS;
  }
  // step 2 (after the sync): map every peer's exchange buffers (cached).
  msort_status peer_bases(RankIO* io, const unsigned char* host, bool pairs,
                          std::vector<const void*>& bk, std::vector<const uint32_t*>& bv) {
    const int p = c->world;
    bk.assign(p, nullptr), bv.assign(p, nullptr);
    for (int j = 0; j < p; ++j) {
      if (j == c->rank) {
        bk[j] = io[0].sk, bv[j] = (const uint32_t*)io[0].sv;
        continue;
      }
      IpcRec r;
      memcpy(&r, host + (size_t)j * kIpcBytes, sizeof(r));
      for (int which = 0; which < (pairs ? 2 : 1); ++which) {
        const cudaIpcMemHandle_t& h = which == 0 ? r.hk : r.hv;
        auto key = std::make_pair(j, std::string(reinterpret_cast<const char*>(&h), sizeof(h)));
        auto it = c->ipc_open.find(key);
        void* base = nullptr;
        if (it != c->ipc_open.end()) {
          base = it->second;
        } else {
          MSORT_CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
          c->ipc_open[key] = base;
        }
        if (which == 0) bk[j] = (const char*)base + r.ok;
        else bv[j] = (const uint32_t*)((const char*)base + r.ov);
      }
    }
    return MSORT_SUCCESS;
  }
};

// Collectives emulated on one device for `world` virtual ranks.
struct EmulColl {
  int p;
  cudaStream_t s;
  int world() const { return p; }
  msort_status allgather_u64(RankIO* io, uint64_t* DistWs::*src, uint64_t* DistWs::*dst,
                             size_t count) {
    PtrTable a{}, b{};
    for (int r = 0; r < p; ++r) a.p[r] = io[r].ws.*src, b.p[r] = io[r].ws.*dst;
    LaunchScope ls(KC_SPLITTER, s);
    int tot = (int)(p * count);
    k_emul_allgather<<<(tot + 255) / 256, 256, 0, s>>>(a, b, p, (int)count);
    MSORT_CUDA_TRY(cudaGetLastError());
    return MSORT_SUCCESS;
  }
  msort_status allreduce_u64(RankIO* io, uint64_t* DistWs::*buf, size_t count) {
    PtrTable a{};
    for (int r = 0; r < p; ++r) a.p[r] = io[r].ws.*buf;
    LaunchScope ls(KC_SPLITTER, s);
    k_emul_allreduce<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(a, p, (int)count);
    MSORT_CUDA_TRY(cudaGetLastError());
    return MSORT_SUCCESS;
  }
  msort_status exchange(RankIO* io, const std::vector<int64_t>& S, msort_dtype kd,
                        msort_dtype vd) {
    const size_t wk = dtype_size(kd);
    auto sp = [&](int r, int j) { return S[(size_t)r * p + j]; };
    LaunchScope ls(KC_EXCHANGE, s);
    for (int me = 0; me < p; ++me) {
      int64_t roff = 0;
      for (int j = 0; j < p; ++j) {
        int64_t rc = sp(me + 1, j) - sp(me, j);
        if (rc > 0) {
          MSORT_CUDA_TRY(cudaMemcpyAsync((char*)io[me].ws.rk + roff * wk,
                                         (char*)io[j].keys + sp(me, j) * wk, rc * wk,
                                         cudaMemcpyDeviceToDevice, s));
          if (vd != MSORT_NONE)
            MSORT_CUDA_TRY(cudaMemcpyAsync((char*)io[me].ws.rv + roff * 4,
                                           (char*)io[j].vals + sp(me, j) * 4, rc * 4,
                                           cudaMemcpyDeviceToDevice, s));
        }
        roff += rc;
      }
    }
    return MSORT_SUCCESS;
  }
  int rank_of(int local) const { return local; }
  // The emulation always takes the device-planned pull path (so it is the one
  // the tests exercise): the shard table is uploaded into rank 0's
  // workspace (its IPC record area, unused in the emulation).
  std::vector<const void*> tab;
  const void* const* reserved_bases(RankIO* io, msort_dtype, bool pairs) {
    if (pairs) return nullptr;
    tab.assign(p, nullptr);
    for (int j = 0; j < p; ++j) tab[j] = io[j].sk;
    auto* d = reinterpret_cast<const void**>(io[0].ws.ipc_all);
    if (cudaMemcpyAsync(d, tab.data(), sizeof(void*) * p, cudaMemcpyHostToDevice, s) !=
        cudaSuccess)
      return nullptr;
    return d;
  }
  msort_status wait(const char* what) {
    cudaError_t e = cudaStreamSynchronize(s);
    return e == cudaSuccess ? MSORT_SUCCESS : cuda_fail(e, what);
  }
  msort_status fetch(void* host, const void* dev, size_t bytes, const char* what) {
    MSORT_CUDA_TRY(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, s));
    return wait(what);
  }
  msort_status barrier(RankIO*) { return MSORT_SUCCESS; }  // one stream: program order
  msort_status ipc_publish(RankIO*, unsigned char*) { return MSORT_SUCCESS; }
  msort_status peer_bases(RankIO* io, const unsigned char*, bool,
                          std::vector<const void*>& bk, std::vector<const uint32_t*>& bv) {
    bk.assign(p, nullptr), bv.assign(p, nullptr);
    for (int j = 0; j < p; ++j) bk[j] = io[j].sk, bv[j] = (const uint32_t*)io[j].sv;
    return MSORT_SUCCESS;
  }
};

template <class K>
static void launch_count(const RankIO& io, int nb, cudaStream_t s) {
  const int warps = nb * B;  // one warp per search
  k4_count<K><<<(warps + 7) / 8, 256, 0, s>>>((const K*)io.sk, (int64_t)io.n, io.ws.lohi, nb,
                                              io.ws.cnt);
}
template <class K>
static void launch_lteq(const RankIO& io, int nb, cudaStream_t s) {
  k4_lteq<K><<<(2 * nb + 7) / 8, 256, 0, s>>>((const K*)io.sk, (int64_t)io.n, io.ws.lohi,
                                              nb, io.ws.lteq);
}

static int rounds_for(msort_dtype kd) { return dtype_size(kd) == 4 ? 4 : 8; }

template <class Coll>
static msort_status dist_run(Coll& C, RankIO* io, int nloc, msort_dtype kd, msort_dtype vd,
                             cudaStream_t s, int64_t* split_out, bool pull_mode) {
  const int p = C.world();
  const int nb = p - 1;
  // D1: local sorts
  for (int l = 0; l < nloc; ++l)
    MSORT_TRY(sort_single_dispatch(io[l].in_keys, io[l].in_vals, io[l].sk, io[l].sv, io[l].n,
                                   kd, vd, io[l].ws.sort_ws, io[l].ws.sort_ws_bytes, s));
  std::vector<int64_t> S((size_t)(p + 1) * p);
  if (p == 1) {
    S[0] = 0, S[1] = (int64_t)io[0].n;
    if (split_out) memcpy(split_out, S.data(), S.size() * 8);
    return MSORT_SUCCESS;
  }
  const uint64_t umax = dtype_size(kd) == 4 ? 0xffffffffull : ~0ull;
  // D2: sizes, then the bucket search, then (lt, eq) and the fill
  for (int l = 0; l < nloc; ++l) {
    LaunchScope ls(KC_SPLITTER, s);
    k4_set_u64<<<1, 1, 0, s>>>(io[l].ws.nsz_send, (uint64_t)io[l].n);
    k4_init<<<(nb + 127) / 128, 128, 0, s>>>(io[l].ws.lohi, nb, umax);
  }
  MSORT_CUDA_TRY(cudaGetLastError());
  MSORT_TRY(C.allgather_u64(io, &DistWs::nsz_send, &DistWs::nsz, 1));
  const int R = rounds_for(kd);
  for (int round = 0; round < R; ++round) {
    for (int l = 0; l < nloc; ++l) {
      LaunchScope ls(KC_SPLITTER, s);
      switch (kd) {
        case MSORT_INT32: launch_count<int32_t>(io[l], nb, s); break;
        case MSORT_UINT32: launch_count<uint32_t>(io[l], nb, s); break;
        case MSORT_INT64: launch_count<int64_t>(io[l], nb, s); break;
        default: launch_count<uint64_t>(io[l], nb, s); break;
      }
    }
    MSORT_CUDA_TRY(cudaGetLastError());
    MSORT_TRY(C.allreduce_u64(io, &DistWs::cnt, (size_t)nb * B));
    for (int l = 0; l < nloc; ++l) {
      LaunchScope ls(KC_SPLITTER, s);
      k4_narrow<<<(nb + 127) / 128, 128, 0, s>>>(io[l].ws.lohi, io[l].ws.cnt, io[l].ws.nsz, p);
    }
    MSORT_CUDA_TRY(cudaGetLastError());
  }
  for (int l = 0; l < nloc; ++l) {
    LaunchScope ls(KC_SPLITTER, s);
    switch (kd) {
      case MSORT_INT32: launch_lteq<int32_t>(io[l], nb, s); break;
      case MSORT_UINT32: launch_lteq<uint32_t>(io[l], nb, s); break;
      case MSORT_INT64: launch_lteq<int64_t>(io[l], nb, s); break;
      default: launch_lteq<uint64_t>(io[l], nb, s); break;
    }
    k4_le_to_eq<<<(nb + 127) / 128, 128, 0, s>>>(io[l].ws.lteq, nb);
  }
  MSORT_CUDA_TRY(cudaGetLastError());
  MSORT_TRY(C.allgather_u64(io, &DistWs::lteq, &DistWs::lteq_all, (size_t)2 * nb));
  for (int l = 0; l < nloc; ++l) {
    LaunchScope ls(KC_SPLITTER, s);
    int tot = (p + 1) * p;
    k4_fill<<<(tot + 127) / 128, 128, 0, s>>>(io[l].ws.lteq_all, io[l].ws.nsz, p, io[l].ws.split);
  }
  MSORT_CUDA_TRY(cudaGetLastError());
  // The one host synchronisation: the exchange sizes are needed on the host.
  const bool pull = pull_mode;
  const size_t wk0 = dtype_size(kd);
  if (pull && vd == MSORT_NONE && p >= 3 && p <= kK5Runs &&
      kway5_scratch_bytes(PullRuns{p, {}, {}, {}}, kd) != SIZE_MAX) {
    // D3 + D4 as ONE K5 launch planned on the device from the split matrix
    // (sync-free once the shard pointers are known on the device: the
    // emulation always, NCCL after msort_comm_reserve)
    const void* const* bases = C.reserved_bases(io, kd, false);
    bool fits = bases != nullptr;
    for (int l = 0; l < nloc && fits; ++l)
      fits = kway5_dev_bytes((int64_t)io[l].n, p, kd) <= io[l].ws.sort_ws_bytes;
    if (fits) {
      msort_status st = MSORT_SUCCESS;
      for (int l = 0; l < nloc && st == MSORT_SUCCESS; ++l)
        st = kway5_dev_dispatch(io[l].ws.split, C.rank_of(l), p, bases, io[l].keys,
                                (int64_t)io[l].n, kd, io[l].ws.sort_ws, io[l].ws.sort_ws_bytes, s);
      // every rank has read the others' segments: exchange buffers are free
      // (the barrier is entered even after a local launch error, so no peer
      // is left waiting in it)
      MSORT_TRY(C.barrier(io));
      if (st != MSORT_SUCCESS) return st;
      if (split_out)  // the only host synchronisation, and only when asked for
        MSORT_TRY(C.fetch(split_out, io[0].ws.split, S.size() * 8, "split matrix"));
      return MSORT_SUCCESS;
    }
  }
  (void)wk0;
  std::vector<unsigned char> ipc_host(pull ? kIpcBytes * (size_t)p : 0);
  if (pull) MSORT_TRY(C.ipc_publish(io, ipc_host.data()));
  MSORT_TRY(C.fetch(S.data(), io[0].ws.split, S.size() * 8, "split matrix"));
  if (split_out) memcpy(split_out, S.data(), S.size() * 8);
  // sanity: every rank's output count equals its input count
  for (int l = 0; l < nloc; ++l) {
    int me = C.rank_of(l);
    int64_t got = 0;
    for (int j = 0; j < p; ++j) got += S[(size_t)(me + 1) * p + j] - S[(size_t)me * p + j];
    if (got != (int64_t)io[l].n) {
      set_error("split matrix inconsistent with local size (ranks disagree on inputs?)");
      return MSORT_ERROR_INVALID_VALUE;
    }
  }
  const size_t wk = dtype_size(kd);
  const bool pairs = vd != MSORT_NONE;
  if (pull) {
    // D3+D4 fused ("pull"): round 1 of the k-way merge reads every rank's
    // sorted segment in place (peer memory over NVLink on a real run), so
    // the segments cross NVLink once, straight into the merge, with no
    // receive-buffer pass through HBM.
    std::vector<const void*> bk;
    std::vector<const uint32_t*> bv;
    MSORT_TRY(C.peer_bases(io, ipc_host.data(), pairs, bk, bv));
    int rounds = 0;
    while ((1 << rounds) < p) ++rounds;
    std::vector<std::vector<int64_t>> offs(nloc);
    std::vector<char> one_pass(nloc, 0);
    for (int l = 0; l < nloc; ++l) {
      const int me = C.rank_of(l);
      offs[l].assign((size_t)p + 1, 0);
      if (io[l].n == 0) continue;
      PullRuns pr{};
      pr.runs = p;
      for (int j = 0; j < p; ++j) {
        const int64_t a = S[(size_t)me * p + j], b = S[(size_t)(me + 1) * p + j];
        pr.k[j] = (const char*)bk[j] + a * wk;
        pr.v[j] = pairs ? bv[j] + a : nullptr;
        pr.n[j] = b - a;
      }
      // keys only, 3..16 runs: the whole D4 is ONE K5 pass reading every
      // segment from its owner (D3 + D4 in one kernel, no receive buffer)
      if (!pairs && p >= 3 && p <= kK5Runs &&
          kway5_scratch_bytes(pr, kd) <= io[l].ws.sort_ws_bytes) {
        MSORT_TRY(kway5_dispatch(pr, io[l].keys, kd, io[l].ws.sort_ws, io[l].ws.sort_ws_bytes, s));
        one_pass[l] = 1;
        continue;
      }
      char* sw = io[l].ws.sort_ws;
      void* tk = sw;
      void* tv = pairs ? sw + align_up(io[l].n * wk, 256) : nullptr;
      void* part = sw + align_up(io[l].n * wk, 256) + (pairs ? align_up(io[l].n * 4, 256) : 0);
      void* ok = rounds == 1 ? io[l].keys : tk;
      void* ov = rounds == 1 ? io[l].vals : tv;
      MSORT_TRY(pull_round_dispatch(pr, ok, ov, offs[l].data(), kd, vd, part, s));
    }
    // every rank has read the others' segments: exchange buffers are free
    MSORT_TRY(C.barrier(io));
    if (rounds > 1) {
      for (int l = 0; l < nloc; ++l) {
        if (io[l].n == 0 || one_pass[l]) continue;
        char* sw = io[l].ws.sort_ws;
        void* tk = sw;
        void* tv = pairs ? sw + align_up(io[l].n * wk, 256) : nullptr;
        void* part = sw + align_up(io[l].n * wk, 256) + (pairs ? align_up(io[l].n * 4, 256) : 0);
        MSORT_TRY(kway_merge_dispatch(tk, tv, io[l].ws.rk, io[l].ws.rv, io[l].keys, io[l].vals,
                                      offs[l].data(), (p + 1) / 2, kd, vd, part, s));
      }
    }
    return MSORT_SUCCESS;
  }
  // D3: exchange
  MSORT_TRY(C.exchange(io, S, kd, vd));
  // D4: k-way merge of the received runs (source-rank order) into keys --
  // one K5 pass for keys only with 3..16 runs, else rounds of K3
  for (int l = 0; l < nloc; ++l) {
    int me = C.rank_of(l);
    std::vector<int64_t> off(p + 1);
    off[0] = 0;
    for (int j = 0; j < p; ++j) off[j + 1] = off[j] + S[(size_t)(me + 1) * p + j] - S[(size_t)me * p + j];
    if (io[l].n == 0) continue;
    char* sw = io[l].ws.sort_ws;  // sort workspace doubles as the ping-pong buffer / K5 scratch
    if (vd == MSORT_NONE && p >= 3 && p <= kK5Runs) {
      PullRuns pr{};
      pr.runs = p;
      for (int j = 0; j < p; ++j) {
        pr.k[j] = (const char*)io[l].ws.rk + off[j] * wk;
        pr.n[j] = off[j + 1] - off[j];
      }
      if (kway5_scratch_bytes(pr, kd) <= io[l].ws.sort_ws_bytes) {
        MSORT_TRY(kway5_dispatch(pr, io[l].keys, kd, sw, io[l].ws.sort_ws_bytes, s));
        continue;
      }
    }
    void* tk = sw;
    void* tv = vd != MSORT_NONE ? sw + align_up(io[l].n * wk, 256) : nullptr;
    void* part = sw + align_up(io[l].n * wk, 256) + (vd != MSORT_NONE ? align_up(io[l].n * 4, 256) : 0);
    MSORT_TRY(kway_merge_dispatch(io[l].ws.rk, io[l].ws.rv, tk, tv, io[l].keys, io[l].vals,
                                  off.data(), p, kd, vd, part, s));
  }
  return MSORT_SUCCESS;
}

msort_status dist_nccl(const void* in_keys, const void* in_vals, void* keys, void* vals, size_t n,
                       msort_dtype kd, msort_dtype vd, msort_comm_s* comm, void* ws,
                       cudaStream_t s, int64_t* split_out) {
  if (comm->aborted) {
    set_error("communicator was aborted after an earlier failure");
    return MSORT_ERROR_NCCL;
  }
  if (comm->world > kMaxWorld) {
    set_error("world too large");
    return MSORT_ERROR_NOT_SUPPORTED;
  }
  const bool pv = vd != MSORT_NONE;
  const int mode = comm->exchange >= 0 ? comm->exchange : exchange_mode();
  const bool pull = mode == 1 && comm->world > 1;
  RankIO io{in_keys, pv ? in_vals : nullptr, keys, pv ? vals : nullptr, n,
            carve(ws, n, kd, vd, comm->world), nullptr, nullptr};
  io.sk = io.keys;
  io.sv = io.vals;
  if (pull) {
    // the sorted shard goes to the communicator's IPC-exportable buffer
    const size_t kb = align_up(n * dtype_size(kd), 256);
    const size_t need = std::max<size_t>(kb + (pv ? align_up(n * 4, 256) : 0), 256);
    if (comm->dbases && (n > comm->reserved_n || dtype_size(kd) > comm->reserved_wk ||
                         (pv && !comm->reserved_vals))) {
      // the peers hold mappings of the reserved buffer: it cannot move
      set_error("pull exchange: n_local exceeds the msort_comm_reserve reservation");
      return MSORT_ERROR_INVALID_VALUE;
    }
    if (need > comm->xbuf_bytes) {
      // the previous call ended with a barrier after every peer's reads, so
      // the old buffer is free; wait for this stream's earlier work too
      MSORT_CUDA_TRY(cudaStreamSynchronize(s));
      if (comm->xbuf) cudaFree(comm->xbuf);
      comm->xbuf = nullptr, comm->xbuf_bytes = 0;
      MSORT_CUDA_TRY(cudaMalloc(&comm->xbuf, need + need / 8));
      comm->xbuf_bytes = need + need / 8;
    }
    io.sk = comm->xbuf;
    io.sv = pv ? static_cast<char*>(comm->xbuf) + kb : nullptr;
  }
  NcclColl C{comm, s};
  return dist_run(C, &io, 1, kd, vd, s, split_out, pull);
}

// msort_comm_reserve: allocate the pull exchange buffer for up to n_max local
// keys (+ 4-byte payloads), publish it through CUDA IPC, open every peer's,
// and keep the table of the p shard pointers on the device.  Collective.
msort_status comm_reserve(msort_comm_s* c, size_t n_max, msort_dtype kd, msort_dtype vd,
                          cudaStream_t s) {
  if (c->aborted) {
    set_error("communicator was aborted after an earlier failure");
    return MSORT_ERROR_NCCL;
  }
  const int p = c->world;
  const bool pv = vd != MSORT_NONE;
  const size_t kb = align_up(n_max * dtype_size(kd), 256);
  const size_t need = std::max<size_t>(kb + (pv ? align_up(n_max * 4, 256) : 0), 256);
  if (need > c->xbuf_bytes) {
    MSORT_CUDA_TRY(cudaStreamSynchronize(s));
    if (c->xbuf) cudaFree(c->xbuf);
    c->xbuf = nullptr, c->xbuf_bytes = 0;
    MSORT_CUDA_TRY(cudaMalloc(&c->xbuf, need));
    c->xbuf_bytes = need;
  }
  // device scratch for the IPC record gather
  unsigned char* rec = nullptr;
  MSORT_CUDA_TRY(scratch_alloc(reinterpret_cast<void**>(&rec), kIpcBytes * (size_t)(p + 1), s));
  struct Free {
    unsigned char* q;
    cudaStream_t s;
    ~Free() { cudaFreeAsync(q, s); }
  } fr{rec, s};
  RankIO io{};
  io.sk = c->xbuf;
  io.sv = pv ? static_cast<char*>(c->xbuf) + kb : nullptr;
  io.ws.ipc_send = rec;
  io.ws.ipc_all = rec + kIpcBytes;
  NcclColl C{c, s};
  std::vector<unsigned char> host(kIpcBytes * (size_t)p);
  MSORT_TRY(C.ipc_publish(&io, host.data()));
  std::vector<const void*> bk;
  std::vector<const uint32_t*> bv;
  MSORT_TRY(C.peer_bases(&io, host.data(), pv, bk, bv));
  if (!c->dbases)
    MSORT_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&c->dbases), sizeof(void*) * p));
  memcpy(c->pinned, bk.data(), sizeof(void*) * p);
  MSORT_CUDA_TRY(cudaMemcpyAsync(c->dbases, c->pinned, sizeof(void*) * p, cudaMemcpyHostToDevice, s));
  MSORT_TRY(wait_stream_nccl(c, s, "reserve"));
  c->reserved_n = n_max;
  c->reserved_wk = dtype_size(kd);
  c->reserved_vals = pv;
  return MSORT_SUCCESS;
}

msort_status dist_emulated(void* const* keys, void* const* vals, const size_t* n, int world,
                           msort_dtype kd, msort_dtype vd, void* const* ws, cudaStream_t s,
                           int64_t* split_out) {
  if (world > kMaxWorld) {
    set_error("world too large");
    return MSORT_ERROR_NOT_SUPPORTED;
  }
  std::vector<RankIO> io(world);
  for (int r = 0; r < world; ++r)
  {
    void* v = vd == MSORT_NONE || !vals ? nullptr : vals[r];
    io[r] = RankIO{keys[r], v, keys[r], v, n[r], carve(ws[r], n[r], kd, vd, world), nullptr,
                   nullptr};
    const bool pull = exchange_mode() == 1 && world > 1;
    io[r].sk = pull ? io[r].ws.rk : io[r].keys;
    io[r].sv = pull ? io[r].ws.rv : io[r].vals;
  }
  EmulColl C{world, s};
  return dist_run(C, io.data(), world, kd, vd, s, split_out, exchange_mode() == 1 && world > 1);
}

// ------------------------------------------------ rank-tree gather (f4)
// The paper's own distribution (fig. mpi-merge-code): every rank
// sorts its shard; then, while more than one rank is active, the upper half
// of the active ranks (right children) send their sorted arrays to rank -
// split and the lower half (left children / parents) merge their own array
// (left, first on ties: merge() of P:516) with the received one.  Rank 0 ends
// with everything.  `split` = active / 2 for the paper's power-of-two worlds
// (P:402); other worlds use ceil(active / 2) parents, the same pairing
// rank <- rank + split with an odd rank out (R12/R13).
// Order of the shards after the tree (ties resolve in this order).
static void tree_rounds(int p, std::vector<std::vector<std::pair<int, int>>>& rounds) {
  rounds.assign(plan::tree_rounds(p), {});
  for (int t = 0; t < (int)rounds.size(); ++t)
    for (int r = 0; r < p; ++r) {
      int peer = -1;
      if (plan::tree_role(p, r, t, &peer) == 1) rounds[t].push_back({r, peer});  // (parent, child)
    }
}

struct TreeBufs {
  void *ak, *av, *bk, *bv;  // [own | received] and the merge target
  void* part;               // K3 scheduler counters
  int64_t cnt;              // elements currently held
};

// Collective-specific pieces of the tree: NCCL send/recv, or device copies
// between the virtual ranks' buffers.
struct TreeNccl {
  msort_comm_s* c;
  cudaStream_t s;
  msort_status move(std::vector<TreeBufs>& tb, int parent, int child, int64_t cnt, msort_dtype kd,
                    msort_dtype vd) {
    const int me = c->rank;
    if (me != parent && me != child) return MSORT_SUCCESS;
    TreeBufs& b = tb[0];
    const size_t wk = dtype_size(kd);
    LaunchScope ls(KC_EXCHANGE, s);
    NcclGroup grp;
    MSORT_NCCL_TRY(grp.start());
    if (me == child) {
      MSORT_NCCL_TRY(ncclSend(b.ak, (size_t)cnt, nccl_type(kd), parent, c->comm, s));
      if (vd != MSORT_NONE)
        MSORT_NCCL_TRY(ncclSend(b.av, (size_t)cnt, ncclUint32, parent, c->comm, s));
    } else {
      MSORT_NCCL_TRY(ncclRecv((char*)b.ak + b.cnt * wk, (size_t)cnt, nccl_type(kd), child,
                              c->comm, s));
      if (vd != MSORT_NONE)
        MSORT_NCCL_TRY(ncclRecv((char*)b.av + b.cnt * 4, (size_t)cnt, ncclUint32, child, c->comm,
                                s));
    }
    MSORT_NCCL_TRY(grp.end());
    return MSORT_SUCCESS;
  }
  int local(int rank) const { return rank == c->rank ? 0 : -1; }
  // Collective agreement before any point-to-point transfer: every rank
  // learns whether all ranks are ready (one all-reduce MIN of a flag and a
  // host wait), so a rank that fails never leaves its peers blocked in a
  // send or receive that it will not post.
  msort_status agree(bool ok, const char* what) {
    uint64_t* d = c->dscratch + 2 * (size_t)c->world;
    uint64_t* h = reinterpret_cast<uint64_t*>(c->pinned + c->pinned_bytes - 64);
    h[0] = ok ? 1 : 0;
    MSORT_CUDA_TRY(cudaMemcpyAsync(d, h, 8, cudaMemcpyHostToDevice, s));
    {
      LaunchScope ls(KC_NCCL, s);
      MSORT_NCCL_TRY(ncclAllReduce(d, d, 1, ncclUint64, ncclMin, c->comm, s));
    }
    MSORT_CUDA_TRY(cudaMemcpyAsync(h + 1, d, 8, cudaMemcpyDeviceToHost, s));
    MSORT_TRY(wait_stream_nccl(c, s, what));
    if (h[1] == 0 && ok) {
      set_error(std::string(what) + ": another rank failed");
      return MSORT_ERROR_OUT_OF_MEMORY;
    }
    return MSORT_SUCCESS;
  }
};
struct TreeEmul {
  cudaStream_t s;
  msort_status move(std::vector<TreeBufs>& tb, int parent, int child, int64_t cnt, msort_dtype kd,
                    msort_dtype vd) {
    const size_t wk = dtype_size(kd);
    LaunchScope ls(KC_EXCHANGE, s);
    MSORT_CUDA_TRY(cudaMemcpyAsync((char*)tb[parent].ak + tb[parent].cnt * wk, tb[child].ak,
                                   cnt * wk, cudaMemcpyDeviceToDevice, s));
    if (vd != MSORT_NONE)
      MSORT_CUDA_TRY(cudaMemcpyAsync((char*)tb[parent].av + tb[parent].cnt * 4, tb[child].av,
                                     cnt * 4, cudaMemcpyDeviceToDevice, s));
    return MSORT_SUCCESS;
  }
  int local(int rank) const { return rank; }
  msort_status agree(bool, const char*) { return MSORT_SUCCESS; }
};

// ranks: the global ranks this process drives (one for NCCL, all for the
// emulation); in_k/in_v per driven rank; nall: every rank's shard size.
template <class Coll>
static msort_status tree_run(Coll& C, const std::vector<int>& ranks,
                             const std::vector<const void*>& in_k,
                             const std::vector<const void*>& in_v,
                             const std::vector<int64_t>& nall, msort_dtype kd, msort_dtype vd,
                             void* root_k, void* root_v, cudaStream_t s) {
  const int p = (int)nall.size();
  const size_t wk = dtype_size(kd);
  const bool pairs = vd != MSORT_NONE;
  std::vector<std::vector<std::pair<int, int>>> rounds;
  tree_rounds(p, rounds);
  // subtree sizes: what each parent will hold at most
  std::vector<int64_t> sub(nall);
  for (auto& r : rounds)
    for (auto& pc : r) sub[pc.first] += sub[pc.second];
  std::vector<TreeBufs> tb(ranks.size());
  std::vector<void*> allocs;
  auto alloc = [&](size_t bytes) -> void* {
    void* q = nullptr;
    if (scratch_alloc(&q, std::max<size_t>(bytes, 256), s) != cudaSuccess) return nullptr;
    allocs.push_back(q);
    return q;
  };
  struct Freer {
    std::vector<void*>* a;
    cudaStream_t s;
    ~Freer() {
      for (void* q : *a) cudaFreeAsync(q, s);
    }
  } freer{&allocs, s};
  std::vector<void*> sws(ranks.size(), nullptr);
  bool ok = true;
  for (size_t l = 0; l < ranks.size(); ++l) {
    const int r = ranks[l];
    const size_t cap = (size_t)sub[r];
    TreeBufs& b = tb[l];
    b.ak = alloc(cap * wk), b.bk = alloc(cap * wk);
    b.av = pairs ? alloc(cap * 4) : nullptr, b.bv = pairs ? alloc(cap * 4) : nullptr;
    b.part = alloc(4096);
    sws[l] = alloc(single_ws_bytes((size_t)nall[r], kd, vd));
    ok = ok && b.ak && b.bk && (!pairs || (b.av && b.bv)) && b.part && sws[l];
  }
  // every rank agrees before the first transfer (a rank that could not
  // allocate must not leave the others waiting in a send / receive)
  MSORT_TRY(C.agree(ok, "tree sort: buffers"));
  if (!ok) {
    set_error("tree sort: out of device memory");
    return MSORT_ERROR_OUT_OF_MEMORY;
  }
  for (size_t l = 0; l < ranks.size(); ++l) {
    const int r = ranks[l];
    TreeBufs& b = tb[l];
    // D1: the local sort (the paper's subsort), into [own | ...]
    MSORT_TRY(sort_single_dispatch(in_k[l], pairs ? in_v[l] : nullptr, b.ak, b.av,
                                   (size_t)nall[r], kd, vd, sws[l],
                                   single_ws_bytes((size_t)nall[r], kd, vd), s));
    b.cnt = nall[r];
  }
  std::vector<int64_t> cnt(nall);  // every rank's count, tracked on every process
  for (size_t t = 0; t < rounds.size(); ++t) {
    const bool last = t + 1 == rounds.size();
    for (auto& pc : rounds[t]) {
      const int parent = pc.first, child = pc.second;
      if (cnt[child] > 0) MSORT_TRY(C.move(tb, parent, child, cnt[child], kd, vd));
      const int lp = C.local(parent);
      // nothing received: nothing to merge, except that the root's last round
      // writes the output
      if (lp >= 0 && (cnt[child] > 0 || (last && parent == 0))) {
        // merge(local, tmp) -> result: runs [0, own) and [own, own + recv)
        TreeBufs& b = tb[(size_t)lp];
        const int64_t off[3] = {0, cnt[parent], cnt[parent] + cnt[child]};
        void* dk = (last && parent == 0) ? root_k : b.bk;
        void* dv = (last && parent == 0) ? root_v : b.bv;
        MSORT_TRY(kway_merge_dispatch(b.ak, b.av, b.bk, b.bv, dk, dv, off, 2, kd, vd, b.part, s));
        if (!(last && parent == 0)) std::swap(b.ak, b.bk), std::swap(b.av, b.bv);
        b.cnt = off[2];
      }
      cnt[parent] += cnt[child];
    }
  }
  const int l0 = C.local(0);
  if (rounds.empty() && l0 >= 0 && nall[0] > 0) {  // one rank: the sorted shard is the result
    MSORT_CUDA_TRY(cudaMemcpyAsync(root_k, tb[(size_t)l0].ak, nall[0] * wk,
                                   cudaMemcpyDeviceToDevice, s));
    if (pairs)
      MSORT_CUDA_TRY(cudaMemcpyAsync(root_v, tb[(size_t)l0].av, nall[0] * 4,
                                     cudaMemcpyDeviceToDevice, s));
  }
  // the buffers are freed on the stream (stream-ordered) by the Freer
  return MSORT_SUCCESS;
}

msort_status tree_nccl(const void* in_keys, const void* in_vals, size_t n, msort_dtype kd,
                       msort_dtype vd, msort_comm_s* comm, void* root_k, void* root_v,
                       size_t root_cap, cudaStream_t s, int64_t* total_out) {
  if (comm->aborted) {
    set_error("communicator was aborted after an earlier failure");
    return MSORT_ERROR_NCCL;
  }
  const int p = comm->world;
  // every rank's (size, root capacity): one all-gather, one host sync; the
  // capacity check is then the same decision on every rank
  uint64_t* d = comm->dscratch;  // [p x (n, cap)] gathered, [2] sent
  uint64_t* h = reinterpret_cast<uint64_t*>(comm->pinned);
  h[0] = (uint64_t)n;
  h[1] = comm->rank == 0 ? (uint64_t)root_cap : 0;
  cudaError_t e = cudaMemcpyAsync(d + 2 * p, h, 16, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "tree sizes");
  {
    LaunchScope ls(KC_NCCL, s);
    MSORT_NCCL_TRY(ncclAllGather(d + 2 * p, d, 2, ncclUint64, comm->comm, s));
  }
  MSORT_CUDA_TRY(cudaMemcpyAsync(comm->pinned + 64, d, 16 * (size_t)p, cudaMemcpyDeviceToHost, s));
  MSORT_TRY(wait_stream_nccl(comm, s, "tree sizes"));
  const uint64_t* g = reinterpret_cast<const uint64_t*>(comm->pinned + 64);
  std::vector<int64_t> nall((size_t)p);
  int64_t total = 0;
  for (int r = 0; r < p; ++r) nall[r] = (int64_t)g[2 * r], total += nall[r];
  const uint64_t cap0 = g[1];
  if (total_out) *total_out = total;
  if ((uint64_t)total > cap0) {  // decided identically on every rank
    set_error("tree sort: root output holds " + std::to_string(cap0) + " elements, need " +
              std::to_string(total));
    return MSORT_ERROR_INVALID_VALUE;
  }
  TreeNccl C{comm, s};
  return tree_run(C, {comm->rank}, {in_keys}, {in_vals}, nall, kd, vd, root_k, root_v, s);
}

msort_status tree_emulated(const void* const* keys, const void* const* vals, const size_t* n,
                           int world, msort_dtype kd, msort_dtype vd, void* root_k, void* root_v,
                           cudaStream_t s) {
  std::vector<int> ranks(world);
  std::vector<const void*> ik(world), iv(world);
  std::vector<int64_t> nall(world);
  for (int r = 0; r < world; ++r) {
    ranks[r] = r, ik[r] = keys[r], iv[r] = vals ? vals[r] : nullptr, nall[r] = (int64_t)n[r];
  }
  TreeEmul C{s};
  return tree_run(C, ranks, ik, iv, nall, kd, vd, root_k, root_v, s);
}

// Process default of the exchange mode (communicators may override it):
// MSORT_EXCHANGE=pull, or msort_debug_set_exchange.  Atomic: a concurrent
// call sees either the old or the new mode.
static std::atomic<int> g_exchange_mode{-1};
int exchange_mode() {
  int m = g_exchange_mode.load(std::memory_order_acquire);
  if (m < 0) {
    const char* e = getenv("MSORT_EXCHANGE");
    m = e && std::string(e) == "pull" ? 1 : 0;
    int expect = -1;
    g_exchange_mode.compare_exchange_strong(expect, m, std::memory_order_acq_rel);
    m = g_exchange_mode.load(std::memory_order_acquire);
  }
  return m;
}
void set_exchange_mode(int m) { g_exchange_mode.store(m, std::memory_order_release); }

msort_status comm_unique_id(void* out) {
  ncclUniqueId id;
  MSORT_NCCL_TRY(ncclGetUniqueId(&id));
  memcpy(out, &id, sizeof(id));
  return MSORT_SUCCESS;
}

// The communicator's page-locked staging and small device scratch.
static msort_status comm_buffers(msort_comm_s* cs) {
  const size_t w = (size_t)cs->world;
  cs->pinned_bytes = std::max<size_t>({8 * (w + 1) * w, kIpcBytes * w, 16 * w + 64}) + 4096;
  if (cudaMallocHost(reinterpret_cast<void**>(&cs->pinned), cs->pinned_bytes) != cudaSuccess) {
    cs->pinned = nullptr;
    set_error("cudaMallocHost (communicator staging)");
    return MSORT_ERROR_OUT_OF_MEMORY;
  }
  if (cudaMalloc(reinterpret_cast<void**>(&cs->dscratch), 8 * (2 * w + 64)) != cudaSuccess) {
    cudaFreeHost(cs->pinned);
    cs->pinned = nullptr, cs->dscratch = nullptr;
    set_error("cudaMalloc (communicator scratch)");
    return MSORT_ERROR_OUT_OF_MEMORY;
  }
  return MSORT_SUCCESS;
}

msort_status comm_init(const void* idp, int rank, int world, msort_comm_s** out) {
  ncclUniqueId id;
  memcpy(&id, idp, sizeof(id));
  ncclComm_t c;
  MSORT_NCCL_TRY(ncclCommInitRank(&c, world, id, rank));
  auto* cs = new msort_comm_s{c, rank, world, {}};
  msort_status st = comm_buffers(cs);
  if (st != MSORT_SUCCESS) {
    ncclCommDestroy(c);
    delete cs;
    return st;
  }
  *out = cs;
  return MSORT_SUCCESS;
}

// Wrap an existing NCCL communicator (e.g. torch's, msort_comm_wrap): rank and
// world come from NCCL itself; the caller keeps ownership.
msort_status comm_wrap(void* nccl_comm, msort_comm_s** out) {
  ncclComm_t c = static_cast<ncclComm_t>(nccl_comm);
  int rank = 0, world = 0;
  MSORT_NCCL_TRY(ncclCommUserRank(c, &rank));
  MSORT_NCCL_TRY(ncclCommCount(c, &world));
  auto* cs = new msort_comm_s{c, rank, world, {}};
  cs->owned = false;
  msort_status st = comm_buffers(cs);
  if (st != MSORT_SUCCESS) {
    delete cs;
    return st;
  }
  *out = cs;
  return MSORT_SUCCESS;
}

msort_status comm_destroy(msort_comm_s* c) {
  if (!c) return MSORT_SUCCESS;
  for (auto& kv : c->ipc_open) cudaIpcCloseMemHandle(kv.second);
  ncclResult_t r = (c->aborted || !c->owned) ? ncclSuccess : ncclCommDestroy(c->comm);
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->dscratch) cudaFree(c->dscratch);
  if (c->xbuf) cudaFree(c->xbuf);
  if (c->dbases) cudaFree(c->dbases);
  delete c;
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
  return MSORT_SUCCESS;
}

int comm_world(msort_comm_s* c) { return c->world; }

}  // namespace msort

extern "C" int msort_debug_set_exchange(int mode) {
  msort::set_exchange_mode(mode ? 1 : 0);
  return 0;
}

extern "C" msort_status msort_comm_set_exchange(msort_comm_t comm, int mode) {
  if (!comm || mode < -1 || mode > 1) {
    msort::set_error("msort_comm_set_exchange: null communicator or mode not in {-1, 0, 1}");
    return MSORT_ERROR_INVALID_VALUE;
  }
  comm->exchange = mode;
  return MSORT_SUCCESS;
}

