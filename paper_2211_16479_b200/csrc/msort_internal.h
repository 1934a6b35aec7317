// msort_internal.h -- host-side plumbing shared by the library's translation
// units (error text, kernel accounting, workspace carving, tile geometry).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <string>

#include "../../include/msort.h"

namespace msort {

// ---------------------------------------------------------------- errors
void set_error(const std::string& s);
msort_status cuda_fail(cudaError_t e, const char* what);
#define MSORT_CUDA_TRY(expr)                                            \
  do {                                                                  \
    cudaError_t _e = (expr);                                            \
    if (_e != cudaSuccess) return ::msort::cuda_fail(_e, #expr);        \
  } while (0)
#define MSORT_TRY(expr)                                                 \
  do {                                                                  \
    msort_status _s = (expr);                                           \
    if (_s != MSORT_SUCCESS) return _s;                                 \
  } while (0)

// ------------------------------------------------------ kernel accounting
enum KernelClass { KC_TILE_SORT = 0, KC_PARTITION = 1, KC_MERGE = 2, KC_SPLITTER = 3,
                   KC_KWAY = 4, KC_NCCL = 5, KC_EXCHANGE = 6, KC_KEY_RANGE = 7 };

// Bracket a kernel launch: counts it, and when profiling is on records a
// pair of CUDA events on the launching stream.
struct LaunchScope {
  LaunchScope(KernelClass kc, cudaStream_t s);
  ~LaunchScope();
  KernelClass kc;
  cudaStream_t s;
  int slot;
};

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// The library's own scratch allocations (the calls without a caller
// workspace): stream-ordered from the library's own memory pool for the
// current device (abi.cu), whose freed blocks are reused by the next call
// instead of being unmapped and mapped again; the default pool is untouched.
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s);

size_t dtype_size(msort_dtype d);
int tile_size_for(msort_dtype kd, msort_dtype vd);

// Single-GPU workspace: [keys n*wk][vals n*4][partition (ntiles+1)*8].
size_t single_ws_bytes(size_t n, msort_dtype kd, msort_dtype vd);

// Distributed extras: receive buffers + splitter scratch.
constexpr int kCandidates = 256;  // candidates per boundary per round (8 bits)
size_t dist_ws_bytes(size_t n, msort_dtype kd, msort_dtype vd, int world);

// Single-GPU sort with explicit workspace (sort_single.cu): sorts in_keys/
// in_vals into keys/vals (the same pointers for an in-place sort).
msort_status tree_emulated(const void* const* keys, const void* const* vals, const size_t* n,
                           int world, msort_dtype kd, msort_dtype vd, void* root_k, void* root_v,
                           cudaStream_t s);
msort_status sort_segmented_dispatch(void* keys, void* vals, const int64_t* off, size_t nseg,
                                     bool dev_off, size_t n, msort_dtype kd, msort_dtype vd,
                                     void* ws, size_t ws_bytes, cudaStream_t s);
msort_status sort_single_dispatch(const void* in_keys, const void* in_vals, void* keys,
                                  void* vals, size_t n, msort_dtype kd, msort_dtype vd, void* ws,
                                  size_t ws_bytes, cudaStream_t s);

// Stable merge of `runs` consecutive sorted runs (run r = [off[r], off[r+1]) of
// src) into dst, ties to the lower run; used by the distributed k-way merge.
// Ping-pongs through tmp; the result lands in dst.  (sort_single.cu)
msort_status kway_merge_dispatch(void* src_k, void* src_v, void* tmp_k, void* tmp_v,
                                 void* dst_k, void* dst_v, const int64_t* off_host, int runs,
                                 msort_dtype kd, msort_dtype vd, void* part_ws, cudaStream_t s);

// Runs of the pull exchange's first merge round: run r is n[r] keys at k[r]
// (payloads at v[r]) -- device pointers, possibly into a peer GPU's memory.
constexpr int kMaxPullRuns = 128;
struct PullRuns {
  int runs;
  const void* k[kMaxPullRuns];
  const uint32_t* v[kMaxPullRuns];
  int64_t n[kMaxPullRuns];
};
// Merges runs (2m, 2m+1) into out (pair m at the sum of the earlier pairs'
// sizes); off_out gets the ceil(runs/2)+1 boundaries of the result.
msort_status pull_round_dispatch(const PullRuns& pr, void* out_k, void* out_v, int64_t* off_out,
                                 msort_dtype kd, msort_dtype vd, void* part_ws, cudaStream_t s);

// D4 in one pass (K5, k5_kway.cuh): stable merge of pr.runs sorted runs of
// keys (run j = pr.n[j] keys at pr.k[j], possibly peer memory; ties to the
// lower run) into dst.  Keys only.  scratch: device memory of at least
// kway5_scratch_bytes(pr, kd) bytes (a small fraction of the keys), which is
// SIZE_MAX when K5 does not take that run count (3..8 by default, see
// Kernels::k5_max_runs) -- the caller then merges by K3 rounds.
constexpr int kK5Runs = 16;
msort_status kway5_dispatch(const PullRuns& pr, void* dst, msort_dtype kd, void* scratch,
                            size_t scratch_bytes, cudaStream_t s);
size_t kway5_scratch_bytes(const PullRuns& pr, msort_dtype kd);
// The same merge planned on the device (k5_plan_dev): rank `me` of p merges
// its segments [S[me][j], S[me+1][j]) of every rank j's sorted shard (split
// matrix `split` and shard table `bases` in device memory) into dst (n_out
// keys).  No host synchronisation.  scratch >= kway5_dev_bytes(n_out, p, kd).
size_t kway5_dev_bytes(int64_t n_out, int p, msort_dtype kd);
msort_status kway5_dev_dispatch(const int64_t* split, int me, int p, const void* const* bases,
                                void* dst, int64_t n_out, msort_dtype kd, void* scratch,
                                size_t scratch_bytes, cudaStream_t s);

// msort_merge_runs: workspace bytes and the call (sort_single.cu).
size_t merge_runs_ws_bytes(size_t n, int p, msort_dtype kd, msort_dtype vd);
msort_status merge_runs_dispatch(const void* ik, const void* iv, const int64_t* off, int p,
                                 void* ok, void* ov, msort_dtype kd, msort_dtype vd, void* ws,
                                 size_t ws_bytes, cudaStream_t s);

// Exchange mode of the distributed sort: 0 = NCCL all-to-all into a receive
// buffer then a local k-way merge; 1 = pull (the first merge round reads the
// peers' sorted segments in place).  (sort_dist.cu, msort_debug_set_exchange)
int exchange_mode();

}  // namespace msort
