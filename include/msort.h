/*
 * msort.h -- C ABI of the B200-native (sm_100a) stable merge sort.
 *
 * The operation (arXiv 2211.16479, /root/reference/PAPER.md; "P:n" = line n):
 * sort an array of integer keys ascending, as merge sort does
 * (P:77-84 [Sequential Merge Sort, steps 1-4], Fig. fig:mergesort P:88-112),
 * stably (equal keys keep their input order -- the tie rule of merge(),
 * P:107, read as "left run first", R1), optionally carrying a
 * payload; and the distributed variant in which each process sorts its shard
 * and the shards are merged across processes (P:398-525 [MPI Merge Sort],
 * Figs. fig:mpi-scatter-code, fig:mpi-merge-code), here as a balanced,
 * globally sorted layout across ranks (R10).
 *
 * Result contract: element i of the input lands at position
 *     pos(i) = #{j : k_j < k_i} + #{j < i : k_j = k_i},
 * which is unique, so results are bit-exact to the CPU oracle (oracle/).
 *
 * Conventions for every call:
 *  - keys/vals/ws are DEVICE pointers on the current CUDA device; the caller
 *    owns them, the library never frees them.  Host pointers are only the
 *    explicitly marked `host` arguments.
 *  - Sorting is in place: the sorted output overwrites keys (and vals).
 *  - Layout: structure of arrays, keys[n] and vals[n], contiguous; pointers
 *    must be aligned to their element size (16-byte alignment is NOT needed).
 *  - Calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy default
 *    stream) and never synchronise, except msort_sort_distributed*, which
 *    synchronises `stream` once to read the split matrix (documented there).
 *    Execution faults surface at the caller's next synchronisation.
 *  - Errors are returned synchronously as msort_status; nothing throws across
 *    the ABI.  msort_last_error() returns thread-local detail text.
 *  - n == 0 or n == 1 is a successful no-op without any launch ("if the input
 *    array has less than two elements, return").
 *  - INVALID_VALUE: NULL pointer with n > 0, misaligned pointer, keys/vals
 *    overlapping, unknown dtype, n > 2^40, workspace too small.
 *    NOT_SUPPORTED: device is not sm_100 or the dtype combination is not built
 *    (payloads: MSORT_UINT32 / MSORT_INT32 only, i.e. 4-byte payloads).
 *  - Thread safety: calls are re-entrant; one msort_comm_t must not be used by
 *    two calls at once (an NCCL rule).
 *
 * There is no CPU fallback: every step runs in the library's sm_100a kernels.
 */
#ifndef MSORT_H
#define MSORT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MSORT_INT32 = 0,
  MSORT_UINT32 = 1,
  MSORT_INT64 = 2,
  MSORT_UINT64 = 3,
  MSORT_NONE = 255 /* "no payload" for val_dtype */
} msort_dtype;

typedef enum {
  MSORT_SUCCESS = 0,
  MSORT_ERROR_INVALID_VALUE = 1,
  MSORT_ERROR_NOT_SUPPORTED = 2,
  MSORT_ERROR_OUT_OF_MEMORY = 3,
  MSORT_ERROR_CUDA = 4,
  MSORT_ERROR_NCCL = 5
} msort_status;

/* A cudaStream_t, passed as an opaque pointer so this header needs no CUDA. */
typedef void *msort_stream_t;

/* Opaque communicator (owns one NCCL communicator).  Caller-owned. */
typedef struct msort_comm_s *msort_comm_t;

/* ---------------------------------------------------------------- single GPU */

/* Stable ascending sort of keys[0..n) in place.  Workspace of
 * msort_workspace_bytes(n, key_dtype, MSORT_NONE, 1) bytes is taken with
 * cudaMallocFromPoolAsync/cudaFreeAsync on `stream` from the library's own
 * memory pool for the current device (created on first use; its freed blocks
 * stay reserved for the next call).  The device's default pool is never
 * modified.  The same holds for every call that allocates scratch itself. */
msort_status msort_sort(void *keys, size_t n, msort_dtype key_dtype, msort_stream_t stream);

/* Stable ascending sort of (keys, vals) pairs by key; vals travel with their
 * keys and equal keys keep input order (P:107 tie rule, R1).
 * val_dtype must be a 4-byte type (MSORT_UINT32 or MSORT_INT32). */
msort_status msort_sort_pairs(void *keys, void *vals, size_t n, msort_dtype key_dtype,
                              msort_dtype val_dtype, msort_stream_t stream);

/* Bytes of device workspace the *_ws calls need: for world <= 1 about
 * n*(wk+wv) (the O(n) extra space of merge sort) plus n/256*8 bytes of
 * merge-path partitions; for world > 1 (n = local count) also an n*(wk+wv)
 * receive buffer and O(world*256) splitter buffers.  For 8-byte keys the
 * single-GPU size also covers the key-range narrowed path (n > 2^16: keys
 * whose values span fewer than 2^32 are sorted as 32-bit offsets from their
 * minimum -- same output, half the key bytes per merge pass; chosen on the
 * device, so the call stays asynchronous) and 256 bytes for
 * the measured range.  bytes: host out. */
msort_status msort_workspace_bytes(size_t n, msort_dtype key_dtype, msort_dtype val_dtype,
                                   int world, size_t *bytes);

/* msort_sort / msort_sort_pairs with caller-supplied device workspace
 * (e.g. from the PyTorch caching allocator).  vals may be NULL with
 * val_dtype == MSORT_NONE.  ws must be 256-byte aligned and at least
 * msort_workspace_bytes(n, key_dtype, val_dtype, 1) bytes; it must not overlap
 * keys/vals.  Nothing is allocated and nothing synchronises, so this call (and
 * msort_sort_out_ws) can be captured into a CUDA graph: a replay sorts whatever
 * the buffers hold (after one uncaptured call has done the library's one-time
 * kernel setup).  The segmented, distributed and host-buffer calls are not
 * capturable (host-side tables / synchronisation). */
msort_status msort_sort_ws(void *keys, void *vals, size_t n, msort_dtype key_dtype,
                           msort_dtype val_dtype, void *ws, size_t ws_bytes,
                           msort_stream_t stream);

/* Out-of-place form (the paper's sorts return a new array):
 * sorts in_keys/in_vals (read only, unchanged) into keys_out/vals_out.  The
 * input may equal the output (then it is msort_sort_ws) but must not
 * partially overlap it.  Same workspace as msort_sort_ws; no extra HBM pass:
 * the tile sort reads the input directly. */
msort_status msort_sort_out_ws(const void *in_keys, const void *in_vals, void *keys_out,
                               void *vals_out, size_t n, msort_dtype key_dtype,
                               msort_dtype val_dtype, void *ws, size_t ws_bytes,
                               msort_stream_t stream);

/* Batched (segmented) sort -- SURVEY.md §8(f) f3, the paper's small-array
 * regime (below a size the parallel overhead dominates, so
 * many small arrays are sorted in one call instead of one call each).
 * Sorts every segment keys[off[i], off[i+1]) (and vals alike) independently,
 * ascending and stable, in place: segment i ends as msort_sort_pairs of that
 * slice alone (P:77-84 applied per segment).
 *   seg_offsets  nseg + 1 int64: off[0] = 0, non-decreasing, off[nseg] = n
 *                (empty segments allowed).  In HOST memory it is read during
 *                the call (from 2^15 segments on it is copied up and
 *                classified on the device, as below); in DEVICE memory
 *                (cudaPointerGetAttributes says so) the segments are
 *                classified and the table checked on the device, and the call
 *                synchronises `stream` once to learn how many long segments
 *                there are.
 *   keys, vals   device arrays of n elements (vals NULL with MSORT_NONE).
 *   ws           device workspace, 256-byte aligned, at least
 *                msort_segmented_workspace_bytes(n, nseg, ...) bytes, not
 *                overlapping keys/vals.
 * Segments of <= 256 elements are sorted one per warp, <= msort_tile_size
 * one per CTA, longer ones by the single-array sort (one after another).
 * With a host table of fewer than 2^15 segments the call is asynchronous on
 * `stream` (its tables are staged through page-locked memory and uploaded on
 * the stream).
 * Errors: INVALID_VALUE for bad offsets (not starting at 0, decreasing, not
 * ending at n -- found on the device for device offsets, before any key is
 * touched), NULL pointers with n > 0, a bad dtype or a short workspace. */
msort_status msort_segmented_workspace_bytes(size_t n, size_t nseg, msort_dtype key_dtype,
                                             msort_dtype val_dtype, size_t *bytes);
msort_status msort_sort_segmented(void *keys, void *vals, size_t n, const int64_t *seg_offsets,
                                  size_t nseg, msort_dtype key_dtype, msort_dtype val_dtype,
                                  void *ws, size_t ws_bytes, msort_stream_t stream);

/* End-to-end sort of HOST arrays (the e2e path of bench.py).  Enqueued on
 * `stream`: host_keys[0..n) (and host_vals) are copied into the caller's
 * device buffers dev_keys (dev_vals), sorted there in place (msort_sort_ws,
 * same workspace), and copied back to host_keys_out (host_vals_out).  With
 * page-locked host buffers the call is asynchronous (returns after enqueue;
 * synchronise the stream before reading host_keys_out); pageable host memory
 * works, but then the copies block the calling thread.  host_keys may equal
 * host_keys_out.  PCIe is full duplex: a caller that alternates two streams
 * and two sets of device buffers overlaps one call's copy-back with the next
 * call's upload.  Errors: as msort_sort_ws, plus INVALID_VALUE for NULL host
 * or device pointers with n > 0. */
msort_status msort_sort_host(const void *host_keys, const void *host_vals, void *host_keys_out,
                             void *host_vals_out, size_t n, msort_dtype key_dtype,
                             msort_dtype val_dtype, void *dev_keys, void *dev_vals, void *ws,
                             size_t ws_bytes, msort_stream_t stream);

/* Stable merge of p sorted runs -- the merge() step of P:107 ("merge the
 * two sorted halves", P:77-84 step 4; the parent's merge(local, tmp) of
 * P:516) generalised to p runs, i.e. D4 of the distributed sort as its own
 * call.  Run j is in_keys[run_offsets[j], run_offsets[j+1]) (and in_vals
 * alike), each sorted ascending; the output keys_out[0, n) (vals_out) holds
 * all n = run_offsets[p] elements in stable order: ties go to the lower run,
 * then the lower index.  Out of place (input and output must not overlap).
 *   run_offsets  HOST array of p + 1 int64, run_offsets[0] = 0,
 *                non-decreasing (empty runs allowed); 1 <= p <= 128.
 *   ws           device workspace of msort_merge_runs_workspace_bytes bytes.
 * Keys only with 3 <= p <= 8: ONE pass over HBM (K5: sample-based tiles,
 * log2(p) merge rounds in shared memory per tile; the environment variable
 * MSORT_K5 = 0 / n <= 16 changes that range); otherwise ceil(log2 p) rounds
 * of the pairwise merge pass.  Asynchronous on `stream`.  Runs that
 * are not sorted give an unspecified permutation (not checked).
 * Errors: INVALID_VALUE for bad offsets, overlapping buffers, a short
 * workspace; as msort_sort_ws otherwise. */
msort_status msort_merge_runs_workspace_bytes(size_t n, int p, msort_dtype key_dtype,
                                              msort_dtype val_dtype, size_t *bytes);
msort_status msort_merge_runs(const void *in_keys, const void *in_vals,
                              const int64_t *run_offsets, int p, void *keys_out, void *vals_out,
                              msort_dtype key_dtype, msort_dtype val_dtype, void *ws,
                              size_t ws_bytes, msort_stream_t stream);

/* --------------------------------------------------------------- multi GPU */

/* Fill `id_out` (host, 128 bytes) with a fresh NCCL unique id.  Rank 0 calls
 * it and broadcasts the bytes over its own process group. */
msort_status msort_comm_unique_id(void *id_out);

/* Create a communicator for `rank` of `world` from the 128-byte id (host).
 * Collective over all ranks; uses the current CUDA device. */
msort_status msort_comm_init(const void *id, int rank, int world, msort_comm_t *out);

/* Wrap an existing NCCL communicator (an ncclComm_t, e.g. the one of torch's
 * NCCL process group) instead of creating one: rank and world are read from
 * it (ncclCommUserRank / ncclCommCount); it must come from the same NCCL
 * library (the torch wheel's libnccl.so.2, which this library links).
 * NON-OWNING: msort_comm_destroy frees only the wrapper, and a failure
 * detected by a distributed call marks the wrapper unusable without aborting
 * the caller's communicator.  The caller must not run its own collectives on
 * the communicator concurrently with a msort call (NCCL's rule for one
 * communicator used from several streams). */
msort_status msort_comm_wrap(void *nccl_comm, msort_comm_t *out);

/* Free a communicator from msort_comm_init (destroys the NCCL communicator)
 * or msort_comm_wrap (frees only the wrapper). */
msort_status msort_comm_destroy(msort_comm_t comm);

/* Exchange mode of the distributed calls on this communicator: 0 = the NCCL
 * all-to-all + local k-way merge, 1 = the fused pull exchange (see
 * msort_debug_set_exchange for both), -1 = the process default (the
 * environment variable MSORT_EXCHANGE=pull or msort_debug_set_exchange; the
 * initial value).  Every rank of the communicator must set the same mode
 * (the two modes run different collectives).  Not synchronised with calls in
 * flight on the communicator: set it between calls.  Errors:
 * MSORT_ERROR_INVALID_VALUE for a null communicator or another mode. */
msort_status msort_comm_set_exchange(msort_comm_t comm, int mode);

/* Reserve the pull exchange (msort_comm_set_exchange(comm, 1)) for calls with up to
 * n_max local elements of these dtypes: the communicator allocates its
 * exchange buffer (cudaMalloc), publishes it through CUDA IPC and opens every
 * peer's, once.  Collective (every rank calls it; synchronises `stream`).
 * Afterwards a pull-mode msort_sort_distributed* call on keys with 3..8 ranks
 * runs WITHOUT any host synchronisation: the splitters (D2) stay on the
 * device, one K5 launch planned on the device from the split matrix reads
 * every rank's segment in place over NVLink (D3 + D4), and only a
 * split_matrix_out request makes the call wait.  A call with n_local above
 * the reservation returns MSORT_ERROR_INVALID_VALUE (before any collective:
 * every rank must respect its reservation, as for matching NCCL counts). */
msort_status msort_comm_reserve(msort_comm_t comm, size_t n_max, msort_dtype key_dtype,
                                msort_dtype val_dtype, msort_stream_t stream);

/* Distributed stable sort (re-designed: local sort, exact
 * splitters by co-rank, one variable all-to-all over NVLink, local k-way
 * merge).  Collective: every rank calls it with the same dtypes; n_local may
 * differ per rank and may be 0.  On return rank r's keys[0..n_local) hold the
 * global stable positions [K_r, K_r + n_local) of the rank-major
 * concatenation of all inputs, K_r = sum_{j<r} n_j (R10/R11).
 * vals: NULL (val_dtype MSORT_NONE) or 4-byte payloads.
 * split_matrix_out: NULL or host (world+1)*world int64: entry (r, j) = number
 * of rank j's elements among the first K_r outputs.
 * Synchronises `stream` once (the exchange sizes are needed on the host) --
 * except in the reserved pull mode (msort_comm_reserve), which does not
 * synchronise unless split_matrix_out is requested.
 * Failure detection: that wait polls the stream and ncclCommGetAsyncError
 * instead of blocking; an NCCL error -- or, with the environment variable
 * MSORT_NCCL_TIMEOUT_S set, a wait longer than that many seconds (a dead or
 * missing peer) -- aborts the communicator (ncclCommAbort) and returns
 * MSORT_ERROR_NCCL; later calls on it return MSORT_ERROR_NCCL at once. */
msort_status msort_sort_distributed(void *keys, void *vals, size_t n_local,
                                    msort_dtype key_dtype, msort_dtype val_dtype,
                                    msort_comm_t comm, msort_stream_t stream,
                                    int64_t *split_matrix_out);

/* As msort_sort_distributed with caller workspace of
 * msort_workspace_bytes(n_local, key_dtype, val_dtype, world) bytes. */
msort_status msort_sort_distributed_ws(void *keys, void *vals, size_t n_local,
                                       msort_dtype key_dtype, msort_dtype val_dtype,
                                       msort_comm_t comm, void *ws, size_t ws_bytes,
                                       msort_stream_t stream, int64_t *split_matrix_out);

/* Out-of-place form of msort_sort_distributed_ws: the local shard is read from
 * in_keys/in_vals (unchanged) and the rank's output slice is written to
 * keys_out/vals_out. */
msort_status msort_sort_distributed_out_ws(const void *in_keys, const void *in_vals,
                                           void *keys_out, void *vals_out, size_t n_local,
                                           msort_dtype key_dtype, msort_dtype val_dtype,
                                           msort_comm_t comm, void *ws, size_t ws_bytes,
                                           msort_stream_t stream, int64_t *split_matrix_out);

/* End-to-end distributed sort of HOST arrays (bench.py's N > 1 e2e path):
 * host_keys[0..n_local) (host_vals) are copied into the caller's device
 * buffers dev_keys (dev_vals), sorted there by msort_sort_distributed_ws (same
 * workspace, same collective contract), and this rank's output slice is
 * copied back to host_keys_out (host_vals_out).  Enqueued on `stream`; with
 * page-locked host buffers the copies are asynchronous -- synchronise the
 * stream before reading host_keys_out (the sort itself synchronises once
 * unless the communicator is reserved for the pull exchange).  Errors: as
 * msort_sort_distributed_ws, plus INVALID_VALUE for NULL host pointers. */
msort_status msort_sort_distributed_host(const void *host_keys, const void *host_vals,
                                         void *host_keys_out, void *host_vals_out,
                                         size_t n_local, msort_dtype key_dtype,
                                         msort_dtype val_dtype, msort_comm_t comm,
                                         void *dev_keys, void *dev_vals, void *ws,
                                         size_t ws_bytes, msort_stream_t stream);

/* Single-process emulation of the distributed sort for `world` virtual ranks
 * whose shards all live on the current device: the same kernels, the same
 * splitter planning and the same k-way merge, with the NCCL collectives
 * replaced by device-side reductions and device-to-device copies.  Used to
 * check the multi-rank path on one GPU.  keys[r], vals[r] (host arrays of
 * device pointers; vals NULL for keys only), n_local[r] (host), ws[r] (host
 * array of device workspaces sized as for msort_sort_distributed_ws).
 * split_matrix_out as above (host, may be NULL).  Synchronises once. */
msort_status msort_sort_distributed_emulated(void *const *keys, void *const *vals,
                                             const size_t *n_local, int world,
                                             msort_dtype key_dtype, msort_dtype val_dtype,
                                             void *const *ws, size_t ws_bytes,
                                             msort_stream_t stream,
                                             int64_t *split_matrix_out);

/* The paper's own distribution, as an output mode:
 * rank-tree gather to rank 0 (the loop of fig. mpi-merge-code).
 * Every rank sorts its shard (in_keys/in_vals, read only); then, while more
 * than one rank is active, the upper half of the active ranks send their
 * sorted arrays to rank - split over NCCL (NVLink) and the lower half merge
 * their own array with the received one (merge() of P:516: the parent's own
 * elements first on ties).  Rank 0 ends with all sum(n_local) elements in
 * root_keys/root_vals (root_capacity elements available there; other ranks
 * may pass NULL and 0).  Ties therefore come out in the TREE's rank order --
 * for p = 2^k the bit-reversed rank order (0, 4, 2, 6, 1, 5, 3, 7 at p = 8),
 * not the balanced call's natural order.  p is any world size: the paper's
 * split = p / 2 halving for powers of two, ceil(active / 2) parents otherwise.
 * Collective; synchronises once (the shard sizes); buffers are allocated on
 * `stream` (cudaMallocAsync) and freed when the call's work completes.
 * *total_out (host, may be NULL) receives sum(n_local).  Errors: as
 * msort_sort_distributed, INVALID_VALUE when root_capacity is too small. */
msort_status msort_sort_distributed_tree(const void *in_keys, const void *in_vals, size_t n_local,
                                         msort_dtype key_dtype, msort_dtype val_dtype,
                                         msort_comm_t comm, void *root_keys, void *root_vals,
                                         size_t root_capacity, msort_stream_t stream,
                                         int64_t *total_out);

/* Single-process emulation of msort_sort_distributed_tree for `world`
 * virtual ranks on the current device (device-to-device copies instead of
 * NCCL send/recv): shards keys[r], vals[r] (host arrays of device pointers,
 * read only), n_local[r]; root_keys/root_vals receive sum(n_local).
 * Asynchronous on `stream`. */
msort_status msort_sort_distributed_tree_emulated(const void *const *keys,
                                                  const void *const *vals,
                                                  const size_t *n_local, int world,
                                                  msort_dtype key_dtype, msort_dtype val_dtype,
                                                  void *root_keys, void *root_vals,
                                                  msort_stream_t stream);

/* --------------------------------------------- splitter planning (host side)
 * The host-side arithmetic of the splitter co-rank, the same
 * functions the device kernels run.  Exported so the multi-process protocol
 * can be tested on CPU over gloo.  All arrays are host arrays.
 *
 * Keys are compared through their order-preserving unsigned image
 * (int32: x ^ 2^31, int64: x ^ 2^63, unsigned: x).  For each boundary
 * r = 1..world-1 the search keeps an inclusive interval [lo_r, hi_r] of images
 * holding v*_r, the image of the key at global position K_r. */

/* Number of search rounds for a key dtype (8 bits per round: 4 or 8). */
int msort_plan_rounds(msort_dtype key_dtype);

/* Candidates per boundary per round (256). */
int msort_plan_candidates_per_round(void);

/* lohi[2*(world-1)] := {0, max image} for every boundary. */
msort_status msort_plan_init(msort_dtype key_dtype, int world, uint64_t *lohi);

/* cand[(world-1)*B] := the B bucket upper ends of each boundary's interval. */
msort_status msort_plan_candidates(int world, const uint64_t *lohi, uint64_t *cand);

/* Given total[(world-1)*B] = sum over ranks of #{keys with image <= cand},
 * narrow each interval to the first bucket whose total exceeds K_r
 * (the last bucket if none).  K[world+1] = prefix sums of the shard sizes. */
msort_status msort_plan_narrow(int world, const uint64_t *K, const uint64_t *total,
                               uint64_t *lohi);

/* Split matrix from the gathered counts: lteq[j*(world-1)*2 + (r-1)*2 + {0,1}]
 * = (#keys < v*_r, #keys == v*_r) on rank j.  out[(world+1)*world]:
 *   s[r][j] = lt_j + clamp(K_r - sum_j' lt_j' - sum_{j'<j} eq_j', 0, eq_j),
 *   s[0][.] = 0, s[world][j] = n_j. */
msort_status msort_plan_fill(int world, const uint64_t *K, const uint64_t *lteq,
                             int64_t *out);

/* The rank-tree schedule of msort_sort_distributed_tree: the
 * number of rounds for `world` ranks, and this rank's role in round t
 * (0 idle, 1 parent: receives from *peer and merges [own | received], own
 * elements first on ties; 2 child: sends its array to *peer).  Host only. */
int msort_plan_tree_rounds(int world);
int msort_plan_tree_role(int world, int rank, int round, int *peer);

/* ------------------------------------------------------- status and timing */

const char *msort_status_string(msort_status s);
const char *msort_last_error(void);

/* Kernel accounting.  The library counts every kernel it launches; when
 * profiling is enabled it also brackets each launch with CUDA events on the
 * launching stream.  msort_profile_read synchronises those events and
 * returns, per kernel class (0 tile_sort, 1 partition, 2 merge_pass,
 * 3 splitter, 4 kway_merge, 5 NCCL collectives, 6 the D3 exchange -- the
 * all-to-all of the sorted segments, or its emulation, 7 key_range -- the
 * range / narrow / widen passes of 8-byte-key sorts), the launch count and
 * total device milliseconds since the last reset.  Host arrays of
 * MSORT_PROFILE_CLASSES. */
#define MSORT_PROFILE_CLASSES 8
void msort_profile_enable(int on);
void msort_profile_reset(void);
msort_status msort_profile_read(int64_t *launches, double *ms);

/* Total launches of the library's OWN kernels (class 5, NCCL, excluded)
 * since process start / the last msort_profile_reset. */
int64_t msort_launch_count(void);

/* Tile size (elements) used for key dtype with/without payload. */
int msort_tile_size(msort_dtype key_dtype, msort_dtype val_dtype);

/* Testing knob for keys-only sorts: how merge levels are grouped into HBM
 * passes.  mode 0 (default): every 2-way level in the fused K3 dataflow;
 * mode 5: every pair of levels as one K6 4-way pass (4-byte keys; tiles from
 * a partition kernel, merged in two rounds by the tile sort's merge engine;
 * 8-byte keys keep mode 0).  Other values select mode 0.  The result is the
 * same in every mode (the stable sort is unique).  Process-wide (an atomic:
 * a concurrent sort sees either mode); overrides the MSORT_QUAD environment
 * variable.  Returns 0. */
int msort_debug_set_quad(int mode);

/* Exchange mode of the distributed sort (D3+D4).  mode 0 (default): one NCCL
 * all-to-all (grouped ncclSend/ncclRecv) into a receive buffer, then the local
 * k-way merge (one K5 pass for keys with 3..8 ranks, K3 rounds otherwise).
 * mode 1 ("pull", the fused exchange): D1 leaves each sorted shard in a
 * buffer the communicator owns (cudaMalloc, IPC-exportable), every rank
 * publishes it through CUDA IPC, and the merge reads the p segments in place
 * from their owners (peer memory over NVLink/NVSwitch): for keys with 3..8
 * ranks D3 and D4 are ONE K5 kernel (no receive buffer, every segment crosses
 * NVLink once, straight into the merge); otherwise the first K3 round reads
 * the peers.  A barrier then frees the exchange buffers.  Validated on one
 * GPU through msort_sort_distributed_emulated (the same kernels, peers =
 * local buffers); environment MSORT_EXCHANGE=pull selects it too.  Returns 0. */
int msort_debug_set_exchange(int mode);

/* Experiment hook (scripts/k1_ab.py; not part of the product path): the tile
 * sort (K1) alone on int32 keys -- every T-key tile of in[0, n) sorted into
 * out (device pointers) by the product kernel (variant 0: 128 threads x 68
 * keys, a per-thread merge-exchange network + merge-path rounds, T = 8704) or
 * its A/B variant (1: 128 x 64, the warp-shuffle bitonic network for the
 * first 2048-key runs, then the same block rounds, T = 8192).  Asynchronous
 * on `stream`; returns T, or -1 on a launch error. */
int msort_debug_tile_sort(const void *in, void *out, int64_t n, int variant, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MSORT_H */
