/*
 * msort_oracle.h -- plain, slow, obviously correct CPU oracle for the stable
 * ascending merge sort of arXiv 2211.16479.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2211_16479_b200/csrc, include/msort.h) and includes nothing from it.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (section in brackets).
 *
 * What it computes.  For keys k_0..k_{n-1} (and optional uint32 payloads
 * v_0..v_{n-1}) the stable ascending sort: element i lands at
 *     pos(i) = #{j : k_j < k_i} + #{j < i : k_j = k_i}.
 * The method reaching it is the textbook top-down merge sort of
 * P:77-84 [Sequential Merge Sort, steps 1-4] and Fig. fig:mergesort P:88-112,
 * with the listing's `right = array[:mid]` read as array[mid:]
 * (reading R2) and ties in merge() taken from the left run
 * (merge() is never listed; reading R1).  No cutoff: the
 * hybrid of Fig. fig:mergesort-2 would make a library sort part
 * of the oracle.
 *
 * Pins (tests/test_oracle.py): brute force over all permutations of tiny
 * inputs, the counting-rank definition pos(i) at medium n, numpy's stable
 * argsort at scale, closed forms (sorted, reversed, all-equal), the worked
 * example and golden values of SURVEY.md §8(c).
 *
 * Error behaviour: functions return 0 on success, -1 on a bad argument
 * (unknown dtype, NULL with n > 0) and -2 when allocation fails.
 */
#ifndef MSORT_ORACLE_H
#define MSORT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Key dtype codes of the oracle (numbered like numpy kinds, own enum). */
enum { ORACLE_INT32 = 0, ORACLE_UINT32 = 1, ORACLE_INT64 = 2, ORACLE_UINT64 = 3 };

/* Stable ascending top-down merge sort, in place on host arrays.
 * keys: n elements of key dtype kd.  vals: NULL (keys only) or n uint32
 * payloads that travel with their keys.  P:77-84, fig:mergesort P:88-112. */
int msort_oracle_sort(void *keys, uint32_t *vals, size_t n, int kd);

/* Stable two-way merge (the never-listed merge() of P:107/P:134/P:516):
 * out = merge(a, b), taking a[i] when a[i] <= b[j] (left first on ties).
 * av/bv/outv may all be NULL (keys only) or all non-NULL. */
int msort_oracle_merge(const void *a, const uint32_t *av, size_t na,
                       const void *b, const uint32_t *bv, size_t nb,
                       void *out, uint32_t *outv, int kd);

/* Reference split matrix of the distributed sort (SURVEY.md §8(a) D2,
 * DESIGN.md reading R10/R11).  shards[j] holds sizes[j] keys of rank j.
 * With the rank-major concatenation stably sorted and K_r = sum_{j<r} n_j,
 * out[r*p + j] (r = 0..p, j = 0..p-1) is the number of shard-j elements
 * among the first K_r outputs.  Computed by definition: concatenate with
 * payload = global index, sort with msort_oracle_sort, count. */
int msort_oracle_split_matrix(const void *const *shards, const size_t *sizes,
                              int p, int kd, int64_t *out);

/* Invariant checker: returns a bit mask,
 *   1 = output not non-decreasing,
 *   2 = payload is not a permutation of [0,n) or out_key[t] != in_key[out_val[t]],
 *   4 = stability violated (equal keys with out_val[t] >= out_val[t+1]).
 * out_vals may be NULL (then only bit 1 is checked).  Returns -1 on bad args. */
int msort_oracle_check(const void *in_keys, const void *out_keys,
                       const uint32_t *out_vals, size_t n, int kd);

/* The paper's own multiprocessing merge sort re-created on host threads
 * (P:255-292 [Multiprocessing Merge Sort], fig:init-mp-ms, fig:mapping):
 * chunks of ceil(n/c), each sorted by msort_oracle_sort on its
 * own thread (the paper's fast_sort), then pairwise merge rounds
 * in parallel ("merge the sorted chunks").  A CPU baseline for
 * bench.py, not a parity authority. */
int msort_oracle_paper_mp(void *keys, uint32_t *vals, size_t n, int kd, int cores);

#ifdef __cplusplus
}
#endif
#endif
