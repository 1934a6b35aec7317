/*
 * msort_oracle.c -- TEST INFRASTRUCTURE ONLY (see msort_oracle.h).
 *
 * A plain, slow, obviously correct CPU implementation of the stable ascending
 * merge sort that arXiv 2211.16479 parallelises.  Every function follows the
 * paper's description step by step; nothing here is blocked, fused or
 * reordered.  It shares nothing with the CUDA path.
 */
#include "msort_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/*
 * ORACLE_IMPL(SUF, T) defines, for key type T:
 *
 *   merge_SUF  -- merge() of P:107: two sorted runs into out, taking the
 *                 left element when left <= right (ties to the left run,
 *                 reading R1), then copying the tail of whichever run is left.
 *   sort_SUF   -- mergesort() of Fig. fig:mergesort, steps of
 *                 P:77-84:
 *                   1. fewer than two elements: return
 *                   2. mid = len // 2; left = [lo, mid), right = [mid, hi)
 *                                                   (reading R2)
 *                   3. sort both halves with the same algorithm
 *                   4. merge the two sorted halves
 *                 The merge writes into the auxiliary buffer (the O(n) extra
 *                 space of P:144) and is copied back.
 */
#define ORACLE_IMPL(SUF, T)                                                        \
  static void merge_##SUF(const T *a, const uint32_t *av, size_t na, const T *b,   \
                          const uint32_t *bv, size_t nb, T *out, uint32_t *outv) { \
    size_t i = 0, j = 0, t = 0;                                                    \
    while (i < na && j < nb) {                                                     \
      if (a[i] <= b[j]) { /* left first on ties: stable */                         \
        out[t] = a[i];                                                             \
        if (outv) outv[t] = av[i];                                                 \
        i++;                                                                       \
      } else {                                                                     \
        out[t] = b[j];                                                             \
        if (outv) outv[t] = bv[j];                                                 \
        j++;                                                                       \
      }                                                                            \
      t++;                                                                         \
    }                                                                              \
    while (i < na) {                                                               \
      out[t] = a[i];                                                               \
      if (outv) outv[t] = av[i];                                                   \
      i++, t++;                                                                    \
    }                                                                              \
    while (j < nb) {                                                               \
      out[t] = b[j];                                                               \
      if (outv) outv[t] = bv[j];                                                   \
      j++, t++;                                                                    \
    }                                                                              \
  }                                                                                \
                                                                                   \
  static void sort_##SUF(T *a, uint32_t *v, T *aux, uint32_t *auxv, size_t lo,     \
                         size_t hi) {                                              \
    size_t n = hi - lo;                                                            \
    if (n < 2) return; /* step 1 */                                                \
    size_t mid = lo + n / 2; /* step 2: mid = len(array) // 2 */                   \
    sort_##SUF(a, v, aux, auxv, lo, mid); /* step 3: left = array[:mid] */         \
    sort_##SUF(a, v, aux, auxv, mid, hi); /*         right = array[mid:] */        \
    merge_##SUF(a + lo, v ? v + lo : NULL, mid - lo, a + mid, v ? v + mid : NULL,  \
                hi - mid, aux + lo, v ? auxv + lo : NULL); /* step 4 */            \
    memcpy(a + lo, aux + lo, n * sizeof(T));                                       \
    if (v) memcpy(v + lo, auxv + lo, n * sizeof(uint32_t));                        \
  }                                                                                \
                                                                                   \
  static int top_sort_##SUF(T *a, uint32_t *v, size_t n) {                         \
    if (n < 2) return 0;                                                           \
    T *aux = (T *)malloc(n * sizeof(T));                                           \
    uint32_t *auxv = v ? (uint32_t *)malloc(n * sizeof(uint32_t)) : NULL;          \
    if (!aux || (v && !auxv)) {                                                    \
      free(aux);                                                                   \
      free(auxv);                                                                  \
      return -2;                                                                   \
    }                                                                              \
    sort_##SUF(a, v, aux, auxv, 0, n);                                             \
    free(aux);                                                                     \
    free(auxv);                                                                    \
    return 0;                                                                      \
  }                                                                                \
                                                                                   \
  static int check_##SUF(const T *in, const T *out, const uint32_t *ov, size_t n) { \
    int bad = 0;                                                                   \
    for (size_t t = 0; t + 1 < n; t++)                                             \
      if (out[t] > out[t + 1]) bad |= 1;                                           \
    if (ov) {                                                                      \
      unsigned char *seen = (unsigned char *)calloc(n ? n : 1, 1);                 \
      if (!seen) return -2;                                                        \
      for (size_t t = 0; t < n; t++) {                                             \
        uint32_t s = ov[t];                                                        \
        if ((size_t)s >= n || seen[s] || in[s] != out[t]) bad |= 2;                \
        else seen[s] = 1;                                                          \
      }                                                                            \
      free(seen);                                                                  \
      for (size_t t = 0; t + 1 < n; t++)                                           \
        if (out[t] == out[t + 1] && ov[t] >= ov[t + 1]) bad |= 4;                  \
    }                                                                              \
    return bad;                                                                    \
  }

ORACLE_IMPL(i32, int32_t)
ORACLE_IMPL(u32, uint32_t)
ORACLE_IMPL(i64, int64_t)
ORACLE_IMPL(u64, uint64_t)

static size_t key_size(int kd) {
  switch (kd) {
    case ORACLE_INT32:
    case ORACLE_UINT32: return 4;
    case ORACLE_INT64:
    case ORACLE_UINT64: return 8;
    default: return 0;
  }
}

int msort_oracle_sort(void *keys, uint32_t *vals, size_t n, int kd) {
  if (!key_size(kd)) return -1;
  if (n > 0 && !keys) return -1;
  switch (kd) {
    case ORACLE_INT32: return top_sort_i32((int32_t *)keys, vals, n);
    case ORACLE_UINT32: return top_sort_u32((uint32_t *)keys, vals, n);
    case ORACLE_INT64: return top_sort_i64((int64_t *)keys, vals, n);
    default: return top_sort_u64((uint64_t *)keys, vals, n);
  }
}

int msort_oracle_merge(const void *a, const uint32_t *av, size_t na, const void *b,
                       const uint32_t *bv, size_t nb, void *out, uint32_t *outv, int kd) {
  if (!key_size(kd)) return -1;
  if ((na && !a) || (nb && !b) || ((na + nb) && !out)) return -1;
  int withv = outv != NULL;
  if (withv && ((na && !av) || (nb && !bv))) return -1;
  switch (kd) {
    case ORACLE_INT32:
      merge_i32((const int32_t *)a, av, na, (const int32_t *)b, bv, nb, (int32_t *)out, outv);
      break;
    case ORACLE_UINT32:
      merge_u32((const uint32_t *)a, av, na, (const uint32_t *)b, bv, nb, (uint32_t *)out, outv);
      break;
    case ORACLE_INT64:
      merge_i64((const int64_t *)a, av, na, (const int64_t *)b, bv, nb, (int64_t *)out, outv);
      break;
    default:
      merge_u64((const uint64_t *)a, av, na, (const uint64_t *)b, bv, nb, (uint64_t *)out, outv);
  }
  return 0;
}

int msort_oracle_check(const void *in_keys, const void *out_keys, const uint32_t *out_vals,
                       size_t n, int kd) {
  if (!key_size(kd)) return -1;
  if (n > 0 && (!in_keys || !out_keys)) return -1;
  switch (kd) {
    case ORACLE_INT32: return check_i32((const int32_t *)in_keys, (const int32_t *)out_keys, out_vals, n);
    case ORACLE_UINT32: return check_u32((const uint32_t *)in_keys, (const uint32_t *)out_keys, out_vals, n);
    case ORACLE_INT64: return check_i64((const int64_t *)in_keys, (const int64_t *)out_keys, out_vals, n);
    default: return check_u64((const uint64_t *)in_keys, (const uint64_t *)out_keys, out_vals, n);
  }
}

/*
 * Split matrix by definition (R10/R11): the distributed output puts
 * global stable positions [K_r, K_{r+1}) of the rank-major concatenation on
 * rank r.  Concatenate the shards in rank order with payload = global index,
 * sort stably, and count, for each prefix of K_r outputs, how many came from
 * each shard.
 */
int msort_oracle_split_matrix(const void *const *shards, const size_t *sizes, int p, int kd,
                              int64_t *out) {
  size_t ks = key_size(kd);
  if (!ks || p < 1 || !sizes || !out) return -1;
  size_t total = 0;
  for (int j = 0; j < p; j++) {
    if (sizes[j] && !shards[j]) return -1;
    total += sizes[j];
  }
  if (total > 0xFFFFFFFFull) return -1;
  unsigned char *cat = (unsigned char *)malloc(total ? total * ks : 1);
  uint32_t *idx = (uint32_t *)malloc(total ? total * sizeof(uint32_t) : 4);
  int *owner = (int *)malloc(total ? total * sizeof(int) : sizeof(int));
  if (!cat || !idx || !owner) {
    free(cat), free(idx), free(owner);
    return -2;
  }
  size_t off = 0;
  for (int j = 0; j < p; j++) {
    if (sizes[j]) memcpy(cat + off * ks, shards[j], sizes[j] * ks);
    for (size_t t = 0; t < sizes[j]; t++) owner[off + t] = j;
    off += sizes[j];
  }
  for (size_t t = 0; t < total; t++) idx[t] = (uint32_t)t;
  int rc = msort_oracle_sort(cat, idx, total, kd);
  if (rc == 0) {
    int64_t *cnt = (int64_t *)calloc((size_t)p, sizeof(int64_t));
    if (!cnt) rc = -2;
    else {
      size_t K = 0, t = 0;
      for (int r = 0; r <= p; r++) {
        /* advance the prefix to K_r outputs, counting their source shards */
        for (; t < K; t++) cnt[owner[idx[t]]]++;
        for (int j = 0; j < p; j++) out[(size_t)r * p + j] = cnt[j];
        if (r < p) K += sizes[r];
      }
      free(cnt);
    }
  }
  free(cat), free(idx), free(owner);
  return rc;
}

/* ---- the paper's multiprocessing merge sort on host threads (baseline) ---- */

typedef struct {
  unsigned char *keys;
  uint32_t *vals;
  size_t n;
  int kd;
  int rc;
} chunk_job;

static void *chunk_sort_main(void *arg) {
  chunk_job *j = (chunk_job *)arg;
  j->rc = msort_oracle_sort(j->keys, j->vals, j->n, j->kd);
  return NULL;
}

typedef struct {
  const unsigned char *a, *b;
  const uint32_t *av, *bv;
  size_t na, nb;
  unsigned char *out;
  uint32_t *outv;
  int kd;
} merge_job;

static void *merge_main(void *arg) {
  merge_job *m = (merge_job *)arg;
  msort_oracle_merge(m->a, m->av, m->na, m->b, m->bv, m->nb, m->out, m->outv, m->kd);
  return NULL;
}

int msort_oracle_paper_mp(void *keys, uint32_t *vals, size_t n, int kd, int cores) {
  size_t ks = key_size(kd);
  if (!ks || cores < 1 || (n && !keys)) return -1;
  if (n < 2) return 0;
  /* size = ceil(len(arr) / processes); chunk i = arr[size*i : size*(i+1)] */
  size_t size = (n + (size_t)cores - 1) / (size_t)cores;
  int c = (int)((n + size - 1) / size);
  size_t *lo = (size_t *)malloc(sizeof(size_t) * (size_t)(c + 1));
  chunk_job *jobs = (chunk_job *)malloc(sizeof(chunk_job) * (size_t)c);
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)c);
  unsigned char *bufk = (unsigned char *)malloc(n * ks);
  uint32_t *bufv = vals ? (uint32_t *)malloc(n * sizeof(uint32_t)) : NULL;
  if (!lo || !jobs || !th || !bufk || (vals && !bufv)) {
    free(lo), free(jobs), free(th), free(bufk), free(bufv);
    return -2;
  }
  for (int i = 0; i <= c; i++) lo[i] = (size_t)i * size < n ? (size_t)i * size : n;
  /* pool.map(fast_sort, arr1): one thread per chunk */
  for (int i = 0; i < c; i++) {
    jobs[i] = (chunk_job){(unsigned char *)keys + lo[i] * ks, vals ? vals + lo[i] : NULL,
                          lo[i + 1] - lo[i], kd, 0};
    pthread_create(&th[i], NULL, chunk_sort_main, &jobs[i]);
  }
  int rc = 0;
  for (int i = 0; i < c; i++) {
    pthread_join(th[i], NULL);
    if (jobs[i].rc) rc = jobs[i].rc;
  }
  /* "merge the sorted chunks": pairwise rounds, pairs merged in parallel */
  unsigned char *src = (unsigned char *)keys, *dst = bufk;
  uint32_t *srcv = vals, *dstv = bufv;
  merge_job *mj = (merge_job *)malloc(sizeof(merge_job) * (size_t)c);
  int runs = c;
  while (rc == 0 && runs > 1) {
    int pairs = (runs + 1) / 2;
    for (int q = 0; q < pairs; q++) {
      size_t a0 = lo[2 * q], a1 = lo[2 * q + 1];
      size_t b1 = (2 * q + 2 <= runs) ? lo[2 * q + 2] : a1;
      mj[q] = (merge_job){src + a0 * ks, src + a1 * ks, srcv ? srcv + a0 : NULL,
                          srcv ? srcv + a1 : NULL, a1 - a0, b1 - a1, dst + a0 * ks,
                          dstv ? dstv + a0 : NULL, kd};
      pthread_create(&th[q], NULL, merge_main, &mj[q]);
    }
    for (int q = 0; q < pairs; q++) pthread_join(th[q], NULL);
    for (int q = 0; q <= pairs; q++) lo[q] = lo[2 * q < runs ? 2 * q : runs];
    runs = pairs;
    unsigned char *t = src; src = dst; dst = t;
    uint32_t *tv = srcv; srcv = dstv; dstv = tv;
  }
  if (rc == 0 && src != (unsigned char *)keys) {
    memcpy(keys, src, n * ks);
    if (vals) memcpy(vals, srcv, n * sizeof(uint32_t));
  }
  free(mj), free(lo), free(jobs), free(th), free(bufk), free(bufv);
  return rc;
}
