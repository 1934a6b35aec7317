// msort_device.cuh -- device building blocks of the sm_100a merge sort.
//
// Everything here is integer comparison and data movement (no tensor cores:
// a sort is not a dense contraction).  "P:n" = /root/reference/PAPER.md line n.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace msort {

// ------------------------------------------------------------- key traits
template <class K>
struct KeyTraits;
template <>
struct KeyTraits<int32_t> {
  using U = uint32_t;
  static __host__ __device__ __forceinline__ int32_t max_key() { return 0x7fffffff; }
  static __host__ __device__ __forceinline__ int32_t min_key() { return (int32_t)0x80000000; }
  static __host__ __device__ __forceinline__ U image(int32_t x) { return (U)x ^ 0x80000000u; }
};
template <>
struct KeyTraits<uint32_t> {
  using U = uint32_t;
  static __host__ __device__ __forceinline__ uint32_t max_key() { return 0xffffffffu; }
  static __host__ __device__ __forceinline__ uint32_t min_key() { return 0u; }
  static __host__ __device__ __forceinline__ U image(uint32_t x) { return x; }
};
template <>
struct KeyTraits<int64_t> {
  using U = uint64_t;
  static __host__ __device__ __forceinline__ int64_t max_key() { return 0x7fffffffffffffffll; }
  static __host__ __device__ __forceinline__ int64_t min_key() { return (int64_t)0x8000000000000000ull; }
  static __host__ __device__ __forceinline__ U image(int64_t x) {
    return (U)x ^ 0x8000000000000000ull;
  }
};
template <>
struct KeyTraits<uint64_t> {
  using U = uint64_t;
  static __host__ __device__ __forceinline__ uint64_t max_key() { return ~0ull; }
  static __host__ __device__ __forceinline__ uint64_t min_key() { return 0ull; }
  static __host__ __device__ __forceinline__ U image(uint64_t x) { return x; }
};

// Key-range narrowing of 8-byte keys (Kernels::sort_narrowed): mm[0] / mm[1]
// = the smallest / largest order-preserving image of a sort's keys.  The
// keys are sorted as 32-bit offsets from mm[0] when they span < 2^32 values.
__device__ __forceinline__ bool range_narrow(const unsigned long long* mm) {
  return mm[1] - mm[0] <= 0xffffffffull;
}
template <class K>
__host__ __device__ __forceinline__ K key_from_image(unsigned long long u) {
  return sizeof(K) == 8 && K(-1) < K(0) ? (K)(u ^ 0x8000000000000000ull) : (K)u;
}

// Shared-memory padding: one spare word per 128 bytes, so that "blocked"
// accesses (thread t touches VT consecutive elements) are conflict-free.
template <class K, bool PAD>
__device__ __forceinline__ int sidx(int i) {
  if constexpr (PAD) return i + i / (int)(128 / sizeof(K));
  else return i;
}
template <class K, int T>
constexpr int padded_len() {
  return T + T / (int)(128 / sizeof(K));
}

// ------------------------------------------------------------ merge path
// Co-rank of diagonal d of the stable A-first merge of A = s[a0, a0+na) and
// B = s[b0, b0+nb):  i(d) = min{ i in [max(0,d-nb), min(d,na)] :
//                               i = min(d,na) or A[i] > B[d-1-i] },
// the number of A elements among the first d outputs of merge(A, B) with
// ties taken from A (R1).
template <class K, bool PAD>
__device__ __forceinline__ int merge_path(const K* s, int a0, int na, int b0, int nb, int d) {
  int lo = d - nb > 0 ? d - nb : 0;
  int hi = d < na ? d : na;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (s[sidx<K, PAD>(a0 + mid)] > s[sidx<K, PAD>(b0 + d - 1 - mid)]) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// Loads of the co-rank searches in global memory (probes).  The fused merge
// pass searches a few chunks ahead of its loads, so a probe's sector would be
// evicted from L2 before the window holding it is staged and then read twice
// from DRAM; with MSORT_PROBE_EVICT_LAST the probes carry an L2 evict_last
// policy.  Plain coherent loads (not .nc): in the fused pass the data was
// written by other CTAs of the same launch (ordered by the acquire that
// precedes the search).
#ifndef MSORT_PROBE_EVICT_LAST
#define MSORT_PROBE_EVICT_LAST 1
#endif
__device__ __forceinline__ uint64_t probe_policy() {
  uint64_t pol = 0;
#if MSORT_PROBE_EVICT_LAST
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#endif
  return pol;
}
template <class K>
__device__ __forceinline__ K probe_ld(const K* p, uint64_t pol) {
  static_assert(sizeof(K) == 4 || sizeof(K) == 8, "4- or 8-byte keys");
#if MSORT_PROBE_EVICT_LAST
  if constexpr (sizeof(K) == 4) {
    uint32_t v;
    asm volatile("ld.global.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return (K)v;
  } else {
    uint64_t v;
    asm volatile("ld.global.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
    return (K)v;
  }
#else
  (void)pol;
  return *reinterpret_cast<const volatile K*>(p);
#endif
}

// Same search over global memory with 64-bit indices.
template <class K>
__device__ __forceinline__ int64_t merge_path_global(const K* __restrict__ a, int64_t na,
                                                     const K* __restrict__ b, int64_t nb,
                                                     int64_t d) {
  int64_t lo = d - nb > 0 ? d - nb : 0;
  int64_t hi = d < na ? d : na;
  const uint64_t pol = probe_policy();
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (probe_ld(a + mid, pol) > probe_ld(b + (d - 1 - mid), pol)) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// The same search restricted to [lo, hi], a bracket known to hold i(d).
template <class K>
__device__ __forceinline__ int64_t merge_path_global_range(const K* __restrict__ a,
                                                           const K* __restrict__ b, int64_t d,
                                                           int64_t lo, int64_t hi) {
  const uint64_t pol = probe_policy();
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (probe_ld(a + mid, pol) > probe_ld(b + (d - 1 - mid), pol)) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// The same search by a group of GS = 2^LG lanes of a warp (lanes gbase ..
// gbase+GS-1; every lane of the warp calls it, `active` false for lanes
// without a search), each lane probing PL candidates per round: a round
// probes C = GS * PL evenly spaced candidates of [lo, hi) -- all of its
// 2C loads in flight at once -- and keeps the bucket where the monotone
// predicate A[i] > B[d-1-i] turns true, so the dependent probe latency is
// paid log_C(range) times instead of log2(range).  Used where a warp has
// fewer searches than lanes and probe latency is on the critical path (small
// sorts: K3's searcher with one chunk per grab).
template <int PL, class K>
__device__ __forceinline__ int64_t merge_path_global_group(const K* __restrict__ a,
                                                           const K* __restrict__ b, int64_t d,
                                                           int64_t lo, int64_t hi, bool active,
                                                           int gl, int LG, int gbase) {
  const uint64_t pol = probe_policy();
  const int GS = 1 << LG;
  const unsigned gm = GS == 32 ? 0xffffffffu : ((1u << GS) - 1u);
  const int64_t C = (int64_t)GS * PL;
  while (__any_sync(0xffffffffu, active && hi > lo)) {
    const bool act = active && hi > lo;
    const int64_t span = hi - lo;
    const int64_t step = (span + C - 1) / C;
    int t1 = PL;  // first candidate of this lane where the predicate holds
    if (act) {
      K av[PL], bv[PL];
#pragma unroll
      for (int t = 0; t < PL; ++t) {
        const int64_t off = step * (gl * PL + t + 1);
        const int64_t p = lo + (off < span ? off : span) - 1;
        av[t] = probe_ld(a + p, pol);
        bv[t] = probe_ld(b + (d - 1 - p), pol);
      }
#pragma unroll
      for (int t = PL - 1; t >= 0; --t)
        if (av[t] > bv[t]) t1 = t;
    }
    const unsigned m = (__ballot_sync(0xffffffffu, t1 < PL) >> gbase) & gm;
    const int f = m ? __ffs(m) - 1 : 0;
    const int tf = __shfl_sync(0xffffffffu, t1, gbase + f);
    if (act) {
      if (m == 0) {
        lo = hi;
      } else {
        const int64_t k = (int64_t)f * PL + tf;  // first candidate where it holds
        const int64_t ok = step * (k + 1), ok0 = step * k;
        const int64_t nlo = k > 0 ? lo + (ok0 < span ? ok0 : span) : lo;
        hi = lo + (ok < span ? ok : span) - 1;
        lo = nlo;
      }
    }
  }
  return lo;
}

// Serial stable merge of VT outputs starting at (ai, bi): take B only when
// B < A (strict), so ties go to A.  Positions are indices into the shared
// buffer s; `pos` records the source position of each output (for payload
// gathers) when TRACK, and `src_idx` (if non-null) maps a position to an
// original index carried from an earlier merge round.
// Branch-free: one shared load per output, at a clamped index (<= lim), so
// the caller only guarantees that s[0..lim] is addressable.
template <class K, bool PAD, bool TRACK, int VT>
__device__ __forceinline__ void serial_merge(const K* s, const int* src_idx, int ai, int aend,
                                             int bi, int bend, int lim, K (&key)[VT],
                                             int (&pos)[VT]) {
  K ak = s[sidx<K, PAD>(min(ai, lim))];
  K bk = s[sidx<K, PAD>(min(bi, lim))];
#pragma unroll
  for (int k = 0; k < VT; ++k) {
    const bool takeB = (bi < bend) && ((ai >= aend) || (bk < ak));
    key[k] = takeB ? bk : ak;
    if constexpr (TRACK) {
      int p = takeB ? bi : ai;
      pos[k] = src_idx ? src_idx[sidx<K, PAD>(p)] : p;
    }
    ai += takeB ? 0 : 1;
    bi += takeB ? 1 : 0;
    if (k + 1 < VT) {
      const K nv = s[sidx<K, PAD>(min(takeB ? bi : ai, lim))];
      ak = takeB ? ak : nv;
      bk = takeB ? nv : bk;
    }
  }
}

// As serial_merge (unpadded, positions tracked as buffer indices), with a
// check-free fast path when neither run can run out within VT steps --
// the common case -- and the checked loop otherwise.
template <class K, bool TRACK, int VT>
__device__ __forceinline__ void serial_merge_fast(const K* s, int ai, int aend, int bi, int bend,
                                                  int lim, K (&key)[VT], int (&pos)[VT]) {
  // warp-uniform choice: a divergent warp would run both paths
  if (__all_sync(__activemask(), ai + VT <= aend && bi + VT <= bend)) {
    K ak = s[ai];
    K bk = s[bi];
#pragma unroll
    for (int k = 0; k < VT; ++k) {
      const bool takeB = bk < ak;
      key[k] = takeB ? bk : ak;
      if constexpr (TRACK) pos[k] = takeB ? bi : ai;
      ai += takeB ? 0 : 1;
      bi += takeB ? 1 : 0;
      if (k + 1 < VT) {
        const K nv = s[takeB ? bi : ai];
        ak = takeB ? ak : nv;
        bk = takeB ? nv : bk;
      }
    }
  } else {
    serial_merge<K, false, TRACK, VT>(s, nullptr, ai, aend, bi, bend, lim, key, pos);
  }
}

// Keys-only merge step kernels on byte offsets into a shared buffer (the
// output value of a keys-only merge is min(a, b) whichever run it came
// from, and each step touches one byte offset: select, add, load).
template <class K>
__device__ __forceinline__ K ld_off(const char* s, uint32_t off) {
  return *reinterpret_cast<const K*>(s + off);
}
// VT outputs of merge(A, B) from byte offsets oa, ob, no end checks: the
// caller guarantees neither run ends within VT steps.
template <class K, int VT>
__device__ __forceinline__ void merge_keys_nocheck(const char* s, uint32_t oa, uint32_t ob,
                                                   K (&key)[VT]) {
  K ak = ld_off<K>(s, oa), bk = ld_off<K>(s, ob);
#pragma unroll
  for (int k = 0; k < VT; ++k) {
    const bool p = bk < ak;
    key[k] = p ? bk : ak;
    if (k + 1 < VT) {
      const uint32_t nx = (p ? ob : oa) + (uint32_t)sizeof(K);
      oa = p ? oa : nx;
      ob = p ? nx : ob;
      const K nv = ld_off<K>(s, nx);
      ak = p ? ak : nv;
      bk = p ? nv : bk;
    }
  }
}
// Same with end checks: a run that is used up reads as "greater than
// anything" (the other run is taken); loads are clamped to `lim`.
template <class K, int VT>
__device__ __forceinline__ void merge_keys_checked(const char* s, uint32_t oa, uint32_t ea,
                                                   uint32_t ob, uint32_t eb, uint32_t lim,
                                                   K (&key)[VT]) {
  K ak = ld_off<K>(s, min(oa, lim)), bk = ld_off<K>(s, min(ob, lim));
#pragma unroll
  for (int k = 0; k < VT; ++k) {
    const bool p = (ob < eb) && ((oa >= ea) || (bk < ak));
    key[k] = p ? bk : ak;
    if (k + 1 < VT) {
      const uint32_t nx = (p ? ob : oa) + (uint32_t)sizeof(K);
      oa = p ? oa : nx;
      ob = p ? nx : ob;
      const K nv = ld_off<K>(s, min(nx, lim));
      ak = p ? ak : nv;
      bk = p ? nv : bk;
    }
  }
}
// Merge-path co-rank (see merge_path) on byte offsets: A at oa (na
// elements), B at ob (nb), diagonal d.
template <class K>
__device__ __forceinline__ int merge_path_off(const char* s, uint32_t oa, int na, uint32_t ob,
                                              int nb, int d) {
  int lo = d - nb > 0 ? d - nb : 0;
  int hi = d < na ? d : na;
  // B[d-1-mid] sits at ob + (d-1)*sz - mid*sz
  const uint32_t obd = ob + (uint32_t)((d - 1) * (int)sizeof(K));
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const uint32_t m = (uint32_t)mid * (uint32_t)sizeof(K);
    if (ld_off<K>(s, oa + m) > ld_off<K>(s, obd - m)) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// 2H outputs of one thread merged as two independent chains: the front chain
// produces outputs 0..H-1 from the co-rank at the thread's first diagonal
// (ai0, bi0) upwards, the back chain outputs 2H-1..H from the co-rank at its
// last diagonal (ai1, bi1) downwards.  Forward, ties take A (R1);
// backward the LAST of equal keys is the B one, so ties take B.  Two
// dependency chains halve the latency of a thread's merge.  Requires that
// no run can run out: ai0+H <= aend, bi0+H <= bend, ai1-H >= a_lo,
// bi1-H >= b_lo (the caller checks, else uses serial_merge).
template <class K, bool TRACK, int H>
__device__ __forceinline__ void dual_merge(const K* s, int ai, int bi, int ai1, int bi1,
                                           K (&key)[2 * H], int (&pos)[2 * H]) {
  K ak = s[ai], bk = s[bi];
  K ak1 = s[ai1 - 1], bk1 = s[bi1 - 1];
#pragma unroll
  for (int k = 0; k < H; ++k) {
    const bool takeB = bk < ak;
    const bool takeB1 = bk1 >= ak1;
    key[k] = takeB ? bk : ak;
    key[2 * H - 1 - k] = takeB1 ? bk1 : ak1;
    if constexpr (TRACK) {
      pos[k] = takeB ? bi : ai;
      pos[2 * H - 1 - k] = takeB1 ? bi1 - 1 : ai1 - 1;
    }
    ai += takeB ? 0 : 1;
    bi += takeB ? 1 : 0;
    ai1 -= takeB1 ? 0 : 1;
    bi1 -= takeB1 ? 1 : 0;
    if (k + 1 < H) {
      const K nv = s[takeB ? bi : ai];
      ak = takeB ? ak : nv;
      bk = takeB ? nv : bk;
      const K nv1 = s[(takeB1 ? bi1 : ai1) - 1];
      ak1 = takeB1 ? ak1 : nv1;
      bk1 = takeB1 ? nv1 : bk1;
    }
  }
}

// ------------------------------------------- mbarrier + 1-D bulk copy (TMA)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
#ifdef MSORT_MBAR_HINT
  // suspend (up to the hint, ns) instead of spinning on the barrier
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase), "n"(MSORT_MBAR_HINT)
      : "memory");
#else
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
#endif
}
// Non-blocking: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
// Global -> shared bulk copy (cp.async.bulk, SASS UBLKCP); dst/src 16-byte
// aligned, bytes a multiple of 16; completion counted on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Shared -> global bulk copy (SASS UBLKCP); completion tracked per issuing
// thread by bulk groups.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {  // sources of all but N groups read
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {  // all but the newest N groups complete
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// Make this thread's generic-proxy shared-memory writes visible to the async
// proxy (the bulk store engine).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// A window src[0, cnt) splits into a <16-byte head, a 16-byte aligned
// interior (moved by one bulk copy) and a <16-byte tail (plain loads).
template <class T>
__device__ __forceinline__ void window_split(const T* src, int cnt, int& head, int& mid) {
  const uintptr_t a = (uintptr_t)src;
  const uintptr_t e = a + (uintptr_t)cnt * sizeof(T);
  uintptr_t ia = (a + 15) & ~(uintptr_t)15;
  uintptr_t ie = e & ~(uintptr_t)15;
  if (ie < ia) ie = ia = e;  // too small for an aligned interior
  head = (int)((ia - a) / sizeof(T));
  mid = (int)((ie - ia) / sizeof(T));
}
template <class T>
__device__ __forceinline__ uint32_t window_bulk_bytes(const T* src, int cnt) {
  int head, mid;
  window_split(src, cnt, head, mid);
  return (uint32_t)mid * sizeof(T);
}
// Stage src[0, cnt) into shared memory at dst (same 16-byte phase as src, see
// stage_offset): the leader issues the bulk copy of the interior (after it
// armed `bar` with the expected bytes), every thread helps with head/tail.
template <class T>
__device__ __forceinline__ void stage_window(T* dst, const T* src, int cnt, uint64_t* bar,
                                             bool leader, int tid, int nthreads) {
  int head, mid;
  window_split(src, cnt, head, mid);
  const int tail = cnt - head - mid;
  if (leader && mid > 0) bulk_g2s(dst + head, src + head, (uint32_t)(mid * sizeof(T)), bar);
  for (int i = tid; i < head + tail; i += nthreads) {
    int j = i < head ? i : head + mid + (i - head);
    dst[j] = src[j];
  }
}
// Element offset (0..16/sizeof(T)-1) at which to place a window starting at
// src so that shared and global addresses share the same 16-byte phase.
template <class T>
__device__ __forceinline__ int stage_offset(const T* src) {
  return (int)(((uintptr_t)src & 15) / sizeof(T));
}

// ------------------------------------------------------ register networks
template <class K>
__device__ __forceinline__ void cmp_swap(K& a, K& b) {
  K lo = a < b ? a : b;
  K hi = a < b ? b : a;
  a = lo;
  b = hi;
}

// Batcher's odd-even merge sort network over N (power of two) registers.
// Keys only: equal integers are indistinguishable, so any network is fine.
// Sorts the first P (a power of two) of the N registers x.
template <int P, int N, class K>
__device__ __forceinline__ void batcher_sort(K (&x)[N]) {
  static_assert(P <= N, "batcher_sort: P <= N");
#pragma unroll
  for (int p = 1; p < P; p <<= 1) {
#pragma unroll
    for (int k = p; k >= 1; k >>= 1) {
#pragma unroll
      for (int j = k % p; j + k < P; j += 2 * k) {
#pragma unroll
        for (int i = 0; i < k; ++i) {
          if (i + j + k < P && (i + j) / (2 * p) == (i + j + k) / (2 * p))
            cmp_swap(x[i + j], x[i + j + k]);
        }
      }
    }
  }
}

// Bitonic sorting network over the first P (a power of two) of N registers;
// three plain counted loops that always unroll completely.
template <int P, int N, class K>
__device__ __forceinline__ void bitonic_sort(K (&x)[N]) {
#pragma unroll
  for (int k = 2; k <= P; k *= 2) {
#pragma unroll
    for (int j = k / 2; j > 0; j /= 2) {
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const int l = i ^ j;
        if (l > i) {
          if ((i & k) == 0) cmp_swap(x[i], x[l]);
          else cmp_swap(x[l], x[i]);
        }
      }
    }
  }
}

// Keys-only network for any N: bitonic on the largest power of two P <= N,
// then each remaining element is inserted by a compare-exchange chain.
// Insertion of x[M] into the sorted x[0..M) by a compare-exchange chain,
// then of x[M+1] ..., x[N-1]; template recursion keeps every index a
// compile-time constant (registers, never local memory) at any size.
template <int I, class K, int N>
struct InsertChain {
  static __device__ __forceinline__ void run(K (&x)[N]) {
    cmp_swap(x[I], x[I + 1]);
    InsertChain<I - 1, K, N>::run(x);
  }
};
template <class K, int N>
struct InsertChain<-1, K, N> {
  static __device__ __forceinline__ void run(K (&)[N]) {}
};
template <int M, int N, class K>
struct InsertAll {
  static __device__ __forceinline__ void run(K (&x)[N]) {
    InsertChain<M - 1, K, N>::run(x);
    InsertAll<M + 1, N, K>::run(x);
  }
};
template <int N, class K>
struct InsertAll<N, N, K> {
  static __device__ __forceinline__ void run(K (&)[N]) {}
};

template <int N, class K>
__device__ __forceinline__ void keys_network(K (&x)[N]) {
  constexpr int P = N >= 128 ? 128 : N >= 64 ? 64 : N >= 32 ? 32 : N >= 16 ? 16 : (N >= 8 ? 8 : (N >= 4 ? 4 : (N >= 2 ? 2 : 1)));
  static_assert(N < 256, "keys_network: N < 256");
  bitonic_sort<P>(x);
  InsertAll<P, N, K>::run(x);
}

// Warp-shuffle bitonic sorting network, keys only (the north_star's
// "warp-shuffle sorting networks"): the warp's 32 * VW keys, VW per lane,
// end sorted in BLOCKED order (lane l holds ranks [l VW, (l + 1) VW)).
// Batcher's bitonic network over i = lane * VW + k: for each block size, the
// half-cleaner strides j; element i and its partner i ^ j are put in
// ascending order when (i & size) == 0, descending otherwise.  Strides below
// VW pair registers of one lane (compare-exchange in registers); larger
// strides pair the same register of lanes lane ^ (j / VW), exchanged by
// __shfl_xor_sync -- no shared memory, no bank conflicts.  Keys only: equal
// keys are indistinguishable, so the (unstable) network gives the sort.
// One stage (block size SIZE, stride J) of the network; the stages are
// instantiated one by one (template recursion) so that every register index
// is a compile-time constant at any VW.
template <int VW, int SIZE, int J>
struct WarpBitonicStage {
  template <class K>
  static __device__ __forceinline__ void run(K (&key)[VW], int lane) {
    if constexpr (J < VW) {
#pragma unroll
      for (int k = 0; k < VW; ++k) {
        if ((k & J) == 0) {
          const int p = k | J;
          const bool up = ((lane * VW + k) & SIZE) == 0;
          const K lo = key[k] < key[p] ? key[k] : key[p];
          const K hi = key[k] < key[p] ? key[p] : key[k];
          key[k] = up ? lo : hi;
          key[p] = up ? hi : lo;
        }
      }
    } else {
      constexpr int lm = J / VW;
      const bool lower = (lane & lm) == 0;
#pragma unroll
      for (int k = 0; k < VW; ++k) {
        const K o = __shfl_xor_sync(0xffffffffu, key[k], lm);
        const bool up = ((lane * VW + k) & SIZE) == 0;
        const bool keep_small = up == lower;  // lower lane of an ascending pair: the min
        key[k] = keep_small ? (o < key[k] ? o : key[k]) : (o < key[k] ? key[k] : o);
      }
    }
    if constexpr (J > 1) {
      WarpBitonicStage<VW, SIZE, J / 2>::run(key, lane);
    } else if constexpr (SIZE < 32 * VW) {
      WarpBitonicStage<VW, SIZE * 2, SIZE>::run(key, lane);
    }
  }
};

template <int VW, class K>
__device__ __forceinline__ void warp_bitonic_keys(K (&key)[VW], int lane) {
  static_assert((VW & (VW - 1)) == 0, "VW: power of two");
  WarpBitonicStage<VW, 2, 1>::run(key, lane);
}

// Odd-even transposition sort: swaps only adjacent elements and only when
// strictly greater, so it is stable -- used when a payload index travels.
template <int N, class K>
__device__ __forceinline__ void odd_even_transposition_sort(K (&x)[N], int (&idx)[N]) {
#pragma unroll
  for (int r = 0; r < N; ++r) {
#pragma unroll
    for (int i = r & 1; i + 1 < N; i += 2) {
      bool sw = x[i] > x[i + 1];
      K a = sw ? x[i + 1] : x[i];
      K b = sw ? x[i] : x[i + 1];
      int ia = sw ? idx[i + 1] : idx[i];
      int ib = sw ? idx[i] : idx[i + 1];
      x[i] = a, x[i + 1] = b, idx[i] = ia, idx[i + 1] = ib;
    }
  }
}

}  // namespace msort
