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
  static __host__ __device__ __forceinline__ U image(int32_t x) { return (U)x ^ 0x80000000u; }
};
template <>
struct KeyTraits<uint32_t> {
  using U = uint32_t;
  static __host__ __device__ __forceinline__ uint32_t max_key() { return 0xffffffffu; }
  static __host__ __device__ __forceinline__ U image(uint32_t x) { return x; }
};
template <>
struct KeyTraits<int64_t> {
  using U = uint64_t;
  static __host__ __device__ __forceinline__ int64_t max_key() { return 0x7fffffffffffffffll; }
  static __host__ __device__ __forceinline__ U image(int64_t x) {
    return (U)x ^ 0x8000000000000000ull;
  }
};
template <>
struct KeyTraits<uint64_t> {
  using U = uint64_t;
  static __host__ __device__ __forceinline__ uint64_t max_key() { return ~0ull; }
  static __host__ __device__ __forceinline__ U image(uint64_t x) { return x; }
};

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

// Same search over global memory with 64-bit indices.
template <class K>
__device__ __forceinline__ int64_t merge_path_global(const K* __restrict__ a, int64_t na,
                                                     const K* __restrict__ b, int64_t nb,
                                                     int64_t d) {
  int64_t lo = d - nb > 0 ? d - nb : 0;
  int64_t hi = d < na ? d : na;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) > __ldg(b + (d - 1 - mid))) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// Serial stable merge of VT outputs starting at (ai, bi): take B only when
// B < A (strict), so ties go to A.  Positions are indices into the shared
// buffer s; `pos` records the source position of each output (for payload
// gathers) when TRACK, and `src_idx` (if non-null) maps a position to an
// original index carried from an earlier merge round.
template <class K, bool PAD, bool TRACK, int VT>
__device__ __forceinline__ void serial_merge(const K* s, const int* src_idx, int ai, int aend,
                                             int bi, int bend, K (&key)[VT], int (&pos)[VT]) {
  K ak = ai < aend ? s[sidx<K, PAD>(ai)] : K(0);
  K bk = bi < bend ? s[sidx<K, PAD>(bi)] : K(0);
#pragma unroll
  for (int k = 0; k < VT; ++k) {
    bool takeB = (bi < bend) && ((ai >= aend) || (bk < ak));
    key[k] = takeB ? bk : ak;
    if constexpr (TRACK) {
      int p = takeB ? bi : ai;
      pos[k] = src_idx ? src_idx[sidx<K, PAD>(p)] : p;
    }
    if (takeB) {
      ++bi;
      if (bi < bend) bk = s[sidx<K, PAD>(bi)];
    } else {
      ++ai;
      if (ai < aend) ak = s[sidx<K, PAD>(ai)];
    }
  }
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
template <int N, class K>
__device__ __forceinline__ void batcher_sort(K (&x)[N]) {
#pragma unroll
  for (int p = 1; p < N; p <<= 1) {
#pragma unroll
    for (int k = p; k >= 1; k >>= 1) {
#pragma unroll
      for (int j = k % p; j + k < N; j += 2 * k) {
#pragma unroll
        for (int i = 0; i < k; ++i) {
          if (i + j + k < N && (i + j) / (2 * p) == (i + j + k) / (2 * p))
            cmp_swap(x[i + j], x[i + j + k]);
        }
      }
    }
  }
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
