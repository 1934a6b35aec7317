// seg_sort.cuh -- batched (segmented) sorts: many independent small arrays
// sorted in one call (the paper's small-array regime,
// P:332 / P:565, where per-array parallel overhead dominates).
//
// Segments are binned by length (Kernels::sort_segmented):
//   len <= 256       one WARP per segment (this file), found on the device
//                    from the offsets table: the warp holds the segment in
//                    registers (1 or 8 keys per lane for <= 32 / <= 256) and
//                    sorts it with a bitonic network whose cross-lane stages
//                    are __shfl_xor_sync exchanges;
//   len <= T         one CTA per segment: the tile-sort kernels (K1) with a
//                    segment descriptor instead of a tile index (128 x 17
//                    threads x keys up to 2176, the K1 tile shape up to T);
//   len >  T         K1 on the segment's tiles, then ONE fused merge launch
//                    for all such segments (SegFused, k3_merge.cuh).
// Stability: the warp network compares (key, original index) -- indices are
// unique, so the (unstable) bitonic network yields the stable order; with
// keys only equal keys are indistinguishable and the key alone decides.
#pragma once

#include "msort_device.cuh"

namespace msort {

// (key, idx) < (key', idx') lexicographically: the stable order (P:107 with
// ties to the earlier element, R1).
template <class K, bool PAIRS>
__device__ __forceinline__ bool seg_less(K a, int ia, K b, int ib) {
  if constexpr (PAIRS) return a < b || (a == b && ia < ib);
  else return a < b;
}

// One warp sorts one segment of at most 32 * VW elements: keys[base, base +
// cnt).  Element i of the segment lives in lane i / VW, register i % VW
// ("blocked"); the padding (MAX key, index >= cnt) sorts after every real
// element.
template <class K, bool PAIRS, int VW>
__device__ __forceinline__ void warp_sort_segment(K* __restrict__ keys,
                                                  uint32_t* __restrict__ vals, int64_t base,
                                                  int cnt, int lane) {
  constexpr int N = 32 * VW;
  static_assert((VW & (VW - 1)) == 0, "VW: power of two");
  K key[VW];
  int idx[VW];
#pragma unroll
  for (int k = 0; k < VW; ++k) {
    const int i = lane * VW + k;
    key[k] = i < cnt ? keys[base + i] : KeyTraits<K>::max_key();
    idx[k] = i;
  }
  // Bitonic sorting network over i = lane * VW + k (Batcher): for each block
  // size `size`, half-cleaner strides j; element i and its partner i ^ j are
  // put in ascending order when (i & size) == 0, descending otherwise.
#pragma unroll
  for (int size = 2; size <= N; size <<= 1) {
#pragma unroll
    for (int j = size >> 1; j > 0; j >>= 1) {
      if (j < VW) {
        // partner in the same lane
#pragma unroll
        for (int k = 0; k < VW; ++k) {
          const int p = k ^ j;
          if (p > k) {
            const bool up = ((lane * VW + k) & size) == 0;
            const bool sw = up ? seg_less<K, PAIRS>(key[p], idx[p], key[k], idx[k])
                               : seg_less<K, PAIRS>(key[k], idx[k], key[p], idx[p]);
            if (sw) {
              const K tk = key[k];
              key[k] = key[p], key[p] = tk;
              const int ti = idx[k];
              idx[k] = idx[p], idx[p] = ti;
            }
          }
        }
      } else {
        // partner in lane ^ (j / VW), same register
        const int lm = j / VW;
        const bool lower = (lane & lm) == 0;
#pragma unroll
        for (int k = 0; k < VW; ++k) {
          const K ok = __shfl_xor_sync(0xffffffffu, key[k], lm);
          int oi = idx[k];
          if constexpr (PAIRS) oi = __shfl_xor_sync(0xffffffffu, idx[k], lm);
          const bool up = ((lane * VW + k) & size) == 0;
          // the lower lane of an ascending pair keeps the smaller element
          const bool keep_small = up == lower;
          const bool other_less = seg_less<K, PAIRS>(ok, oi, key[k], idx[k]);
          if (keep_small == other_less) key[k] = ok, idx[k] = oi;
        }
      }
    }
  }
  uint32_t v[PAIRS ? VW : 1];
  if constexpr (PAIRS) {
#pragma unroll
    for (int k = 0; k < VW; ++k)
      if (idx[k] < cnt) v[k] = vals[base + idx[k]];
    __syncwarp();  // every lane has read its payloads before any is overwritten
  }
#pragma unroll
  for (int k = 0; k < VW; ++k) {
    const int i = lane * VW + k;
    if (i < cnt) {
      keys[base + i] = key[k];
      if constexpr (PAIRS) vals[base + i] = v[k];
    }
  }
}

// Segments of 2..256 elements straight from the offsets table: warp w of the
// grid takes segment w, sorts it with a 32- or 256-element network by its
// length (warp-uniform), and leaves longer or trivial segments alone (the
// CTA-per-segment and merge paths take those).
template <class K, bool PAIRS>
__global__ void __launch_bounds__(128)
    kseg_warp_sort(K* __restrict__ keys, uint32_t* __restrict__ vals,
                   const int64_t* __restrict__ off, int64_t nseg) {
  const int lane = threadIdx.x & 31;
  const int64_t s = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (s >= nseg) return;  // warp-uniform
  const int64_t base = off[s];
  const int64_t len = off[s + 1] - base;
  if (len < 2 || len > 256) return;
  if (len <= 32) warp_sort_segment<K, PAIRS, 1>(keys, vals, base, (int)len, lane);
  else warp_sort_segment<K, PAIRS, 8>(keys, vals, base, (int)len, lane);
}

// Device-resident offsets: classify every segment (and check the table:
// off[0] = 0, non-decreasing, off[nseg] = n).  counts[0..2] = entries
// appended to the lists of (offset, length) for lengths in (w8, m], (m, t]
// and > t; counts[3] = segments of 2..w8 elements (the warp kernel's); counts[4]
// != 0 flags a bad table.  List order is arbitrary (segments are independent).
__global__ void __launch_bounds__(256)
    kseg_classify(const int64_t* __restrict__ off, int64_t nseg, int64_t n, int64_t w8, int64_t m,
                  int64_t t, int64_t* __restrict__ lm, int64_t* __restrict__ ll,
                  int64_t* __restrict__ lx, unsigned long long* __restrict__ counts) {
  // list capacities: a valid table has at most n / (bound + 1) such segments
  const unsigned long long cap[3] = {(unsigned long long)(n / (w8 + 1) + 1),
                                     (unsigned long long)(n / (m + 1) + 1),
                                     (unsigned long long)(n / (t + 1) + 1)};
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // whole warps iterate together (ballot-aggregated small count)
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < nseg;
       base += stride) {
    const int64_t i = base + lane;
    bool small = false;
    if (i < nseg) {
      const int64_t o0 = off[i], o1 = off[i + 1], len = o1 - o0;
      const bool bad = len < 0 || o0 < 0 || o1 > n || (i == 0 && o0 != 0) ||
                       (i == nseg - 1 && o1 != n);
      if (bad) atomicOr(counts + 4, 1ull);
      small = !bad && len >= 2 && len <= w8;
      if (!bad && len > w8) {
        const int c = len <= m ? 0 : len <= t ? 1 : 2;
        int64_t* l = c == 0 ? lm : c == 1 ? ll : lx;
        const unsigned long long k = atomicAdd(counts + c, 1ull);
        if (k < cap[c]) l[2 * k] = o0, l[2 * k + 1] = len;
        else atomicOr(counts + 4, 1ull);  // overlapping segments: not a valid table
      }
    }
    const unsigned b = __ballot_sync(0xffffffffu, small);
    if (lane == 0 && b) atomicAdd(counts + 3, (unsigned long long)__popc(b));
  }
}

}  // namespace msort
