// seg_sort.cuh -- batched (segmented) sorts: many independent small arrays
// sorted in one call (the paper's small-array regime,
// P:332 / P:565, where per-array parallel overhead dominates).
//
// Segments are binned by length (Kernels::sort_segmented):
//   len <= 32        kseg_tiny_sort, found on the device from the offsets
//                    table: a warp sorts 4 segments at once, one register
//                    each, with a 32-element bitonic network whose stages are
//                    __shfl_xor_sync exchanges between lanes;
//   len <= 256       kseg_mid_sort: one warp per segment, 2/4/8 keys per
//                    lane, a 64/128/256-element bitonic network (in-lane
//                    stages for strides below the keys per lane, shuffles
//                    above);
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

// Segments of 2..32 elements straight from the offsets table.  Warp w of the
// grid takes segments [w*S, w*S + S) and sorts the short ones TOGETHER:
// register j of every lane holds element `lane` of segment j, and one
// 32-element bitonic network runs on all S registers (S independent shuffle
// chains: S loads in flight and S-way ILP for these latency-bound segments).
// Longer or trivial segments are left to the other kernels.
#ifndef MSORT_SEG_PER_WARP
#define MSORT_SEG_PER_WARP 4
#endif
constexpr int kSegPerWarp = MSORT_SEG_PER_WARP;
template <class K, bool PAIRS>
__global__ void __launch_bounds__(128)
    kseg_tiny_sort(K* __restrict__ keys, uint32_t* __restrict__ vals,
                   const int64_t* __restrict__ off, int64_t nseg) {
  constexpr int S = kSegPerWarp;
  const int lane = threadIdx.x & 31;
  const int64_t s0 = ((int64_t)blockIdx.x * 4 + (threadIdx.x >> 5)) * S;
  if (s0 >= nseg) return;  // warp-uniform
  // the S + 1 boundaries, one lane each
  int64_t ob = 0;
  if (lane <= S && s0 + lane <= nseg) ob = off[s0 + lane];
  int64_t base[S];
  int cnt[S];
  K key[S];
  int idx[S];
#pragma unroll
  for (int j = 0; j < S; ++j) {
    const int64_t a = __shfl_sync(0xffffffffu, ob, j), e = __shfl_sync(0xffffffffu, ob, j + 1);
    const int64_t l = s0 + j < nseg ? e - a : 0;
    base[j] = a;
    cnt[j] = l >= 2 && l <= 32 ? (int)l : 0;
    key[j] = lane < cnt[j] ? keys[a + lane] : KeyTraits<K>::max_key();
    idx[j] = lane;
  }
  // one 32-element bitonic network per register (element index = lane)
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int st = size >> 1; st > 0; st >>= 1) {
      // the lower lane of an ascending pair keeps the smaller element
      const bool keep_small = ((lane & size) == 0) == ((lane & st) == 0);
#pragma unroll
      for (int j = 0; j < S; ++j) {
        const K ok = __shfl_xor_sync(0xffffffffu, key[j], st);
        int oi = idx[j];
        if constexpr (PAIRS) oi = __shfl_xor_sync(0xffffffffu, idx[j], st);
        if (keep_small == seg_less<K, PAIRS>(ok, oi, key[j], idx[j])) key[j] = ok, idx[j] = oi;
      }
    }
  }
  uint32_t v[PAIRS ? S : 1];
  if constexpr (PAIRS) {
#pragma unroll
    for (int j = 0; j < S; ++j)
      if (lane < cnt[j]) v[j] = vals[base[j] + idx[j]];
    __syncwarp();  // all payloads read before any is overwritten
  }
#pragma unroll
  for (int j = 0; j < S; ++j)
    if (lane < cnt[j]) {
      keys[base[j] + lane] = key[j];
      if constexpr (PAIRS) vals[base[j] + lane] = v[j];
    }
}

// Segments of 33..256 elements: one warp per (offset, length) descriptor,
// the smallest network that holds the segment: 64, 128 or 256 elements (2, 4
// or 8 keys per lane; the choice is warp-uniform).
template <class K, bool PAIRS>
__global__ void __launch_bounds__(128)
    kseg_mid_sort(K* __restrict__ keys, uint32_t* __restrict__ vals,
                  const int64_t* __restrict__ desc, int64_t cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t d = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (d >= cnt) return;
  const int64_t base = desc[2 * d];
  // the segment length as a ballot (a warp-uniform value the compiler can see
  // as such): the network chosen by it runs in convergent code, so its
  // shuffles need no per-shuffle WARPSYNC / ENDCOLLECTIVE
  const int len = (int)desc[2 * d + 1];
  const unsigned cls = __ballot_sync(0xffffffffu, lane == 0 ? len > 64 : false) |
                       (__ballot_sync(0xffffffffu, lane == 0 ? len > 128 : false) << 1);
  if (cls == 0) warp_sort_segment<K, PAIRS, 2>(keys, vals, base, len, lane);
  else if (cls == 1) warp_sort_segment<K, PAIRS, 4>(keys, vals, base, len, lane);
  else warp_sort_segment<K, PAIRS, 8>(keys, vals, base, len, lane);
}

// Device-resident offsets: classify every segment (and check the table:
// off[0] = 0, non-decreasing, off[nseg] = n).  counts[c] = entries appended to
// list c of (offset, length) for lengths in (32, 256], (256, m], (m, t] and
// > t; counts[4] = segments of 2..32 elements (kseg_tiny_sort reads those from
// the table itself); counts[5] != 0 flags a bad table.  List order is
// arbitrary (segments are independent).
__global__ void __launch_bounds__(256)
    kseg_classify(const int64_t* __restrict__ off, int64_t nseg, int64_t n, int64_t m, int64_t t,
                  int64_t* __restrict__ l0, int64_t* __restrict__ l1, int64_t* __restrict__ l2,
                  int64_t* __restrict__ l3, unsigned long long* __restrict__ counts) {
  // list capacities: a valid table has at most n / (lower bound + 1) such segments
  const unsigned long long cap[4] = {
      (unsigned long long)(n / 33 + 1), (unsigned long long)(n / 257 + 1),
      (unsigned long long)(n / (m + 1) + 1), (unsigned long long)(n / (t + 1) + 1)};
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // whole warps iterate together (ballot-aggregated tiny count)
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < nseg;
       base += stride) {
    const int64_t i = base + lane;
    int c = -1;  // list of this lane's segment (4: tiny, counted only)
    int64_t o0 = 0, len = 0;
    if (i < nseg) {
      o0 = off[i];
      const int64_t o1 = off[i + 1];
      len = o1 - o0;
      const bool bad = len < 0 || o0 < 0 || o1 > n || (i == 0 && o0 != 0) ||
                       (i == nseg - 1 && o1 != n);
      if (bad) atomicOr(counts + 5, 1ull);
      else if (len >= 2) c = len <= 32 ? 4 : len <= 256 ? 0 : len <= m ? 1 : len <= t ? 2 : 3;
    }
    // one atomic per class per warp; lanes of a class write at base + rank
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const unsigned b = __ballot_sync(0xffffffffu, c == k);
      if (!b) continue;
      unsigned long long at = 0;
      if (lane == __ffs(b) - 1) at = atomicAdd(counts + k, (unsigned long long)__popc(b));
      at = __shfl_sync(0xffffffffu, at, __ffs(b) - 1);
      if (c == k && k < 4) {
        const unsigned long long slot = at + __popc(b & ((1u << lane) - 1));
        int64_t* l = k == 0 ? l0 : k == 1 ? l1 : k == 2 ? l2 : l3;
        if (slot < cap[k]) l[2 * slot] = o0, l[2 * slot + 1] = len;
        else atomicOr(counts + 5, 1ull);  // overlapping segments: not a valid table
      }
    }
  }
}

}  // namespace msort
