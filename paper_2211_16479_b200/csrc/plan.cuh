// plan.cuh -- splitter co-rank arithmetic of the distributed sort (D2),
// shared verbatim by the device kernels and the exported host helpers
// (msort_plan_*), so the multi-process protocol can be tested on CPU.
//
// The paper's MPI merge sort pairs ranks in a tree and funnels everything to
// rank 0 (Fig. fig:mpi-merge-code).  Here every rank keeps a
// balanced slice of the globally sorted output (R10): rank r owns
// global stable positions [K_r, K_{r+1}), K_r = sum_{j<r} n_j, and the split
// matrix s[r][j] counts rank j's elements before position K_r.
//
// Search: v*_r = the key image at global position K_r = the smallest image u
// with sum_j #{x in shard j : image(x) <= u} > K_r.  Each round splits the
// inclusive interval [lo, hi] into B buckets; bucket b's upper end is the
// candidate c_b; the new interval is the first bucket whose global count
// exceeds K_r (the last one if none -- then v* ends at the maximum image and
// the fill below still yields s[r][j] = n_j).
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define MSORT_HD __host__ __device__ __forceinline__
#else
#define MSORT_HD inline
#endif

namespace msort {
namespace plan {

// Upper end of bucket b of [lo, hi] split into B buckets of width
// step = (hi - lo) / B + 1; the last bucket ends at hi.  No overflow: for
// b < B-1, step*(b+1) <= (2^64/B + 1)*(B-1) < 2^64.
MSORT_HD uint64_t candidate(uint64_t lo, uint64_t hi, int b, int B) {
  if (b >= B - 1) return hi;
  uint64_t width = hi - lo;
  uint64_t step = width / (uint64_t)B + 1;
  uint64_t off = step * (uint64_t)(b + 1) - 1;
  return off >= width ? hi : lo + off;
}

// New interval from the global counts le[b] = #{image <= candidate b}.
MSORT_HD void narrow(uint64_t& lo, uint64_t& hi, const uint64_t* le, int B, uint64_t K) {
  int sel = B - 1;
  for (int b = 0; b < B; ++b) {
    if (le[b] > K) {
      sel = b;
      break;
    }
  }
  uint64_t nlo = sel == 0 ? lo : candidate(lo, hi, sel - 1, B) + 1;
  uint64_t nhi = candidate(lo, hi, sel, B);
  if (nlo > nhi) nlo = nhi;  // only when an earlier bucket collapsed onto hi
  lo = nlo;
  hi = nhi;
}

// s[r][j] for 0 < r < world from the gathered counts of boundary r:
//   s[r][j] = lt_j + clamp(K_r - sum lt - sum_{j'<j} eq_j', 0, eq_j),
// i.e. ties at v*_r are handed out in rank order (lower rank first), which is
// the stable order of the rank-major concatenation (R11).
// Layout of the gathered counts: lteq[(t*(world-1) + (r-1))*2 + {0: lt, 1: eq}].
MSORT_HD int64_t fill_one(uint64_t K, const uint64_t* lteq, int world, int r, int j) {
  const int nb = world - 1;
  uint64_t sum_lt = 0, eq_before = 0;
  for (int t = 0; t < world; ++t) sum_lt += lteq[(t * nb + (r - 1)) * 2 + 0];
  for (int t = 0; t < j; ++t) eq_before += lteq[(t * nb + (r - 1)) * 2 + 1];
  const uint64_t lt = lteq[(j * nb + (r - 1)) * 2 + 0];
  const uint64_t eq = lteq[(j * nb + (r - 1)) * 2 + 1];
  // K >= sum lt holds for the exact v*; the clamp also covers K >= N.
  int64_t rem = (int64_t)K - (int64_t)sum_lt - (int64_t)eq_before;
  if (rem < 0) rem = 0;
  if (rem > (int64_t)eq) rem = (int64_t)eq;
  return (int64_t)lt + rem;
}

// The paper's merge tree (f4): with `active` ranks left, split =
// ceil(active / 2) (= active / 2, the paper's, for powers of two); ranks in
// [split, active) send to rank - split, ranks below active - split receive
// from rank + split.  Rounds until one rank is active:
inline int tree_rounds(int world) {
  int r = 0;
  for (int a = world; a > 1; a = (a + 1) / 2) ++r;
  return r;
}
// This rank's role in round t: 0 idle, 1 parent (receives from *peer and
// merges [own | received], own first on ties), 2 child (sends to *peer).
inline int tree_role(int world, int rank, int t, int* peer) {
  int a = world;
  for (int i = 0; i < t; ++i) a = (a + 1) / 2;
  if (a <= 1) return 0;
  const int split = (a + 1) / 2;
  if (rank >= split && rank < a) {
    *peer = rank - split;
    return 2;
  }
  if (rank < a - split) {
    *peer = rank + split;
    return 1;
  }
  return 0;
}

}  // namespace plan
}  // namespace msort
