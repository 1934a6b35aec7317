// k3_merge.cuh -- K3, the global merge pass (SURVEY.md §8(a) S2+S3).
//
// Merges run pairs (A, B) into one run with the stable merge() of P:107 (ties
// take the left run, R1).  The output of a merge level is cut into
// tiles of Tm elements; tile q covers diagonals [q*Tm, (q+1)*Tm) of its pair
// and needs the merge-path co-rank
//     i(d) = min{ i : i = min(d, |A|) or A[i] > B[d-1-i] }
// at its two boundary diagonals (K2, fused here).
//
// One persistent, warp-specialised kernel; work is handed out dynamically in
// chunks of CH consecutive tiles through a global atomic counter.  Roles:
//   warp 1      co-rank searcher: grabs `grab` (<= kGrab) chunks at a time and
//               binary-searches their boundary co-ranks in global memory (one
//               lane each) into a ring of chunk descriptors (mbarriers);
//   warp 0      TMA producer: stages A[i0,i1) and B[j0,j1) of each tile into an
//               S-stage shared ring with cp.async.bulk (UBLKCP) + mbarrier;
//   warps 2..   mergers: per thread a merge-path search in shared memory and
//               a branch-free serial merge of VT outputs; the output overwrites
//               the consumed stage and leaves by one bulk store.
// At start every warp helps with the first chunk's co-ranks (32-way
// cooperative searches).
//
// Two work sources (the Src template parameter):
//   SinglePass  - one merge level (also the distributed k-way merge rounds);
//   FusedPasses - ALL merge levels of a sort in one launch, as a dataflow:
//                 a chunk of level p starts as soon as the two level-(p-1)
//                 pairs it reads are complete (per-pair completion counters,
//                 release/acquire at GPU scope), so there is no idle gap or
//                 tail at level boundaries except where a level depends on
//                 the whole previous one.
#pragma once

#include <type_traits>

#include "msort_device.cuh"

namespace msort {

// ---------------------------------------------------------------- pair maps
// Where output tile q sits: its run pair starts at A0 (global index), run A
// has na elements, run B (immediately after A) nb, and the tile's first
// output diagonal is dl inside the pair.  The pair's output occupies
// [A0, A0+na+nb) of the destination.
struct UniformPairs {  // runs of length L (the last ones may be short)
  int64_t n, L;
  __device__ __forceinline__ void locate(int64_t q, int T, int64_t& A0, int64_t& na,
                                         int64_t& nb, int64_t& dl) const {
    int64_t d = q * T;
    int64_t m = d / (2 * L);
    A0 = m * 2 * L;
    na = min(L, n - A0);
    int64_t B0 = A0 + L;
    nb = B0 < n ? min(L, n - B0) : 0;
    dl = d - A0;
  }
  // runs A and B of tile q's pair (output at A0): contiguous in src
  template <class T>
  __device__ __forceinline__ const T* ra(const T* src, int64_t, int64_t A0, int64_t, bool) const {
    return src + A0;
  }
  template <class T>
  __device__ __forceinline__ const T* rb(const T* src, int64_t, int64_t A0, int64_t na,
                                         bool) const {
    return src + A0 + na;
  }
};

constexpr int kMaxPairs = 64;
struct ExplicitPairs {  // arbitrary consecutive runs, pairs (2m, 2m+1)
  int npairs;
  int64_t first_tile[kMaxPairs + 1];
  int64_t off[2 * kMaxPairs + 1];
  __device__ __forceinline__ void locate(int64_t q, int T, int64_t& A0, int64_t& na,
                                         int64_t& nb, int64_t& dl) const {
    int m = 0;
    while (m + 1 < npairs && first_tile[m + 1] <= q) ++m;
    A0 = off[2 * m];
    na = off[2 * m + 1] - A0;
    nb = off[2 * m + 2] - off[2 * m + 1];
    dl = (q - first_tile[m]) * T;
  }
  template <class T>
  __device__ __forceinline__ const T* ra(const T* src, int64_t, int64_t A0, int64_t, bool) const {
    return src + A0;
  }
  template <class T>
  __device__ __forceinline__ const T* rb(const T* src, int64_t, int64_t A0, int64_t na,
                                         bool) const {
    return src + A0 + na;
  }
};

// Runs that live in different buffers -- on a multi-GPU run, in the peers'
// memory (NVLink/NVSwitch, mapped into this process): pair m merges run
// a[m] (na[m] keys) with run b[m] (nb[m]) into the output at out[m].  The
// first k-way merge round of the distributed sort reads the p sorted segments
// straight from their owners this way ("pull" exchange).
struct PeerPairs {
  int npairs;
  int64_t first_tile[kMaxPairs + 1];
  int64_t out[kMaxPairs];
  int64_t na[kMaxPairs], nb[kMaxPairs];
  const void* ka[kMaxPairs];
  const void* kb[kMaxPairs];
  const uint32_t* va[kMaxPairs];
  const uint32_t* vb[kMaxPairs];
  __device__ __forceinline__ int find(int64_t q) const {
    int m = 0;
    while (m + 1 < npairs && first_tile[m + 1] <= q) ++m;
    return m;
  }
  __device__ __forceinline__ void locate(int64_t q, int T, int64_t& A0, int64_t& na_,
                                         int64_t& nb_, int64_t& dl) const {
    const int m = find(q);
    A0 = out[m], na_ = na[m], nb_ = nb[m];
    dl = (q - first_tile[m]) * T;
  }
  // keys (vals = false) or payloads (vals = true) of tile q's runs
  template <class T>
  __device__ __forceinline__ const T* ra(const T*, int64_t q, int64_t, int64_t, bool vals) const {
    const int m = find(q);
    return vals ? reinterpret_cast<const T*>(va[m]) : static_cast<const T*>(ka[m]);
  }
  template <class T>
  __device__ __forceinline__ const T* rb(const T*, int64_t q, int64_t, int64_t, bool vals) const {
    const int m = find(q);
    return vals ? reinterpret_cast<const T*>(vb[m]) : static_cast<const T*>(kb[m]);
  }
};

#ifndef MSORT_K3_CHUNK
#define MSORT_K3_CHUNK 8
#endif
#ifndef MSORT_K3_GRAB
#define MSORT_K3_GRAB 3
#endif
constexpr int kChunk = MSORT_K3_CHUNK;  // tiles per dynamically scheduled chunk
constexpr int kGrab = MSORT_K3_GRAB;    // chunks taken per atomic
#ifndef MSORT_K3_RING1
#define MSORT_K3_RING1 2
#endif
// chunk-descriptor ring slots when a grab is one chunk (the searcher may run
// kRing1 - 1 chunks ahead of the producer); <= the 2 * kGrab slots allocated
constexpr int kRing1 = MSORT_K3_RING1;
static_assert(kRing1 >= 2 && kRing1 <= 2 * kGrab, "ring of single-chunk grabs");
constexpr int kMaxFusedPasses = 48;

struct TileMeta {
  int64_t out;  // output index of the tile's first element (-1: stop)
  int64_t q;    // tile index within its level
  int na, nb, offA, offB, offAv, offBv, tot, pass;
};

struct ChunkDesc {
  int64_t q0;  // first tile
  int cnt;     // tiles in the chunk (0: no more work)
  int pass;    // merge level
  int64_t co[kChunk + 1];  // co-ranks of its boundary diagonals
};

constexpr size_t align_up_c(size_t x, size_t a) { return (x + a - 1) / a * a; }

template <class K, bool PAIRS, int NC, int VT, int S>
struct K3Layout {
  static constexpr int Tm = NC * VT;
  static constexpr int EK = 16 / sizeof(K);
  static constexpr int R = 2 * kGrab;      // chunk ring: two searcher rounds
  static constexpr int SKE = Tm + 4 * EK;  // keys per stage (windows + phase slack)
  static constexpr int SVE = Tm + 16;      // payloads per stage
  static constexpr size_t bars = 0;  // full[S], empty[S], sfull[R], sempty[R], outr[S]
  static constexpr size_t meta = align_up_c(8 * (3 * S + 2 * R), 16);
  static constexpr size_t ring = align_up_c(meta + sizeof(TileMeta) * S, 16);
  static constexpr size_t corank = ring + sizeof(ChunkDesc) * R;  // NC+1 ints
  static constexpr size_t misc = align_up_c(corank + 4 * (NC + 1), 16);
  static constexpr size_t stage_k = align_up_c(misc + 16, 128);
  static constexpr size_t stage_v = align_up_c(stage_k + (size_t)S * SKE * sizeof(K), 128);
  static constexpr size_t bytes = align_up_c(stage_v + (PAIRS ? (size_t)S * SVE * 4 : 0), 128);
};

// ------------------------------------------------------------ work sources
template <class K, class PM>
struct SinglePass {
  static constexpr bool kFused = false;
  PM pm;
  const K* src_k;
  const uint32_t* src_v;
  K* dst_k;
  uint32_t* dst_v;
  int64_t ntiles;
  int ch;    // tiles per chunk (1..kChunk; small sorts use small chunks)
  int grab;  // chunks per atomic grab (1..kGrab)
  __device__ __forceinline__ int64_t nchunks() const { return (ntiles + ch - 1) / ch; }
  __device__ __forceinline__ void chunk(int64_t g, int& pass, int64_t& q0, int& cnt) const {
    pass = 0;
    q0 = g * ch;
    cnt = (int)min((int64_t)ch, ntiles - q0);
  }
  __device__ __forceinline__ int64_t tiles(int) const { return ntiles; }
  __device__ __forceinline__ void wait_ready(int, int64_t, int, int, int) const {}
  __device__ __forceinline__ void locate(int, int64_t q, int Tm, int64_t& A0, int64_t& na,
                                         int64_t& nb, int64_t& dl) const {
    pm.locate(q, Tm, A0, na, nb, dl);
  }
  __device__ __forceinline__ const K* srck(int) const { return src_k; }
  __device__ __forceinline__ const uint32_t* srcv(int) const { return src_v; }
  // runs A / B (keys, payloads) of tile q, whose pair's output starts at A0
  __device__ __forceinline__ const K* pa(int, int64_t q, int64_t A0, int64_t na) const {
    return pm.ra(src_k, q, A0, na, false);
  }
  __device__ __forceinline__ const K* pb(int, int64_t q, int64_t A0, int64_t na) const {
    return pm.rb(src_k, q, A0, na, false);
  }
  __device__ __forceinline__ const uint32_t* pva(int, int64_t q, int64_t A0, int64_t na) const {
    return pm.ra(src_v, q, A0, na, true);
  }
  __device__ __forceinline__ const uint32_t* pvb(int, int64_t q, int64_t A0, int64_t na) const {
    return pm.rb(src_v, q, A0, na, true);
  }
  __device__ __forceinline__ K* dstk(int, int64_t) const { return dst_k; }
  __device__ __forceinline__ uint32_t* dstv(int, int64_t) const { return dst_v; }
  __device__ __forceinline__ void tile_done(int, int64_t, int) const {}
};

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_gpu_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

#ifdef MSORT_K3_TRACE
// Tuning builds only: per-tile publish times (index pass * ntiles + q) and
// per-chunk times (grab, inputs ready, co-ranks searched, CTA) of the last
// fused K3 launch.
constexpr int kK3TraceTiles = 1 << 20, kK3TraceChunks = 1 << 18;
__device__ unsigned long long g_k3_tiles[kK3TraceTiles];
__device__ unsigned long long g_k3_chunks[kK3TraceChunks * 4];
__device__ __forceinline__ unsigned long long gtimer2() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void k3_trace_chunk(int64_t g, int slot, unsigned long long v) {
  if (g < kK3TraceChunks) g_k3_chunks[g * 4 + slot] = v;
}
#define K3_TRACE_CHUNK(g, slot, v) k3_trace_chunk((g), (slot), (v))
#else
#define K3_TRACE_CHUNK(g, slot, v) ((void)0)
#endif

// All merge levels of one sort: level p merges runs of L_p = T * 2^p from
// buffer bk[p & 1] into bk[(p+1) & 1]; every level has the same tile count.
template <class K>
struct FusedPasses {
  static constexpr bool kFused = true;
  K* bk[2];
  uint32_t* bv[2];
  int64_t n, T, ntiles;
  int P;
  int ch;          // tiles per chunk (1..kChunk; small sorts use small chunks)
  int grab;        // chunks per atomic grab (1..kGrab)
  unsigned* done;  // per level, per pair: tiles completed
  int64_t pair_base[kMaxFusedPasses + 1];
  // key-range gate (Kernels::sort_narrowed): with gate set the launch does
  // nothing unless range_narrow(gate) == gate_want
  const unsigned long long* gate;
  int gate_want;
  __device__ __forceinline__ int64_t cpp() const { return (ntiles + ch - 1) / ch; }
  __device__ __forceinline__ int64_t nchunks() const { return (int64_t)P * cpp(); }
  __device__ __forceinline__ void chunk(int64_t g, int& pass, int64_t& q0, int& cnt) const {
    const int64_t c = cpp();
    pass = (int)(g / c);
    q0 = (g % c) * ch;
    cnt = (int)min((int64_t)ch, ntiles - q0);
  }
  __device__ __forceinline__ int64_t tiles(int) const { return ntiles; }
  __device__ __forceinline__ int64_t L(int pass) const { return T << pass; }
  __device__ __forceinline__ void locate(int pass, int64_t q, int Tm, int64_t& A0, int64_t& na,
                                         int64_t& nb, int64_t& dl) const {
    UniformPairs{n, L(pass)}.locate(q, Tm, A0, na, nb, dl);
  }
  __device__ __forceinline__ int64_t pair_of(int pass, int64_t q, int Tm) const {
    return q * Tm / (2 * L(pass));
  }
  __device__ __forceinline__ unsigned pair_tiles(int pass, int64_t m, int Tm) const {
    const int64_t len = min(2 * L(pass), n - m * 2 * L(pass));
    return (unsigned)((len + Tm - 1) / Tm);
  }
  // Level p >= 1 reads the outputs of level-(p-1) pairs 2m, 2m+1: wait until
  // those are complete (the whole warp returns together).
  __device__ __forceinline__ void wait_ready(int pass, int64_t q0, int cnt, int lane,
                                             int Tm) const {
    if (pass == 0) return;
    const int64_t m0 = pair_of(pass, q0, Tm), m1 = pair_of(pass, q0 + cnt - 1, Tm);
    const int64_t np = pair_base[pass] - pair_base[pass - 1];  // pairs of level p-1
    const int64_t last = min(2 * m1 + 1, np - 1);
    for (int64_t dp = 2 * m0 + lane; dp <= last; dp += 32) {
      const unsigned need = pair_tiles(pass - 1, dp, Tm);
      const unsigned* c = done + pair_base[pass - 1] + dp;
      while (ld_acquire_gpu(c) < need) __nanosleep(256);
    }
    __syncwarp();
  }
  __device__ __forceinline__ const K* srck(int p) const { return bk[p & 1]; }
  __device__ __forceinline__ const uint32_t* srcv(int p) const { return bv[p & 1]; }
  __device__ __forceinline__ const K* pa(int p, int64_t, int64_t A0, int64_t) const {
    return bk[p & 1] + A0;
  }
  __device__ __forceinline__ const K* pb(int p, int64_t, int64_t A0, int64_t na) const {
    return bk[p & 1] + A0 + na;
  }
  __device__ __forceinline__ const uint32_t* pva(int p, int64_t, int64_t A0, int64_t) const {
    return bv[p & 1] + A0;
  }
  __device__ __forceinline__ const uint32_t* pvb(int p, int64_t, int64_t A0, int64_t na) const {
    return bv[p & 1] + A0 + na;
  }
  __device__ __forceinline__ K* dstk(int p, int64_t) const { return bk[(p + 1) & 1]; }
  __device__ __forceinline__ uint32_t* dstv(int p, int64_t) const { return bv[(p + 1) & 1]; }
  // Called by one thread after the tile's output (bulk store waited for,
  // scalar stores ordered by a CTA barrier) is complete.
  __device__ __forceinline__ void tile_done(int pass, int64_t q, int Tm) const {
#ifndef MSORT_K3_NOPROXYFENCE
    fence_proxy_async_global();
#endif
    red_release_gpu_add(done + pair_base[pass] + pair_of(pass, q, Tm), 1u);
#ifdef MSORT_K3_TRACE
    const int64_t ti = (int64_t)pass * ntiles + q;
    if (ti < kK3TraceTiles) g_k3_tiles[ti] = gtimer2();
#endif
  }
};

// All merge levels of a BATCH of segments (msort_sort_segmented, segments
// longer than a tile) in one dataflow launch.  Segment s (in the order of the
// host's list: level count descending) occupies [off[s], off[s] + len[s]) of
// both buffers and tiles [tile0[s], tile0[s+1]) of every level -- a segment
// has ceil(len / Tm) output tiles at every level, since 2L is a multiple of
// Tm.  Level p of segment s merges runs of L_p = T * 2^p starting at off[s];
// segments with fewer levels drop out of the tail of the tile range (level p
// covers tiles [0, ntl[p])).  Segment s with P_s levels was tile-sorted into
// buffer P_s & 1 and level p reads buffer (P_s - p) & 1, so its last level
// writes buffer 0, the caller's array.  Completion counters: done[p * ntiles
// + first tile of the level-p pair] counts that pair's finished tiles.
constexpr int kMaxSegLevels = 48;
template <class K>
struct SegFused {
  static constexpr bool kFused = true;
  K* bk[2];
  uint32_t* bv[2];
  const int64_t* off;    // [nseg] first element of each segment
  const int64_t* len;    // [nseg] its length
  const int64_t* tile0;  // [nseg + 1] first output tile of each segment
  const int* lev;        // [nseg] its number of merge levels P_s
  int nseg;
  int64_t T, ntiles;
  int P;
  int ch, grab;
  unsigned* done;
  int64_t ntl[kMaxSegLevels];          // tiles of level p (a prefix of the segments)
  int64_t cbase[kMaxSegLevels + 1];    // first chunk of level p
  __host__ __device__ __forceinline__ int64_t nchunks() const { return cbase[P]; }
  __device__ __forceinline__ void chunk(int64_t g, int& pass, int64_t& q0, int& cnt) const {
    int p = 0;
    while (p + 1 < P && cbase[p + 1] <= g) ++p;
    pass = p;
    q0 = (g - cbase[p]) * ch;
    cnt = (int)min((int64_t)ch, ntl[p] - q0);
  }
  __device__ __forceinline__ int64_t tiles(int pass) const { return ntl[pass]; }
  __device__ __forceinline__ int seg_of(int64_t q) const {
    int lo = 0, hi = nseg - 1;  // last s with tile0[s] <= q
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (tile0[mid] <= q) lo = mid;
      else hi = mid - 1;
    }
    return lo;
  }
  __device__ __forceinline__ int64_t L(int pass) const { return T << pass; }
  __device__ __forceinline__ void locate(int pass, int64_t q, int Tm, int64_t& A0, int64_t& na,
                                         int64_t& nb, int64_t& dl) const {
    const int s = seg_of(q);
    const int64_t d = (q - tile0[s]) * Tm, l = len[s], Lp = L(pass);
    const int64_t m = d / (2 * Lp);
    A0 = off[s] + m * 2 * Lp;
    na = min(Lp, l - m * 2 * Lp);
    nb = max((int64_t)0, min(Lp, l - m * 2 * Lp - Lp));
    dl = d - m * 2 * Lp;
  }
  __device__ __forceinline__ int src_buf(int pass, int64_t q) const {
    return (lev[seg_of(q)] - pass) & 1;
  }
  __device__ __forceinline__ const K* pa(int p, int64_t q, int64_t A0, int64_t) const {
    return bk[src_buf(p, q)] + A0;
  }
  __device__ __forceinline__ const K* pb(int p, int64_t q, int64_t A0, int64_t na) const {
    return bk[src_buf(p, q)] + A0 + na;
  }
  __device__ __forceinline__ const uint32_t* pva(int p, int64_t q, int64_t A0, int64_t) const {
    return bv[src_buf(p, q)] + A0;
  }
  __device__ __forceinline__ const uint32_t* pvb(int p, int64_t q, int64_t A0, int64_t na) const {
    return bv[src_buf(p, q)] + A0 + na;
  }
  __device__ __forceinline__ K* dstk(int p, int64_t q) const { return bk[src_buf(p, q) ^ 1]; }
  __device__ __forceinline__ uint32_t* dstv(int p, int64_t q) const {
    return bv[src_buf(p, q) ^ 1];
  }
  // first tile and tile count of the level-p pair holding tile q
  __device__ __forceinline__ void pair_tiles(int pass, int64_t q, int Tm, int64_t& first,
                                             unsigned& cnt) const {
    const int s = seg_of(q);
    const int64_t t = q - tile0[s], per = 2 * L(pass) / Tm;  // tiles per full pair
    first = tile0[s] + t / per * per;
    cnt = (unsigned)min(per, tile0[s + 1] - first);
  }
  // Level p >= 1 reads the level-(p-1) pairs covering each tile's level-p
  // pair: wait until they are complete (the whole warp returns together).
  __device__ __forceinline__ void wait_ready(int pass, int64_t q0, int cnt, int lane,
                                             int Tm) const {
    if (pass == 0) return;  // tile-sorted before this launch
    const int64_t half = L(pass) / Tm;  // tiles per full level-(p-1) pair
    // every level-(p-1) pair start in [first pair of q0, end of q0+cnt-1's pair)
    int64_t f0, f1;
    unsigned c0, c1;
    pair_tiles(pass, q0, Tm, f0, c0);
    pair_tiles(pass, q0 + cnt - 1, Tm, f1, c1);
    const int64_t end = f1 + c1;
    for (int64_t f = f0; f < end;) {
      // f is the first tile of a level-(p-1) pair: its segment and size
      const int s = seg_of(f);
      const int64_t segend = tile0[s + 1];
      // pairs of this segment start at tile0[s] + j * half
      const int64_t npairs = (min(end, segend) - f + half - 1) / half;
      for (int64_t j = lane; j < npairs; j += 32) {
        const int64_t pf = f + j * half;
        const unsigned need = (unsigned)min(half, segend - pf);
        const unsigned* c = done + (int64_t)(pass - 1) * ntiles + pf;
        while (ld_acquire_gpu(c) < need) __nanosleep(256);
      }
      f = min(end, segend);
    }
    __syncwarp();
  }
  __device__ __forceinline__ void tile_done(int pass, int64_t q, int Tm) const {
    int64_t first;
    unsigned cnt;
    pair_tiles(pass, q, Tm, first, cnt);
#ifndef MSORT_K3_NOPROXYFENCE
    fence_proxy_async_global();
#endif
    red_release_gpu_add(done + (int64_t)pass * ntiles + first, 1u);
  }
};

#ifdef MSORT_K3_TRACE
// Tuning builds only (-DMSORT_K3_TRACE): per-CTA timeline of the last K3 launch.
__device__ unsigned long long g_k3_trace[4096 * 8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define K3_TRACE(slot, v) g_k3_trace[(blockIdx.x & 4095) * 8 + (slot)] = (v)
#else
#define K3_TRACE(slot, v) ((void)0)
#endif

#ifdef MSORT_K3_CHECK
// Debug builds only (-DMSORT_K3_CHECK): invariant checks that trap.
#define K3_CHECK(cond, ...)                                                                \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      printf("K3_CHECK failed: %s block %d thread %d: ", #cond, blockIdx.x, threadIdx.x); \
      printf(__VA_ARGS__);                                                                 \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define K3_CHECK(cond, ...) ((void)0)
#endif

// Co-rank of tile q's first diagonal by one warp: each round probes 32
// evenly spaced candidates of [lo, hi) and keeps the bucket holding the
// first one where the (monotone) predicate A[i] > B[d-1-i] turns true.
template <class K, class Src>
__device__ __forceinline__ int64_t corank_warp(const Src& src, int pass, int64_t q, int T,
                                               int lane) {
  int64_t A0, na, nb, dl;
  src.locate(pass, q, T, A0, na, nb, dl);
  const K* a = src.pa(pass, q, A0, na);
  const K* b = src.pb(pass, q, A0, na);
  int64_t lo = dl - nb > 0 ? dl - nb : 0;
  int64_t hi = dl < na ? dl : na;
  const uint64_t pol = probe_policy();
  while (hi > lo) {
    const int64_t span = hi - lo;
    const int64_t step = (span + 31) >> 5;
    const int64_t off = step * (lane + 1);
    const int64_t p = lo + (off < span ? off : span) - 1;
    const bool pred = probe_ld(a + p, pol) > probe_ld(b + (dl - 1 - p), pol);
    const unsigned m = __ballot_sync(0xffffffffu, pred);
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

constexpr int kK3Extra = 96;  // producer, searcher and store warps
#ifndef MSORT_SEARCH_PL
#define MSORT_SEARCH_PL 2  // 1: +1% on 2^24-2^26 (profiles/r02/c2/pl_ab.log); 8: spills, slower
#endif
constexpr int kSearchPL = MSORT_SEARCH_PL;  // probes per lane per round (group searches)

template <class Src>
__device__ __forceinline__ bool k3_gated_off(const Src&) {
  return false;
}
template <class K>
__device__ __forceinline__ bool k3_gated_off(const FusedPasses<K>& f) {
  return f.gate && (int)range_narrow(f.gate) != f.gate_want;
}

template <class K, bool PAIRS, int NC, int VT, int S, int MINB, class Src>
__global__ void __launch_bounds__(NC + kK3Extra, MINB)
    k3_merge_pass(const __grid_constant__ Src src, unsigned long long* __restrict__ ctr) {
  if (k3_gated_off(src)) return;
  using LY = K3Layout<K, PAIRS, NC, VT, S>;
  constexpr int Tm = LY::Tm, EK = LY::EK, CH = kChunk;
  const int G = src.grab;  // chunks per grab (<= kGrab); chunk ring of R = 2G slots
  const int R = G == 1 ? kRing1 : 2 * G;
  constexpr int NW = (NC + kK3Extra) / 32;  // warps per CTA
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + LY::bars);
  uint64_t* empty = full + S;
  uint64_t* sfull = empty + S;
  uint64_t* sempty = sfull + R;
  uint64_t* outr = sempty + R;  // output tile of stage s written, ready to store
  TileMeta* meta = reinterpret_cast<TileMeta*>(smem + LY::meta);
  ChunkDesc* ring = reinterpret_cast<ChunkDesc*>(smem + LY::ring);
  int* corank = reinterpret_cast<int*>(smem + LY::corank);
  int64_t* first_chunk = reinterpret_cast<int64_t*>(smem + LY::misc);
  K* stk = reinterpret_cast<K*>(smem + LY::stage_k);
  uint32_t* stv = reinterpret_cast<uint32_t*>(smem + LY::stage_v);
  constexpr bool DUAL = (VT % 2) == 0;  // even: two chains per thread
  constexpr int H = VT / 2;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nchunks = src.nchunks();
#ifdef MSORT_K3_TRACE
  const unsigned long long t_start = gtimer();
  unsigned long long t_wait = 0;
  int64_t ntile_done = 0;
  if (threadIdx.x == 0) K3_TRACE(0, t_start);
#endif
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s)
      mbar_init(&full[s], 32), mbar_init(&empty[s], 1), mbar_init(&outr[s], NC / 32);
    for (int r = 0; r < R; ++r) mbar_init(&sfull[r], 32), mbar_init(&sempty[r], 1);
    fence_mbar_init();
    *first_chunk = (int64_t)atomicAdd(ctr, (unsigned long long)G);
  }
  __syncthreads();
#ifdef MSORT_K3_TRACE
  if (threadIdx.x == 0) K3_TRACE(2, gtimer() - t_start);
#endif
  {
    // the first chunk's co-ranks, one cooperative search per warp; the other
    // G-1 chunks of this grab go to the searcher
    const int64_t c = *first_chunk;
    if (c >= nchunks) return;  // no work for this CTA (uniform)
    int pass, cnt;
    int64_t q0;
    src.chunk(c, pass, q0, cnt);
    if (threadIdx.x == 0) K3_TRACE_CHUNK(c, 0, gtimer2()), K3_TRACE_CHUNK(c, 3, blockIdx.x);
    if (warp == 0) src.wait_ready(pass, q0, cnt, lane, Tm);
    if (threadIdx.x == 0) K3_TRACE_CHUNK(c, 1, gtimer2());
    __syncthreads();
    for (int w = warp; w <= cnt; w += NW) {
      const int64_t q = q0 + w;
      const int64_t v = q < src.tiles(pass) ? corank_warp<K>(src, pass, q, Tm, lane) : 0;
      if (lane == 0) ring[0].co[w] = v;
    }
    if (threadIdx.x == 0) ring[0].q0 = q0, ring[0].cnt = cnt, ring[0].pass = pass;
  }
#ifdef MSORT_K3_TRACE
  __syncthreads();
  if (threadIdx.x == 0) K3_TRACE_CHUNK(*first_chunk, 2, gtimer2());
#endif
  __syncthreads();
#ifdef MSORT_K3_TRACE
  if (threadIdx.x == 0) K3_TRACE(1, gtimer() - t_start);
#endif

  if (warp == 1) {
    // ------------------------------------------------ co-rank searcher (K2)
    // Round g fills ring slots G*g .. G*g+G-1 (mod R) with the
    // chunks of one grab; lanes 9m..9m+8 search chunk m's CH+1 co-ranks.
    static_assert(kGrab * (kChunk + 1) <= 32, "one lane per co-rank");
    mbar_arrive(&sfull[0]);  // slot 0 (first chunk of grab 0) was filled above
    int64_t c0 = *first_chunk;
    bool done = false;
    for (int64_t g = 0; !done; ++g) {
      if (g > 0) {
        int64_t c = 0;
        if (lane == 0) c = (int64_t)atomicAdd(ctr, (unsigned long long)G);
        c0 = __shfl_sync(0xffffffffu, c, 0);
      }
      const int m = lane / (CH + 1), j = lane % (CH + 1);
      for (int mm = (g == 0 ? 1 : 0); mm < G; ++mm) {
        const int64_t b = g * G + mm;  // ring use index
        const int r = (int)(b % R);
        mbar_wait(&sempty[r], (uint32_t)(((b / R) & 1) ^ 1));
      }
      // The grab's chunks in order, in groups of the same merge level: a later
      // level may read an earlier chunk of this very grab, so each group is
      // published before the next one waits for its inputs.
      int mm0 = g == 0 ? 1 : 0;
      while (mm0 < G && !done) {
        if (c0 + mm0 >= nchunks) {
          const int r = (int)((g * G + mm0) % R);
          if (lane == 0) ring[r].cnt = 0;  // end of work: the producer stops here
          mbar_arrive(&sfull[r]);
          done = true;
          break;
        }
        int pass0, cnt_;
        int64_t q_;
        src.chunk(c0 + mm0, pass0, q_, cnt_);
        int mm1 = mm0 + 1;
        while (mm1 < G && c0 + mm1 < nchunks) {
          int p_, c_;
          int64_t q2;
          src.chunk(c0 + mm1, p_, q2, c_);
          if (p_ != pass0) break;
          ++mm1;
        }
#ifdef MSORT_K3_TRACE
        if (lane == 0)
          for (int mm = mm0; mm < mm1; ++mm)
            K3_TRACE_CHUNK(c0 + mm, 0, gtimer2()), K3_TRACE_CHUNK(c0 + mm, 3, blockIdx.x);
#endif
        for (int mm = mm0; mm < mm1; ++mm) {
          int p_, c_;
          int64_t q2;
          src.chunk(c0 + mm, p_, q2, c_);
          src.wait_ready(p_, q2, c_, lane, Tm);
        }
#ifdef MSORT_K3_TRACE
        if (lane == 0)
          for (int mm = mm0; mm < mm1; ++mm) K3_TRACE_CHUNK(c0 + mm, 1, gtimer2());
#endif
        if (G == 1) {
          // One chunk per grab (small sorts): its <= kChunk + 1 co-ranks are
          // searched by lane GROUPS -- the two edges by 16 lanes each, then
          // the inner ones (inside the edges' bracket) by 32 / (cnt - 1)
          // lanes each -- so the probe latency chain is log_16 of the range,
          // not log2 (the searcher is the critical path of a small sort).
          int p_, cnt1;
          int64_t q01;
          src.chunk(c0 + mm0, p_, q01, cnt1);
          const int e = lane >> 4, gl = lane & 15;
          const int je = e ? cnt1 : 0;
          const bool ve = q01 + je < src.tiles(pass0);
          int64_t A0e = -1, nae = 0, nbe = 0, dle = 0;  // -1: no pair (bracket unused)
          if (ve) src.locate(pass0, q01 + je, Tm, A0e, nae, nbe, dle);
          const K* rae = ve ? src.pa(pass0, q01 + je, A0e, nae) : nullptr;
          const K* rbe = ve ? src.pb(pass0, q01 + je, A0e, nae) : nullptr;
          const int64_t ve_ = merge_path_global_group<kSearchPL>(
              rae, rbe, dle, dle - nbe > 0 ? dle - nbe : 0, dle < nae ? dle : nae, ve, gl, 4,
              e << 4);
          const int64_t v0 = __shfl_sync(0xffffffffu, ve ? ve_ : 0, 0);
          const int64_t a00 = __shfl_sync(0xffffffffu, A0e, 0);
          const int64_t vN = __shfl_sync(0xffffffffu, ve ? ve_ : 0, 16);
          const int64_t a0N = __shfl_sync(0xffffffffu, A0e, 16);
          const int ni = cnt1 - 1;  // inner co-ranks
          int64_t vi = 0;
          int ji = 0;
          bool vin = false;
          if (ni > 0) {
            const int LG = ni == 1 ? 5 : ni == 2 ? 4 : ni <= 4 ? 3 : 2;
            const int grp = lane >> LG;
            ji = 1 + grp;
            vin = grp < ni && q01 + ji < src.tiles(pass0);
            int64_t A0 = 0, na = 0, nb = 0, dl = 0;
            int64_t lo = 0, hi = 0;
            const K* ra = nullptr;
            const K* rbp = nullptr;
            if (vin) {
              src.locate(pass0, q01 + ji, Tm, A0, na, nb, dl);
              ra = src.pa(pass0, q01 + ji, A0, na);
              rbp = src.pb(pass0, q01 + ji, A0, na);
              lo = dl - nb > 0 ? dl - nb : 0;
              hi = dl < na ? dl : na;
              if (a00 == A0) lo = max(lo, v0), hi = min(hi, v0 + (int64_t)ji * Tm);
              if (a0N == A0) lo = max(lo, vN - (int64_t)(cnt1 - ji) * Tm), hi = min(hi, vN);
            }
            vi = merge_path_global_group<kSearchPL>(ra, rbp, dl, lo, hi, vin, lane & ((1 << LG) - 1),
                                         LG, grp << LG);
            vin = vin && (lane & ((1 << LG) - 1)) == 0;
          }
#ifdef MSORT_K3_TRACE
          if (lane == 0) K3_TRACE_CHUNK(c0 + mm0, 2, gtimer2());
#endif
          const int r = (int)((g * G + mm0) % R);
          if (lane == 0) ring[r].co[0] = v0;
          if (lane == 16) ring[r].co[cnt1] = vN;
          if (vin) ring[r].co[ji] = vi;
          if (lane == 0) ring[r].q0 = q01, ring[r].cnt = cnt1, ring[r].pass = p_;
          mbar_arrive(&sfull[r]);
          mm0 = mm0 + 1;
          continue;
        }
        // Two rounds: the chunk's first and last co-ranks by full searches,
        // then the inner ones inside the bracket those give (co-ranks are
        // monotone: i(d) <= i(d + x) <= i(d) + x within one pair), so the
        // inner probes fall in the windows the chunk is about to stage
        // instead of all over the runs (ncu: fewer stray DRAM sectors).
        int64_t v = 0;
        int cntm = 0;
        int64_t q0m = 0;
        int64_t A0 = -1, na = 0, nb = 0, dl = 0;
        bool valid = false;
        if (m >= mm0 && m < mm1) {
          int p_;
          src.chunk(c0 + m, p_, q0m, cntm);
          valid = j <= cntm && q0m + j < src.tiles(pass0);
          if (valid) src.locate(pass0, q0m + j, Tm, A0, na, nb, dl);
        }
        const K* ra = valid ? src.pa(pass0, q0m + j, A0, na) : nullptr;
        const K* rbp = valid ? src.pb(pass0, q0m + j, A0, na) : nullptr;
        const bool edge = j == 0 || j == cntm;
        if (valid && edge) v = merge_path_global(ra, na, rbp, nb, dl);
        const int l0 = m * (CH + 1) < 32 ? m * (CH + 1) : 0;
        const int le = l0 + cntm < 32 ? l0 + cntm : 0;
        const int64_t v0 = __shfl_sync(0xffffffffu, v, l0);
        const int64_t a00 = __shfl_sync(0xffffffffu, A0, l0);
        const int64_t ve = __shfl_sync(0xffffffffu, v, le);
        const int64_t a0e = __shfl_sync(0xffffffffu, A0, le);
        if (valid && !edge) {
          int64_t lo = dl - nb > 0 ? dl - nb : 0;
          int64_t hi = dl < na ? dl : na;
          if (a00 == A0) {  // same pair as the chunk's first tile
            lo = max(lo, v0);
            hi = min(hi, v0 + (int64_t)j * Tm);
          }
          if (a0e == A0) {  // same pair as the chunk's last boundary
            lo = max(lo, ve - (int64_t)(cntm - j) * Tm);
            hi = min(hi, ve);
          }
          v = merge_path_global_range(ra, rbp, dl, lo, hi);
        }
#ifdef MSORT_K3_TRACE
        __syncwarp();
        if (lane == 0)
          for (int mm = mm0; mm < mm1; ++mm) K3_TRACE_CHUNK(c0 + mm, 2, gtimer2());
#endif
        for (int mm = mm0; mm < mm1; ++mm) {
          const int r = (int)((g * G + mm) % R);
          if (m == mm && j <= cntm) ring[r].co[j] = v;
          if (lane == 0) {
            int p_, c_;
            int64_t q2;
            src.chunk(c0 + mm, p_, q2, c_);
            ring[r].q0 = q2, ring[r].cnt = c_, ring[r].pass = p_;
          }
          mbar_arrive(&sfull[r]);
        }
        mm0 = mm1;
      }
    }
  } else if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    int64_t k = 0;  // tiles issued by this CTA
    for (int64_t b = 0;; ++b) {
      const int r = (int)(b % R);
      mbar_wait(&sfull[r], (uint32_t)((b / R) & 1));
      const ChunkDesc& cd = ring[r];
      const int ccnt = cd.cnt;
      const int pass = cd.pass;
      if (ccnt == 0) {
        // no more chunks: tell the mergers to stop
        const int s = (int)(k % S);
        mbar_wait(&empty[s], (uint32_t)(((k / S) & 1) ^ 1));
        if (lane == 0) meta[s].out = -1;
        mbar_arrive(&full[s]);
        break;
      }
      // inputs written by other SMs (generic or bulk stores) were acquired by
      // the searcher; order them before this thread's bulk (async-proxy) loads
      if constexpr (Src::kFused) fence_proxy_async_global();
      for (int j = 0; j < ccnt; ++j, ++k) {
        const int64_t q = cd.q0 + j;
        const int s = (int)(k % S);
        int64_t A0, na_all, nb_all, d0;
        src.locate(pass, q, Tm, A0, na_all, nb_all, d0);
        const int64_t tot_all = na_all + nb_all;
        const int64_t d1 = min(d0 + Tm, tot_all);
        const int64_t i0 = cd.co[j];
        const int64_t i1 = d1 == tot_all ? na_all : cd.co[j + 1];
        const int64_t j0 = d0 - i0, j1 = d1 - i1;
        const int na = (int)(i1 - i0), nb = (int)(j1 - j0);
        const K* a = src.pa(pass, q, A0, na_all) + i0;
        const K* bp = src.pb(pass, q, A0, na_all) + j0;
        const int offA = stage_offset(a);
        const int offB = (offA + na + EK - 1) / EK * EK + stage_offset(bp);
        K3_CHECK(i0 >= 0 && i0 <= i1 && i1 <= na_all && j0 >= 0 && j0 <= j1 && j1 <= nb_all &&
                     offB + nb <= LY::SKE && na + nb <= Tm,
                 "pass %d q %lld j %d ccnt %d i0 %lld i1 %lld na_all %lld nb_all %lld d0 %lld\n",
                 pass, (long long)q, j, ccnt, (long long)i0, (long long)i1, (long long)na_all,
                 (long long)nb_all, (long long)d0);
        const uint32_t* av = nullptr;
        const uint32_t* bv = nullptr;
        int offAv = 0, offBv = 0;
        if constexpr (PAIRS) {
          av = src.pva(pass, q, A0, na_all) + i0;
          bv = src.pvb(pass, q, A0, na_all) + j0;
          offAv = stage_offset(av);
          offBv = (offAv + na + 3) / 4 * 4 + stage_offset(bv);
        }
        if (j + 1 == ccnt) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&sempty[r]);  // chunk descriptor consumed
        }
#ifdef MSORT_K3_TRACE
        const unsigned long long tw0 = gtimer();
#endif
        mbar_wait(&empty[s], (uint32_t)(((k / S) & 1) ^ 1));
#ifdef MSORT_K3_TRACE
        t_wait += gtimer() - tw0;
#endif
        K* sk = stk + (size_t)s * LY::SKE;
        uint32_t* sv = stv + (size_t)s * LY::SVE;
        if (lane == 0) {
          meta[s] = TileMeta{A0 + d0, q, na, nb, offA, offB, offAv, offBv, na + nb, pass};
          uint32_t tx = window_bulk_bytes(a, na) + window_bulk_bytes(bp, nb);
          if constexpr (PAIRS) tx += window_bulk_bytes(av, na) + window_bulk_bytes(bv, nb);
          mbar_expect_tx(&full[s], tx);  // before the copies that complete it
        }
        stage_window(sk + offA, a, na, &full[s], lane == 0, lane, 32);
        stage_window(sk + offB, bp, nb, &full[s], lane == 0, lane, 32);
        if constexpr (PAIRS) {
          stage_window(sv + offAv, av, na, &full[s], lane == 0, lane, 32);
          stage_window(sv + offBv, bv, nb, &full[s], lane == 0, lane, 32);
        }
        mbar_arrive(&full[s]);  // all 32 lanes: their head/tail stores are released
      }
    }
#ifdef MSORT_K3_TRACE
    if (lane == 0) K3_TRACE(7, t_wait);
#endif
  } else if (warp == 2) {
    // ------------------------------------------------------------ store warp
    // Lane 0 writes each merged tile out of its stage (bulk store of the
    // 16-byte aligned middle, plain stores of the <16-byte head and tail),
    // hands the stage back once the store has read it, and publishes the
    // tile's completion (fused levels) one tile later, when its store is done.
    if (lane == 0) {
      bool pend = false;
      int ppass = 0;
      int64_t pq = 0;
      for (int64_t k = 0;; ++k) {
        const int s = (int)(k % S);
        const uint32_t par = (uint32_t)((k / S) & 1);
        if constexpr (Src::kFused) {
          // never sit on an unpublished tile: another chunk (maybe this CTA's
          // own next one) may be waiting for it
          if (pend && !mbar_test(&outr[s], par)) {
            bulk_wait_all();
            src.tile_done(ppass, pq, Tm);
            pend = false;
          }
        }
        mbar_wait(&outr[s], par);
        const TileMeta m = meta[s];
        if (m.out < 0) break;
        K* sk = stk + (size_t)s * LY::SKE;
        uint32_t* sv = stv + (size_t)s * LY::SVE;
        K* gk = src.dstk(m.pass, m.q) + m.out;
        const int phk = stage_offset(gk);
        int hk, mk;
        window_split(gk, m.tot, hk, mk);
        if (mk) bulk_s2g(gk + hk, sk + phk + hk, (uint32_t)(mk * sizeof(K)));
        uint32_t* gv = nullptr;
        int phv = 0, hv = 0, mv = 0;
        if constexpr (PAIRS) {
          gv = src.dstv(m.pass, m.q) + m.out;
          phv = stage_offset(gv);
          window_split(gv, m.tot, hv, mv);
          if (mv) bulk_s2g(gv + hv, sv + phv + hv, (uint32_t)(mv * 4));
        }
        bulk_commit();
        for (int i = 0; i < m.tot - mk; ++i) {
          const int j = i < hk ? i : i + mk;
          gk[j] = sk[phk + j];
        }
        if constexpr (PAIRS)
          for (int i = 0; i < m.tot - mv; ++i) {
            const int j = i < hv ? i : i + mv;
            gv[j] = sv[phv + j];
          }
        bulk_wait_read<0>();     // this tile's store has read the stage
        mbar_arrive(&empty[s]);  // ... so it goes back to the producer
        if constexpr (Src::kFused) {
          if (pend) {
            bulk_wait<1>();  // the previous tile's store is complete
            src.tile_done(ppass, pq, Tm);
          }
          pend = true, ppass = m.pass, pq = m.q;
        }
      }
      bulk_wait_all();
      if constexpr (Src::kFused)
        if (pend) src.tile_done(ppass, pq, Tm);
    }
  } else {
    // ------------------------------------------------------------ mergers
    const int ct = threadIdx.x - kK3Extra;  // 0..NC-1
    for (int64_t k = 0;; ++k) {
      const int s = (int)(k % S);
#ifdef MSORT_K3_TRACE
      const unsigned long long tw0 = gtimer();
#endif
      mbar_wait(&full[s], (uint32_t)((k / S) & 1));
#ifdef MSORT_K3_TRACE
      t_wait += gtimer() - tw0;
      if (k == 0 && ct == 0) K3_TRACE(3, gtimer() - t_start);
#endif
      const TileMeta m = meta[s];
      if (m.out < 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&outr[s]);  // pass the stop on to the store warp
        break;
      }
      K* sk = stk + (size_t)s * LY::SKE;
      uint32_t* sv = stv + (size_t)s * LY::SVE;
      K key[VT];
      int pos[VT];
      const int d = ct * VT;
      const int aend = m.offA + m.na, bend = m.offB + m.nb;
      if constexpr (DUAL) {
        // co-rank of my first diagonal; the one of my last comes from the
        // next thread through shared memory
        const int i0 = d < m.tot ? merge_path<K, false>(sk, m.offA, m.na, m.offB, m.nb, d) : 0;
        corank[ct] = i0;
        named_bar_sync(1, NC);
        const int d1 = min(d + VT, m.tot);
        const int i1 = d + VT < m.tot ? corank[ct + 1] : m.na;
        const int ai0 = m.offA + i0, bi0 = m.offB + d - i0;
        const int ai1 = m.offA + i1, bi1 = m.offB + d1 - i1;
        if (d1 - d == VT && ai0 + H <= aend && bi0 + H <= bend && ai1 - H >= m.offA &&
            bi1 - H >= m.offB) {
          dual_merge<K, PAIRS, H>(sk, ai0, bi0, ai1, bi1, key, pos);
        } else if (d < m.tot) {
          serial_merge<K, false, PAIRS, VT>(sk, nullptr, ai0, aend, bi0, bend, LY::SKE - 1, key,
                                            pos);
        }
      } else if (d < m.tot) {
        int i = merge_path<K, false>(sk, m.offA, m.na, m.offB, m.nb, d);
        serial_merge_fast<K, PAIRS, VT>(sk, m.offA + i, aend, m.offB + d - i, bend,
                                        LY::SKE - 1, key, pos);
      }
      uint32_t val[PAIRS ? VT : 1];
      if constexpr (PAIRS) {
#pragma unroll
        for (int t = 0; t < VT; ++t) {
          if (d + t < m.tot) {
            const int p = pos[t];
            val[t] = sv[p < m.offB ? m.offAv + (p - m.offA) : m.offBv + (p - m.offB)];
          }
        }
      }
      named_bar_sync(1, NC);  // everyone is done reading stage s: overwrite it
      // The output keeps its global 16-byte phase so the aligned middle leaves
      // by one bulk store (TMA, cp.async.bulk.global.shared).
      const int phk = stage_offset(src.dstk(m.pass, m.q) + m.out);
      int phv = 0;
      if constexpr (PAIRS) phv = stage_offset(src.dstv(m.pass, m.q) + m.out);
#pragma unroll
      for (int t = 0; t < VT; ++t) {
        if (d + t < m.tot) {
          sk[phk + d + t] = key[t];
          if constexpr (PAIRS) sv[phv + d + t] = val[t];
        }
      }
      fence_proxy_async_smem();  // visible to the bulk-store engine
      __syncwarp();
      if (lane == 0) mbar_arrive(&outr[s]);
#ifdef MSORT_K3_TRACE
      ++ntile_done;
#endif
    }
#ifdef MSORT_K3_TRACE
    if (ct == 0) K3_TRACE(4, gtimer() - t_start), K3_TRACE(6, t_wait), K3_TRACE(5, ntile_done);
#endif
  }
}

}  // namespace msort
