// k0_small.cuh -- K0, the small-n sort in ONE launch.
//
// The paper's small-array regime: below some size the parallel machinery's
// fixed costs dominate (P:332, P:565 -- multiprocessing loses to the
// sequential sort at 10^4 keys).  On the GPU the general path costs two
// kernels (tile sort + fused merge levels), each latency-bound at this size
// (2^16 int32: ~25 us each).  K0 sorts n <= CL * NT * VT keys (CL <= 16 CTAs
// of one thread-block CLUSTER) in a single launch, keys only:
//   1. each CTA sorts its chunk of Q = ceil(n / CL) keys: a per-thread
//      register network on VT keys, then log2(NT) merge-path rounds in
//      shared memory (the recursion of P:77-84 bottom-up, merge() of P:107
//      with ties to the left run);
//   2. ONE CL-way merge step ACROSS the cluster (MW, the default): the CL
//      sorted chunks stay in their CTAs' shared memory (DSMEM, distributed
//      shared memory); every chunk is sampled every kK0S keys, each CTA ranks
//      its own samples among all CL sample lists (a local copy), and the
//      sample of merged rank t*g starts output tile t (K5's sample-bounded
//      tiles, k5_kway.cuh: a tile never exceeds S(g + CL) - CL keys); CTA t
//      finds its tile's exact start/end STATE per chunk by one DSMEM probe
//      round (16 lanes x S/16) inside the S keys between two samples, copies its
//      CL windows in (16-byte DSMEM vectors) and merges them in log2(CL)
//      in-CTA rounds (K5's engine, ping-pong buffers, one barrier per round),
//      writing HBM from the last round.  Three cluster barriers in all, the
//      last one split (arrive after the window copies, wait before exit).
//      C1 (2^16 int32): 26.6 -> 22.0 us per CUDA-graph replay against the
//      pairwise levels (profiles/r02/k0mw/); S = 64 (half the samples to
//      copy and rank, 4 probes per lane): 22.0 -> 20.5 us.
//      The round-2 variant (MW = false, MSORT_K0=3): log2(CL) pairwise merge
//      levels across the cluster -- co-ranks by 32-ary DSMEM searches, the
//      two windows copied in, a per-thread merge, one cluster barrier per level.
// No workspace, no memset, no second launch.  Equal keys are
// indistinguishable (keys only), so the result is the stable sort.
#pragma once

#include <cooperative_groups.h>

namespace msort {

#ifdef MSORT_K0_TRACE
// Tuning builds only (-DMSORT_K0_TRACE): globaltimer per CTA and phase.
__device__ unsigned long long g_k0_trace[16 * 32];  // [CTA][slot]
__device__ __forceinline__ void k0_mark(int slot) {
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_k0_trace[blockIdx.x * 32 + slot] = t;
  }
  __syncwarp();  // reconverge: a diverged warp takes the slow path of every later shuffle
}
__device__ __forceinline__ void k0_note(int slot, unsigned long long v) {
  if ((threadIdx.x & 31) == 0) {
    if (v == 1) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    g_k0_trace[blockIdx.x * 32 + slot] = v;
  }
  __syncwarp();
}
#else
__device__ __forceinline__ void k0_mark(int) {}
__device__ __forceinline__ void k0_note(int, unsigned long long) {}
#endif

// 512 threads x 8 keys per CTA, up to 16 CTAs (a non-portable cluster size,
// schedulable on B200): C1 (2^16 int32) 38.9 -> 30.7 us per sort (CUDA-graph
// replay) against 512 x 16 x 8 CTAs; 1024 x 4 x 16: 34.8, 256 x 16 x 16:
// 34.8 (profiles/r02/k0/).
#ifndef MSORT_K0_NT
#define MSORT_K0_NT 512
#endif
#ifndef MSORT_K0_VT
#define MSORT_K0_VT 8
#endif
#ifndef MSORT_K0_MAXCL
#define MSORT_K0_MAXCL 16
#endif
constexpr int kK0NT = MSORT_K0_NT, kK0VT = MSORT_K0_VT, kK0Chunk = kK0NT * kK0VT;  // keys per CTA
constexpr int kK0MaxCL = MSORT_K0_MAXCL;  // cluster size (> 8: non-portable, B200 allows 16)
constexpr int64_t kK0MaxN = (int64_t)kK0MaxCL * kK0Chunk;  // 65536 = 2^16
static_assert(kK0MaxN >= 65536, "K0 covers C1 (2^16 keys)");
// Multiway step (MW): sample stride S, merge-round outputs per thread VT2
// (a multiple of the 16-byte vector width; the tile bound S(g+CL)-CL <=
// Q + (S-1) CL keys must fit the round's threads: (bound)/VT2 + CL/2 <= NT).
#ifndef MSORT_K0_S
#define MSORT_K0_S 64
#endif
#ifndef MSORT_K0_VT2
#define MSORT_K0_VT2 12
#endif
constexpr int kK0S = MSORT_K0_S, kK0VT2 = MSORT_K0_VT2;
static_assert(kK0S % 16 == 0 && kK0S <= 64, "a tile state is finished by one probe round of 16 lanes");
constexpr int kK0TileMax = kK0Chunk + (kK0S - 1) * kK0MaxCL;  // S (g + CL) - CL, g <= Q / S
static_assert(kK0TileMax / kK0VT2 + kK0MaxCL / 2 + 1 <= kK0NT / 32 * 31,
              "MW tile fits one round of output threads (31 per warp)");
constexpr int kK0MWKeys = kK0TileMax + 12 * kK0MaxCL + 16;  // tile + per-run slack (layout)
constexpr int kK0SampStride = kK0Chunk / kK0S;  // >= samples of one chunk (ceil(Q / S), Q <= kK0Chunk)
static_assert((kK0SampStride & (kK0SampStride - 1)) == 0 && kK0SampStride % 32 == 0,
              "sample lists: a power of two, whole warps");

// Shared-memory buffers are plain arrays of kK0Chunk keys plus slack: a
// thread's VT keys leave as 16-byte vector stores, and the cross-cluster
// window copies move 16-byte vectors (a chunk holds Q keys, Q a multiple of
// the vector width, so no vector straddles two chunks).
template <class K>
constexpr int k0_padded() {
  return kK0Chunk + 16;
}
template <class K>
constexpr int k0_vec() {
  return 16 / (int)sizeof(K);
}

// VT outputs [d, d + VT) of merge(A, B) into key[] (ties to A); A = s[a0, a0+na),
// B = s[b0, b0+nb), s[0..lim] addressable.
template <class K, int VT>
__device__ __forceinline__ void k0_merge_thread(const K* s, int a0, int na, int b0, int nb, int d,
                                                int lim, K (&key)[VT]) {
  const int i = merge_path<K, false>(s, a0, na, b0, nb, d);
  int pos[VT];
  serial_merge<K, false, false, VT>(s, nullptr, a0 + i, a0 + na, b0 + d - i, b0 + nb, lim, key,
                                    pos);
}

// Key g of the cluster's global view (chunk g / Q, offset g % Q); n <= 2^16
// keeps every index in 32 bits.
template <class K>
__device__ __forceinline__ K k0_at(const K* const* chunk, int Q, int g) {
  const int c = g / Q;
  return chunk[c][g - c * Q];
}

template <class K>
__device__ __forceinline__ int k0_corank_dsmem(const K* const* chunk, int Q, int a_start, int na,
                                               int b_start, int nb, int d, int lane) {
  int lo = d - nb > 0 ? d - nb : 0, hi = d < na ? d : na;
  while (hi > lo) {  // i(d) = min{i : i = min(d, na) or A[i] > B[d-1-i]}
    const int span = hi - lo;
    const int step = (span + 31) >> 5;
    const int off = step * (lane + 1);
    const int q = lo + (off < span ? off : span) - 1;
    const bool pred = k0_at(chunk, Q, a_start + q) > k0_at(chunk, Q, b_start + d - 1 - q);
    const unsigned m = __ballot_sync(0xffffffffu, pred);
    if (m == 0) {
      lo = hi;
    } else {
      const int f = __ffs(m) - 1;
      const int pf = __shfl_sync(0xffffffffu, q, f);
      const int pp = __shfl_sync(0xffffffffu, q, f > 0 ? f - 1 : 0);
      hi = pf;
      if (f > 0) lo = pp + 1;
    }
  }
  return lo;
}

// Number of a[0, m) that precede v in the stable order: a[x] <= v (INCL) or
// a[x] < v; 1 <= m <= kK0SampStride (fixed-depth, branch-free binary
// lifting; U searches in lock step so their loads overlap).
template <class K, bool INCL, int U>
__device__ __forceinline__ void k0_rank_in(const K* a, int m, const K (&v)[U], int (&pos)[U]) {
#pragma unroll
  for (int k = 0; k < U; ++k) pos[k] = 0;
#pragma unroll
  for (int step = kK0SampStride; step > 0; step >>= 1) {
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int t = pos[k] + step;
      const K y = a[(t < m ? t : m) - 1];
      if (t <= m && (INCL ? !(v[k] < y) : y < v[k])) pos[k] = t;
    }
  }
}
template <class K>
__device__ __forceinline__ int k0_rank1(const K* a, int m, K v, bool incl) {
  if (m == 0) return 0;
  const K vv[1] = {v};
  int pos[1];
  if (incl) k0_rank_in<K, true, 1>(a, m, vv, pos);
  else k0_rank_in<K, false, 1>(a, m, vv, pos);
  return pos[0];
}

// A tile boundary: the merged sample x = (key v, chunk k, index i); k < 0:
// the end of every chunk.
template <class K>
struct K0Bound {
  K v;
  int k, i;
};

// Phase 2 of K0 (MW): one CL-way merge of the cluster's sorted chunks (see
// the header).  mine = this CTA's sorted chunk (read by the peers, left
// untouched), mysam = room for its samples (published), sam = room for every
// chunk's samples (list j at j * kK0SampStride), sk = the merge area
// (kK0MWKeys keys).  Ends with the cluster barrier that keeps mine alive
// until every peer has copied from it.
template <class K, int VT2>
__device__ __forceinline__ void k0_multiway(const K* mine, int Q, int N, int CL, K* mysam, K* sam,
                                            K* sk, K* sk2, K* __restrict__ out) {
  namespace cg = cooperative_groups;
  constexpr int NT = kK0NT, S = kK0S, EK = k0_vec<K>(), MCL = kK0MaxCL, SS = kK0SampStride;
  constexpr unsigned F = 0xffffffffu;
  constexpr uint32_t Z = sizeof(K);
  __shared__ const K* chunk[MCL];        // the peers' chunks (DSMEM)
  __shared__ const K* psam[MCL];         // the peers' samples (DSMEM)
  __shared__ K0Bound<K> s_bnd[2];        // my tile's start / end (written by peers)
  __shared__ int s_rank[SS];             // merged ranks of my samples
  __shared__ int s_state[2][MCL];        // tile start / end state per chunk
  __shared__ int s_len[4][MCL];          // run sizes per round (K5 layout)
  __shared__ int s_off[4][MCL];          // run offsets (keys) per round
  __shared__ int s_tp[4][MCL / 2 + 1];   // first thread of each pair per round
  __shared__ int s_vpre[MCL + 1];        // window vectors before chunk j
  __shared__ int s_out, s_sh;
  cg::cluster_group cluster = cg::this_cluster();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = blockIdx.x;  // the grid is one cluster
  const int RR = __ffs(CL) - 1;  // CL is a power of two
  auto clen = [&](int j) { const int l = N - j * Q; return l <= 0 ? 0 : (l < Q ? l : Q); };
  auto nsam = [&](int j) { return (clen(j) + S - 1) / S; };
  const int mc = nsam(c);
  __syncthreads();  // my chunk is complete
  // ---- publish my samples (keys 0, S, 2S, ...) and the DSMEM pointers
  for (int q = tid; q < mc; q += NT) mysam[q] = mine[q * S];
  if (tid < CL) {
    chunk[tid] = cluster.map_shared_rank(mine, tid);
    psam[tid] = cluster.map_shared_rank(static_cast<const K*>(mysam), tid);
  }
  if (tid < 2) s_bnd[tid].k = -1;
  for (int q = tid; q < SS; q += NT) s_rank[q] = 0;
  cluster.sync();  // every chunk sorted and sampled
  k0_mark(3);
  // ---- every chunk's samples, 16-byte vectors over DSMEM
  {
    constexpr int VPL = SS / EK;
    for (int e = tid; e < CL * VPL; e += NT) {
      const int j = e / VPL, v = e % VPL;
      if (v * EK < nsam(j))
        *reinterpret_cast<uint4*>(sam + j * SS + v * EK) =
            *reinterpret_cast<const uint4*>(psam[j] + v * EK);
    }
  }
  __syncthreads();
  k0_mark(7);
  // ---- merged rank of my samples in the stable order (key, chunk, index):
  // warp j counts list j's samples before each of mine
  if (warp < CL && nsam(warp) > 0) {
    constexpr int U = SS / 32;
    const int j = warp, m = nsam(j);
    const K* a = sam + j * SS;
    K v[U];
    int cnt[U];
#pragma unroll
    for (int k = 0; k < U; ++k) v[k] = sam[c * SS + min(lane + 32 * k, SS - 1)];
    if (j < c) k0_rank_in<K, true, U>(a, m, v, cnt);
    else k0_rank_in<K, false, U>(a, m, v, cnt);
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int q = lane + 32 * k;
      if (q < mc) atomicAdd(&s_rank[q], j == c ? q : cnt[k]);
    }
  }
  __syncthreads();
  k0_mark(8);
  // ---- the sample of merged rank t g starts tile t and ends tile t - 1
  {
    int M = 0;
    for (int j = 0; j < CL; ++j) M += nsam(j);
    const int g = (M + CL - 1) / CL;  // merged samples per tile
    for (int q = tid; q < mc; q += NT) {
      const int r = s_rank[q];
      if (r % g == 0) {
        const int t = r / g;
        const K0Bound<K> b{sam[c * SS + q], c, q * S};
        *cluster.map_shared_rank(&s_bnd[0], t) = b;
        if (t > 0) *cluster.map_shared_rank(&s_bnd[1], t - 1) = b;
      }
    }
  }
  cluster.sync();  // every tile knows its bounds
  k0_mark(4);
  // ---- exact state of both bounds per chunk, 16 lanes per (bound, chunk):
  // r samples of chunk j precede x, so its state lies in [(r-1) S + 1, r S]
  {
    const int task = warp * 2 + (lane >> 4), sub = lane & 15;
    if (warp < CL) {  // tasks 0 .. 2 CL - 1, whole warps
      const int b = task / CL, j = task % CL;
      const K0Bound<K> x = s_bnd[b];
      const int lj = clen(j);
      constexpr int PR = S / 16;  // probes per lane (16 lanes cover the S - 1 keys)
      int st = -1, lo = 0;
      bool pr[PR];
#pragma unroll
      for (int u = 0; u < PR; ++u) pr[u] = false;
      if (x.k < 0) {
        st = lj;
      } else if (j == x.k) {
        st = x.i;
      } else {
        const int r = k0_rank1<K>(sam + j * SS, nsam(j), x.v, j < x.k);
        if (r == 0) {
          st = 0;
        } else {
          lo = (r - 1) * S + 1;
          const int hi = min(r * S, lj);
#pragma unroll
          for (int u = 0; u < PR; ++u) {
            if (lo + sub + 16 * u < hi) {
              const K y = chunk[j][lo + sub + 16 * u];
              pr[u] = j < x.k ? !(x.v < y) : y < x.v;
            }
          }
        }
      }
      const unsigned hm = 0xffffu << (lane & 16);
      int cnt = 0;
#pragma unroll
      for (int u = 0; u < PR; ++u) cnt += __popc(__ballot_sync(F, pr[u]) & hm);
      if (st < 0) st = lo + cnt;
      if (sub == 0) s_state[b][j] = st;
    }
  }
  __syncthreads();
  k0_mark(9);
  // ---- layout (K5's), one warp per round r < RR (lane j = run j of the
  // round, a group of 2^r chunks) and warp RR for the copy: round r's pair m
  // is [MIN | run 2m+1 | MAX .. MIN | run 2m | MAX] (B below A), round 0's
  // runs at their chunks' 16-byte phase; thread ranges per pair and round
  if (warp <= RR) {
    auto scan_excl = [&](int v) {  // over lanes 0..15 (CL <= 16 runs)
      int inc = v;
#pragma unroll
      for (int d = 1; d < MCL; d <<= 1) {
        const int t = __shfl_up_sync(F, inc, d);
        if (lane >= d) inc += t;
      }
      return inc - v;
    };
    const int a = lane < CL ? s_state[0][lane] : 0;
    const int l0 = lane < CL ? s_state[1][lane] - a : 0;
    int out0 = a;
#pragma unroll
    for (int d = 1; d < MCL; d <<= 1) out0 += __shfl_xor_sync(F, out0, d);
    if (warp == RR) {
      const int nv = l0 > 0 ? (a + l0 + EK - 1) / EK - a / EK : 0;
      const int vp = scan_excl(nv);
      if (lane < CL) s_vpre[lane] = vp;
      if (lane == CL - 1) s_vpre[CL] = vp + nv;
      if (lane == 0) {
        s_out = out0;
        s_sh = stage_offset(out + out0);
      }
    } else {
      const int r = warp, nr = CL >> r, np = nr / 2;
      // run j of round r = chunks [j 2^r, (j+1) 2^r); lane j of the next round
      // = chunks [j 2^(r+1), ...): group sums by xor-reduction, then gathered
      int gs = l0;
      for (int d = 1; d < (1 << r); d <<= 1) gs += __shfl_xor_sync(F, gs, d);
      int gs2 = gs + __shfl_xor_sync(F, gs, 1 << r);
      const int l = __shfl_sync(F, gs, (lane << r) & 31);
      const int l2 = __shfl_sync(F, gs2, (lane << (r + 1)) & 31);
      const int ph = r == 0 ? a % EK : 0;
      const int fp = lane < nr ? (ph + l + 8) & ~3 : 0;  // MIN slot, phase, run, MAX, rounding
      const int base = __shfl_sync(F, scan_excl(__shfl_sync(F, fp, lane ^ 1)), lane ^ 1);
      if (lane < nr) {
        s_off[r][lane] = base + 4 + ph;
        s_len[r][lane] = l;
      }
      const int shr = r + 1 == RR ? stage_offset(out + out0) : 0;  // last round: output phase
      const int cnt = lane < np ? (l2 + shr + VT2 - 1) / VT2 : 0;
      const int tp = scan_excl(cnt);
      if (lane < np) s_tp[r][lane] = tp;
      if (lane == np - 1) s_tp[r][np] = tp + cnt;
    }
  }
  __syncthreads();
  k0_mark(20);
  // ---- the CL windows, 16-byte vectors over DSMEM, each at its phase (U
  // loads in flight per thread)
  {
    constexpr int U = 3;
    const int nvt = s_vpre[CL];
    k0_note(21, (unsigned long long)nvt);
    for (int e0 = tid; e0 < nvt; e0 += U * NT) {
      uint4 w[U];
      K* dst[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = e0 + u * NT;
        dst[u] = nullptr;
        if (e < nvt) {
          int j = 0;
#pragma unroll
          for (int q = 1; q < MCL; ++q)
            if (q < CL && s_vpre[q] <= e) j = q;
          const int a = s_state[0][j];
          const int v0 = a / EK, v = v0 + (e - s_vpre[j]);
          w[u] = *reinterpret_cast<const uint4*>(chunk[j] + v * EK);
          dst[u] = sk + s_off[0][j] - a % EK + (v - v0) * EK;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (dst[u]) *reinterpret_cast<uint4*>(dst[u]) = w[u];
    }
  }
  // my DSMEM reads are done (their values are in hand): peers may leave once
  // every thread of the cluster got here (relaxed: nothing to publish; the
  // matching wait is at the end)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  __syncthreads();
  k0_mark(10);
  if (tid < CL) {
    sk[s_off[0][tid] - 1] = KeyTraits<K>::min_key();
    sk[s_off[0][tid] + s_len[0][tid]] = KeyTraits<K>::max_key();
  }
  __syncthreads();
  k0_mark(5);
  // ---- log2(CL) rounds of pairwise merges (k5_merge's engine, ping-pong
  // between sk and sk2: one barrier per round).  Output thread o = 31 warp +
  // lane (lanes 0..30) merges VT2 outputs; lane 31 only searches the co-rank
  // at the next warp's first diagonal, so every thread's end co-rank is its
  // neighbour's start (a shuffle, no shared-memory exchange).  The last round
  // stores to HBM, its diagonals shifted by the output phase so that every
  // full thread's VT2 outputs leave as 16-byte vectors.
  K key[VT2];
  K* go = out + s_out;
  const int o = warp * 31 + lane;
#pragma unroll 1
  for (int r = 0; r < RR; ++r) {
    const char* sb = reinterpret_cast<const char*>((r & 1) ? sk2 : sk);
    K* dk = (r & 1) ? sk : sk2;
    const int npair = CL >> (r + 1);
    int m = 0;
#pragma unroll
    for (int q = 1; q < MCL / 2; ++q)
      if (q < npair && s_tp[r][q] <= o) m = q;
    const bool in = o < s_tp[r][npair];
    const int la = s_len[r][2 * m], lb = s_len[r][2 * m + 1], len = la + lb;
    const uint32_t oa = (uint32_t)s_off[r][2 * m] * Z, ob = (uint32_t)s_off[r][2 * m + 1] * Z;
    const bool last = r + 1 == RR;
    const int sh = last ? s_sh : 0;
    int d = 0, cnt = 0, i0 = 0;
    if (in) {
      d = max(0, (o - s_tp[r][m]) * VT2 - sh);
      cnt = min((o - s_tp[r][m] + 1) * VT2 - sh, len) - d;
      i0 = merge_path_off<K>(sb, oa, la, ob, lb, d);
    }
    const int nx = __shfl_down_sync(F, i0, 1);
    const bool act = in && lane < 31;
    if (act) {
      const int i1 = d + cnt == len ? la : nx;
      merge_keys_dual<K, VT2>(sb, oa + (uint32_t)i0 * Z, oa + (uint32_t)la * Z,
                              ob + (uint32_t)(d - i0) * Z, oa + (uint32_t)i1 * Z,
                              ob + (uint32_t)(d + cnt - i1) * Z, ob - Z, key);
    }
    if (last) {
      if (act) put_outputs<K, VT2>(go + d, key, cnt);  // full threads: 16-byte aligned
      break;
    }
    if (act) put_outputs<K, VT2>(dk + s_off[r + 1][m] + d, key, cnt);
    if (tid < npair) {
      dk[s_off[r + 1][tid] - 1] = KeyTraits<K>::min_key();
      dk[s_off[r + 1][tid] + s_len[r + 1][tid]] = KeyTraits<K>::max_key();
    }
    __syncthreads();
    k0_mark(11 + r);
  }
  k0_mark(6);
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // my chunk outlives the peers' copies
}

// Grid = CL CTAs forming one cluster (CL = 1: a single CTA, no cluster).
// Shared memory: three padded buffers of kK0Chunk keys (two ping-pong, one
// scratch).  SHFL: each warp first sorts its 32 x 16 keys with the
// warp-shuffle bitonic network (warp_bitonic_keys), so the shared-memory
// merge rounds start from runs of 512; otherwise (the A/B variant) every
// thread sorts its 16 keys in registers and the rounds start from 16.
// MW: phase 2 is the one-step CL-way merge (k0_multiway; shared memory: two
// chunk buffers, every chunk's samples, the merge area -- k0_smem_keys);
// otherwise the pairwise cluster levels (three chunk buffers).
template <class K, bool MW>
constexpr int k0_smem_keys() {
  return MW ? 2 * k0_padded<K>() + (kK0MaxCL + 1) * kK0SampStride + 2 * kK0MWKeys
            : 3 * k0_padded<K>();
}
template <class K, bool SHFL, bool MW>
__global__ void __launch_bounds__(kK0NT, 1)
    k0_small_sort(const K* __restrict__ in, K* __restrict__ out, int64_t n, int CL) {
  namespace cg = cooperative_groups;
  constexpr int NT = kK0NT, VT = kK0VT, C = kK0Chunk, CP = k0_padded<K>();
  extern __shared__ __align__(16) unsigned char smem[];
  K* buf[2] = {reinterpret_cast<K*>(smem), reinterpret_cast<K*>(smem) + CP};
  K* win = reinterpret_cast<K*>(smem) + 2 * CP;
  __shared__ const K* chunk[kK0MaxCL];
  __shared__ int64_t s_co[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = blockIdx.x;
  const int N = (int)n;  // <= 2^16
  constexpr int EK = k0_vec<K>();
  const int Q = ((N + CL - 1) / CL + EK - 1) / EK * EK;  // keys per chunk, whole vectors
  const int base = c * Q;
  const int len = N - base <= 0 ? 0 : min(Q, N - base);
  // the chunk's sort only spans the warps / rounds that hold real keys:
  // runs double from w0 while w < CP2 (Q rounded up to a power of two >=
  // the first run)
  // ---- 1. the chunk, padded to C keys with the maximum key (the padding
  // sorts last, so the first len keys are the sorted chunk)
  k0_mark(0);
  K key[VT];
  int w0;
  if constexpr (SHFL) w0 = 32 * VT;
  else w0 = VT;
  int CP2 = w0;  // from Q, not len: every CTA runs the same rounds (same buffer parity)
  while (CP2 < Q) CP2 *= 2;
  const bool active = tid * VT < CP2;  // this thread holds keys of the padded chunk
  if constexpr (SHFL) {
    // warp w takes keys [32 VT w, 32 VT (w + 1)), lane-striped loads.  Every
    // warp runs the network (warps past the chunk sort MAX padding): in
    // convergent code the shuffles need no per-shuffle WARPSYNC /
    // ENDCOLLECTIVE, which a warp-dependent branch around them costs.
#pragma unroll
    for (int k = 0; k < VT; ++k) {
      const int i = warp * 32 * VT + k * 32 + lane;
      key[k] = i < len ? in[base + i] : KeyTraits<K>::max_key();
    }
    warp_bitonic_keys<VT>(key, lane);
    k0_mark(1);
  } else {
#pragma unroll
    for (int k = 0; k < VT; ++k) {
      const int i = tid * VT + k;
      key[k] = i < len ? in[base + i] : KeyTraits<K>::max_key();
    }
    keys_network<VT>(key);
  }
  int cur = 0;
  if (active) {
#pragma unroll
    store_vec<K, VT>(buf[0] + tid * VT, key);
  }
#pragma unroll 1
  for (int w = w0; w < CP2; w *= 2) {
    __syncthreads();
    if (active) {
      const K* src = buf[cur];
      const int d0 = tid * VT, g0 = d0 / (2 * w) * (2 * w);
      k0_merge_thread<K, VT>(src, g0, w, g0 + w, w, d0 - g0, CP2 - 1, key);
      store_vec<K, VT>(buf[cur ^ 1] + d0, key);
    }
    cur ^= 1;
  }
  k0_mark(2);
  if (CL == 1) {
    __syncthreads();
    for (int i = tid; i < len; i += NT) out[base + i] = buf[cur][i];
    return;
  }
  cg::cluster_group cluster = cg::this_cluster();
  if constexpr (MW) {
    // ---- 2. one CL-way merge step across the cluster (DSMEM)
    K* mysam = reinterpret_cast<K*>(smem) + 2 * CP;
    K* sam = mysam + kK0SampStride;
    K* sk = sam + kK0MaxCL * kK0SampStride;
    k0_multiway<K, kK0VT2>(buf[cur], Q, N, CL, mysam, sam, sk, sk + kK0MWKeys, out);
    k0_mark(31);
    return;
  }
  // ---- 2. merge levels across the cluster (DSMEM)
  if (tid < CL) chunk[tid] = cluster.map_shared_rank(buf[cur], tid);
  cluster.sync();  // every chunk sorted; DSMEM pointers published
  k0_mark(3);
  int lvl = 0;
  for (int span = 1; span < CL; span *= 2, ++lvl) {  // runs of `span` chunks
    // my pair: chunks [m 2 span, (m + 1) 2 span); A = first span, B = next
    const int m = c / (2 * span);
    const int a_start = m * 2 * span * Q;
    const int b_start = a_start + span * Q;
    const int a_end = min(N, b_start), b_end = min(N, b_start + span * Q);
    const int na = max(0, a_end - a_start), nb = max(0, b_end - b_start);
    const int d0 = base - a_start, d1 = d0 + len;  // my outputs in the pair
    if (warp < 2) {
      const int d = warp == 0 ? d0 : d1;
      const int i = d >= na + nb ? na
                                 : k0_corank_dsmem<K>(chunk, Q, a_start, na, b_start, nb, d, lane);
      if (lane == 0) s_co[warp] = i;
    }
    __syncthreads();
    k0_mark(4 + 3 * lvl);
    const int i0 = (int)s_co[0], i1 = (int)s_co[1];
    const int la = i1 - i0, lb = len - la;
    const int j0 = d0 - i0;
    // the two windows, from the peers: A[i0, i1) then B[j0, j0 + lb), as
    // 16-byte vectors (the vectors holding them; a vector never straddles
    // two chunks).  In win each window keeps its global phase mod EK: A at
    // pa = ga mod EK, B at pb = (first vector after A) * EK + gb mod EK.
    const int ga = a_start + i0, gb = b_start + j0;
    const int pa = ga % EK;
    const int wb = la > 0 ? (pa + la + EK - 1) / EK : 0;  // first win vector of B
    const int pb = wb * EK + gb % EK;
    {
      const int va0 = ga / EK, nva = la > 0 ? (ga + la + EK - 1) / EK - va0 : 0;
      const int vb0 = gb / EK, nvb = lb > 0 ? (gb + lb + EK - 1) / EK - vb0 : 0;
      const int ca = ga / Q, cb = gb / Q;
      const int ea = (ca + 1) * Q, eb = (cb + 1) * Q;  // first key of the next chunk
      for (int e = tid; e < nva + nvb; e += NT) {
        const bool inA = e < nva;
        const int g = (inA ? va0 + e : vb0 + (e - nva)) * EK;
        const int c0 = inA ? ca : cb;
        const int c1 = g < (inA ? ea : eb) ? c0 : c0 + 1;
        const uint4 v = *reinterpret_cast<const uint4*>(chunk[c1] + (g - c1 * Q));
        *reinterpret_cast<uint4*>(win + (inA ? e : wb + (e - nva)) * EK) = v;
      }
    }
    __syncthreads();
    k0_mark(5 + 3 * lvl);
    const bool last = 2 * span >= CL;
    const int d = tid * VT;
    if (d < len) {
      k0_merge_thread<K, VT>(win, pa, la, pb, lb, d, CP - 1, key);
      const int e = min(VT, len - d);
      K* dst = buf[cur ^ 1];
      if (e == VT) {
        store_vec<K, VT>(dst + d, key);
      } else {
#pragma unroll
        for (int k = 0; k < VT; ++k)
          if (k < e) dst[d + k] = key[k];
      }
    }
    if (last) {  // the sorted slice leaves by coalesced stores
      __syncthreads();
      const K* o = buf[cur ^ 1];
      for (int i = tid; i < len; i += NT) out[base + i] = o[i];
      break;
    }
    cur ^= 1;
    if (tid < CL) chunk[tid] = cluster.map_shared_rank(buf[cur], tid);
    k0_mark(6 + 3 * lvl);
    cluster.sync();  // level written everywhere; nobody still reads the old buffers
  }
  k0_mark(30);
  // keep every CTA's shared memory alive until the peers' last reads are done
  cluster.sync();
  k0_mark(31);
}

}  // namespace msort
