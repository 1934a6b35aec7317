// k5_kway.cuh -- K5, the one-pass stable p-way merge.
//
// The distributed sort ends with p sorted runs on each rank (one segment from
// every rank, in source-rank order); D4 merges them into the rank's output.
// The paper does the corresponding final merges pairwise up its rank tree
// (merge(local, tmp)); here all p runs are merged in ONE pass over HBM:
// every key is read once and written once (2 n wk bytes), instead of once per
// level of a pairwise merge tree (ceil(log2 p) passes).  Ties go to the lower
// run (source rank), so the result is the stable order of the rank-major
// concatenation (R10/R11).  Keys only (any keys-only output is
// unique; equal keys are indistinguishable).  Included by sort_single.cu
// after merge_keys_dual / put_outputs.
//
// Tiles.  Run j is sampled every S keys (its keys at 0, S, 2S, ...); the
// samples of all runs, merged stably (ties to the lower run, then the lower
// index; k5_sample_level, payload = sample id), are in the stable order of
// the output.  Every g-th merged sample starts a tile; tile t's start STATE
// is the number of keys of each run that precede its sample x = (key v,
// run k, index i) in the stable order:
//     c_j = #{R_j <= v} (j < k),   c_k = i,   c_j = #{R_j < v} (j > k),
// found by a binary search per run inside the S keys between the run's
// samples around x (k5_bounds).  Between two consecutive
// tile starts lie g merged samples, and run j contributes fewer than
// (q_j + 1) S keys when q_j of them are its own, so a tile holds at most
//     S (g + p) - p  keys  <=  C (the tile capacity)
// by the choice of S -- no tile is ever cut, whatever the key distribution.
//
// Merge (k5_merge, one CTA per tile, K6's engine generalised): the tile's p
// windows arrive by TMA bulk copies (cp.async.bulk, SASS UBLKCP) between
// MIN/MAX sentinels; ceil(log2 p) rounds of pairwise merges in shared memory
// (round r merges adjacent groups of 2^r runs, lower group first on ties:
// each thread VT outputs as two merge chains, merge_keys_dual); the last
// round writes at the destination's 16-byte phase and the tile leaves by one
// bulk store.  The runs may live in other GPUs' memory (the pull exchange:
// peer pointers mapped through CUDA IPC), so the exchange and the merge are
// one kernel and the segments cross NVLink once, straight into the merge.
#pragma once

namespace msort {

constexpr int kK5MaxRuns = 16;
#ifndef MSORT_K5_G
#define MSORT_K5_G 8  // merged samples per K5 tile, per run
#endif
#ifndef MSORT_K5_MINB
#define MSORT_K5_MINB 6  // K5 CTAs per SM the register budget allows (4-byte keys)
#endif  // runs merged in one pass (more: K3 rounds first)

// Runs of one K5 merge: run j = n[j] keys at k[j] (device pointers, possibly
// into a peer GPU's memory).
struct K5Runs {
  int p;
  const void* k[kK5MaxRuns];
  int64_t n[kK5MaxRuns];
  int64_t soff[kK5MaxRuns + 1];  // first sample of run j in the sample arrays
  int64_t S;                      // sample stride
  int64_t g;                      // merged samples per tile
  int64_t ntiles;                 // T (tile t = [state t, state t+1))
};

// The kernels take the geometry by value (host-planned) or as a pointer into
// device memory (planned on the device by k5_plan_dev: no host round trip).
__device__ __forceinline__ const K5Runs& k5r(const K5Runs& r) { return r; }
__device__ __forceinline__ const K5Runs& k5r(const K5Runs* r) { return *r; }

// Shape of the merge CTA: NT threads x VT keys per thread and round;
// capacity C = (31 NT / 32 - P2 / 2) * VT keys for P2 (p rounded up to a
// power of two) runs, so that a round's ceil(len / VT) output threads per
// pair fit in the 31 output lanes of each warp.
template <int NT, int VT>
struct K5Shape {
  static constexpr int cap(int P2) { return (NT / 32 * 31 - P2 / 2) * VT; }  // 31 output threads per warp
  // keys of shared memory: capacity + per-run slack (<= 3 phase + 2
  // sentinels + 3 rounding) + guard
  static constexpr int keys(int P2) { return cap(P2) + 8 * P2 + 16; }
};

// ---------------------------------------------------------------- partition
// Run j's samples are its keys at 0, S, 2S, ...; sample x = (run k, index
// m) is stored at skey[soff[k] + m] with id x.  The sample runs are merged
// stably (ties to the lower run, then the lower index) in ceil(log2 p) small
// levels; every g-th merged sample starts a tile.

// first index in [lo, hi) with a[i] > v (UPPER) or a[i] >= v
template <class K, bool UPPER>
__device__ __forceinline__ int64_t k5_bound(const K* __restrict__ a, int64_t lo, int64_t hi, K v) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const K x = a[mid];
    if (UPPER ? !(v < x) : (x < v)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int k5_run_of(const K5Runs& R, int64_t x) {
  int k = 0;
  while (k + 1 < R.p && R.soff[k + 1] <= x) ++k;
  return k;
}

// skey[x] = the sample's key, sid[x] = x (its id: run and index follow from
// soff).
template <class K, class RS>
__global__ void __launch_bounds__(256)
    k5_samples(const __grid_constant__ RS Rin, K* __restrict__ skey,
               uint32_t* __restrict__ sid) {
  const K5Runs& R = k5r(Rin);
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= R.soff[R.p]) return;
  const int k = k5_run_of(R, x);
  skey[x] = static_cast<const K*>(R.k[k])[(x - R.soff[k]) * R.S];
  sid[x] = (uint32_t)x;
}

// One level of the sample merge: runs q = [ro[q], ro[q+1]) of (ik, iv); pair
// m = (runs 2m, 2m+1) merged stably (ties to run 2m) into (ok, ov) at the
// same place (a lone last run is copied).  One CTA per output chunk of <= Q
// samples of one pair: the chunk's two co-ranks by 32-ary warp searches in
// global memory (L2-resident arrays), both windows staged in shared memory,
// each thread merges VT outputs there (merge path + serial merge).
constexpr int kK5LvlNT = 256, kK5LvlVT = 8, kK5LvlQ = kK5LvlNT * kK5LvlVT;
struct K5Level {
  int q;                            // runs at this level
  int64_t ro[kK5MaxRuns + 1];       // their offsets
  int64_t c0[kK5MaxRuns / 2 + 2];   // first chunk of each pair (prefix)
};
__device__ __forceinline__ const K5Level& k5l(const K5Level& l) { return l; }
__device__ __forceinline__ const K5Level& k5l(const K5Level* l) { return *l; }

template <class K>
__device__ __forceinline__ int64_t k5_corank_warp(const K* __restrict__ A, int64_t na,
                                                  const K* __restrict__ B, int64_t nb, int64_t d,
                                                  int lane) {
  int64_t lo = d - nb > 0 ? d - nb : 0, hi = d < na ? d : na;
  while (hi > lo) {  // i(d) = min{i : i = min(d, na) or A[i] > B[d-1-i]}
    const int64_t span = hi - lo;
    const int64_t step = (span + 31) >> 5;
    const int64_t off = step * (lane + 1);
    const int64_t q = lo + (off < span ? off : span) - 1;
    const bool pred = A[q] > B[d - 1 - q];
    const unsigned m = __ballot_sync(0xffffffffu, pred);
    if (m == 0) {
      lo = hi;
    } else {
      const int f = __ffs(m) - 1;
      const int64_t pf = __shfl_sync(0xffffffffu, q, f);
      const int64_t pp = __shfl_sync(0xffffffffu, q, f > 0 ? f - 1 : 0);
      hi = pf;
      if (f > 0) lo = pp + 1;
    }
  }
  return lo;
}

template <class K, class LS>
__global__ void __launch_bounds__(kK5LvlNT)
    k5_sample_level(const __grid_constant__ LS Lin, const K* __restrict__ ik,
                    const uint32_t* __restrict__ iv, K* __restrict__ ok,
                    uint32_t* __restrict__ ov) {
  const K5Level& L = k5l(Lin);
  constexpr int Q = kK5LvlQ, VT = kK5LvlVT;
  __shared__ K sk[Q + 2];
  __shared__ uint32_t sv[Q + 2];
  __shared__ int64_t s_co[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int npair = (L.q + 1) / 2;
  if ((int64_t)blockIdx.x >= L.c0[npair]) return;  // upper-bound grid (device-planned)
  int m = 0;
  while (m + 1 < npair && L.c0[m + 1] <= (int64_t)blockIdx.x) ++m;
  const int64_t a0 = L.ro[2 * m], a1 = L.ro[min(2 * m + 1, L.q)];
  const int64_t b1 = L.ro[min(2 * m + 2, L.q)];
  const int64_t na = a1 - a0, nb = b1 - a1;
  const int64_t d0 = ((int64_t)blockIdx.x - L.c0[m]) * Q;
  const int64_t d1 = min(d0 + Q, na + nb);
  const K* A = ik + a0;
  const K* B = ik + a1;
  if (warp < 2) {
    const int64_t d = warp == 0 ? d0 : d1;
    const int64_t i = d == na + nb ? na : k5_corank_warp<K>(A, na, B, nb, d, lane);
    if (lane == 0) s_co[warp] = i;
  }
  __syncthreads();
  const int64_t i0 = s_co[0], i1 = s_co[1];
  const int la = (int)(i1 - i0), lb = (int)((d1 - i1) - (d0 - i0));
  const int64_t j0 = d0 - i0;
  for (int e = tid; e < la + lb; e += kK5LvlNT) {
    const int64_t src = e < la ? a0 + i0 + e : a1 + j0 + (e - la);
    sk[e] = ik[src];
    sv[e] = iv[src];
  }
  __syncthreads();
  const int d = tid * VT, tot = la + lb;
  if (d < tot) {
    int lo = d - lb > 0 ? d - lb : 0, hi = d < la ? d : la;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (sk[mid] > sk[la + d - 1 - mid]) hi = mid;
      else lo = mid + 1;
    }
    int i = lo, j = la + (d - lo);
    const int e = min(d + VT, tot);
    for (int o = d; o < e; ++o) {
      const bool takeB = j < tot && (i >= la || sk[j] < sk[i]);
      const int src = takeB ? j : i;
      ok[a0 + d0 + o] = sk[src];
      ov[a0 + d0 + o] = sv[src];
      i += takeB ? 0 : 1;
      j += takeB ? 1 : 0;
    }
  }
}

// states[t * p + j] for t = 0..T: tile t's start state (t = T: the ends).
// One thread per (t, j): the merged sample x = mid[t g] = (key v, run k,
// index i);
//     c_j = #{R_j <= v} (j < k),   c_k = i,   c_j = #{R_j < v} (j > k),
// searched only between run j's samples around x: with r = rank_j(x) (the
// number of run j's samples before x, by a search in its sample array), the
// sample at (r - 1) S precedes x and the one at r S does not, so
// c_j in [(r - 1) S + 1, r S]  (c_j = 0 when r = 0).
template <class K, class RS>
__global__ void __launch_bounds__(256)
    k5_bounds(const __grid_constant__ RS Rin, const K* __restrict__ skey,
              const K* __restrict__ mkey, const uint32_t* __restrict__ mid,
              int64_t* __restrict__ states) {
  const K5Runs& R = k5r(Rin);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int p = R.p;
  if (i >= (R.ntiles + 1) * p) return;
  const int64_t t = i / p;
  const int j = (int)(i - t * p);
  int64_t c;
  if (t == 0) {
    c = 0;
  } else if (t == R.ntiles) {
    c = R.n[j];
  } else {
    const int64_t x = mid[t * R.g];
    const int k = k5_run_of(R, x);
    if (j == k) {
      c = (x - R.soff[k]) * R.S;  // x itself starts the tile
    } else {
      const K v = mkey[t * R.g];
      const int64_t r =
          (j < k ? k5_bound<K, true>(skey, R.soff[j], R.soff[j + 1], v)
                 : k5_bound<K, false>(skey, R.soff[j], R.soff[j + 1], v)) - R.soff[j];
      const K* run = static_cast<const K*>(R.k[j]);
      const int64_t lo = r == 0 ? 0 : (r - 1) * R.S + 1, hi = min(r * R.S, R.n[j]);
      c = j < k ? k5_bound<K, true>(run, lo, hi, v)   // lower runs: keys <= v first
                : k5_bound<K, false>(run, lo, hi, v); // higher runs: keys < v first
    }
  }
  states[i] = c;
}

// ------------------------------------------------------- device planning
// The geometry of one K5 merge planned on the device (one thread), so the
// distributed pull path needs no host round trip: rank `me`'s runs are the
// segments [S[me][j], S[me+1][j]) of every rank j's sorted shard (the split
// matrix S, (p+1) x p int64, on the device), at bases[j] (device table of the
// ranks' shard pointers, possibly peer memory).  Fills the K5Runs (the
// sample stride S and fill g come from the host: they depend on p only) and
// the sample-merge levels; the kernels are launched with upper-bound grids.
constexpr int kK5MaxLevels = 4;
struct K5Geo {
  K5Runs R;
  K5Level L[kK5MaxLevels];
  int levels;
};
__global__ void k5_plan_dev(K5Geo* __restrict__ G, const int64_t* __restrict__ split, int me,
                            int p, const void* const* __restrict__ bases, int wk, int64_t S,
                            int64_t g) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  K5Runs& R = G->R;
  R.p = p, R.S = S, R.g = g;
  R.soff[0] = 0;
  for (int j = 0; j < p; ++j) {
    const int64_t a = split[(int64_t)me * p + j], b = split[(int64_t)(me + 1) * p + j];
    R.k[j] = static_cast<const char*>(bases[j]) + a * wk;
    R.n[j] = b - a;
    R.soff[j + 1] = R.soff[j] + (R.n[j] + S - 1) / S;
  }
  const int64_t M = R.soff[p];
  R.ntiles = M == 0 ? 0 : max((int64_t)1, (M + g - 1) / g);
  K5Level L{};
  L.q = p;
  for (int j = 0; j <= p; ++j) L.ro[j] = R.soff[j];
  int levels = 0;
  while ((1 << levels) < p) ++levels;
  G->levels = levels;
  for (int lv = 0; lv < levels && lv < kK5MaxLevels; ++lv) {
    const int npair = (L.q + 1) / 2;
    int64_t ch = 0;
    for (int m = 0; m < npair; ++m) {
      L.c0[m] = ch;
      const int64_t len = L.ro[min(2 * m + 2, L.q)] - L.ro[2 * m];
      ch += (len + kK5LvlQ - 1) / kK5LvlQ;
    }
    L.c0[npair] = ch;
    G->L[lv] = L;
    K5Level N{};
    N.q = npair;
    for (int m = 0; m <= N.q; ++m) N.ro[m] = L.ro[min(2 * m, L.q)];
    L = N;
  }
}

// ---------------------------------------------------------------- merge
// One CTA per tile; P2 = p rounded up to a power of two (runs p..P2-1 are
// empty), R = log2(P2) rounds: round r has P2 >> r runs; run i of round r =
// the merge of runs 2i, 2i+1 of round r-1; round r's pair m = (run 2m = A,
// run 2m+1 = B) sits in shared memory as [MIN | B | MAX .. MIN | A | MAX]
// (B below A: merge_keys_dual clamps A at its MAX and B at its MIN sentinel
// with one bound each).  The layout is computed with warp shuffles (lane j =
// run j; sizes from the tile's states): warp 0 lays out round 0, arms the
// barrier and issues the window copies, while warps 1.. lay out the later
// rounds and the thread ranges under the copies' latency.  Output thread
// o = 31 warp + lane (lanes 0..30) merges VT outputs; lane 31 only searches
// the co-rank at the next warp's first diagonal, so every thread's end
// co-rank is its neighbour's start (a shuffle): two barriers per round.
template <class K, int NT, int VT, int MINB, int P2, class RS>
__global__ void __launch_bounds__(NT, MINB)
    k5_merge(const __grid_constant__ RS Rin, const int64_t* __restrict__ states,
             K* __restrict__ dst) {
  const K5Runs& R = k5r(Rin);
  if ((int64_t)blockIdx.x >= R.ntiles) return;  // upper-bound grid (device-planned)
  constexpr int RR = __builtin_ctz(P2);  // rounds
  constexpr int NW = NT / 32;
  static_assert(NW >= 2 && P2 <= 32, "a layout warp besides warp 0; one lane per run");
  constexpr uint32_t Z = sizeof(K);
  constexpr unsigned F = 0xffffffffu;
  extern __shared__ __align__(16) unsigned char smem[];
  K* sk = reinterpret_cast<K*>(smem);
  const char* sb = reinterpret_cast<const char*>(smem);
  __shared__ uint64_t bar;
  __shared__ int s_len[RR + 1][P2];     // run sizes per round (round RR: the tile)
  __shared__ int s_off[RR][P2];         // run offsets (keys) per round
  __shared__ int s_tp[RR][P2 / 2 + 1];  // first output thread of each pair per round
  __shared__ int64_t s_src[P2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int p = R.p;
  const int64_t t = blockIdx.x;

  if (tid == 0) {
    mbar_init(&bar, 32);
    fence_mbar_init();
  }
  auto scan_excl = [&](int v) {  // exclusive prefix over lanes 0..P2-1
    int inc = v;
#pragma unroll
    for (int d = 1; d < P2; d <<= 1) {
      const int x = __shfl_up_sync(F, inc, d);
      if (lane >= d) inc += x;
    }
    return inc - v;
  };
  // every warp: lane j < p holds run j's window [a, b) of this tile
  int64_t a = 0, b = 0;
  if (lane < p) a = states[t * p + lane], b = states[(t + 1) * p + lane];
  const int l0 = (int)(b - a);
  int64_t out = a;
#pragma unroll
  for (int d = 1; d < P2; d <<= 1) out += __shfl_xor_sync(F, out, d);
  out = __shfl_sync(F, out, 0);  // lanes 0..P2-1 summed their group
  const int sh = stage_offset(dst + out);  // the output's 16-byte phase
  __syncthreads();  // barrier initialised
  if (warp == 0) {
    const K* g = lane < p ? static_cast<const K*>(R.k[lane]) + a : nullptr;
    const int ph = lane < p ? stage_offset(g) : 0;
    const int fp = lane < P2 ? (ph + l0 + 8) & ~3 : 0;  // MIN slot, phase, run, MAX, rounding
    const int base = __shfl_sync(F, scan_excl(__shfl_sync(F, fp, lane ^ 1)), lane ^ 1);
    const int o0 = base + 4 + ph;
    uint32_t tx = lane < p ? window_bulk_bytes(g, l0) : 0u;
#pragma unroll
    for (int d = 1; d < P2; d <<= 1) tx += __shfl_xor_sync(F, tx, d);
    if (lane < P2) {
      s_off[0][lane] = o0;
      s_len[0][lane] = l0;
      s_src[lane] = a;
      sk[o0 - 1] = KeyTraits<K>::min_key();
      sk[o0 + l0] = KeyTraits<K>::max_key();
    }
    if (lane == 0) mbar_expect_tx(&bar, tx);
    __syncwarp();
    for (int j = 0; j < p; ++j)
      stage_window(sk + s_off[0][j], static_cast<const K*>(R.k[j]) + s_src[j], s_len[0][j], &bar,
                   lane == 0, lane, 32);
    mbar_arrive(&bar);
  } else {
    for (int r = warp - 1; r < RR; r += NW - 1) {
      // run j of round r = runs [j 2^r, (j+1) 2^r) of round 0: group sums by
      // xor-reduction, gathered from the group's first lane
      int gs = l0;
      for (int d = 1; d < (1 << r); d <<= 1) gs += __shfl_xor_sync(F, gs, d);
      const int gs2 = gs + __shfl_xor_sync(F, gs, 1 << r);
      const int nr = P2 >> r, np = nr / 2;
      const int l = __shfl_sync(F, gs, (lane << r) & 31);
      const int l2 = __shfl_sync(F, gs2, (lane << (r + 1)) & 31);
      if (r > 0) {
        const int fp = lane < nr ? (l + 8) & ~3 : 0;
        const int base = __shfl_sync(F, scan_excl(__shfl_sync(F, fp, lane ^ 1)), lane ^ 1);
        if (lane < nr) {
          s_off[r][lane] = base + 4;
          s_len[r][lane] = l;
        }
      }
      // the last round's diagonals are shifted by the output phase sh
      // (thread k: [k VT - sh, (k+1) VT - sh)), so every full thread's
      // outputs start 16-byte aligned in the phase-matched output buffer
      const int shr = r + 1 == RR ? sh : 0;
      const int cnt = lane < np ? (l2 + shr + VT - 1) / VT : 0;
      const int tp = scan_excl(cnt);
      if (lane < np) s_tp[r][lane] = tp;
      if (lane == np - 1) s_tp[r][np] = tp + cnt;
      if (r + 1 == RR && lane == 0) s_len[RR][0] = l2;
    }
  }
  __syncthreads();  // layout and round-0 sentinels visible
  mbar_wait(&bar, 0);

  K key[VT];
  const int tot = s_len[RR][0];
  const int o = warp * 31 + lane;
#pragma unroll 1
  for (int r = 0; r < RR; ++r) {
    const int npair = P2 >> (r + 1);
    int m = 0;
#pragma unroll
    for (int q = 1; q < P2 / 2; ++q)
      if (q < npair && s_tp[r][q] <= o) m = q;
    const bool in = o < s_tp[r][npair];
    const int la = s_len[r][2 * m], lb = s_len[r][2 * m + 1], len = la + lb;
    const uint32_t oa = (uint32_t)s_off[r][2 * m] * Z, ob = (uint32_t)s_off[r][2 * m + 1] * Z;
    const int shr = r + 1 == RR ? sh : 0;
    int d = 0, c = 0, i0 = 0;
    if (in) {
      d = max(0, (o - s_tp[r][m]) * VT - shr);
      c = min((o - s_tp[r][m] + 1) * VT - shr, len) - d;
      i0 = merge_path_off<K>(sb, oa, la, ob, lb, d);
    }
    const int nx = __shfl_down_sync(F, i0, 1);
    const bool act = in && lane < 31;
    if (act) {
      const int i1 = d + c == len ? la : nx;
      merge_keys_dual<K, VT>(sb, oa + (uint32_t)i0 * Z, oa + (uint32_t)la * Z,
                             ob + (uint32_t)(d - i0) * Z, oa + (uint32_t)i1 * Z,
                             ob + (uint32_t)(d + c - i1) * Z, ob - Z, key);
    }
    __syncthreads();  // every thread has read its inputs: the buffer is free
    if (r + 1 < RR) {
      if (act) put_outputs<K, VT>(sk + s_off[r + 1][m] + d, key, c);
      if (tid < npair) {
        sk[s_off[r + 1][tid] - 1] = KeyTraits<K>::min_key();
        sk[s_off[r + 1][tid] + s_len[r + 1][tid]] = KeyTraits<K>::max_key();
      }
      __syncthreads();
    } else {
      if (act) put_outputs<K, VT>(sk + sh + d, key, c);  // full threads: (sh + d) % 4 == 0
    }
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (tid < 32) {
    K* go = dst + out;
    int h, mid;
    window_split(go, tot, h, mid);
    if (tid == 0 && mid) {
      bulk_s2g(go + h, sk + sh + h, (uint32_t)(mid * sizeof(K)));
      bulk_commit();
    }
    for (int i = tid; i < tot - mid; i += 32) {
      const int j = i < h ? i : i + mid;
      go[j] = sk[sh + j];
    }
    if (tid == 0 && mid) bulk_wait_read<0>();  // shared memory must outlive the copy's reads
  }
}

}  // namespace msort
