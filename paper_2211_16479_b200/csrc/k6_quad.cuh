// k6_quad.cuh -- K6 (experimental): two merge levels per HBM pass with the
// tile-sort kernel's merge engine.  Included by sort_single.cu after
// merge_keys_dual.
//
// A 4-way pass merges groups of four consecutive runs A, B, C, D of length L
// into runs of 4L: X = merge(A, B), Y = merge(C, D), out = merge(X, Y), every
// merge the stable merge() of P:107 (ties to the left run, R1).
// A tile is the stretch of the output between two 4-way prefix "states"
// (keys of A, B, C, D before it) found by the partition kernels below; it
// holds at most Tm = NT2 * VT keys.  One CTA per tile, K1-style: the four
// windows arrive by TMA bulk copies between MIN/MAX sentinels, round 1 merges
// A+B and C+D (each thread VT outputs of X or of Y as two merge chains,
// merge_keys_dual) into registers, they go back to shared memory as 16-byte
// vectors for the round-2 pair, round 2 merges X+Y at the destination's
// 16-byte phase, and the tile leaves by one bulk store.  Opt-in (quad mode 5):
// 2% faster than the fused 2-way levels on 2^28 int32.
#pragma once

#ifndef MSORT_K6_NT2
#define MSORT_K6_NT2 126  // round-2 threads (Tm = MSORT_K6_NT2 x 68; CTA = +2 threads)
#endif

namespace msort {

struct K6Tile {
  int64_t out;     // output index of the tile's first key
  int64_t src[4];  // first key of each window in the source
  int64_t n[4];    // window lengths (A, B, C, D)
};

// NT1 threads; a tile holds Tm = NT2 * VT keys with NT2 = NT1 - 2, so that
// round 1 (X and Y each ending with a partial thread) fits in NT1 threads
template <int NT2, int VT>
struct K6Shape {
  static constexpr int Tm = NT2 * VT;
  static constexpr int NT1 = NT2 + 2;
  static_assert(NT1 % 32 == 0, "NT2 + 2 threads: whole warps");
  // keys: [MIN | B | MAX .. MIN | A | MAX .. MIN | D | MAX .. MIN | C | MAX ..]
  // each window rounded up to 4 keys plus 2 sentinel slots (round 1); round 2
  // reuses the start as [MIN | Y | MAX .. MIN | X | MAX]
  static constexpr int KEYS = Tm + 4 * 12 + 16;
};

// A thread's c <= VT merge outputs (front chain key[0, H), back chain
// key[VT-1-k] = output c-1-k) into o[0, c): vectors when the thread is full
// and o is 16-byte aligned, else element by element.
template <class K, int VT>
__device__ __forceinline__ void put_outputs(K* o, const K (&key)[VT], int c, bool aligned = true) {
  if (c == VT && aligned) {
    store_vec<K, VT>(o, key);
    return;
  }
  constexpr int H = VT / 2;
#pragma unroll
  for (int k = 0; k < H; ++k) {
    if (k < c) o[k] = key[k];
    if (k < c) o[c - 1 - k] = key[VT - 1 - k];
  }
}

#ifndef MSORT_K6_MINB
#define MSORT_K6_MINB (MSORT_K6_NT2 > 126 ? 3 : 6)
#endif
template <class K, int NT2, int VT>
__device__ __forceinline__ void k6_tile(const K* __restrict__ src, K* __restrict__ dst,
                                        const K6Tile& t, uint64_t* bar, uint32_t phase);

// One tile per CTA (tiles with out < 0 are skipped: their pieces come in the
// cut list), or -- with ntiles_dev -- a grid-stride loop over a device-counted list.
template <class K, int NT2, int VT>
__global__ void __launch_bounds__(K6Shape<NT2, VT>::NT1, MSORT_K6_MINB)
    k6_quad_pass(const K* __restrict__ src, K* __restrict__ dst,
                 const K6Tile* __restrict__ tiles,
                 const unsigned long long* __restrict__ ntiles_dev) {
  __shared__ uint64_t bar;  // the tile's TMA loads (one phase per tile)
  if (threadIdx.x == 0) {
    mbar_init(&bar, 32);
    fence_mbar_init();
  }
  __syncthreads();
  if (ntiles_dev == nullptr) {
    const K6Tile t = tiles[blockIdx.x];
    if (t.out >= 0) k6_tile<K, NT2, VT>(src, dst, t, &bar, 0);
    return;
  }
  const int64_t cnt = (int64_t)*ntiles_dev;
  uint32_t phase = 0;
  for (int64_t i = blockIdx.x; i < cnt; i += gridDim.x, phase ^= 1) {
    const K6Tile t = tiles[i];
    k6_tile<K, NT2, VT>(src, dst, t, &bar, phase);
    __syncthreads();  // shared memory is reused by the next tile
  }
}

template <class K, int NT2, int VT>
__device__ __forceinline__ void k6_tile(const K* __restrict__ src, K* __restrict__ dst,
                                        const K6Tile& t, uint64_t* bar, uint32_t phase) {
  using SH = K6Shape<NT2, VT>;
  constexpr int NT1 = SH::NT1;
  constexpr uint32_t Z = sizeof(K);
  extern __shared__ __align__(16) unsigned char smem[];
  K* sk = reinterpret_cast<K*>(smem);
  const char* sb = reinterpret_cast<const char*>(smem);
  const int tid = threadIdx.x;
  const int na = (int)t.n[0], nb = (int)t.n[1], nc = (int)t.n[2], nd = (int)t.n[3];
  const int nx = na + nb, ny = nc + nd, tot = nx + ny;
  // round-1 layout (key indices): B, A, D, C, each window at its global
  // 16-byte phase (TMA bulk copies) with a MIN slot before it and a MAX after
  auto up4 = [](int x) { return (x + 3) & ~3; };
  const K* gA = src + t.src[0];
  const K* gB = src + t.src[1];
  const K* gC = src + t.src[2];
  const K* gD = src + t.src[3];
  const int oB = 4 + stage_offset(gB);
  const int oA = up4(oB + nb + 2) + stage_offset(gA);
  const int oD = up4(oA + na + 2) + stage_offset(gD);
  const int oC = up4(oD + nd + 2) + stage_offset(gC);
  __shared__ int cr[NT1 + 1];  // co-ranks of the threads' first diagonals
  if (tid < 4) {
    const int o = tid == 0 ? oA : tid == 1 ? oB : tid == 2 ? oC : oD;
    const int c = tid == 0 ? na : tid == 1 ? nb : tid == 2 ? nc : nd;
    sk[o - 1] = KeyTraits<K>::min_key();
    sk[o + c] = KeyTraits<K>::max_key();
  }
  __syncthreads();
  if (tid < 32) {
    if (tid == 0)
      mbar_expect_tx(bar, window_bulk_bytes(gA, na) + window_bulk_bytes(gB, nb) +
                               window_bulk_bytes(gC, nc) + window_bulk_bytes(gD, nd));
    __syncwarp();
    stage_window(sk + oA, gA, na, bar, tid == 0, tid, 32);
    stage_window(sk + oB, gB, nb, bar, tid == 0, tid, 32);
    stage_window(sk + oC, gC, nc, bar, tid == 0, tid, 32);
    stage_window(sk + oD, gD, nd, bar, tid == 0, tid, 32);
    mbar_arrive(bar);
  }
  mbar_wait(bar, phase);
  K key[VT];
  // ---- round 1: X = merge(A, B) by threads [0, tx), Y = merge(C, D) after
  const int tx = (nx + VT - 1) / VT, ty = (ny + VT - 1) / VT;
  const bool isx = tid < tx;
  const bool act1 = isx || tid < tx + ty;
  int d1 = 0, c1 = 0, i0 = 0;
  const int ra = isx ? oA : oC, rb = isx ? oB : oD;
  const int la = isx ? na : nc, lb = isx ? nb : nd;
  const int kk = isx ? nx : ny;
  const uint32_t oa1 = (uint32_t)ra * Z, ob1 = (uint32_t)rb * Z;
  if (act1) {
    d1 = (isx ? tid : tid - tx) * VT;
    c1 = min(VT, kk - d1);
    i0 = merge_path_off<K>(sb, oa1, la, ob1, lb, d1);
    cr[tid] = i0;
  }
  __syncthreads();
  if (act1) {
    // the co-rank at my last diagonal: the next thread's first, or the end
    const int i1 = d1 + c1 == kk ? la : cr[tid + 1];
    merge_keys_dual<K, VT>(sb, oa1 + (uint32_t)i0 * Z, oa1 + (uint32_t)la * Z,
                           ob1 + (uint32_t)(d1 - i0) * Z, oa1 + (uint32_t)i1 * Z,
                           ob1 + (uint32_t)(d1 + c1 - i1) * Z, ob1 - Z, key);
  }
  __syncthreads();
  // round-2 layout: [MIN | Y | MAX | MIN | X | MAX], runs 16-byte aligned so
  // a full thread's VT outputs leave as vectors (VT * 4 bytes apart: 17
  // vector slots for VT = 68, odd -- conflict-free quarter-warps)
  const int oY = 4, oX = up4(oY + ny + 2);
  if (act1) {
    K* o = sk + (isx ? oX : oY) + d1;
    put_outputs<K, VT>(o, key, c1);
  }
  if (tid == 0) {
    sk[oY - 1] = KeyTraits<K>::min_key(), sk[oY + ny] = KeyTraits<K>::max_key();
    sk[oX - 1] = KeyTraits<K>::min_key(), sk[oX + nx] = KeyTraits<K>::max_key();
  }
  __syncthreads();
  // ---- round 2: out = merge(X, Y)
  const bool act2 = tid < NT2 && tid * VT < tot;
  int d2 = 0, c2 = 0, j0 = 0;
  const uint32_t oa2 = (uint32_t)oX * Z, ob2 = (uint32_t)oY * Z;
  if (act2) {
    d2 = tid * VT;
    c2 = min(VT, tot - d2);
    j0 = merge_path_off<K>(sb, oa2, nx, ob2, ny, d2);
    cr[tid] = j0;
  }
  __syncthreads();
  if (act2) {
    const int j1 = d2 + c2 == tot ? nx : cr[tid + 1];
    merge_keys_dual<K, VT>(sb, oa2 + (uint32_t)j0 * Z, oa2 + (uint32_t)nx * Z,
                           ob2 + (uint32_t)(d2 - j0) * Z, oa2 + (uint32_t)j1 * Z,
                           ob2 + (uint32_t)(d2 + c2 - j1) * Z, ob2 - Z, key);
  }
  __syncthreads();
  // the tile leaves by one bulk store: outputs at the destination's phase
  K* gout = dst + t.out;
  const int ph = stage_offset(gout);
  if (act2) put_outputs<K, VT>(sk + ph + d2, key, c2, ph == 0);
  fence_proxy_async_smem();
  __syncthreads();
  if (tid < 32) {
    int h, mid;
    window_split(gout, tot, h, mid);
    if (tid == 0 && mid) {
      bulk_s2g(gout + h, sk + ph + h, (uint32_t)(mid * sizeof(K)));
      bulk_commit();
    }
    for (int i = tid; i < tot - mid; i += 32) {
      const int j = i < h ? i : i + mid;
      gout[j] = sk[ph + j];
    }
    if (tid == 0 && mid) bulk_wait_read<0>();  // smem must outlive the copy's reads
  }
}

// ------------------------------------------------------------ partition
// Tiles of a 4-way pass (keys only).  Group g = runs 4g..4g+3 of length L
// (A, B, C, D; the last group may be short), X = merge(A, B), Y = merge(C, D).
// A UNIT of group g covers X keys [k XS, (k+1) XS); its start STATE is the
// prefix of the stable 4-way order ending just before X[k XS]:
//     (a, b) = co-rank of merge(A, B) at x = k XS (ties to A), v = X[x],
//     c = #C < v, d = #D < v     (C/D keys equal to v follow it: A<B<C<D),
// so a unit holds XS keys of X and the Y keys between two X samples.  A unit
// with more than YS keys of Y is cut at Y-side states (w = Y[y]: (c, d) =
// co-rank of merge(C, D) at y, a = #A <= w, b = #B <= w) every YS keys of Y,
// so every tile holds <= XS + YS <= Tm keys.
struct K6Pass {
  const void* src;
  int64_t n, L;
  int64_t groups, upg;  // groups; units per full group (ceil(2L / XS))
  int64_t nunits;
  int xs, ys;
};

template <class K>
__device__ __forceinline__ void k6_group(const K6Pass& P, int64_t g, int64_t (&st)[5]) {
#pragma unroll
  for (int r = 0; r <= 4; ++r) st[r] = min(P.n, g * 4 * P.L + (int64_t)r * P.L);
}
template <class K>
__device__ __forceinline__ void k6_unit(const K6Pass& P, int64_t u, int64_t& g, int64_t& k) {
  g = min(u / P.upg, P.groups - 1);
  k = u - g * P.upg;
}
// first i in [lo, hi) with r[i] > v (UPPER) or r[i] >= v
template <class K, bool UPPER>
__device__ __forceinline__ int64_t k6_bound(const K* __restrict__ r, int64_t lo, int64_t hi, K v) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (UPPER ? !(v < r[mid]) : (r[mid] < v)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
// co-rank of diagonal x of merge(P, Q), ties to P, searched inside [lo, hi]
template <class K>
__device__ __forceinline__ int64_t k6_corank(const K* __restrict__ P, int64_t np,
                                             const K* __restrict__ Q, int64_t nq, int64_t x,
                                             int64_t lo = 0, int64_t hi = INT64_MAX) {
  lo = max(lo, x - nq > 0 ? x - nq : (int64_t)0);
  hi = min(hi, x < np ? x : np);
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (Q[x - 1 - mid] < P[mid]) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// states[u] = start state of unit u (a, b, c, d).  Two launches: COARSE
// computes every 32nd unit of a group by full searches; the others search
// only inside the bracket of their coarse neighbours (states are monotone),
// so their probes fall in a small region that the neighbouring threads share
// (the partition is bound by its random probe traffic, not by latency).
constexpr int kK6Coarse = 32;
template <class K, bool COARSE>
__global__ void __launch_bounds__(128)
    k6_states(const K6Pass P, int64_t* __restrict__ states) {
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= P.nunits) return;
  int64_t g, k;
  k6_unit<K>(P, u, g, k);
  if (COARSE != (k % kK6Coarse == 0)) return;
  int64_t st[5];
  k6_group<K>(P, g, st);
  const K* src = static_cast<const K*>(P.src);
  const K* A = src + st[0];
  const K* B = src + st[1];
  const K* C = src + st[2];
  const K* D = src + st[3];
  const int64_t na = st[1] - st[0], nb = st[2] - st[1], nc = st[3] - st[2], nd = st[4] - st[3];
  // bracket: the coarse states before and after (the group's ends at its edges)
  int64_t lo[4] = {0, 0, 0, 0}, hi[4] = {na, nb, nc, nd};
  if (!COARSE) {
    const int64_t u0 = u - k % kK6Coarse, u1 = u0 + kK6Coarse;
#pragma unroll
    for (int r = 0; r < 4; ++r) lo[r] = states[4 * u0 + r];
    int64_t g1 = -1, k1 = 0;
    if (u1 < P.nunits) k6_unit<K>(P, u1, g1, k1);
    if (g1 == g) {
#pragma unroll
      for (int r = 0; r < 4; ++r) hi[r] = states[4 * u1 + r];
    }
  }
  int64_t a = 0, b = 0, c = 0, d = 0;
  const int64_t x = k * P.xs;
  if (x >= na + nb) {
    a = na, b = nb, c = nc, d = nd;
  } else if (x > 0) {
    a = k6_corank(A, na, B, nb, x, max(lo[0], x - hi[1]), min(hi[0], x - lo[1]));
    b = x - a;
    const K v = (a < na && (b >= nb || !(B[b] < A[a]))) ? A[a] : B[b];
    c = k6_bound<K, false>(C, lo[2], hi[2], v);
    d = k6_bound<K, false>(D, lo[3], hi[3], v);
  }
  int64_t* o = states + 4 * u;
  o[0] = a, o[1] = b, o[2] = c, o[3] = d;
}

// End state of unit u: the next unit's start in the same group, else the group end.
template <class K>
__device__ __forceinline__ void k6_end(const K6Pass& P, const int64_t* states, int64_t u, int64_t g,
                                       const int64_t (&st)[5], int64_t (&e)[4]) {
  int64_t g2 = -1, k2 = 0;
  if (u + 1 < P.nunits) k6_unit<K>(P, u + 1, g2, k2);
  if (g2 == g) {
#pragma unroll
    for (int r = 0; r < 4; ++r) e[r] = states[4 * (u + 1) + r];
  } else {
#pragma unroll
    for (int r = 0; r < 4; ++r) e[r] = st[r + 1] - st[r];
  }
}

__device__ __forceinline__ void k6_put(K6Tile* t, const int64_t (&st)[5], const int64_t (&s0)[4],
                                       const int64_t (&s1)[4]) {
  t->out = st[0] + s0[0] + s0[1] + s0[2] + s0[3];
#pragma unroll
  for (int r = 0; r < 4; ++r) t->src[r] = st[r] + s0[r], t->n[r] = s1[r] - s0[r];
}

// tiles[u] = unit u when its Y part fits (else out = -1 and its YS-pieces
// are listed as (u, j) in cuts[], counted in *ncut).
template <class K>
__global__ void __launch_bounds__(128)
    k6_tiles(const K6Pass P, const int64_t* __restrict__ states, K6Tile* __restrict__ tiles,
             int64_t* __restrict__ cuts, unsigned long long* __restrict__ ncut) {
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= P.nunits) return;
  int64_t g, k;
  k6_unit<K>(P, u, g, k);
  int64_t st[5], s0[4], s1[4];
  k6_group<K>(P, g, st);
#pragma unroll
  for (int r = 0; r < 4; ++r) s0[r] = states[4 * u + r];
  k6_end<K>(P, states, u, g, st, s1);
  const int64_t ysz = (s1[2] + s1[3]) - (s0[2] + s0[3]);
  if (ysz <= P.ys) {
    k6_put(tiles + u, st, s0, s1);
    return;
  }
  tiles[u].out = -1;
  const int64_t m = (ysz + P.ys - 1) / P.ys;
  const unsigned long long j0 = atomicAdd(ncut, (unsigned long long)m);
  for (int64_t j = 0; j < m; ++j) cuts[2 * (j0 + j)] = u, cuts[2 * (j0 + j) + 1] = j;
}

// Y-side state at y of unit u's group (searches inside the unit's bounds)
template <class K>
__device__ __forceinline__ void k6_ystate(const K6Pass& P, const int64_t (&st)[5],
                                          const int64_t (&s0)[4], const int64_t (&s1)[4],
                                          int64_t y, int64_t (&o)[4]) {
  const K* src = static_cast<const K*>(P.src);
  const K* A = src + st[0];
  const K* B = src + st[1];
  const K* C = src + st[2];
  const K* D = src + st[3];
  const int64_t nc = st[3] - st[2], nd = st[4] - st[3];
  const int64_t c = k6_corank(C, nc, D, nd, y);
  const int64_t d = y - c;
  const K w = (c < nc && (d >= nd || !(D[d] < C[c]))) ? C[c] : D[d];
  o[0] = k6_bound<K, true>(A, s0[0], s1[0], w);
  o[1] = k6_bound<K, true>(B, s0[1], s1[1], w);
  o[2] = c, o[3] = d;
}

// the pieces of the oversized units (grid-stride over *ncut)
template <class K>
__global__ void __launch_bounds__(128)
    k6_cut_tiles(const K6Pass P, const int64_t* __restrict__ states,
                 const int64_t* __restrict__ cuts, const unsigned long long* __restrict__ ncut,
                 K6Tile* __restrict__ extra) {
  const int64_t cnt = (int64_t)*ncut;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = cuts[2 * i], j = cuts[2 * i + 1];
    int64_t g, k;
    k6_unit<K>(P, u, g, k);
    int64_t st[5], s0[4], s1[4], a[4], b[4];
    k6_group<K>(P, g, st);
#pragma unroll
    for (int r = 0; r < 4; ++r) s0[r] = states[4 * u + r];
    k6_end<K>(P, states, u, g, st, s1);
    const int64_t y0 = s0[2] + s0[3], y1 = s1[2] + s1[3];
    const int64_t ya = y0 + j * P.ys, yb = ya + P.ys;
    if (j == 0) {
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r] = s0[r];
    } else {
      k6_ystate<K>(P, st, s0, s1, ya, a);
    }
    if (yb >= y1) {
#pragma unroll
      for (int r = 0; r < 4; ++r) b[r] = s1[r];
    } else {
      k6_ystate<K>(P, st, s0, s1, yb, b);
    }
    k6_put(extra + i, st, a, b);
  }
}

}  // namespace msort
