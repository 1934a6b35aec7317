// k3x_merge.cuh -- K3X: two merge levels per HBM pass (keys only).
//
// A 4-way pass merges groups of four consecutive runs A, B, C, D of length L
// (group g = runs 4g..4g+3) into runs of 4L -- the same result as two 2-way
// levels X = merge(A, B), Y = merge(C, D), out = merge(X, Y) (every merge the
// stable merge() of P:107 with ties to the left run, R1, so ties
// go A < B < C < D), but each key crosses HBM once instead of twice.
//
// Boundaries without nested searches.  A boundary STATE (a, b, c, d) counts
// the keys of A..D before it.  Two kinds are cheap:
//   X-side state at x: (a, b) = co-rank of merge(A, B) at x, v = X[x];
//                      c = #C < v, d = #D < v  (C/D keys equal to v follow X[x]);
//   Y-side state at y: (c, d) = co-rank of merge(C, D) at y, w = Y[y];
//                      a = #A <= w, b = #B <= w  (A/B keys equal to w precede Y[y]).
// Each is a prefix of the stable 4-way order (the position of the sampled key
// X[x] or Y[y] in the output).  A work UNIT is the stretch between X-side
// states at x = (u-1) S and u S (unit 0 starts at the zero state, the last
// ends at the group's end): at most S keys of X plus the keys of Y in that
// value range.  A unit whose size exceeds CAP is cut further at Y-side states
// every M keys of Y (M = CAP - S), so every super-tile holds <= CAP keys.
//
// One persistent, warp-specialised kernel (the K3 pipeline):
//   warp 1  searcher: grabs chunks of U units; computes their states in
//           order (the chunk's first by full searches, the rest bracketed /
//           galloping from the previous one, so the probes fall in the data
//           the chunk is about to stage) and posts super-tiles to a ring;
//   warp 0  producer: stages a super-tile's four windows by TMA bulk copies;
//   warps 3.. mergers: phase 1 -- every thread merges VT outputs of X or of Y
//           (merge-path co-rank in shared memory) into an X|Y buffer; phase 2
//           -- merge X and Y over the consumed input windows (at the
//           destination's 16-byte phase);
//   warp 2  store: bulk copy of the output back to HBM.
#pragma once

#include "msort_device.cuh"

namespace msort {

struct XState {
  int64_t c[4];
};

#ifdef MSORT_K3X_TRACE
// tuning builds: per CTA, ns spent waiting: [0] mergers on full, [1] producer
// on tfull (searcher), [2] producer on empty (store), [3] searcher on tempty
// (ring full), [4] store on outr, [5] kernel span, [6] tiles
__device__ unsigned long long g_k3x_trace[1024 * 8];
__device__ __forceinline__ unsigned long long xt_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define XT_BEGIN(v) const unsigned long long v = xt_now()
#define XT_ADD(slot, v) atomicAdd(&g_k3x_trace[(blockIdx.x & 1023) * 8 + (slot)], xt_now() - (v))
#else
#define XT_BEGIN(v) ((void)0)
#define XT_ADD(slot, v) ((void)0)
#endif

struct XTile {
  int64_t g;    // group (-1: stop)
  XState s0, s1;
};

template <class K, int NC, int VT, int S>
struct K3XLayout {
  static constexpr int CAP = NC * VT;       // merge capacity of the CTA
  static constexpr int CAPT = CAP - VT;     // keys per super-tile (max): phase 1 fits NC threads
  static constexpr int XS = CAP / 2 - 128;  // unit: X keys between X-side states
  static constexpr int YM = CAPT - XS;      // Y keys between Y-side cuts
  static constexpr int EK = 16 / sizeof(K);
  static constexpr int SIN = CAP + 8 * EK;  // four input windows (+ phase slack)
  static constexpr int RT = 64;             // super-tile descriptor ring
  static constexpr size_t bars = 0;         // full[S], empty[S], outr[S], tfull[RT], tempty[RT]
  static constexpr size_t desc = align_up_c(8 * (3 * S + 2 * RT), 16);
  static constexpr size_t meta = align_up_c(desc + sizeof(XTile) * RT, 16);
  static constexpr size_t chunk = align_up_c(meta + 64 * S, 16);  // searcher: 32 states
  static constexpr size_t stage = align_up_c(chunk + 32 * 32, 128);
  static constexpr size_t stage_keys = (size_t)(SIN + CAP);
  static constexpr size_t bytes = align_up_c(stage + (size_t)S * stage_keys * sizeof(K), 128);
};

struct XMeta {
  int64_t out;  // output index of the first key (-1: stop)
  int n[4];
  int off[4];
  int tot;
};

// first i in [lo, n) with r[i] >= v (UPPER: r[i] > v), galloping from lo
template <class K, bool UPPER>
__device__ __forceinline__ int64_t x_gallop(const K* __restrict__ r, int64_t lo, int64_t n, K v) {
  auto before = [&](int64_t i) { return UPPER ? !(v < r[i]) : (r[i] < v); };
  int64_t step = 1, probe = lo;
  while (probe < n && before(probe)) {
    lo = probe + 1;
    probe = lo + step;
    step <<= 1;
  }
  int64_t hi = probe < n ? probe : n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (before(mid)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// first i in [lo, hi) with r[i] >= v (UPPER: r[i] > v), by bisection
template <class K, bool UPPER>
__device__ __forceinline__ int64_t x_bound(const K* __restrict__ r, int64_t lo, int64_t hi, K v) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (UPPER ? !(v < r[mid]) : (r[mid] < v)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// co-rank (ties to P) of diagonal x of merge(P, Q) inside [lo, hi]
template <class K>
__device__ __forceinline__ int64_t x_corank(const K* __restrict__ P, const K* __restrict__ Q,
                                            int64_t x, int64_t lo, int64_t hi) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (Q[x - 1 - mid] < P[mid]) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

__device__ __forceinline__ XState shfl_state(const XState& s, int src_lane) {
  XState r;
#pragma unroll
  for (int i = 0; i < 4; ++i) r.c[i] = __shfl_sync(0xffffffffu, s.c[i], src_lane);
  return r;
}

#ifndef MSORT_X_MINB
#define MSORT_X_MINB 2
#endif
template <class K, int NC, int VT, int S>
__global__ void __launch_bounds__(NC + 96, MSORT_X_MINB)
    k3x_pass(const K* __restrict__ src, K* __restrict__ dst, int64_t n, int64_t L,
             int64_t ngroups, int64_t units_per_group, unsigned long long* __restrict__ ctr) {
  using LY = K3XLayout<K, NC, VT, S>;
  constexpr int EK = LY::EK, RT = LY::RT, CAP = LY::CAP;
  constexpr int U = 31;  // units per grab (<= 31: one lane per unit start + the end)
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + LY::bars);
  uint64_t* empty = full + S;
  uint64_t* outr = empty + S;
  uint64_t* tfull = outr + S;
  uint64_t* tempty = tfull + RT;
  XTile* ring = reinterpret_cast<XTile*>(smem + LY::desc);
  XMeta* meta = reinterpret_cast<XMeta*>(smem + LY::meta);
  K* stg = reinterpret_cast<K*>(smem + LY::stage);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s)
      mbar_init(&full[s], 32), mbar_init(&empty[s], 1), mbar_init(&outr[s], NC / 32);
    for (int r = 0; r < RT; ++r) mbar_init(&tfull[r], 1), mbar_init(&tempty[r], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t nunits = ngroups * units_per_group;
  XT_BEGIN(tk);

  if (warp == 1) {
    // ------------------------------------------------------------ searcher
    // A chunk of U consecutive units: lane l computes the start state of
    // unit u0 + l (l = 0..U); lanes 0 and U search the whole runs, the inner
    // lanes inside the bracket those give (states are monotone), so their
    // probes fall in the data the chunk stages next.  Lane 0 then posts the
    // units' super-tiles in order (cutting oversized units at Y-side states).
    XState* cs = reinterpret_cast<XState*>(smem + LY::chunk);
    int64_t t = 0;  // super-tiles posted (lane 0)
    auto post = [&](int64_t g, const XState& a, const XState& b) {
      const int r = (int)(t % RT);
      XT_BEGIN(t0);
      mbar_wait(&tempty[r], (uint32_t)(((t / RT) & 1) ^ 1));
      XT_ADD(3, t0);
      ring[r].g = g, ring[r].s0 = a, ring[r].s1 = b;
      mbar_arrive(&tfull[r]);
      ++t;
    };
    auto geom = [&](int64_t g, int64_t (&off)[5]) {
#pragma unroll
      for (int i = 0; i <= 4; ++i) off[i] = min(n, g * 4 * L + (int64_t)i * L);
    };
    // X-side state at x of group g: the position of X[x] in the output (the
    // group's end state for x >= |X|), searched inside the bracket [lo, hi].
    auto xstate = [&](int64_t g, int64_t x, const XState& lo, const XState& hi) {
      int64_t off[5];
      geom(g, off);
      const K* A = src + off[0];
      const K* B = src + off[1];
      const K* C = src + off[2];
      const K* D = src + off[3];
      const int64_t na = off[1] - off[0], nb = off[2] - off[1], nc = off[3] - off[2],
                    nd = off[4] - off[3];
      XState st;
      if (x >= na + nb) {
        st.c[0] = na, st.c[1] = nb, st.c[2] = nc, st.c[3] = nd;
        return st;
      }
      const int64_t ilo = max(max(x - nb, (int64_t)0), lo.c[0]);
      const int64_t ihi = min(min(x, na), hi.c[0]);
      const int64_t i = x_corank(A, B, x, ilo, ihi);
      const int64_t j = x - i;
      const K v = (i < na && (j >= nb || !(B[j] < A[i]))) ? A[i] : B[j];
      st.c[0] = i, st.c[1] = j;
      const bool br = hi.c[2] < nc || lo.c[2] > 0;  // bracketed: gallop, else bisect
      st.c[2] = br ? x_gallop<K, false>(C, lo.c[2], min(nc, hi.c[2]), v)
                   : x_bound<K, false>(C, 0, nc, v);
      st.c[3] = br ? x_gallop<K, false>(D, lo.c[3], min(nd, hi.c[3]), v)
                   : x_bound<K, false>(D, 0, nd, v);
      return st;
    };
    auto start_state = [&](int64_t u, const XState& lo, const XState& hi) {
      const int64_t g = u / units_per_group, k = u % units_per_group;
      if (k == 0) {
        XState z;
        z.c[0] = z.c[1] = z.c[2] = z.c[3] = 0;
        return z;
      }
      return xstate(g, (k - 1) * (int64_t)LY::XS, lo, hi);
    };
    XState zero, inf;
#pragma unroll
    for (int i = 0; i < 4; ++i) zero.c[i] = 0, inf.c[i] = INT64_MAX / 4;
    // Static split: CTA b takes units [b*per, (b+1)*per), so each chunk's
    // first state is the previous chunk's last (one full search per CTA per
    // pass; every later edge is bracketed from the carried state).
    const int64_t per = (nunits + gridDim.x - 1) / gridDim.x;
    const int64_t ubeg = min(nunits, (int64_t)blockIdx.x * per);
    const int64_t uend = min(nunits, ubeg + per);
    XState carry = zero;
    int64_t carry_u = -1;
    for (int64_t u0 = ubeg; u0 < uend; u0 += U) {
      const int nu = (int)min((int64_t)U, uend - u0);
      // edges (lanes 0 and nu), then the bracketed inner lanes
      const int64_t gfirst = u0 / units_per_group, glast = (u0 + nu) / units_per_group;
      XState mine;
      if (lane == 0) mine = carry_u == u0 ? carry : start_state(u0, zero, inf);
      const XState e0 = shfl_state(mine, 0);
      if (lane == nu) {
        // bracket from the chunk's first state when in the same group
        const bool same = glast == gfirst && (u0 % units_per_group) != 0;
        XState hi = inf;
        if (same)
          hi.c[0] = e0.c[0] + (int64_t)nu * LY::XS;  // at most nu*XS more keys of A
        mine = start_state(u0 + lane, same ? e0 : zero, hi);
      }
      const XState e1 = shfl_state(mine, nu);
      carry = e1, carry_u = u0 + nu;
      if (lane > 0 && lane < nu) {
        const int64_t g = (u0 + lane) / units_per_group;
        mine = start_state(u0 + lane, g == gfirst ? e0 : zero, g == glast ? e1 : inf);
      }
      if (lane <= nu) cs[lane] = mine;
      __syncwarp();
      if (lane == 0) {
        for (int l = 0; l < nu; ++l) {
          const int64_t u = u0 + l;
          const int64_t g = u / units_per_group, k = u % units_per_group;
          int64_t off[5];
          geom(g, off);
          const XState s0 = cs[l];
          XState s1;
          if (k + 1 < units_per_group) {
            s1 = cs[l + 1];
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) s1.c[i] = off[i + 1] - off[i];
          }
          const int64_t xk = (s1.c[0] - s0.c[0]) + (s1.c[1] - s0.c[1]);
          const int64_t yk = (s1.c[2] - s0.c[2]) + (s1.c[3] - s0.c[3]);
          if (xk + yk == 0) continue;
          if (xk + yk <= LY::CAPT) {
            post(g, s0, s1);
            continue;
          }
          // an oversized unit: cut it at Y-side states every YM keys of Y
          const K* A = src + off[0];
          const K* B = src + off[1];
          const K* C = src + off[2];
          const K* D = src + off[3];
          const int64_t nc = off[3] - off[2], nd = off[4] - off[3];
          XState a = s0;
          const int64_t y0 = s0.c[2] + s0.c[3], y1 = s1.c[2] + s1.c[3];
          for (int64_t y = y0 + LY::YM; y < y1; y += LY::YM) {
            XState b;
            const int64_t lo = max(max(s0.c[2], y - s1.c[3]), a.c[2]);
            const int64_t hi = min(s1.c[2], y - s0.c[3]);
            const int64_t i = x_corank(C, D, y, lo, hi);
            const int64_t j = y - i;
            const K w = (i < nc && (j >= nd || !(D[j] < C[i]))) ? C[i] : D[j];
            b.c[2] = i, b.c[3] = j;
            b.c[0] = x_gallop<K, true>(A, a.c[0], s1.c[0], w);
            b.c[1] = x_gallop<K, true>(B, a.c[1], s1.c[1], w);
            post(g, a, b);
            a = b;
          }
          post(g, a, s1);
        }
      }
      __syncwarp();
    }
    if (lane == 0) {
      XState z{};
      post(-1, z, z);
    }
    (void)ctr;
  } else if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    int64_t k = 0;
    for (int64_t t = 0;; ++t) {
      const int r = (int)(t % RT);
      XT_BEGIN(t0);
      mbar_wait(&tfull[r], (uint32_t)((t / RT) & 1));
      if (lane == 0) XT_ADD(1, t0);
      const XTile d = ring[r];
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[r]);
      const int s = (int)(k % S);
      XT_BEGIN(t1);
      mbar_wait(&empty[s], (uint32_t)(((k / S) & 1) ^ 1));
      if (lane == 0) XT_ADD(2, t1);
      if (d.g < 0) {
        if (lane == 0) meta[s].out = -1;
        mbar_arrive(&full[s]);
        break;
      }
      K* sk = stg + (size_t)s * LY::stage_keys;
      XMeta m;
      int64_t pos = 0;
      const K* p[4];
      m.tot = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        p[i] = src + min(n, d.g * 4 * L + (int64_t)i * L) + d.s0.c[i];
        m.n[i] = (int)(d.s1.c[i] - d.s0.c[i]);
        m.tot += m.n[i];
        pos += d.s0.c[i];
      }
      m.out = d.g * 4 * L + pos;
      int o = 0;
      uint32_t tx = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        o = (o + EK - 1) / EK * EK + stage_offset(p[i]);
        m.off[i] = o;
        tx += window_bulk_bytes(p[i], m.n[i]);
        o += m.n[i];
      }
      if (lane == 0) {
        meta[s] = m;
        mbar_expect_tx(&full[s], tx);
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 4; ++i)
        stage_window(sk + m.off[i], p[i], m.n[i], &full[s], lane == 0, lane, 32);
      mbar_arrive(&full[s]);
      ++k;
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------ store warp
    if (lane == 0) {
      for (int64_t k = 0;; ++k) {
        const int s = (int)(k % S);
        XT_BEGIN(t0);
        mbar_wait(&outr[s], (uint32_t)((k / S) & 1));
        XT_ADD(4, t0);
        const XMeta m = meta[s];
        if (m.out < 0) break;
        K* sk = stg + (size_t)s * LY::stage_keys;
        K* g = dst + m.out;
        const int ph = stage_offset(g);
        int h, mid;
        window_split(g, m.tot, h, mid);
        if (mid) bulk_s2g(g + h, sk + ph + h, (uint32_t)(mid * sizeof(K)));
        bulk_commit();
        for (int i = 0; i < m.tot - mid; ++i) {
          const int j = i < h ? i : i + mid;
          g[j] = sk[ph + j];
        }
        bulk_wait_read<0>();
        mbar_arrive(&empty[s]);
      }
      bulk_wait_all();
    }
  } else {
    // ------------------------------------------------------------ mergers
    const int ct = threadIdx.x - 96;
    for (int64_t k = 0;; ++k) {
      const int s = (int)(k % S);
      XT_BEGIN(t0);
      mbar_wait(&full[s], (uint32_t)((k / S) & 1));
      if (ct == 0) XT_ADD(0, t0);
      const XMeta m = meta[s];
      if (m.out < 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&outr[s]);
        break;
      }
#ifdef MSORT_K3X_TRACE
      if (ct == 0) atomicAdd(&g_k3x_trace[(blockIdx.x & 1023) * 8 + 6], 1ull);
#endif
      K* sk = stg + (size_t)s * LY::stage_keys;
      K* xy = sk + LY::SIN;
      K key[VT];
      int pos[VT];
      const int nx = m.n[0] + m.n[1], ny = m.n[2] + m.n[3];
      const int t1 = (nx + VT - 1) / VT;
      {  // phase 1: X -> xy[0, nx), Y -> xy[nx, nx + ny)
        const bool n1 = ct < t1;
        const int d = n1 ? ct * VT : (ct - t1) * VT;
        const int kk = n1 ? nx : ny;
        if (d < kk) {
          const int oa = n1 ? m.off[0] : m.off[2], ca = n1 ? m.n[0] : m.n[2];
          const int ob = n1 ? m.off[1] : m.off[3], cb = n1 ? m.n[1] : m.n[3];
          const int i = merge_path<K, false>(sk, oa, ca, ob, cb, d);
          serial_merge_fast<K, false, VT>(sk, oa + i, oa + ca, ob + d - i, ob + cb, LY::SIN - 1,
                                          key, pos);
          K* o = xy + (n1 ? 0 : nx) + d;
          const int c = min(VT, kk - d);
#pragma unroll
          for (int j = 0; j < VT; ++j)
            if (j < c) o[j] = key[j];
        }
      }
      named_bar_sync(1, NC);
      {  // phase 2: merge(X, Y) over the consumed inputs
        const int d = ct * VT;
        if (d < m.tot) {
          const int i = merge_path<K, false>(xy, 0, nx, nx, ny, d);
          serial_merge_fast<K, false, VT>(xy, i, nx, nx + d - i, nx + ny, CAP - 1, key, pos);
          K* o = sk + stage_offset(dst + m.out) + d;
          const int c = min(VT, m.tot - d);
#pragma unroll
          for (int j = 0; j < VT; ++j)
            if (j < c) o[j] = key[j];
        }
      }
      fence_proxy_async_smem();
      named_bar_sync(1, NC);
      if (lane == 0) mbar_arrive(&outr[s]);
    }
    if (ct == 0) XT_ADD(5, tk);
  }
}

}  // namespace msort
