// k3q_merge.cuh -- K3Q: two merge levels in one HBM pass (keys only).
//
// A 2-way merge level moves every key through HBM twice (read + write), so
// a sort costs ~ (1 + levels) full passes.  K3Q merges four consecutive runs
// A, B, C, D (group g = runs 4g..4g+3 of length L) into one run of 4L in one
// pass: inside a CTA a three-node merge tree streams
//     node1: X = merge(A, B)   node2: Y = merge(C, D)   node3: out = merge(X, Y)
// through shared-memory rings (A..D filled by TMA bulk copies, X/Y written by
// node1/node2), so X and Y never touch HBM.  Every node is the stable merge()
// of P:107 with ties to the left input (R1), so the tree is the
// 4-way stable merge with ties in run order A < B < C < D -- i.e. the same
// result as two 2-way levels.
//
// Work: each group's output is cut into S segments at boundaries found by K2Q
// (regular sampling of the four runs, then lower/upper-bound searches and a
// rank-order fill of ties, as the distributed splitter D2 does); CTAs take
// segments from an atomic counter.  A segment is processed in steps:
//   phase A  node1 and node2 top X and Y up to XCAP keys (one combined batch of
//            <= Tm outputs; thread t merges VT outputs of one node from its
//            merge-path co-rank, searched in the rings);
//   phase B  node3 merges up to Tm outputs of X and Y into an output stage,
//            which the store warp writes back with a bulk copy.
// The producer warp refills A..D after each phase A and computes the exact
// consumption of each node (co-rank of the batch end, searched on the real
// keys).  Used-up inputs are followed by VT maximum-key sentinels, so the
// serial merges need no end checks (keys only: taking a sentinel on a tie
// with a real maximum key outputs the same value; consumption is not taken
// from the merge cursors but from the producer's exact searches).
#pragma once

#include "msort_device.cuh"

namespace msort {

struct QuadState {
  int64_t c[4];  // keys of runs A..D before the boundary
};

constexpr int kQuadMaxSeg = 32;    // segments per group (K2Q: one CTA per group)
constexpr int kQuadSamples = 1024;  // regular samples per group

// ------------------------------------------------------------------- K2Q
// Segment boundaries of one 4-way pass.  Group g's boundary k (0..S) is
// states[g*(S_full+1) + k]; 0 and S are the group's ends.  Boundary k aims at
// output diagonal d_k = k*|G|/S: its splitter v_k is the sample of rank
// k*ns/S among ns regular samples (proportional to run sizes); the state is
// lb_i(v_k) (keys < v_k) for every run, plus keys equal to v_k taken in run
// order up to d_k, clamped to [lb, ub] -- monotone in k, so segments tile the
// output exactly; their sizes are near |G|/S for any data (ties included).
template <class K>
__global__ void __launch_bounds__(256)
    k2q_partition(const K* __restrict__ src, int64_t n, int64_t L, int S_full, int S_last,
                  int64_t ngroups, QuadState* __restrict__ states) {
  __shared__ K smp[kQuadSamples];
  __shared__ int64_t bnd[kQuadMaxSeg][8];
  const int64_t g = blockIdx.x;
  const int S = g == ngroups - 1 ? S_last : S_full;
  QuadState* out = states + g * (S_full + 1);
  int64_t off[5], m[4], tot = 0;
#pragma unroll
  for (int i = 0; i <= 4; ++i) off[i] = min(n, g * 4 * L + (int64_t)i * L);
#pragma unroll
  for (int i = 0; i < 4; ++i) m[i] = off[i + 1] - off[i], tot += m[i];
  const int tid = threadIdx.x;
  if (tid == 0) {
    QuadState z, e;
#pragma unroll
    for (int i = 0; i < 4; ++i) z.c[i] = 0, e.c[i] = m[i];
    out[0] = z;
    out[S] = e;
  }
  if (S <= 1) return;
  int ns[4], nsum = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) ns[i] = (int)((kQuadSamples * m[i]) / tot), nsum += ns[i];
  for (int j = tid; j < kQuadSamples; j += 256) {
    int i = 0, jj = j;
    while (i < 4 && jj >= ns[i]) jj -= ns[i], ++i;
    K v = KeyTraits<K>::max_key();
    if (i < 4) v = src[off[i] + ((2 * (int64_t)jj + 1) * m[i]) / (2 * (int64_t)ns[i])];
    smp[j] = v;
  }
  __syncthreads();
  for (int k = 2; k <= kQuadSamples; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < kQuadSamples; i += 256) {
        const int l = i ^ j;
        if (l > i) {
          const K a = smp[i], b = smp[l];
          if ((a > b) == ((i & k) == 0)) smp[i] = b, smp[l] = a;
        }
      }
      __syncthreads();
    }
  for (int q = tid; q < (S - 1) * 8; q += 256) {
    const int k = q / 8 + 1, s = q % 8, i = s >> 1;
    const bool upper = s & 1;
    const K v = smp[(int)(((int64_t)k * nsum) / S)];
    const K* r = src + off[i];
    int64_t lo = 0, hi = m[i];
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (upper ? !(v < r[mid]) : (r[mid] < v)) lo = mid + 1;
      else hi = mid;
    }
    bnd[k][s] = lo;
  }
  __syncthreads();
  for (int k = 1 + tid; k < S; k += 256) {
    const int64_t d = (tot * k) / S;
    int64_t lb = 0, ub = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) lb += bnd[k][2 * i], ub += bnd[k][2 * i + 1];
    QuadState st;
    int64_t rem = d < lb ? 0 : (d > ub ? ub - lb : d - lb);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t eq = bnd[k][2 * i + 1] - bnd[k][2 * i];
      const int64_t take = rem < eq ? rem : eq;
      st.c[i] = bnd[k][2 * i] + take;
      rem -= take;
    }
    out[k] = st;
  }
}

// ------------------------------------------------------------------- K3Q
constexpr int pow2_ceil(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}
template <class K, int NT, int VT>
struct QuadLayout {
  static constexpr int Z = sizeof(K);
  static constexpr int Tm = NT * VT;                  // outputs per phase (max)
  static constexpr int CAP = Tm - VT - 2;             // phase-A batch cap (keeps one thread free)
  static constexpr int XCAP = Tm - VT - 2;            // X / Y fill target
  // input rings: a phase A reads <= CAP + 1 past the consumed point and may
  // run on the refill of the step before last (<= 2 CAP + VT + 2 ahead)
  static constexpr int R = pow2_ceil(2 * CAP + 2 * VT + 4);
  static constexpr uint32_t RB = (uint32_t)R * Z;     // input ring bytes
  static constexpr uint32_t MASK = RB - 1;
  // X / Y rings hold <= XCAP keys + VT sentinels
  static constexpr int RX = pow2_ceil(XCAP + VT + 1);
  static constexpr uint32_t RXB = (uint32_t)RX * Z;
  static constexpr uint32_t XMASK = RXB - 1;
  static constexpr int EK = 16 / Z;
  static constexpr int SK = Tm + 2 * EK;              // keys per output stage
  static constexpr uint32_t ringx = 4 * RB;           // A, B, C, D, then X, Y
  static constexpr uint32_t stage = 4 * RB + 2 * RXB;
  static constexpr uint32_t stage_bytes = (uint32_t)((SK * Z + 127) / 128 * 128);
  static constexpr uint32_t misc = stage + 2 * stage_bytes;
  static constexpr uint32_t bytes = misc + 256;
};

// Shared control block of a K3Q CTA.
struct QuadCtl {
  uint64_t ld_bar[2];    // refills (alternating): producer lanes' cp.async + bulk tx
  uint64_t full[2];      // output stage written (mergers -> store warp)
  uint64_t empty[2];     // output stage read (store warp -> mergers)
  int64_t seg;           // current segment (-1: no more)
  int64_t s0[4], s1[4];  // its boundary states
  int nA[4];             // consumption of A..D by the coming phase A (producer)
  int nx3;               // X consumed by the coming phase B (producer)
  int64_t meta_out[2];   // stage s: absolute output index of its first key
  int meta_cnt[2];
};

// Global -> shared copy of 4 or 8 bytes (cp.async, SASS LDGSTS): the head and
// tail of a window that the 16-byte bulk copy cannot move.
template <class T>
__device__ __forceinline__ void cp_async_elem(T* dst, const T* src) {
  if constexpr (sizeof(T) == 4)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src)
                 : "memory");
}
// This thread's arrival on `bar` fires when its earlier cp.async copies land.
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// Stage src[0, cnt) at dst (same 16-byte phase): the 16-byte aligned middle
// by one bulk copy (lane 0), head and tail by per-lane cp.async; nothing
// blocks.  Completion: tx bytes + each lane's arrive.noinc on `bar`.
template <class T>
__device__ __forceinline__ void stage_async(T* dst, const T* src, int cnt, uint64_t* bar,
                                            int lane) {
  int head, mid;
  window_split(src, cnt, head, mid);
  if (lane == 0 && mid > 0) bulk_g2s(dst + head, src + head, (uint32_t)(mid * sizeof(T)), bar);
  for (int i = lane; i < cnt - mid; i += 32) {
    const int j = i < head ? i : i + mid;
    cp_async_elem(dst + j, src + j);
  }
}

template <class K>
__device__ __forceinline__ K ldsK(const char* sb, uint32_t off) {
  return *reinterpret_cast<const K*>(sb + off);
}

// Co-rank (merge path, ties to A) of diagonal d of merge(A, B), A = na keys
// of ring (ba, oa), B = nb keys of ring (bb, ob); ring offsets wrap at MASK.
template <class K, uint32_t MASK>
__device__ __forceinline__ int corank_rings(const char* sb, uint32_t ba, uint32_t oa, int na,
                                            uint32_t bb, uint32_t ob, int nb, int d) {
  constexpr uint32_t Z = sizeof(K);
  int lo = d - nb > 0 ? d - nb : 0;
  int hi = d < na ? d : na;
  const uint32_t obd = ob + (uint32_t)(d - 1) * Z;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const uint32_t mz = (uint32_t)mid * Z;
    if (ldsK<K>(sb, ba + ((oa + mz) & MASK)) > ldsK<K>(sb, bb + ((obd - mz) & MASK))) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// VT outputs of merge(A, B) from ring cursors (oa, ob): no end checks (used
// up inputs are followed by maximum-key sentinels).
template <class K, int VT, uint32_t MASK>
__device__ __forceinline__ void merge_rings(const char* sb, uint32_t ba, uint32_t oa, uint32_t bb,
                                            uint32_t ob, K (&key)[VT]) {
  constexpr uint32_t Z = sizeof(K);
  K ak = ldsK<K>(sb, ba + oa), bk = ldsK<K>(sb, bb + ob);
#pragma unroll
  for (int k = 0; k < VT; ++k) {
    const bool p = bk < ak;
    key[k] = p ? bk : ak;
    if (k + 1 < VT) {
      const uint32_t nx = ((p ? ob : oa) + Z) & MASK;
      const K nv = ldsK<K>(sb, (p ? bb : ba) + nx);
      oa = p ? oa : nx;
      ob = p ? nx : ob;
      ak = p ? ak : nv;
      bk = p ? nv : bk;
    }
  }
}

template <class K, int NT, int VT>
__global__ void __launch_bounds__(NT + 64)
    k3q_pass(const K* __restrict__ src, K* __restrict__ dst, int64_t n, int64_t L, int S_full,
             int64_t nseg, const QuadState* __restrict__ states,
             unsigned long long* __restrict__ ctr) {
  using LY = QuadLayout<K, NT, VT>;
  constexpr uint32_t Z = sizeof(K), MASK = LY::MASK, RB = LY::RB, XMASK = LY::XMASK;
  constexpr int Tm = LY::Tm;
  extern __shared__ __align__(16) unsigned char smem[];
  const char* sb = reinterpret_cast<const char*>(smem);
  K* stk = reinterpret_cast<K*>(smem + LY::stage);
  QuadCtl& C = *reinterpret_cast<QuadCtl*>(smem + LY::misc);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // rings A B C D (RB bytes, MASK) then X Y (RXB bytes, XMASK)
  auto rb = [](int i) { return i < 4 ? (uint32_t)i * RB : LY::ringx + (uint32_t)(i - 4) * LY::RXB; };
  auto put = [&](int ring, uint32_t off, K v) {
    *reinterpret_cast<K*>(smem + rb(ring) + (off & (ring < 4 ? MASK : XMASK))) = v;
  };
  constexpr int BAR_MP = 1;  // named barrier: mergers + producer
  if (threadIdx.x == 0) {
    mbar_init(&C.ld_bar[0], 32), mbar_init(&C.ld_bar[1], 32);
    mbar_init(&C.full[0], NT / 32), mbar_init(&C.full[1], NT / 32);
    mbar_init(&C.empty[0], 1), mbar_init(&C.empty[1], 1);
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 1) {
    // ------------------------------------------------------------ store warp
    if (lane == 0) {
      for (int64_t k = 0;; ++k) {
        const int s = (int)(k & 1);
        mbar_wait(&C.full[s], (uint32_t)((k >> 1) & 1));
        const int cnt = C.meta_cnt[s];
        if (cnt < 0) break;
        K* g = dst + C.meta_out[s];
        const K* st = stk + (size_t)s * LY::SK + stage_offset(g);
        int h, mid;
        window_split(g, cnt, h, mid);
        if (mid) bulk_s2g(g + h, st + h, (uint32_t)mid * Z);
        bulk_commit();
        for (int i = 0; i < cnt - mid; ++i) {
          const int j = i < h ? i : i + mid;
          g[j] = st[j];
        }
        bulk_wait_read<0>();
        mbar_arrive(&C.empty[s]);
      }
      bulk_wait_all();
    }
    return;
  }

  const bool prod = warp == 0;
  const int mt = threadIdx.x - 64;  // merger thread 0..NT-1
  int64_t step = 0;                 // steps so far (output stage ring)
  int64_t nref = 0;                 // producer: refills issued (ld_bar[id & 1])
  int loaded[4];                    // producer: keys of each run loaded (end + 1: + sentinels)

  auto wait_refill = [&](int64_t id) {
    mbar_wait(&C.ld_bar[id & 1], (uint32_t)((id >> 1) & 1));
  };

  for (;;) {
    // ---------------------------------------------------- segment set-up
    if (prod && lane == 0) {
      const int64_t sg = (int64_t)atomicAdd(ctr, 1ull);
      C.seg = sg < nseg ? sg : -1;
      if (sg < nseg) {
        const int64_t g = sg / S_full, k = sg % S_full;
        const QuadState a = states[g * (S_full + 1) + k], b = states[g * (S_full + 1) + k + 1];
#pragma unroll
        for (int i = 0; i < 4; ++i) C.s0[i] = a.c[i], C.s1[i] = b.c[i];
      }
    }
    named_bar_sync(BAR_MP, NT + 32);
    const int64_t seg = C.seg;
    if (seg < 0) break;
    // the segment's state, replicated in every thread's registers
    const int64_t gbase = (seg / S_full) * 4 * L;
    const K* run[4];
    uint32_t ph[4];  // ring byte offset of each run's first segment key
    int end[4], cons[4];
    int64_t out_pos = gbase, out_end = gbase;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      run[i] = src + min(n, gbase + (int64_t)i * L) + C.s0[i];
      ph[i] = (uint32_t)((uintptr_t)run[i]) & MASK;
      end[i] = (int)(C.s1[i] - C.s0[i]);
      cons[i] = 0;
      out_pos += C.s0[i], out_end += C.s1[i];
    }
    int xp = 0, xc = 0, yp = 0, yc = 0;

    // Producer: load run i up to min(end, cons + R - VT - 1) (ring room for
    // the sentinels) and write VT sentinels once the segment's end is in.
    auto refill = [&]() {
      uint64_t* bar = &C.ld_bar[nref & 1];
      uint32_t tx = 0;
      int from[4], cnt[4], p1[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        from[i] = loaded[i];
        const int to = max(from[i], min(end[i], cons[i] + LY::R - VT - 1));
        cnt[i] = to - from[i];
        const uint32_t o0 = (ph[i] + (uint32_t)from[i] * Z) & MASK;
        p1[i] = min(cnt[i], (int)((RB - o0) / Z));
        tx += window_bulk_bytes(run[i] + from[i], p1[i]) +
              window_bulk_bytes(run[i] + from[i] + p1[i], cnt[i] - p1[i]);
      }
      if (lane == 0) mbar_expect_tx(bar, tx);
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t o0 = (ph[i] + (uint32_t)from[i] * Z) & MASK;
        K* r = reinterpret_cast<K*>(smem + rb(i));
        stage_async(r + o0 / Z, run[i] + from[i], p1[i], bar, lane);
        if (cnt[i] > p1[i])
          stage_async(r, run[i] + from[i] + p1[i], cnt[i] - p1[i], bar, lane);
        loaded[i] = from[i] + cnt[i];
        if (loaded[i] == end[i]) {
          for (int j = lane; j < VT; j += 32)
            put(i, ph[i] + (uint32_t)(end[i] + j) * Z, KeyTraits<K>::max_key());
          loaded[i] = end[i] + 1;
        }
      }
      cp_async_arrive_noinc(bar);
      ++nref;
    };

    if (prod) {
#pragma unroll
      for (int i = 0; i < 4; ++i) loaded[i] = 0;
      refill();
      // an empty input pair: its node's output is sentinels from the start
      for (int j = lane; j < VT; j += 32) {
        if (end[0] + end[1] == 0) put(4, (uint32_t)j * Z, KeyTraits<K>::max_key());
        if (end[2] + end[3] == 0) put(5, (uint32_t)j * Z, KeyTraits<K>::max_key());
      }
      wait_refill(nref - 1);
    }
    named_bar_sync(BAR_MP, NT + 32);

    // ----------------------------------------------------------- steps
    while (out_pos < out_end) {
      // phase A: node1 / node2 top X and Y up to XCAP keys
      const int abrem = (end[0] - cons[0]) + (end[1] - cons[1]);
      const int cdrem = (end[2] - cons[2]) + (end[3] - cons[3]);
      int kA = max(0, min(LY::XCAP - (xp - xc), abrem));
      int kC = max(0, min(LY::XCAP - (yp - yc), cdrem));
      if (kA + kC > LY::CAP) {
        kA = min(kA, LY::CAP - min(kC, LY::CAP / 2));
        kC = min(kC, LY::CAP - kA);
      }
      if (prod) {
        if (lane < 2) {  // exact consumption of the batch: co-rank of its end
          const bool n1 = lane == 0;
          const int k = n1 ? kA : kC;
          const uint32_t oa = n1 ? (ph[0] + (uint32_t)cons[0] * Z) & MASK
                                 : (ph[2] + (uint32_t)cons[2] * Z) & MASK;
          const uint32_t ob = n1 ? (ph[1] + (uint32_t)cons[1] * Z) & MASK
                                 : (ph[3] + (uint32_t)cons[3] * Z) & MASK;
          const int na = n1 ? end[0] - cons[0] : end[2] - cons[2];
          const int nb = n1 ? end[1] - cons[1] : end[3] - cons[3];
          const int c = corank_rings<K, MASK>(sb, n1 ? rb(0) : rb(2), oa, na,
                                              n1 ? rb(1) : rb(3), ob, nb, k);
          C.nA[2 * lane] = c, C.nA[2 * lane + 1] = k - c;
        }
      } else {
        const int tA = (kA + VT - 1) / VT;
        const bool n1 = mt < tA;
        const int d = n1 ? mt * VT : (mt - tA) * VT;
        const int kk = n1 ? kA : kC;
        if (d < kk) {
          // (register arrays indexed by constants only: select the node's pair)
          const uint32_t ra = n1 ? rb(0) : rb(2), rbb = n1 ? rb(1) : rb(3);
          const uint32_t oa = n1 ? (ph[0] + (uint32_t)cons[0] * Z) & MASK
                                 : (ph[2] + (uint32_t)cons[2] * Z) & MASK;
          const uint32_t ob = n1 ? (ph[1] + (uint32_t)cons[1] * Z) & MASK
                                 : (ph[3] + (uint32_t)cons[3] * Z) & MASK;
          const int na = n1 ? end[0] - cons[0] : end[2] - cons[2];
          const int nb = n1 ? end[1] - cons[1] : end[3] - cons[3];
          const int c = corank_rings<K, MASK>(sb, ra, oa, na, rbb, ob, nb, d);
          K key[VT];
          merge_rings<K, VT, MASK>(sb, ra, (oa + (uint32_t)c * Z) & MASK, rbb,
                                   (ob + (uint32_t)(d - c) * Z) & MASK, key);
          const int ring = n1 ? 4 : 5;
          const uint32_t base = (uint32_t)((n1 ? xp : yp) + d) * Z;
          const int cnt = min(VT, kk - d);
#pragma unroll
          for (int j = 0; j < VT; ++j)
            if (j < cnt) put(ring, base + (uint32_t)j * Z, key[j]);
          // the batch that uses the node's inputs up appends its sentinels
          if (d + cnt == kk && kk == (n1 ? abrem : cdrem))
#pragma unroll
            for (int j = 0; j < VT; ++j)
              put(ring, base + (uint32_t)(cnt + j) * Z, KeyTraits<K>::max_key());
        }
      }
      named_bar_sync(BAR_MP, NT + 32);  // phase A done
#pragma unroll
      for (int i = 0; i < 4; ++i) cons[i] += C.nA[i];
      const bool abdone = kA == abrem, cddone = kC == cdrem;
      xp += kA, yp += kC;
      const int xav = xp - xc, yav = yp - yc;
      int k3 = (int)min((int64_t)Tm, out_end - out_pos);
      if (!abdone) k3 = min(k3, xav - 1);
      if (!cddone) k3 = min(k3, yav - 1);
      k3 = max(k3, 0);
      const int s = (int)(step & 1);
      if (prod) {
        refill();  // ring room freed by phase A
        wait_refill(nref - 2);  // the next phase A may read up to the previous refill
      } else {
        // phase B: node3 merges X and Y into output stage s
        if (step >= 2) mbar_wait(&C.empty[s], (uint32_t)(((step >> 1) - 1) & 1));
        const int d = mt * VT;
        K* st = stk + (size_t)s * LY::SK + stage_offset(dst + out_pos);
        if (d < k3) {
          const uint32_t ox = ((uint32_t)xc * Z) & XMASK, oy = ((uint32_t)yc * Z) & XMASK;
          const int c = corank_rings<K, XMASK>(sb, rb(4), ox, xav, rb(5), oy, yav, d);
          K key[VT];
          merge_rings<K, VT, XMASK>(sb, rb(4), (ox + (uint32_t)c * Z) & XMASK, rb(5),
                                    (oy + (uint32_t)(d - c) * Z) & XMASK, key);
          const int cnt = min(VT, k3 - d);
#pragma unroll
          for (int j = 0; j < VT; ++j)
            if (j < cnt) st[d + j] = key[j];
        }
        // X consumed by this batch: the last merger thread is idle in phase B
        // (k3 <= Tm - VT - 3), so it searches the batch end's co-rank
        if (mt == NT - 1)
          C.nx3 = corank_rings<K, XMASK>(sb, rb(4), ((uint32_t)xc * Z) & XMASK, xav, rb(5),
                                         ((uint32_t)yc * Z) & XMASK, yav, k3);
        fence_proxy_async_smem();
        if (mt == 0) C.meta_out[s] = out_pos, C.meta_cnt[s] = k3;
      }
      named_bar_sync(BAR_MP, NT + 32);  // phase B done
      if (!prod && lane == 0) mbar_arrive(&C.full[s]);
      const int nx3 = C.nx3;
      xc += nx3, yc += k3 - nx3;
      out_pos += k3;
      ++step;
    }
    if (prod) wait_refill(nref - 1);  // rings are reused by the next segment
    named_bar_sync(BAR_MP, NT + 32);
  }
  // stop the store warp
  if (!prod) {
    const int s = (int)(step & 1);
    if (mt == 0) {
      if (step >= 2) mbar_wait(&C.empty[s], (uint32_t)(((step >> 1) - 1) & 1));
      C.meta_cnt[s] = -1;
    }
    named_bar_sync(2, NT);
    if (lane == 0) mbar_arrive(&C.full[s]);
  }
}

}  // namespace msort
