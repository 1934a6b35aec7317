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
//   2. log2(CL) merge levels ACROSS the cluster: the level's runs are the
//      concatenations of 2^l consecutive chunks, read from the other CTAs'
//      shared memory (DSMEM, distributed shared memory); each CTA produces
//      its own Q outputs -- the merge-path co-ranks of its first and last
//      diagonal by 32-ary warp searches over DSMEM, the two windows copied
//      into local shared memory, a per-thread merge -- and a cluster barrier
//      separates the levels.  The last level writes the output to HBM.
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
}
#else
__device__ __forceinline__ void k0_mark(int) {}
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

// Grid = CL CTAs forming one cluster (CL = 1: a single CTA, no cluster).
// Shared memory: three padded buffers of kK0Chunk keys (two ping-pong, one
// scratch).  SHFL: each warp first sorts its 32 x 16 keys with the
// warp-shuffle bitonic network (warp_bitonic_keys), so the shared-memory
// merge rounds start from runs of 512; otherwise (the A/B variant) every
// thread sorts its 16 keys in registers and the rounds start from 16.
template <class K, bool SHFL>
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
  // ---- 2. merge levels across the cluster (DSMEM)
  cg::cluster_group cluster = cg::this_cluster();
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
