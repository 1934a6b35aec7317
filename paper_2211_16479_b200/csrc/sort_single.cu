// sort_single.cu -- single-GPU stable merge sort for sm_100a.
//
//   K1 k1_tile_sort   : each T-element tile sorted in registers + shared
//                       memory: the base case of the recursion, the
//                       chunk sort of the multiprocessing variant;
//                       T plays `SMALLEST_ARRAY_SIZE` (reading R17).
//   K3 k3_merge_pass  : one persistent, warp-specialised kernel per merge
//                       level: merges run pairs of length L into 2L with the
//                       stable merge() of P:107 (ties to the left run, R1).
//                       Warp 0 stages windows with TMA bulk copies
//                       (cp.async.bulk + mbarrier), warp 1 computes the
//                       merge-path co-ranks (K2) of the CTA's tiles ahead of
//                       use, warps 2.. merge from shared memory and write
//                       through a shared buffer with TMA bulk stores.
//   S4 placement      : K1's destination is picked from the parity of the
//                       merge-pass count so that the last pass lands in keys.
//
// "P:n" = /root/reference/PAPER.md line n.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "k3_merge.cuh"
#include "msort_device.cuh"
#include "networks.cuh"
#include "msort_internal.h"
#include "seg_sort.cuh"

namespace msort {

// VT outputs of the stable merge of A (from ai) and B (from bi) in s, ties to
// A, with the in-tile index of each output gathered through src_idx; no end
// checks -- the caller guarantees neither run ends within VT steps.
template <class K, int VT>
__device__ __forceinline__ void merge_pairs_nocheck(const K* s, const int* src_idx, int ai, int bi,
                                                    K (&key)[VT], int (&idx)[VT]) {
  K ak = s[ai], bk = s[bi];
#pragma unroll
  for (int k = 0; k < VT; ++k) {
    const bool takeB = bk < ak;
    key[k] = takeB ? bk : ak;
    idx[k] = src_idx[takeB ? bi : ai];
    ai += takeB ? 0 : 1;
    bi += takeB ? 1 : 0;
    if (k + 1 < VT) {
      const K nv = s[takeB ? bi : ai];
      ak = takeB ? ak : nv;
      bk = takeB ? nv : bk;
    }
  }
}

// A K1 input key: KW == K, or (the key-range narrowed sort, sort_narrowed)
// an 8-byte key narrowed on the fly to its offset from the range minimum mm[0].
template <class K, class KW>
__device__ __forceinline__ K k1_in(const KW* p, const unsigned long long* mm) {
  if constexpr (std::is_same<K, KW>::value) return *p;
  else return (K)(KeyTraits<KW>::image(*p) - mm[0]);
}

// ----------------------------------------------------------------- K1
// NT threads x VT items (VT odd: "blocked" shared accesses at stride VT are
// bank-conflict free without padding).  KW: the input key type (see k1_in).
template <class K, bool PAIRS, int NT, int VT, class KW = K>
__global__ void __launch_bounds__(NT)
    k1_tile_sort(const KW* __restrict__ in_k, const uint32_t* __restrict__ in_v,
                 K* __restrict__ out_k, uint32_t* __restrict__ out_v, int64_t n,
                 const int64_t* __restrict__ seg, const unsigned long long* __restrict__ gate = nullptr,
                 int gate_want = 0) {
  if (gate && (int)range_narrow(gate) != gate_want) return;  // key-range gate (sort_narrowed)
  constexpr int T = NT * VT;
  extern __shared__ __align__(16) unsigned char smem[];
  K* sk = reinterpret_cast<K*>(smem);                 // T keys
  int* si = reinterpret_cast<int*>(sk + T);           // PAIRS: original in-tile index
  uint32_t* sv = reinterpret_cast<uint32_t*>(si + T);  // PAIRS: payload staging

  const int tid = threadIdx.x;
  // tile blockIdx.x of the array, or (segmented sorts, seg_sort.cuh) the
  // segment of descriptor blockIdx.x: (offset, length <= T)
  const int64_t base = seg ? seg[2 * blockIdx.x] : (int64_t)blockIdx.x * T;
  const int cnt = seg ? (int)seg[2 * blockIdx.x + 1] : (int)min((int64_t)T, n - base);

  K key[VT];
  int idx[VT];
  if constexpr (PAIRS) {
    // Load the tile; pad the partial last tile with the maximum key AFTER the
    // real elements, so the stable order keeps real keys first.
#pragma unroll 4
    for (int i = tid; i < T; i += NT) {
      sk[i] = i < cnt ? k1_in<K>(in_k + base + i, gate) : KeyTraits<K>::max_key();
      if (i < cnt) sv[i] = in_v[base + i];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < VT; ++k) {
      key[k] = sk[tid * VT + k];
      idx[k] = tid * VT + k;
    }
  } else {
    // Keys only: which thread holds which key before the network does not
    // matter (equal keys are indistinguishable), so load straight into
    // registers, striped (coalesced), padding with the maximum key.
#pragma unroll
    for (int k = 0; k < VT; ++k) {
      const int i = k * NT + tid;
      key[k] = i < cnt ? k1_in<K>(in_k + base + i, gate) : KeyTraits<K>::max_key();
    }
  }
  // Per-thread register network.
  if constexpr (PAIRS) odd_even_transposition_sort<VT>(key, idx);
  else keys_network<VT>(key);

  // In-block merge rounds: runs of w -> 2w, merge path per thread.
  // While a merge group (2w outputs, 2w/VT threads) fits in one warp the
  // round needs only warp-level synchronisation.
#pragma unroll 1
  for (int w = VT; w < T; w *= 2) {
    const bool in_warp = 2 * w <= 32 * VT;
    if (in_warp) __syncwarp();
    else __syncthreads();
#pragma unroll
    for (int k = 0; k < VT; ++k) {
      sk[tid * VT + k] = key[k];
      if constexpr (PAIRS) si[tid * VT + k] = idx[k];
    }
    if (in_warp) __syncwarp();
    else __syncthreads();
    const int tpg = 2 * w / VT;  // threads per merge group
    const int g0 = (tid / tpg) * 2 * w;
    const int d = (tid % tpg) * VT;
    if constexpr (!PAIRS) {
      constexpr uint32_t Z = sizeof(K);
      const char* sb = reinterpret_cast<const char*>(sk);
      const uint32_t oa0 = (uint32_t)g0 * Z, ob0 = oa0 + (uint32_t)w * Z;
      const int i = merge_path_off<K>(sb, oa0, w, ob0, w, d);
      const uint32_t oa = oa0 + (uint32_t)i * Z, ob = ob0 + (uint32_t)(d - i) * Z;
      const uint32_t ea = ob0, eb = ob0 + (uint32_t)w * Z;
      if (__all_sync(0xffffffffu, oa + VT * Z <= ea && ob + VT * Z <= eb))
        merge_keys_nocheck<K, VT>(sb, oa, ob, key);
      else
        merge_keys_checked<K, VT>(sb, oa, ea, ob, eb, (uint32_t)(T - 1) * Z, key);
      continue;
    }
    int i = merge_path<K, false>(sk, g0, w, g0 + w, w, d);
    if constexpr (PAIRS) {
      const int ai = g0 + i, bi = g0 + w + d - i;
      // check-free steps when no lane's run can end within VT outputs (the
      // common case), else the checked merge
      if (__all_sync(0xffffffffu, ai + VT <= g0 + w && bi + VT <= g0 + 2 * w))
        merge_pairs_nocheck<K, VT>(sk, si, ai, bi, key, idx);
      else
        serial_merge<K, false, true, VT>(sk, si, ai, g0 + w, bi, g0 + 2 * w, T - 1, key, idx);
    } else {
      serial_merge_fast<K, false, VT>(sk, g0 + i, g0 + w, g0 + w + d - i, g0 + 2 * w, T - 1,
                                      key, idx);
    }
  }

  __syncthreads();
#pragma unroll
  for (int k = 0; k < VT; ++k) {
    sk[tid * VT + k] = key[k];
    if constexpr (PAIRS) si[tid * VT + k] = idx[k];
  }
  __syncthreads();
#pragma unroll 4
  for (int i = tid; i < cnt; i += NT) {
    out_k[base + i] = sk[i];
    if constexpr (PAIRS) out_v[base + i] = sv[si[i]];
  }
}

// Keys-only K1.  Each thread sorts VT keys in registers (k1_network: Batcher's
// merge-exchange network, networks.cuh), then log2(NT) merge-path rounds in
// shared memory double the runs.  In round r (runs of w = VT << r) pair
// m = (run 2m = A, run 2m+1 = B) is laid out as
//     [ B (w) | pad | A (w) | pad ]        (K1Layout, in 16-byte vectors)
// with a MAX key right after each run and a MIN key right before it, so a run
// that is used up reads as its sentinel and the merges (merge_keys_dual) need
// no end checks: no thread diverges.  (With equal keys indistinguishable, a
// sentinel that ties with a real MIN / MAX key outputs the right value; the
// cursor that could step over its sentinel on such a tie is clamped.)  Every
// run starts 16-byte aligned, so a thread's VT keys leave as 16-byte vector
// stores (store_vec), and the paddings keep those stores free of bank
// conflicts.  Rounds whose merge groups fit in a warp use a per-warp region
// and only warp synchronisation.
//
// The same VT outputs as two independent chains of VT/2 (twice the loads in
// flight per thread): the front chain from the co-rank at the thread's first
// diagonal (oa, ob) upwards, ties to A, A clamped at its MAX sentinel ea; the
// back chain from the co-rank at its last diagonal (oa1, ob1 = one past the
// last elements) downwards, taking the LAST of equal keys (B's), B clamped at
// its MIN sentinel bmin (each run has a MIN key in front of it, K1Layout).
template <class K, int VT>
__device__ __forceinline__ void merge_keys_dual(const char* s, uint32_t oa, uint32_t ea,
                                                uint32_t ob, uint32_t oa1, uint32_t ob1,
                                                uint32_t bmin, K (&key)[VT]) {
  static_assert(VT % 2 == 0, "two chains of VT/2");
  constexpr int H = VT / 2;
  constexpr uint32_t Z = sizeof(K);
  uint32_t pa = oa1 - Z, pb = ob1 - Z;
  K ak = ld_off<K>(s, oa), bk = ld_off<K>(s, ob);
  K ax = ld_off<K>(s, pa), bx = ld_off<K>(s, pb);
#pragma unroll
  for (int k = 0; k < H; ++k) {
    const bool p = bk < ak;
    key[k] = p ? bk : ak;
    const bool q = ax > bx;
    key[VT - 1 - k] = q ? ax : bx;
    if (k + 1 < H) {
      const uint32_t nx = min((p ? ob : oa) + Z, ea);  // B lies below ea
      oa = p ? oa : nx;
      ob = p ? nx : ob;
      const uint32_t ny = max((q ? pa : pb) - Z, bmin);  // A lies above bmin
      pa = q ? ny : pa;
      pb = q ? pb : ny;
      const K nv = ld_off<K>(s, nx);
      const K nw = ld_off<K>(s, ny);
      ak = p ? ak : nv;
      bk = p ? nv : bk;
      ax = q ? nw : ax;
      bx = q ? bx : nw;
    }
  }
}

// VT keys of a thread stored as 16-byte vectors (4 x 32-bit or 2 x 64-bit
// keys; VT a multiple of the width, dst 16-byte aligned).  A thread's run
// starts every VT keys, i.e. 4*VT bytes apart for int32: with VT = 68 that is
// 17 vector slots, odd, so the 8 lanes of each quarter-warp phase hit 8
// different slot groups -- conflict-free (2-key vectors would be 2-way).
template <class K>
struct VecOf {
  static constexpr int W = 16 / sizeof(K);
};
template <class K, int W>
struct __align__(16) KVec {
  K x[W];
};
template <class K, int VT>
__device__ __forceinline__ void store_vec(K* dst, const K (&key)[VT]) {
  constexpr int W = VecOf<K>::W;
  static_assert(VT % W == 0, "VT: multiple of the 16-byte vector width");
#pragma unroll
  for (int k = 0; k < VT; k += W) {
    KVec<K, W> v;
#pragma unroll
    for (int j = 0; j < W; ++j) v.x[j] = key[k + j];
    *reinterpret_cast<KVec<K, W>*>(dst + k) = v;
  }
}

}  // namespace msort
#include "k6_quad.cuh"
#include "k5_kway.cuh"
#include "k0_small.cuh"
namespace msort {

// Compare-exchange of the keys-only register network (min and max; any
// network is fine for keys only -- equal integers are indistinguishable).
struct CmpSwapKeys {
  template <class K>
  __device__ __forceinline__ void operator()(K& a, K& b, int) const {
    const K lo = a < b ? a : b, hi = a < b ? b : a;
    a = lo;
    b = hi;
  }
};

template <int VT, class K>
__device__ __forceinline__ void k1_network(K (&key)[VT]) {
  if constexpr (MergeExchange<VT>::kHave)
    MergeExchange<VT>::run(key, CmpSwapKeys{});
  else
    keys_network<VT>(key);
}

// Round-r pair layout of the keys-only K1 in 16-byte vectors (V = vectors per
// thread).  Pair m of a region starts at start(r, m) with its B run, A follows
// at start + aoff(r); each run is followed by >= 1 vector of MAX sentinels.
// The paddings are chosen so that the 8 lanes of every quarter-warp store
// their V-vector runs into 8 different bank groups when V = 1 mod 8 (V = 17:
// 68 int32 / 34 int64 keys per thread): the thread runs start V apart, so
// only the run / pair boundaries can collide -- round 0 staggers the pairs
// (stride 2V+2, +1 every second pair), round 1 alternates strides 4V+6 and
// 4V+4 with A at 2V+2, round 2 puts A at 4V+8 (a bank group half a turn from B); from round
// 3 on a quarter-warp lies inside one run.
struct K1Layout {
  template <int V>
  static constexpr __host__ __device__ int start(int r, int m) {
    return r == 0 ? (2 * V + 2) * m + (m >> 1)
         : r == 1 ? (4 * V + 5) * m + (m & 1)
         : r == 2 ? (8 * V + 9) * m
                  : ((2 * V << r) + 2) * m;
  }
  template <int V>
  static constexpr __host__ __device__ int aoff(int r) {
    return r == 0 ? V + 1 : r == 1 ? 2 * V + 2 : r == 2 ? 4 * V + 8 : (V << r) + 1;
  }
};

template <class K, int NT, int VT>
struct K1KeysShape {
  static constexpr int T = NT * VT;
  static constexpr int NW = NT / 32;
  static constexpr int W = VecOf<K>::W;      // keys per vector (= sentinel slot)
  static constexpr int V = VT / W;           // vectors per thread
  static constexpr int ROUNDS = __builtin_ctz(NT);
  static constexpr int cmax(int a, int b) { return a > b ? a : b; }
  // per-warp region (in-warp rounds: 16 >> r pairs) and the whole-block
  // region (block rounds: NT >> (r+1) pairs), in vectors
  static constexpr int wreg(int r) {
    return r > 4 ? 0 : cmax(K1Layout::start<V>(r, 16 >> r), wreg(r + 1));
  }
  static constexpr int breg(int r) {
    return r >= ROUNDS ? 0 : cmax(r > 4 ? K1Layout::start<V>(r, NT >> (r + 1)) : 0, breg(r + 1));
  }
  static constexpr int WREGV = wreg(0);
  // block rounds' co-rank exchange (NT ints) after the block region, in ints
  // from the start of shared memory (guard vector included)
  static constexpr int CRANK = (1 + breg(0)) * 4;
  static constexpr size_t smem =
      (size_t)cmax(cmax(NW * WREGV, breg(0) + NT / 4), T / W) * 16 + 16;
  static_assert((NT & (NT - 1)) == 0 && NT >= 32, "NT: power of two >= 32");
};

// SHFL (the A/B variant of SURVEY §8(a) S1 / north_star (1), VT a power of
// two): each warp sorts its 32 x VT keys with the warp-shuffle bitonic
// network (warp_bitonic_keys, no shared memory) instead of the per-thread
// network + the five in-warp merge rounds; the block rounds then start from
// runs of 32 VT.
template <class K, int NT, int VT, bool SHFL = false, class KW = K>
__global__ void __launch_bounds__(NT)
    k1_tile_sort_keys(const KW* __restrict__ in_k, K* __restrict__ out_k, int64_t n,
                      const int64_t* __restrict__ seg,
                      const unsigned long long* __restrict__ gate = nullptr, int gate_want = 0) {
  if (gate && (int)range_narrow(gate) != gate_want) return;  // key-range gate (sort_narrowed)
  using SH = K1KeysShape<K, NT, VT>;
  static_assert(VT % VecOf<K>::W == 0, "keys-only K1 stores 16-byte vectors");
  constexpr int T = SH::T;
  constexpr uint32_t Z = sizeof(K);
  extern __shared__ __align__(16) unsigned char smem[];
  // one guard vector in front: the MIN sentinel of the first run
  K* sk = reinterpret_cast<K*>(smem + 16);
  const char* sb = reinterpret_cast<const char*>(smem);  // byte offsets include the guard
  const int tid = threadIdx.x, warp = tid >> 5;
  // tile blockIdx.x, or the segment of descriptor blockIdx.x (as in k1_tile_sort)
  const int64_t base = seg ? seg[2 * blockIdx.x] : (int64_t)blockIdx.x * T;
  const int cnt = seg ? (int)seg[2 * blockIdx.x + 1] : (int)min((int64_t)T, n - base);

  // Which thread holds which key before the network does not matter (keys
  // only), so load straight into registers, striped (coalesced); the partial
  // last tile is padded with the maximum key.
  K key[VT];
#pragma unroll
  for (int k = 0; k < VT; ++k) {
    const int i = k * NT + tid;
    key[k] = i < cnt ? k1_in<K>(in_k + base + i, gate) : KeyTraits<K>::max_key();
  }
  int r0 = 0;
  if constexpr (SHFL) {
    warp_bitonic_keys<VT>(key, tid & 31);  // the warp's 32 VT keys, blocked
    r0 = 5;
  } else {
    k1_network<VT>(key);
  }

#pragma unroll 1
  for (int r = r0; r < SH::ROUNDS; ++r) {
    const int w = VT << r;
    const bool in_warp = (2 << r) <= 32;
    // region origin of this round's pairs (vectors)
    const int org = in_warp ? warp * SH::WREGV : 0;
    const int mbase = in_warp ? (warp * 32) >> (r + 1) : 0;  // first pair of the region
    if (in_warp) __syncwarp();
    else __syncthreads();
    {
      // my VT keys: run rho = tid >> r at offset (tid mod 2^r) * VT
      const int rho = tid >> r;
      const int pos = (tid & ((1 << r) - 1)) * VT;
      const int m = (rho >> 1) - mbase;
      constexpr int W = SH::W;
      const int run = org + K1Layout::start<SH::V>(r, m) + ((rho & 1) ? 0 : K1Layout::aoff<SH::V>(r));
      const int at = run * W + pos;
      store_vec<K, VT>(sk + at, key);
      if (pos + VT == w) sk[at + VT] = KeyTraits<K>::max_key();  // sentinels
      if (pos == 0) sk[at - 1] = KeyTraits<K>::min_key();
    }
    if (in_warp) __syncwarp();
    else __syncthreads();
    const int m = (tid >> (r + 1)) - mbase;
    const int d = (tid & ((2 << r) - 1)) * VT;
    const uint32_t ob0 = (uint32_t)(1 + org + K1Layout::start<SH::V>(r, m)) * 16u;
    const uint32_t oa0 = ob0 + (uint32_t)K1Layout::aoff<SH::V>(r) * 16u;
    const int i = merge_path_off<K>(sb, oa0, w, ob0, w, d);
    // co-rank at my last diagonal d + VT: the next thread's (shuffle inside
    // a warp, shared memory across warps), or w at the end of the pair
    int i1 = __shfl_down_sync(0xffffffffu, i, 1);
    if (!in_warp) {
      int* cr = reinterpret_cast<int*>(smem) + SH::CRANK;
      cr[tid] = i;
      __syncthreads();
      if ((tid & 31) == 31 && tid + 1 < NT) i1 = cr[tid + 1];
    }
    if (d + VT == 2 * w) i1 = w;
    merge_keys_dual<K, VT>(sb, oa0 + (uint32_t)i * Z, oa0 + (uint32_t)w * Z,
                           ob0 + (uint32_t)(d - i) * Z, oa0 + (uint32_t)i1 * Z,
                           ob0 + (uint32_t)(d + VT - i1) * Z, ob0 - Z, key);
  }

  __syncthreads();
  store_vec<K, VT>(sk + tid * VT, key);
  __syncthreads();
#pragma unroll 4
  for (int i = tid; i < cnt; i += NT) out_k[base + i] = sk[i];
}

// ----------------------------------------------------------------- K3
// k3_merge.cuh: the persistent merge pass with fused co-rank search (K2).

// A/B hook of the tile sort alone (scripts/k1_ab.py): sorts every tile of
// in[0, n) (int32) into out with the product K1 (variant 0: 128 x 68, T =
// 8704) or the warp-shuffle variant (1: 128 x 64, T = 8192).  Returns the
// tile size, or -1 on a launch error.  Not part of the product path.
extern "C" int msort_debug_tile_sort(const void* in, void* out, int64_t n, int variant,
                                     void* stream) {
  using namespace msort;
  cudaStream_t s = (cudaStream_t)stream;
  if (variant == 0) {
    using SH = K1KeysShape<int32_t, 128, 68>;
    static bool init = false;
    if (!init) {
      cudaFuncSetAttribute(k1_tile_sort_keys<int32_t, 128, 68, false>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SH::smem);
      init = true;
    }
    const int64_t nt = (n + SH::T - 1) / SH::T;
    {
      LaunchScope ls(KC_TILE_SORT, s);
      k1_tile_sort_keys<int32_t, 128, 68, false><<<(unsigned)nt, 128, SH::smem, s>>>(
          (const int32_t*)in, (int32_t*)out, n, nullptr);
    }
    return cudaGetLastError() == cudaSuccess ? SH::T : -1;
  }
  using SH = K1KeysShape<int32_t, 128, 64>;
  static bool init1 = false;
  if (!init1) {
    cudaFuncSetAttribute(k1_tile_sort_keys<int32_t, 128, 64, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SH::smem);
    init1 = true;
  }
  const int64_t nt = (n + SH::T - 1) / SH::T;
  {
    LaunchScope ls(KC_TILE_SORT, s);
    k1_tile_sort_keys<int32_t, 128, 64, true><<<(unsigned)nt, 128, SH::smem, s>>>(
        (const int32_t*)in, (int32_t*)out, n, nullptr);
  }
  return cudaGetLastError() == cudaSuccess ? SH::T : -1;
}

#ifdef MSORT_K0_TRACE
extern "C" int msort_debug_k0_trace(unsigned long long* host) {
  return (int)cudaMemcpyFromSymbol(host, g_k0_trace, sizeof(unsigned long long) * 16 * 32);
}
#endif
#ifdef MSORT_K3_TRACE
extern "C" int msort_debug_k3_trace(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_k3_trace, sizeof(unsigned long long) * n);
}
extern "C" int msort_debug_k3_trace2(unsigned long long* tiles, int nt, unsigned long long* chunks,
                                     int nc) {
  int e = (int)cudaMemcpyFromSymbol(tiles, g_k3_tiles, sizeof(unsigned long long) * nt);
  if (e) return e;
  return (int)cudaMemcpyFromSymbol(chunks, g_k3_chunks, sizeof(unsigned long long) * nc * 4);
}
extern "C" int msort_debug_k3_trace_clear() {
  void *pt = nullptr, *pc = nullptr;
  cudaError_t e = cudaGetSymbolAddress(&pt, g_k3_tiles);
  if (!e) e = cudaGetSymbolAddress(&pc, g_k3_chunks);
  if (!e) e = cudaMemset(pt, 0, sizeof(unsigned long long) * kK3TraceTiles);
  if (!e) e = cudaMemset(pc, 0, sizeof(unsigned long long) * kK3TraceChunks * 4);
  return (int)e;
}
#endif

// ------------------------------------------------------------ host driver
#ifndef MSORT_K3_NC
#define MSORT_K3_NC 512  // merging threads per K3 CTA (4-byte keys only; 256 otherwise)
#endif
#ifndef MSORT_K1_NT
#define MSORT_K1_NT 128  // keys-only K1 threads (4-byte keys)
#endif
#ifndef MSORT_K3P_VT
#define MSORT_K3P_VT 17  // 4-byte keys + payload: outputs per merger
#endif
#ifndef MSORT_K3P_NC
#define MSORT_K3P_NC 256  // 4-byte keys + payload: mergers per CTA
#endif
#ifndef MSORT_K1P_NT
#define MSORT_K1P_NT 512  // pairs K1 threads, 4-byte keys (x 17 keys)
#endif
#ifndef MSORT_K1P8_NT
// pairs K1 threads, 8-byte keys (x 17 keys): 256 (T = 4352, 70 KB of shared
// memory, 3 CTAs/SM) -- C3 K1 1.98 -> 1.29 ms for one more merge level
// (+0.24 ms): C3 5.36 -> 4.91 ms.  4-byte keys keep 512 (T = 8704): 256 gives
// K1 2.13 -> 1.74 but a 15th level, C4 7.24 -> 7.20 (noise).
#define MSORT_K1P8_NT 256
#endif
#ifndef MSORT_K1_VT
#define MSORT_K1_VT 68  // keys-only K1 items per thread (NT x VT = 8704)
#endif
#ifndef MSORT_K3_VT
#define MSORT_K3_VT 17  // outputs per merging thread (even: two chains per thread)
#endif

#ifndef MSORT_K3_GRABDIV
#define MSORT_K3_GRABDIV 4  // grabs of kGrab chunks per CTA per level below which grabs are single
#endif
#ifndef MSORT_K3_CHDIV
#define MSORT_K3_CHDIV 2  // full chunks per CTA per level below which chunks shrink
#endif
#ifndef MSORT_QUAD
#define MSORT_QUAD 0  // keys only, 4-byte keys: 5 = two merge levels per HBM pass (K6)
#endif
// Merge-level grouping for keys-only sorts: 0 = every level in the fused
// 2-way dataflow (default), 5 = K6 4-way passes (opt-in experiment).  The
// environment variable MSORT_QUAD sets it once; msort_debug_set_quad (tests)
// overrides it.  Atomic: concurrent sorts read a consistent value.
static std::atomic<int> g_quad_mode{-1};
static int quad_mode() {
  int m = g_quad_mode.load(std::memory_order_relaxed);
  if (m < 0) {
    const char* e = getenv("MSORT_QUAD");
    int v = e ? atoi(e) : MSORT_QUAD;
    if (v != 5) v = 0;
    g_quad_mode.compare_exchange_strong(m, v);
    m = g_quad_mode.load(std::memory_order_relaxed);
  }
  return m;
}

// Scheduler state in the workspace: 64 chunk counters (one per launch of a
// sort) then the per-level, per-pair completion counters of the fused merge.
constexpr int kMaxLaunches = 64;

// Page-locked staging buffers for host tables uploaded by a call (segment
// descriptors): a small ring per device, each buffer with its own event.  A
// call takes a buffer whose previous upload has completed (growing it if
// needed), so it only waits when every buffer of its device is still in
// flight; the lease records the buffer's event on the caller's stream.
struct StageBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaEvent_t ev = nullptr;
  bool held = false;
};
constexpr int kStageRing = 4;
static std::mutex g_stage_mu;
static StageBuf g_stage[64][kStageRing];

struct StageLease {
  int dev = -1, slot = -1;
  void* ptr = nullptr;
  ~StageLease() {  // an early return before release(): nothing was enqueued
    if (slot >= 0) {
      std::lock_guard<std::mutex> lk(g_stage_mu);
      g_stage[dev][slot].held = false;
    }
  }
  msort_status release(cudaStream_t s) {
    cudaError_t e;
    {
      std::lock_guard<std::mutex> lk(g_stage_mu);
      e = cudaEventRecord(g_stage[dev][slot].ev, s);
      g_stage[dev][slot].held = false;
    }
    slot = -1;
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord (staging)");
    return MSORT_SUCCESS;
  }
};

static msort_status staging_acquire(size_t bytes, StageLease& L) {
  int dev = 0;
  MSORT_CUDA_TRY(cudaGetDevice(&dev));
  if (dev >= 64) {
    set_error("device index >= 64");
    return MSORT_ERROR_NOT_SUPPORTED;
  }
  for (int attempt = 0;; ++attempt) {
    int pick = -1;
    {
      std::lock_guard<std::mutex> lk(g_stage_mu);
      // a free buffer whose last upload is complete (or never used)
      for (int i = 0; i < kStageRing && pick < 0; ++i) {
        StageBuf& b = g_stage[dev][i];
        if (b.held) continue;
        if (!b.ev) {
          cudaError_t e = cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming);
          if (e != cudaSuccess) return cuda_fail(e, "cudaEventCreate (staging)");
          pick = i;
        } else if (cudaEventQuery(b.ev) == cudaSuccess) {
          pick = i;
        }
      }
      (void)cudaGetLastError();  // cudaErrorNotReady from the queries
      if (pick < 0 && attempt > 0) {
        for (int i = 0; i < kStageRing && pick < 0; ++i)
          if (!g_stage[dev][i].held) pick = i;  // waited for below
      }
      if (pick >= 0) {
        StageBuf& b = g_stage[dev][pick];
        b.held = true;
        L.dev = dev, L.slot = pick;
      }
    }
    if (pick < 0) {
      if (attempt > 1000000) {
        set_error("staging: every buffer held");
        return MSORT_ERROR_NOT_SUPPORTED;
      }
      std::this_thread::yield();
      continue;
    }
    StageBuf& b = g_stage[dev][pick];
    MSORT_CUDA_TRY(cudaEventSynchronize(b.ev));  // immediate unless every buffer was busy
    if (bytes > b.cap) {
      if (b.p) cudaFreeHost(b.p);
      b.p = nullptr, b.cap = 0;
      const size_t cap = std::max<size_t>(bytes + bytes / 2, 1 << 16);
      MSORT_CUDA_TRY(cudaHostAlloc(&b.p, cap, cudaHostAllocDefault));
      b.cap = cap;
    }
    L.ptr = b.p;
    return MSORT_SUCCESS;
  }
}

template <class K, bool PAIRS>
struct Kernels {
  // K1 shape.  Pairs: 512 threads x 17 (odd: conflict-free blocked shared
  // accesses; the stable odd-even transposition network is quadratic, so
  // threads keep few items).  Keys only: fewer threads with more items each
  // -- a register network level is cheaper than a shared-memory merge round
  // (and each thread's co-rank search is amortised over more outputs).
  // (4-byte keys: 128 x 68 -- 1.53 ms vs 1.74 for 256 x 34 and 1.99 for 64 x
  // 136 on 2^28 int32; 8-byte keys keep 256 x 34: twice the registers per key)
  static constexpr int VT = PAIRS ? 17 : (sizeof(K) == 4 ? MSORT_K1_VT : 34);
  static constexpr int NT1 =
      PAIRS ? (sizeof(K) == 8 ? MSORT_K1P8_NT : MSORT_K1P_NT) : (sizeof(K) == 4 ? MSORT_K1_NT : 256);
  static constexpr int T = NT1 * VT;  // tile sort size
  // 4-byte keys: 512 mergers x 17 = one 8704-key output tile (= T) per stage,
  // 2 CTAs/SM -- half the tiles (and co-rank searches) of 256 x 17, measured
  // 5.35 vs 5.71 ms for the 15 levels of 2^28; wider records
  // keep 256 mergers so three stages fit in shared memory.
  static constexpr bool WIDE3 = sizeof(K) == 4 && !PAIRS;
  // 8-byte keys (with or without payload): 512 mergers and two stages, one
  // CTA/SM (C3: 4.25 -> 3.67 ms of merging); 4-byte keys with a payload keep
  // 256 mergers and three stages (512 x 2 stages: C4 5.40 -> 6.10 ms).
  static constexpr bool WIDE8 = sizeof(K) == 8;
  static constexpr int NC = WIDE3 ? MSORT_K3_NC : (WIDE8 ? 512 : MSORT_K3P_NC);
  static constexpr int VT3 = PAIRS ? (sizeof(K) == 4 ? MSORT_K3P_VT : 17) : MSORT_K3_VT;
  static constexpr int Tm = NC * VT3;  // merge output tile (divides 2T)
#ifndef MSORT_K3_S
#define MSORT_K3_S 3
#endif
#ifndef MSORT_K3P_S
#define MSORT_K3P_S 3  // 4-byte keys + payload
#endif
#ifndef MSORT_K3P_MINB
#define MSORT_K3P_MINB 2
#endif
  static constexpr int S = WIDE3 ? MSORT_K3_S : (WIDE8 ? 2 : MSORT_K3P_S);  // stage ring depth
  using LY = K3Layout<K, PAIRS, NC, VT3, S>;
  // CTAs per SM the register budget is tuned for (shared memory allows 4 for
  // 4-byte keys without payload, 2-3 otherwise)
#ifndef MSORT_K3_MINB
#define MSORT_K3_MINB 2
#endif
  static constexpr int MINB = WIDE3 ? MSORT_K3_MINB : (WIDE8 ? 1 : MSORT_K3P_MINB);  // CTAs/SM for registers
  static constexpr size_t k1_smem =
      PAIRS ? (size_t)T * sizeof(K) + (size_t)T * 8 : K1KeysShape<K, NT1, VT>::smem;
  static constexpr size_t k3_smem = LY::bytes;
  static_assert((2 * T) % Tm == 0, "pair boundaries must be tile boundaries");
  using Fused = FusedPasses<K>;
  using Explicit = SinglePass<K, ExplicitPairs>;
  using Peer = SinglePass<K, PeerPairs>;

  // K6 (4-byte keys only, quad mode 5): 128 threads x 68 keys, tiles of
  // <= XS keys of X plus <= YS keys of Y (XS + YS = Tm = 126 x 68)
  static constexpr int kK6NT2 = MSORT_K6_NT2, kK6VT = 68;
  using K6S = K6Shape<kK6NT2, kK6VT>;
  // X keys per unit: 7/15 of the tile, so a unit of random keys (as many Y
  // keys as X keys, +- a few sqrt) fits without a cut
  static constexpr int kK6XS = K6S::Tm * 7 / 15, kK6YS = K6S::Tm - kK6XS;
  static bool k6_mode() { return sizeof(K) == 4 && quad_mode() == 5; }
  static int64_t k6_units_max(int64_t n) { return n / kK6XS + n / (4 * (int64_t)T) + 2; }
  static_assert(kK6XS >= 3998, "msort_workspace_bytes sizes the K6 area for XS >= 3998");
  static int64_t k6_extra_max(int64_t n) { return n / kK6YS + k6_units_max(n) + 1; }
  // Per-device grid sizes, set once by init() / k6_init() (release) and read
  // by any thread (acquire): 0 = not initialised on that device yet.
  static std::atomic<int>& k6_grid_slot(int dev) {
    static std::atomic<int> g[64];
    return g[dev & 63];
  }
  static int k6_grid(int dev) { return k6_grid_slot(dev).load(std::memory_order_acquire); }
  static std::atomic<int>& grid3_slot(int dev) {
    static std::atomic<int> g[64];
    return g[dev & 63];
  }
  static int grid3(int dev) { return grid3_slot(dev).load(std::memory_order_acquire); }

  // Tiles per scheduled chunk for a level of `tiles` output tiles: kChunk
  // when every CTA gets >= 2 full chunks per level (few searches, long bulk
  // streams), else smaller -- a small sort is latency-bound and a level takes
  // as long as its longest chunk.
  static int chunk_tiles(int64_t tiles, int dev) {
    const int64_t per = tiles / (MSORT_K3_CHDIV * (int64_t)std::max(grid3(dev), 1));
    return (int)std::max<int64_t>(1, std::min<int64_t>(kChunk, per));
  }
  // Chunks per atomic grab: kGrab only when every CTA gets >= MSORT_K3_GRABDIV
  // grabs per level, else 1 -- a grab of kGrab full chunks is 24 tiles, and
  // with ~1-2 grabs per CTA and level the level waits for the CTAs that got
  // one more (2^26 int32: 2.04 -> 1.64 ms); with one chunk per grab the
  // searcher's lanes search that chunk's co-ranks in groups (k3_merge.cuh).
  static int grab_for(int64_t tiles, int ch, int dev) {
    if (ch < kChunk) return 1;
    const int64_t need =
        (int64_t)MSORT_K3_GRABDIV * std::max(grid3(dev), 1) * (int64_t)ch * kGrab;
    return tiles >= need ? kGrab : 1;
  }

  // Kernel attributes are set lazily, per kernel instance and device, the
  // first time a call needs that kernel (a first call only pays for what it
  // launches).
  template <class Src>
  static msort_status k3_ready(int dev) {
    static std::atomic<bool> done[64];
    if (done[dev & 63].load(std::memory_order_acquire)) return MSORT_SUCCESS;
    auto k = k3_merge_pass<K, PAIRS, NC, VT3, S, MINB, Src>;
    MSORT_CUDA_TRY(
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k3_smem));
    done[dev & 63].store(true, std::memory_order_release);
    return MSORT_SUCCESS;
  }

  // K1 and the persistent merge kernel's grid (every CTA of the fused
  // levels must be resident: grid = SMs x occupancy).
  static msort_status init() {
    int dev = 0;
    MSORT_CUDA_TRY(cudaGetDevice(&dev));
    if (grid3(dev)) return MSORT_SUCCESS;
    if constexpr (PAIRS)
      MSORT_CUDA_TRY(cudaFuncSetAttribute(k1_tile_sort<K, PAIRS, NT1, VT>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)k1_smem));
    else
      MSORT_CUDA_TRY(cudaFuncSetAttribute(k1_tile_sort_keys<K, NT1, VT>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)k1_smem));
    MSORT_TRY(k3_ready<Fused>(dev));
    int sms = 0, occ = 0;
    MSORT_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    MSORT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &occ, k3_merge_pass<K, PAIRS, NC, VT3, S, MINB, Fused>, NC + kK3Extra, k3_smem));
    if (occ < 1) {
      set_error("merge pass kernel does not fit on an SM");
      return MSORT_ERROR_NOT_SUPPORTED;
    }
    grid3_slot(dev).store(sms * occ, std::memory_order_release);
    return MSORT_SUCCESS;
  }

  // K6 (opt-in): its attribute and grid, on first use
  static msort_status k6_init(int dev) {
    if constexpr (!PAIRS && sizeof(K) == 4) {
      if (k6_grid(dev)) return MSORT_SUCCESS;
      auto k6 = k6_quad_pass<K, kK6NT2, kK6VT>;
      MSORT_CUDA_TRY(cudaFuncSetAttribute(k6, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(K6S::KEYS * sizeof(K))));
      int o6 = 0, sms = 0;
      MSORT_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      MSORT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o6, k6, K6S::NT1,
                                                                   K6S::KEYS * sizeof(K)));
      k6_grid_slot(dev).store(sms * std::max(o6, 1), std::memory_order_release);
    }
    return MSORT_SUCCESS;
  }

  template <class Src>
  static msort_status launch_k3(const Src& src, int64_t nchunks, unsigned long long* ctr,
                                cudaStream_t s, KernelClass kc) {
    int dev = 0;
    MSORT_CUDA_TRY(cudaGetDevice(&dev));
    MSORT_TRY(k3_ready<Src>(dev));
    const int64_t grid = std::min<int64_t>(grid3(dev), (nchunks + src.grab - 1) / src.grab);
    {
      LaunchScope ls(kc, s);
      k3_merge_pass<K, PAIRS, NC, VT3, S, MINB, Src>
          <<<(unsigned)grid, NC + kK3Extra, k3_smem, s>>>(src, ctr);
    }
    MSORT_CUDA_TRY(cudaGetLastError());
#ifdef MSORT_K3_CHECK
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      fprintf(stderr, "K3 failed: chunks %lld grid %lld: %s\n", (long long)nchunks,
              (long long)grid, cudaGetErrorString(e));
      return cuda_fail(e, "k3 (debug sync)");
    }
#endif
    return MSORT_SUCCESS;
  }

  // K1 of the narrowed sort: reads the caller's 8-byte keys (KW) and narrows
  // them on the fly (k1_in); its attribute is set on first use per device.
  template <class KW>
  static msort_status k1_wide(const KW* in, const uint32_t* in_v, K* ok, uint32_t* ov, size_t n,
                              int64_t ntiles, const unsigned long long* gate, int want,
                              cudaStream_t s) {
    int dev = 0;
    MSORT_CUDA_TRY(cudaGetDevice(&dev));
    static std::atomic<bool> ready[64];
    if (!ready[dev & 63].load(std::memory_order_acquire)) {
      if constexpr (PAIRS)
        MSORT_CUDA_TRY(cudaFuncSetAttribute(k1_tile_sort<K, PAIRS, NT1, VT, KW>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)k1_smem));
      else
        MSORT_CUDA_TRY(cudaFuncSetAttribute(k1_tile_sort_keys<K, NT1, VT, false, KW>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)k1_smem));
      ready[dev & 63].store(true, std::memory_order_release);
    }
    LaunchScope ls(KC_TILE_SORT, s);
    if constexpr (PAIRS)
      k1_tile_sort<K, PAIRS, NT1, VT, KW>
          <<<(unsigned)ntiles, NT1, k1_smem, s>>>(in, in_v, ok, ov, (int64_t)n, nullptr, gate,
                                                   want);
    else
      k1_tile_sort_keys<K, NT1, VT, false, KW>
          <<<(unsigned)ntiles, NT1, k1_smem, s>>>(in, ok, (int64_t)n, nullptr, gate, want);
    return MSORT_SUCCESS;
  }

  // Sort in_k/in_v into out_k/out_v (in == out: in place; K1 reads a whole
  // tile into shared memory before writing it back, so that is safe).
  // gate / gate_want: the key-range gate of sort_narrowed (every launch of
  // this sort does nothing unless range_narrow(gate) == gate_want); the
  // caller guarantees n > kK0MaxN, so no K0, and K6 is not used.
  // wide / wide_kind (4-byte keys of the narrowed sort only): K1 reads the
  // caller's 8-byte keys (1 int64, 2 uint64) and narrows them on the fly
  // (k1_in, gate = the range); in_k is then unused.
  static msort_status sort(const K* in_k, const uint32_t* in_v, K* keys, uint32_t* vals,
                           size_t n, void* ws, size_t ws_bytes, cudaStream_t s,
                           const unsigned long long* gate = nullptr, int gate_want = 0,
                           const void* wide = nullptr, int wide_kind = 0) {
    MSORT_TRY(init());
    if (n < 2) {
      if (n == 1 && in_k != keys) {
        MSORT_CUDA_TRY(cudaMemcpyAsync(keys, in_k, sizeof(K), cudaMemcpyDeviceToDevice, s));
        if (PAIRS)
          MSORT_CUDA_TRY(cudaMemcpyAsync(vals, in_v, 4, cudaMemcpyDeviceToDevice, s));
      }
      return MSORT_SUCCESS;
    }
    if constexpr (!PAIRS) {
      // small keys-only sorts: the whole sort in one cluster launch (K0)
      if ((int64_t)n <= kK0MaxN && k0_enabled() && (int64_t)n <= k0_limit())
        return small_sort(in_k, keys, (int64_t)n, s);
    }
    const int64_t ntiles = (int64_t)((n + T - 1) / T);
    int passes = 0;
    while ((int64_t(1) << passes) < ntiles) ++passes;
    int dev = 0;
    MSORT_CUDA_TRY(cudaGetDevice(&dev));
    // K6 (opt-in, 4-byte keys only): every pair of levels as one 4-way pass;
    // otherwise (the default) every level runs in the fused 2-way dataflow.
    int nq = 0;
    int64_t Lq = T;
    if constexpr (!PAIRS) {
      if (k6_mode() && !gate) {
        MSORT_TRY(k6_init(dev));
        nq = passes / 2, Lq = (int64_t)T << (2 * nq);
      }
    }
    const int left = passes - 2 * nq;  // 2-way levels
    if (passes > kMaxFusedPasses) {
      set_error("too many merge levels");
      return MSORT_ERROR_NOT_SUPPORTED;
    }
    char* w = static_cast<char*>(ws);
    K* wk = reinterpret_cast<K*>(w);
    w += align_up(n * sizeof(K), 256);
    uint32_t* wv = nullptr;
    if (PAIRS) {
      wv = reinterpret_cast<uint32_t*>(w);
      w += align_up(n * sizeof(uint32_t), 256);
    }
    auto* ctr = reinterpret_cast<unsigned long long*>(w);
    auto* done = reinterpret_cast<unsigned*>(ctr + kMaxLaunches);
    char* const k6ws = w + align_up(((size_t)n / T + 2 + 2 * 64) * sizeof(int64_t), 256);
    (void)ws_bytes;

    K* bk[2] = {keys, wk};
    uint32_t* bv[2] = {vals, wv};
    // S4: pick K1's destination so the last pass lands in keys
    int cur = (nq + left) % 2;
    bool k1_done = false;
    if constexpr (std::is_same<K, uint32_t>::value) {
      if (wide_kind != 0) {
        if (wide_kind == 1)
          MSORT_TRY(k1_wide<int64_t>(static_cast<const int64_t*>(wide), in_v, bk[cur], bv[cur], n,
                                     ntiles, gate, gate_want, s));
        else
          MSORT_TRY(k1_wide<uint64_t>(static_cast<const uint64_t*>(wide), in_v, bk[cur], bv[cur],
                                      n, ntiles, gate, gate_want, s));
        k1_done = true;
      }
    }
    if (!k1_done) {
      LaunchScope ls(KC_TILE_SORT, s);
      if constexpr (PAIRS)
        k1_tile_sort<K, PAIRS, NT1, VT>
            <<<(unsigned)ntiles, NT1, k1_smem, s>>>(in_k, in_v, bk[cur], bv[cur], (int64_t)n,
                                                     nullptr, gate, gate_want);
      else
        k1_tile_sort_keys<K, NT1, VT>
            <<<(unsigned)ntiles, NT1, k1_smem, s>>>(in_k, bk[cur], (int64_t)n, nullptr, gate,
                                                     gate_want);
    }
    MSORT_CUDA_TRY(cudaGetLastError());
#ifdef MSORT_K3_CHECK
    {
      cudaError_t e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) fprintf(stderr, "K1 failed: %s\n", cudaGetErrorString(e));
      if (e != cudaSuccess) return cuda_fail(e, "k1 (debug sync)");
    }
#endif
    if (passes == 0) return MSORT_SUCCESS;
    if constexpr (!PAIRS) {
      if (nq > 0)
        MSORT_CUDA_TRY(cudaMemsetAsync(ctr, 0, kMaxLaunches * sizeof(unsigned long long), s));
      int64_t L = T;
      if constexpr (sizeof(K) == 4) {
      if (k6_mode() && nq > 0) {
        // K6 (k6_quad.cuh): partition (unit states, tiles, cut pieces), then
        // the 4-way pass over the unit tiles and over the pieces
        char* kw = k6ws;
        int64_t* states = reinterpret_cast<int64_t*>(kw);
        const int64_t NUmax = k6_units_max((int64_t)n);
        K6Tile* tiles = reinterpret_cast<K6Tile*>(kw + align_up(32 * NUmax, 256));
        int64_t* cuts = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(tiles) +
                                                   align_up(sizeof(K6Tile) * NUmax, 256));
        const int64_t EXmax = k6_extra_max((int64_t)n);
        K6Tile* extra = reinterpret_cast<K6Tile*>(reinterpret_cast<char*>(cuts) +
                                                  align_up(16 * EXmax, 256));
        auto* ncut = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(extra) +
                                                            align_up(sizeof(K6Tile) * EXmax, 256));
        for (int q = 0; q < nq; ++q, L *= 4) {
          K6Pass P{};
          P.src = bk[cur], P.n = (int64_t)n, P.L = L;
          P.groups = ((int64_t)n + 4 * L - 1) / (4 * L);
          P.xs = kK6XS, P.ys = kK6YS;
          P.upg = (2 * L + kK6XS - 1) / kK6XS;
          const int64_t last0 = (P.groups - 1) * 4 * L;
          const int64_t nx_last = std::min<int64_t>((int64_t)n, last0 + 2 * L) - last0;
          P.nunits = (P.groups - 1) * P.upg + std::max<int64_t>(1, (nx_last + kK6XS - 1) / kK6XS);
          MSORT_CUDA_TRY(cudaMemsetAsync(ncut, 0, 8, s));
          const unsigned gb = (unsigned)((P.nunits + 127) / 128);
          {
            LaunchScope ls(KC_PARTITION, s);
            k6_states<K, true><<<gb, 128, 0, s>>>(P, states);
            k6_states<K, false><<<gb, 128, 0, s>>>(P, states);
            k6_tiles<K><<<gb, 128, 0, s>>>(P, states, tiles, cuts, ncut);
            k6_cut_tiles<K><<<(unsigned)(k6_grid(dev) / 8 + 1), 128, 0, s>>>(P, states, cuts, ncut,
                                                                           extra);
          }
          MSORT_CUDA_TRY(cudaGetLastError());
          {
            LaunchScope ls(KC_MERGE, s);
            k6_quad_pass<K, kK6NT2, kK6VT><<<(unsigned)P.nunits, K6S::NT1, K6S::KEYS * sizeof(K),
                                             s>>>(bk[cur], bk[cur ^ 1], tiles, nullptr);
            k6_quad_pass<K, kK6NT2, kK6VT><<<(unsigned)k6_grid(dev), K6S::NT1,
                                             K6S::KEYS * sizeof(K), s>>>(bk[cur], bk[cur ^ 1],
                                                                         extra, ncut);
          }
          MSORT_CUDA_TRY(cudaGetLastError());
#ifdef MSORT_K3_CHECK
          {
            cudaError_t e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) return cuda_fail(e, "k6 (debug sync)");
          }
#endif
          cur ^= 1;
        }
        if (left == 0) return MSORT_SUCCESS;
      }
      }
    }
#ifdef MSORT_K3_PERPASS
    // tuning variant: one launch per merge level
    MSORT_CUDA_TRY(cudaMemsetAsync(ctr, 0, kMaxLaunches * 8, s));
    for (int p = 0; p < passes; ++p) {
      SinglePass<K, UniformPairs> sp{};
      sp.pm = UniformPairs{(int64_t)n, (int64_t)T << p};
      sp.src_k = bk[cur], sp.src_v = bv[cur], sp.dst_k = bk[cur ^ 1], sp.dst_v = bv[cur ^ 1];
      sp.ntiles = (int64_t)((n + Tm - 1) / Tm);
      sp.ch = chunk_tiles(sp.ntiles, dev);
      sp.grab = grab_for(sp.ntiles, sp.ch, dev);
      MSORT_TRY(launch_k3(sp, (sp.ntiles + sp.ch - 1) / sp.ch, ctr + p, s, KC_MERGE));
      cur ^= 1;
    }
    return MSORT_SUCCESS;
#endif
    // All merge levels in one dataflow launch (k3_merge.cuh, FusedPasses).
    Fused f{};
    f.bk[0] = bk[cur], f.bk[1] = bk[cur ^ 1];
    f.bv[0] = bv[cur], f.bv[1] = bv[cur ^ 1];
    f.n = (int64_t)n, f.T = Lq, f.ntiles = (int64_t)((n + Tm - 1) / Tm), f.P = left;
    f.done = done;
    f.gate = gate, f.gate_want = gate_want;
    int64_t pb = 0;
    for (int p = 0; p < left; ++p) {
      f.pair_base[p] = pb;
      const int64_t twoL = (int64_t)2 * Lq << p;
      pb += ((int64_t)n + twoL - 1) / twoL;
    }
    f.pair_base[left] = pb;
    MSORT_CUDA_TRY(cudaMemsetAsync(ctr, 0, kMaxLaunches * 8 + pb * 4, s));
    f.ch = chunk_tiles(f.ntiles, dev);
    f.grab = grab_for(f.ntiles, f.ch, dev);
    return launch_k3(f, (int64_t)left * ((f.ntiles + f.ch - 1) / f.ch), ctr, s, KC_MERGE);
  }

  // ---- K0: n <= kK0MaxN keys in one launch (k0_small.cuh) -------------
  // MSORT_K0 (environment): 0 disables K0; 1 (default) the one-step
  // multiway cluster merge for clusters of 4 or more CTAs and the pairwise
  // cluster level below (2^13 keys: 14.4 vs 16.4 us, profiles/r02/k0mw/);
  // 4 the multiway step at every cluster size; 3 the pairwise cluster levels
  // (round-2 A/B variant); 2 the pairwise levels without the warp-shuffle
  // network
  static int k0_mode() {
    const char* e = getenv("MSORT_K0");
    const int m = e && *e ? atoi(e) : 1;
    return m < 0 || m > 4 ? 1 : m;
  }
  static bool k0_enabled() { return k0_mode() != 0; }
  template <bool SHFL, bool MW>
  static msort_status k0_attr(int dev) {
    static std::atomic<bool> done[64];
    if (!done[dev & 63].load(std::memory_order_acquire)) {
      constexpr size_t smem = (size_t)k0_smem_keys<K, MW>() * sizeof(K);
      MSORT_CUDA_TRY(cudaFuncSetAttribute(k0_small_sort<K, SHFL, MW>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      if (kK0MaxCL > 8)
        MSORT_CUDA_TRY(cudaFuncSetAttribute(k0_small_sort<K, SHFL, MW>,
                                            cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      done[dev & 63].store(true, std::memory_order_release);
    }
    return MSORT_SUCCESS;
  }
  template <bool SHFL, bool MW>
  static bool k0_fits16(int dev) {
    if (k0_attr<SHFL, MW>(dev) != MSORT_SUCCESS) return false;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)kK0MaxCL, 1, 1);
    cfg.blockDim = dim3(kK0NT, 1, 1);
    cfg.dynamicSmemBytes = (size_t)k0_smem_keys<K, MW>() * sizeof(K);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)kK0MaxCL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nc = 0;
    const bool ok = cudaOccupancyMaxActiveClusters(&nc, k0_small_sort<K, SHFL, MW>, &cfg) ==
                        cudaSuccess && nc > 0;
    cudaGetLastError();  // a refused query is not an error of this call
    return ok;
  }
  // Largest n K0 takes on this device: kK0MaxN when a cluster of kK0MaxCL
  // CTAs (16: non-portable) is schedulable, else what 8 CTAs hold (the
  // general path takes the rest).  Queried once per device (every variant
  // is checked, so the limit does not depend on MSORT_K0).
  static int64_t k0_limit() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    static std::atomic<int64_t> lim[64];
    int64_t v = lim[dev & 63].load(std::memory_order_acquire);
    if (v) return v;
    v = (int64_t)std::min(kK0MaxCL, 8) * kK0Chunk;
    if (kK0MaxCL > 8 && k0_fits16<true, true>(dev) && k0_fits16<true, false>(dev) &&
        k0_fits16<false, false>(dev))
      v = kK0MaxN;
    lim[dev & 63].store(v, std::memory_order_release);
    return v;
  }
  static msort_status small_sort(const K* in, K* out, int64_t n, cudaStream_t s) {
    int dev = 0;
    MSORT_CUDA_TRY(cudaGetDevice(&dev));
    int CL = 1;
    while ((int64_t)CL * kK0Chunk < n) CL *= 2;
    int mode = k0_mode();
    if (mode == 1) mode = CL >= 4 ? 4 : 3;
    if (mode == 2) MSORT_TRY((k0_attr<false, false>(dev)));
    else if (mode == 3) MSORT_TRY((k0_attr<true, false>(dev)));
    else MSORT_TRY((k0_attr<true, true>(dev)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)CL, 1, 1);
    cfg.blockDim = dim3(kK0NT, 1, 1);
    cfg.dynamicSmemBytes =
        (size_t)(mode == 4 ? k0_smem_keys<K, true>() : k0_smem_keys<K, false>()) * sizeof(K);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = CL > 1 ? 1 : 0;
    {
      LaunchScope ls(KC_TILE_SORT, s);
      if (mode == 2)
        MSORT_CUDA_TRY(cudaLaunchKernelEx(&cfg, k0_small_sort<K, false, false>, in, out, n, CL));
      else if (mode == 3)
        MSORT_CUDA_TRY(cudaLaunchKernelEx(&cfg, k0_small_sort<K, true, false>, in, out, n, CL));
      else
        MSORT_CUDA_TRY(cudaLaunchKernelEx(&cfg, k0_small_sort<K, true, true>, in, out, n, CL));
    }
    return MSORT_SUCCESS;
  }

  // Batched sort of independent segments [off[i], off[i+1]) of keys/vals, in
  // place (seg_sort.cuh, include/msort.h msort_sort_segmented).  Segments are
  // binned by length: one warp per segment up to 256 elements (bitonic network
  // with warp shuffles), one CTA per segment up to T (the tile-sort kernels
  // reading a segment descriptor), and every longer segment through ONE
  // tile-sort launch per buffer parity plus ONE fused merge launch over all
  // of them (SegFused: all levels of all long segments as one dataflow).
  static constexpr int kSegW8 = 256;  // warp classes: <= 32 (VW = 1), <= 256 (VW = 8)
  static constexpr int64_t kSegUploadMin = 1 << 15;  // host tables this long are classified on the device
  static constexpr int kSegNTM = 128, kSegVTM = 17, kSegM = kSegNTM * kSegVTM;  // CTA class
  using SegF = SegFused<K>;
  // off: nseg + 1 offsets, in host memory (dev_off false) or device memory.
  static msort_status sort_segmented(K* keys, uint32_t* vals, const int64_t* off, size_t nseg,
                                     bool dev_off, int64_t n, void* ws, size_t ws_bytes,
                                     cudaStream_t s) {
    MSORT_TRY(init());
    int dev = 0;
    MSORT_CUDA_TRY(cudaGetDevice(&dev));
    // ---- workspace: [ping-pong keys n][vals n][device lists][staged][done][ctr]
    char* w = static_cast<char*>(ws);
    char* const wend = w + ws_bytes;
    K* wk = reinterpret_cast<K*>(w);
    w += align_up((size_t)n * sizeof(K), 256);
    uint32_t* wv = nullptr;
    if (PAIRS) {
      wv = reinterpret_cast<uint32_t*>(w);
      w += align_up((size_t)n * 4, 256);
    }
    // Many segments with a host table: a host pass over them costs ~3 ns
    // each, so upload the table (page-locked staging) and classify it on the
    // device like a device-resident table (one synchronisation).
    if (!dev_off && (int64_t)nseg >= kSegUploadMin) {
      int64_t* doff = reinterpret_cast<int64_t*>(w);
      w += align_up(8 * (nseg + 1), 256);
      StageLease lease;
      MSORT_TRY(staging_acquire(8 * (nseg + 1), lease));
      int64_t* h = static_cast<int64_t*>(lease.ptr);
      std::memcpy(h, off, 8 * (nseg + 1));
      const cudaError_t e =
          cudaMemcpyAsync(doff, h, 8 * (nseg + 1), cudaMemcpyHostToDevice, s);
      MSORT_TRY(lease.release(s));
      if (e != cudaSuccess) return cuda_fail(e, "segment table upload");
      off = doff;
      dev_off = true;
    }
    // ---- classification.  Segments of <= 32 elements are found by the tiny
    // kernel itself from the offsets table; the longer ones are listed: the
    // warp bin (<= 256) and the CTA bins (<= 2176, <= T) as (offset, length)
    // descriptors, long segments as (offset, length) on the host (their
    // tables are built here).
    std::vector<int64_t> mid[3], xl;  // bins: <= 256, <= 2176, <= T
    const int64_t* md[3] = {nullptr, nullptr, nullptr};
    int64_t nb[3] = {0, 0, 0}, ntiny = 0;
    if (!dev_off) {
      for (size_t i = 0; i < nseg; ++i) {
        const int64_t len = off[i + 1] - off[i];
        if (len <= 32) {
          ntiny += len >= 2;
          continue;
        }
        auto& v = len <= T ? mid[len <= kSegW8 ? 0 : len <= kSegM ? 1 : 2] : xl;
        v.push_back(off[i]);
        v.push_back(len);
      }
      for (int c = 0; c < 3; ++c) nb[c] = (int64_t)mid[c].size() / 2;
    } else {
      // on the device (kseg_classify), then one synchronisation for the
      // counts and the long segments' list
      const int64_t cap[4] = {n / 33 + 1, n / (kSegW8 + 1) + 1, n / (kSegM + 1) + 1,
                              n / (T + 1) + 1};
      int64_t* lists[4];
      for (int c = 0; c < 4; ++c) {
        lists[c] = reinterpret_cast<int64_t*>(w);
        w += align_up((size_t)cap[c] * 16, 256);
      }
      auto* counts = reinterpret_cast<unsigned long long*>(w);
      w += 256;
      if (w > wend) {
        set_error("segmented sort: workspace too small");
        return MSORT_ERROR_INVALID_VALUE;
      }
      MSORT_CUDA_TRY(cudaMemsetAsync(counts, 0, 6 * 8, s));
      {
        LaunchScope ls(KC_PARTITION, s);
        const int64_t blocks = std::min<int64_t>(((int64_t)nseg + 255) / 256, 148 * 8);
        kseg_classify<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(
            off, (int64_t)nseg, n, kSegM, T, lists[0], lists[1], lists[2], lists[3], counts);
      }
      MSORT_CUDA_TRY(cudaGetLastError());
      unsigned long long hc[6];
      MSORT_CUDA_TRY(cudaMemcpyAsync(hc, counts, sizeof(hc), cudaMemcpyDeviceToHost, s));
      MSORT_CUDA_TRY(cudaStreamSynchronize(s));
      if (hc[5]) {
        set_error("seg_offsets must start at 0, not decrease and end at n");
        return MSORT_ERROR_INVALID_VALUE;
      }
      ntiny = (int64_t)hc[4];
      for (int c = 0; c < 3; ++c) nb[c] = (int64_t)hc[c], md[c] = lists[c];
      xl.resize(2 * hc[3]);
      if (hc[3]) {
        MSORT_CUDA_TRY(cudaMemcpyAsync(xl.data(), lists[3], hc[3] * 16, cudaMemcpyDeviceToHost, s));
        MSORT_CUDA_TRY(cudaStreamSynchronize(s));
      }
    }
    const int64_t nxl = (int64_t)xl.size() / 2;
    // long segments: level count P_s, ordered by it (descending, stable) so
    // that level p's segments are a prefix of the tile range
    auto levels = [](int64_t len) {
      const int64_t t = (len + T - 1) / T;
      int P = 0;
      while ((int64_t(1) << P) < t) ++P;
      return P;
    };
    std::vector<int64_t> xo(nxl);
    for (int64_t j = 0; j < nxl; ++j) xo[j] = j;
    std::stable_sort(xo.begin(), xo.end(), [&](int64_t x, int64_t y) {
      return levels(xl[2 * x + 1]) > levels(xl[2 * y + 1]);
    });
    int Pmax = 0;
    int64_t k1t = 0, n_even_tiles = 0;
    for (int64_t j = 0; j < nxl; ++j) {
      const int64_t len = xl[2 * j + 1], t = (len + T - 1) / T;
      const int P = levels(len);
      Pmax = std::max(Pmax, P);
      k1t += t;
      if ((P & 1) == 0) n_even_tiles += t;
    }
    if (Pmax > kMaxSegLevels) {
      set_error("segment too long");
      return MSORT_ERROR_NOT_SUPPORTED;
    }
    // ---- staging (int64 words): [host offsets only: the offsets table (when
    // there are short segments), CTA-bin descriptors] K1 tile descriptors of
    // the long segments (even-level ones first), long-segment tables off[nxl]
    // len[nxl] tile0[nxl+1] lev[nxl] (int32, packed)
    const int64_t w_off = (!dev_off && ntiny) ? (int64_t)nseg + 1 : 0;
    const int64_t w_desc = w_off + (dev_off ? 0 : 2 * (nb[0] + nb[1] + nb[2])), w_k1 = 2 * k1t;
    const int64_t w_tab = nxl ? 3 * nxl + 1 + (nxl + 1) / 2 : 0;
    const int64_t words = w_desc + w_k1 + w_tab;
    int64_t* dstage = reinterpret_cast<int64_t*>(w);
    w += align_up((size_t)words * 8, 256);
    StageLease lease;  // early returns before release() hand it back unused
    MSORT_TRY(staging_acquire((size_t)words * 8, lease));
    int64_t* h = static_cast<int64_t*>(lease.ptr);
    if (w_off) std::memcpy(h, off, (size_t)w_off * 8);
    if (!dev_off) {
      int64_t at = w_off;
      for (int c = 0; c < 3; ++c) {
        if (nb[c]) std::memcpy(h + at, mid[c].data(), (size_t)nb[c] * 16);
        md[c] = dstage + at;
        at += 2 * nb[c];
      }
    }
    int64_t ntl_all = 0;
    {
      int64_t pe = w_desc, po = w_desc + 2 * n_even_tiles;  // K1 tiles: even P_s, then odd
      int64_t* toff = h + w_desc + w_k1;
      int64_t* tlen = toff + nxl;
      int64_t* tt0 = tlen + nxl;
      int* tlev = reinterpret_cast<int*>(tt0 + nxl + 1);
      for (int64_t j = 0; j < nxl; ++j) {
        const int64_t o = xl[2 * xo[j]], len = xl[2 * xo[j] + 1];
        const int P = levels(len);
        int64_t& pp = (P & 1) ? po : pe;
        for (int64_t t = 0; t * T < len; ++t) {
          h[pp++] = o + t * T;
          h[pp++] = std::min<int64_t>(T, len - t * T);
        }
        toff[j] = o, tlen[j] = len, tt0[j] = ntl_all, tlev[j] = P;
        ntl_all += (len + Tm - 1) / Tm;
      }
      if (nxl) tt0[nxl] = ntl_all;
    }
    unsigned* done = reinterpret_cast<unsigned*>(w);
    w += align_up((size_t)std::max(Pmax, 1) * ntl_all * 4, 256);
    auto* ctr = reinterpret_cast<unsigned long long*>(w);
    w += 256;
    if (w > wend) {
      set_error("segmented sort: workspace too small");
      return MSORT_ERROR_INVALID_VALUE;
    }
    if (words)
      MSORT_CUDA_TRY(cudaMemcpyAsync(dstage, h, (size_t)words * 8, cudaMemcpyHostToDevice, s));
    MSORT_TRY(lease.release(s));
    // ---- launches
    if (ntiny) {
      LaunchScope ls(KC_TILE_SORT, s);
      const int64_t per_cta = 4 * kSegPerWarp;  // 4 warps x kSegPerWarp segments
      kseg_tiny_sort<K, PAIRS><<<(unsigned)((nseg + per_cta - 1) / per_cta), 128, 0, s>>>(
          keys, vals, dev_off ? off : dstage, (int64_t)nseg);
    }
    if (nb[0]) {
      LaunchScope ls(KC_TILE_SORT, s);
      kseg_mid_sort<K, PAIRS><<<(unsigned)((nb[0] + 3) / 4), 128, 0, s>>>(keys, vals, md[0], nb[0]);
    }
    if (nb[1]) {
      LaunchScope ls(KC_TILE_SORT, s);
      constexpr size_t sm = (size_t)kSegM * sizeof(K) + (PAIRS ? (size_t)kSegM * 8 : 0);
      k1_tile_sort<K, PAIRS, kSegNTM, kSegVTM>
          <<<(unsigned)nb[1], kSegNTM, sm, s>>>(keys, vals, keys, vals, 0, md[1]);
    }
    auto k1_desc = [&](const int64_t* d, int64_t cnt_, K* ok, uint32_t* ov) {
      LaunchScope ls(KC_TILE_SORT, s);
      if constexpr (PAIRS)
        k1_tile_sort<K, PAIRS, NT1, VT>
            <<<(unsigned)cnt_, NT1, k1_smem, s>>>(keys, vals, ok, ov, 0, d);
      else
        k1_tile_sort_keys<K, NT1, VT><<<(unsigned)cnt_, NT1, k1_smem, s>>>(keys, ok, 0, d);
    };
    if (nb[2]) k1_desc(md[2], nb[2], keys, vals);
    if (nxl) {
      // long segments: K1 into buffer P_s & 1, then all levels of all of them
      if (n_even_tiles) k1_desc(dstage + w_desc, n_even_tiles, keys, vals);
      if (k1t > n_even_tiles)
        k1_desc(dstage + w_desc + 2 * n_even_tiles, k1t - n_even_tiles, wk, wv);
      MSORT_CUDA_TRY(cudaGetLastError());
      SegF f{};
      f.bk[0] = keys, f.bk[1] = wk, f.bv[0] = vals, f.bv[1] = wv;
      const int64_t* tab = dstage + w_desc + w_k1;
      f.off = tab, f.len = tab + nxl, f.tile0 = tab + 2 * nxl;
      f.lev = reinterpret_cast<const int*>(tab + 3 * nxl + 1);
      f.nseg = (int)nxl, f.T = T, f.ntiles = ntl_all, f.P = Pmax, f.done = done;
      f.ch = chunk_tiles(ntl_all, dev);
      f.grab = grab_for(f.ntiles, f.ch, dev);
      f.cbase[0] = 0;
      int64_t act = nxl;  // segments with more than p levels (a prefix of xo)
      for (int p = 0; p < Pmax; ++p) {
        while (act > 0 && levels(xl[2 * xo[act - 1] + 1]) <= p) --act;
        f.ntl[p] = 0;
        for (int64_t j = 0; j < act; ++j) f.ntl[p] += (xl[2 * xo[j] + 1] + Tm - 1) / Tm;
        f.cbase[p + 1] = f.cbase[p] + (f.ntl[p] + f.ch - 1) / f.ch;
      }
      MSORT_CUDA_TRY(cudaMemsetAsync(done, 0, (size_t)Pmax * ntl_all * 4 + 256, s));
      MSORT_TRY(launch_k3(f, f.nchunks(), ctr, s, KC_MERGE));
    }
    MSORT_CUDA_TRY(cudaGetLastError());
    return MSORT_SUCCESS;
  }

  // First k-way round straight from the runs' owners (pull exchange): pair
  // m = runs (2m, 2m+1), each possibly in another GPU's memory, merged into
  // out at the sum of the earlier pairs' sizes (ties to the lower run).
  // Writes the run boundaries of the result (ceil(runs/2) runs) to off_out.
  static msort_status pull(const PullRuns& pr, K* out_k, uint32_t* out_v, int64_t* off_out,
                           unsigned long long* ctr, cudaStream_t s) {
    MSORT_TRY(init());
    int dev = 0;
    MSORT_CUDA_TRY(cudaGetDevice(&dev));
    if (pr.runs > 2 * kMaxPairs) {
      set_error("pull merge: too many runs");
      return MSORT_ERROR_NOT_SUPPORTED;
    }
    Peer src{};
    PeerPairs& pm = src.pm;
    pm.npairs = (pr.runs + 1) / 2;
    int64_t tiles = 0, out = 0;
    for (int m = 0; m < pm.npairs; ++m) {
      const int a = 2 * m, b = 2 * m + 1 < pr.runs ? 2 * m + 1 : -1;
      pm.first_tile[m] = tiles;
      pm.out[m] = out;
      off_out[m] = out;
      pm.na[m] = pr.n[a];
      pm.nb[m] = b >= 0 ? pr.n[b] : 0;
      pm.ka[m] = pr.k[a];
      pm.kb[m] = b >= 0 ? pr.k[b] : pr.k[a];
      pm.va[m] = PAIRS ? pr.v[a] : nullptr;
      pm.vb[m] = PAIRS ? (b >= 0 ? pr.v[b] : pr.v[a]) : nullptr;
      tiles += (pm.na[m] + pm.nb[m] + Tm - 1) / Tm;
      out += pm.na[m] + pm.nb[m];
    }
    pm.first_tile[pm.npairs] = tiles;
    off_out[pm.npairs] = out;
    if (tiles == 0) return MSORT_SUCCESS;
    src.dst_k = out_k, src.dst_v = out_v, src.ntiles = tiles;
    src.ch = chunk_tiles(tiles, dev);
    src.grab = grab_for(src.ntiles, src.ch, dev);
    MSORT_CUDA_TRY(cudaMemsetAsync(ctr, 0, kMaxLaunches * sizeof(unsigned long long), s));
    return launch_k3(src, (tiles + src.ch - 1) / src.ch, ctr, s, KC_KWAY);
  }

  // ---- K5: one-pass p-way merge (keys only; k5_kway.cuh) -------------
  static constexpr int K5NT = sizeof(K) == 4 ? 128 : 256;
  static constexpr int K5VT = sizeof(K) == 4 ? 68 : 34;
  static constexpr int K5MINB = sizeof(K) == 4 ? MSORT_K5_MINB : 2;
  using K5S = K5Shape<K5NT, K5VT>;
  // shared memory for any p (the capacity, and with it the buffer, is
  // largest for two runs)
  static constexpr size_t k5_smem = (size_t)K5S::keys(2) * sizeof(K);
  static int P2of(int p) {
    int P2 = 1;
    while (P2 < p) P2 <<= 1;
    return P2;
  }
  // Tile geometry for p runs of the given sizes: fills R.S, R.g, R.soff,
  // R.ntiles; returns the scratch bytes the partition needs.
  static size_t k5_plan(K5Runs& R) {
    const int p = R.p;
    const int64_t C = K5S::cap(P2of(p));
    R.g = MSORT_K5_G * (int64_t)p;  // merged samples per tile (utilisation g / (g + p))
    R.S = std::max<int64_t>(1, (C + p) / (R.g + p));  // tile <= S (g + p) - p <= C
    R.soff[0] = 0;
    for (int j = 0; j < p; ++j) R.soff[j + 1] = R.soff[j] + (R.n[j] + R.S - 1) / R.S;
    const int64_t M = R.soff[p];
    R.ntiles = std::max<int64_t>(1, (M + R.g - 1) / R.g);
    return 3 * align_up((size_t)M * sizeof(K), 256) + 3 * align_up((size_t)M * 4, 256) +
           align_up((size_t)(R.ntiles + 1) * p * 8, 256);
  }
  // Merge the runs of R (R.p in [2, kK5MaxRuns], R.k/R.n set) into dst in one
  // pass.  scratch: >= the bytes k5_plan returns, device memory not
  // overlapping the runs or dst.
  // Largest run count merged by K5 automatically: 8 (measured on 2^28 keys:
  // one K5 pass beats the ceil(log2 p) K3 rounds for p = 3..8 -- e.g. 1.12
  // vs 1.22 ms at p = 8 -- but not at 16: 1.74 vs 1.62 ms).  The environment
  // variable MSORT_K5 overrides it for A/B runs and tests: 0 = never, n =
  // up to n runs (<= 16).
  static int k5_max_runs() {
    const char* e = getenv("MSORT_K5");
    if (!e || !*e) return 8;
    return std::min(atoi(e), kK5MaxRuns);
  }
  static msort_status kway5(K5Runs R, K* dst, char* scratch, size_t scratch_bytes,
                            cudaStream_t s) {
    const int p = R.p;
    if (p < 2 || p > kK5MaxRuns) {
      set_error("k5: run count out of range");
      return MSORT_ERROR_NOT_SUPPORTED;
    }
    const size_t need = k5_plan(R);
    if (need > scratch_bytes) {
      set_error("k5: scratch too small");
      return MSORT_ERROR_INVALID_VALUE;
    }
    const int64_t M = R.soff[p];
    if (M == 0) return MSORT_SUCCESS;  // every run empty
    if (M >= ((int64_t)1 << 32)) {
      set_error("k5: too many samples");
      return MSORT_ERROR_NOT_SUPPORTED;
    }
    int dev = 0;
    MSORT_CUDA_TRY(cudaGetDevice(&dev));
    MSORT_TRY(k5_init(dev));
    const K5Bufs B = k5_carve(scratch, M, R.ntiles, p);
    // the sample-merge levels, planned here
    K5Level lv[kK5MaxLevels];
    int64_t lch[kK5MaxLevels];
    int levels = 0;
    {
      K5Level L{};
      L.q = p;
      for (int j = 0; j <= p; ++j) L.ro[j] = R.soff[j];
      while ((1 << levels) < p) ++levels;
      for (int l = 0; l < levels; ++l) {
        const int npair = (L.q + 1) / 2;
        int64_t ch = 0;
        for (int m = 0; m < npair; ++m) {
          L.c0[m] = ch;
          const int64_t len = L.ro[std::min(2 * m + 2, L.q)] - L.ro[2 * m];
          ch += (len + kK5LvlQ - 1) / kK5LvlQ;
        }
        L.c0[npair] = ch;
        lv[l] = L, lch[l] = ch;
        K5Level N{};
        N.q = npair;
        for (int m = 0; m <= N.q; ++m) N.ro[m] = L.ro[std::min(2 * m, L.q)];
        L = N;
      }
    }
    return k5_launch(R, lv, lch, levels, p, M, R.ntiles, B, dst, s);
  }

  // Scratch of one K5 merge for M samples and T tiles (k5_plan's layout).
  struct K5Bufs {
    K *skey, *tkey, *mkey;
    uint32_t *sid, *tid, *mid;
    int64_t* states;
  };
  static K5Bufs k5_carve(char* w, int64_t M, int64_t T, int p) {
    auto take = [&](size_t b) {
      char* q = w;
      w += align_up(b, 256);
      return q;
    };
    K5Bufs B;
    B.skey = reinterpret_cast<K*>(take((size_t)M * sizeof(K)));
    B.tkey = reinterpret_cast<K*>(take((size_t)M * sizeof(K)));
    B.mkey = reinterpret_cast<K*>(take((size_t)M * sizeof(K)));
    B.sid = reinterpret_cast<uint32_t*>(take((size_t)M * 4));
    B.tid = reinterpret_cast<uint32_t*>(take((size_t)M * 4));
    B.mid = reinterpret_cast<uint32_t*>(take((size_t)M * 4));
    B.states = reinterpret_cast<int64_t*>(take((size_t)(T + 1) * p * 8));
    return B;
  }

  // The K5 launches for a geometry given by value (RS = K5Runs, LS =
  // K5Level) or by device pointers (const K5Runs*, const K5Level*); Mgrid /
  // Tgrid / lch are the exact counts or, device-planned, upper bounds.
  template <class RS, class LS>
  static msort_status k5_launch(const RS& R, const LS* lv, const int64_t* lch, int levels, int p,
                                int64_t Mgrid, int64_t Tgrid, const K5Bufs& B, K* dst,
                                cudaStream_t s) {
    {
      LaunchScope ls(KC_PARTITION, s);
      k5_samples<K, RS><<<(unsigned)((Mgrid + 255) / 256), 256, 0, s>>>(R, B.skey, B.sid);
      // ceil(log2 p) levels of pairwise merges of the sample runs (ties to
      // the lower run), ping-ponging so the last lands in (mkey, mid); the
      // unmerged samples (skey) stay for the rank searches of k5_bounds
      const K* ck = B.skey;
      const uint32_t* cv = B.sid;
      for (int l = 0; l < levels; ++l) {
        const bool to_m = (levels - 1 - l) % 2 == 0;  // the last level writes (mkey, mid)
        K* nk = to_m ? B.mkey : B.tkey;
        uint32_t* nv = to_m ? B.mid : B.tid;
        if (lch[l] > 0)
          k5_sample_level<K, LS><<<(unsigned)lch[l], kK5LvlNT, 0, s>>>(lv[l], ck, cv, nk, nv);
        ck = nk, cv = nv;
      }
      const int64_t nb = (Tgrid + 1) * p;
      k5_bounds<K, RS><<<(unsigned)((nb + 255) / 256), 256, 0, s>>>(R, B.skey, ck, cv, B.states);
    }
    MSORT_CUDA_TRY(cudaGetLastError());
    if (Tgrid > 0) {
      LaunchScope ls(KC_KWAY, s);
      const int P2 = P2of(p);
      const unsigned T = (unsigned)Tgrid;
      if (P2 <= 2) k5_merge<K, K5NT, K5VT, K5MINB, 2, RS><<<T, K5NT, k5_smem, s>>>(R, B.states, dst);
      else if (P2 == 4) k5_merge<K, K5NT, K5VT, K5MINB, 4, RS><<<T, K5NT, k5_smem, s>>>(R, B.states, dst);
      else if (P2 == 8) k5_merge<K, K5NT, K5VT, K5MINB, 8, RS><<<T, K5NT, k5_smem, s>>>(R, B.states, dst);
      else k5_merge<K, K5NT, K5VT, K5MINB, 16, RS><<<T, K5NT, k5_smem, s>>>(R, B.states, dst);
    }
    MSORT_CUDA_TRY(cudaGetLastError());
#ifdef MSORT_K3_CHECK
    {
      cudaError_t e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) return cuda_fail(e, "k5 (debug sync)");
    }
#endif
    return MSORT_SUCCESS;
  }

  // K5 planned on the device (k5_plan_dev): rank `me` of p merges its
  // segments of every rank's sorted shard (split matrix `split` and shard
  // table `bases`, both device memory) into dst, n_out keys in all.  No host
  // synchronisation: the grids are upper bounds from n_out.  scratch: >=
  // k5_dev_bytes(n_out, p).
  static void k5_dev_geometry(int64_t n_out, int p, int64_t& S, int64_t& g, int64_t& Mmax,
                              int64_t& Tmax) {
    const int64_t C = K5S::cap(P2of(p));
    g = MSORT_K5_G * (int64_t)p;
    S = std::max<int64_t>(1, (C + p) / (g + p));
    Mmax = n_out / S + p;  // sum of ceil(n_j / S) <= n_out / S + p
    Tmax = std::max<int64_t>(1, (Mmax + g - 1) / g);
  }
  static size_t k5_dev_bytes(int64_t n_out, int p) {
    int64_t S, g, Mmax, Tmax;
    k5_dev_geometry(n_out, p, S, g, Mmax, Tmax);
    return 3 * align_up((size_t)Mmax * sizeof(K), 256) + 3 * align_up((size_t)Mmax * 4, 256) +
           align_up((size_t)(Tmax + 1) * p * 8, 256) + align_up(sizeof(K5Geo), 256);
  }
  static msort_status kway5_dev(const int64_t* split, int me, int p, const void* const* bases,
                                K* dst, int64_t n_out, char* scratch, size_t scratch_bytes,
                                cudaStream_t s) {
    if (p < 2 || p > kK5MaxRuns) {
      set_error("k5: run count out of range");
      return MSORT_ERROR_NOT_SUPPORTED;
    }
    if (k5_dev_bytes(n_out, p) > scratch_bytes) {
      set_error("k5: scratch too small");
      return MSORT_ERROR_INVALID_VALUE;
    }
    int64_t S, g, Mmax, Tmax;
    k5_dev_geometry(n_out, p, S, g, Mmax, Tmax);
    if (Mmax >= ((int64_t)1 << 32)) {
      set_error("k5: too many samples");
      return MSORT_ERROR_NOT_SUPPORTED;
    }
    int dev = 0;
    MSORT_CUDA_TRY(cudaGetDevice(&dev));
    MSORT_TRY(k5_init(dev));
    const K5Bufs B = k5_carve(scratch, Mmax, Tmax, p);
    K5Geo* G = reinterpret_cast<K5Geo*>(
        scratch + 3 * align_up((size_t)Mmax * sizeof(K), 256) + 3 * align_up((size_t)Mmax * 4, 256) +
        align_up((size_t)(Tmax + 1) * p * 8, 256));
    {
      LaunchScope ls(KC_PARTITION, s);
      k5_plan_dev<<<1, 32, 0, s>>>(G, split, me, p, bases, (int)sizeof(K), S, g);
    }
    MSORT_CUDA_TRY(cudaGetLastError());
    const K5Level* lv[kK5MaxLevels];
    int64_t lch[kK5MaxLevels];
    int levels = 0;
    while ((1 << levels) < p) ++levels;
    for (int l = 0; l < levels; ++l) lv[l] = &G->L[l], lch[l] = (Mmax + kK5LvlQ - 1) / kK5LvlQ + p;
    const K5Runs* Rp = &G->R;
    return k5_launch(Rp, lv, lch, levels, p, Mmax, Tmax, B, dst, s);
  }
  template <class RS>
  static msort_status k5_attr() {
    auto set = [](auto f) {
      return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k5_smem);
    };
    MSORT_CUDA_TRY(set(k5_merge<K, K5NT, K5VT, K5MINB, 2, RS>));
    MSORT_CUDA_TRY(set(k5_merge<K, K5NT, K5VT, K5MINB, 4, RS>));
    MSORT_CUDA_TRY(set(k5_merge<K, K5NT, K5VT, K5MINB, 8, RS>));
    MSORT_CUDA_TRY(set(k5_merge<K, K5NT, K5VT, K5MINB, 16, RS>));
    return MSORT_SUCCESS;
  }
  static msort_status k5_init(int dev) {
    static std::atomic<bool> done[64];
    if (done[dev & 63].load(std::memory_order_acquire)) return MSORT_SUCCESS;
    MSORT_TRY(k5_attr<K5Runs>());
    MSORT_TRY(k5_attr<const K5Runs*>());
    done[dev & 63].store(true, std::memory_order_release);
    return MSORT_SUCCESS;
  }

  // Merge `runs` consecutive runs src[off[r], off[r+1]) into dst with rounds of
  // pairwise merges (ties to the lower run: merge() left-first at every
  // round keeps the lower run on the left).
  static msort_status kway(K* src_k, uint32_t* src_v, K* tmp_k, uint32_t* tmp_v, K* dst_k,
                           uint32_t* dst_v, const int64_t* off_in, int runs,
                           unsigned long long* ctr, cudaStream_t s,
                           KernelClass kc = KC_KWAY) {
    MSORT_TRY(init());
    int dev = 0;
    MSORT_CUDA_TRY(cudaGetDevice(&dev));
    const int64_t n = off_in[runs] - off_in[0];
    if (runs <= 1 || n == 0) {
      if (n > 0 && src_k != dst_k) {
        MSORT_CUDA_TRY(cudaMemcpyAsync(dst_k, src_k + off_in[0], n * sizeof(K),
                                       cudaMemcpyDeviceToDevice, s));
        if (PAIRS)
          MSORT_CUDA_TRY(cudaMemcpyAsync(dst_v, src_v + off_in[0], n * sizeof(uint32_t),
                                         cudaMemcpyDeviceToDevice, s));
      }
      return MSORT_SUCCESS;
    }
    if ((runs + 1) / 2 > kMaxPairs) {
      set_error("k-way merge: too many runs");
      return MSORT_ERROR_NOT_SUPPORTED;
    }
    int rounds = 0;
    while ((1 << rounds) < runs) ++rounds;
    MSORT_CUDA_TRY(cudaMemsetAsync(ctr, 0, kMaxLaunches * sizeof(unsigned long long), s));
    // Ping-pong src -> (tmp|dst) ... so that the last round writes dst.
    int64_t off[2 * kMaxPairs + 2];
    for (int r = 0; r <= runs; ++r) off[r] = off_in[r] - off_in[0];
    K* ck = src_k + off_in[0];
    uint32_t* cv = PAIRS ? src_v + off_in[0] : nullptr;
    for (int round = 0; round < rounds; ++round) {
      // rounds-1-round remaining after this one: alternate so the last hits dst
      const bool to_dst = ((rounds - 1 - round) % 2) == 0;
      K* nk = to_dst ? dst_k : tmp_k;
      uint32_t* nv = to_dst ? dst_v : tmp_v;
      Explicit src{};
      ExplicitPairs& pm = src.pm;
      pm.npairs = (runs + 1) / 2;
      int64_t tiles = 0;
      for (int m = 0; m < pm.npairs; ++m) {
        pm.first_tile[m] = tiles;
        int64_t a = off[2 * m], bmid = off[std::min(2 * m + 1, runs)],
                e = off[std::min(2 * m + 2, runs)];
        pm.off[2 * m] = a;
        pm.off[2 * m + 1] = bmid;
        pm.off[2 * m + 2] = e;
        tiles += (e - a + Tm - 1) / Tm;
      }
      pm.first_tile[pm.npairs] = tiles;
      src.src_k = ck, src.src_v = cv, src.dst_k = nk, src.dst_v = nv, src.ntiles = tiles;
      // empty pairs own no tiles; locate() picks the last pair whose first
      // tile <= q, which is never an empty one
      if (tiles > 0) {
        src.ch = chunk_tiles(tiles, dev);
        src.grab = grab_for(src.ntiles, src.ch, dev);
        MSORT_TRY(launch_k3(src, (tiles + src.ch - 1) / src.ch, ctr + round, s, kc));
      }
      int nr = pm.npairs;
      for (int m = 0; m <= nr; ++m) off[m] = off[std::min(2 * m, runs)];
      runs = nr;
      ck = nk;
      cv = nv;
    }
    return MSORT_SUCCESS;
  }
};

// ---- key-range narrowing (8-byte keys) ----------------------------------
// The paper's arrays are numpy integers (int64) drawn from
// [0, n) with n <= 10^7, and C3's keys lie in [0, 1000): 8-byte
// keys that span fewer than 2^32 values.  Such a sort runs on 32-bit keys:
// key -> image(key) - min image, the 4-byte sort (half the key bytes of every
// merge pass, the 4-byte tile shape), then back.  The map is monotone and
// injective, so the output (keys, payload order: the stable order) is the
// one the 8-byte sort gives.  The choice is made on the device: both the
// narrowed and the 8-byte sort are enqueued, every kernel of each gated on
// the measured range (k_key_range), so the call stays asynchronous and
// graph-capturable; the path not taken launches kernels that return at once.
// The narrowing itself happens as the 4-byte sort's K1 loads the keys (k1_in).
template <class K>
__global__ void __launch_bounds__(256) k_key_range(const K* __restrict__ k, int64_t n,
                                                   unsigned long long* __restrict__ mm) {
  unsigned long long lo = ~0ull, hi = 0;
  const int64_t stride = (int64_t)gridDim.x * 256;
  int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    unsigned long long u[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) u[j] = KeyTraits<K>::image(k[i + j * stride]);
#pragma unroll
    for (int j = 0; j < 4; ++j) lo = min(lo, u[j]), hi = max(hi, u[j]);
  }
  for (; i < n; i += stride) {
    const unsigned long long u = KeyTraits<K>::image(k[i]);
    lo = min(lo, u), hi = max(hi, u);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, d));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, d));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&mm[0], lo);
    atomicMax(&mm[1], hi);
  }
}
template <class K>
__global__ void __launch_bounds__(256) k_key_widen(const uint32_t* __restrict__ u, int64_t n,
                                                   const unsigned long long* __restrict__ mm,
                                                   K* __restrict__ k) {
  if (!range_narrow(mm)) return;
  const unsigned long long lo = mm[0];
  const int64_t stride = (int64_t)gridDim.x * 256;
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += stride)
    k[i] = key_from_image<K>(lo + u[i]);
}

// MSORT_NARROW=0 (environment) disables the narrowing (A/B, tests)
static bool narrow_enabled() {
  const char* e = getenv("MSORT_NARROW");
  return !(e && *e == '0');
}

// Workspace (single_ws_bytes for 8-byte keys): [ 32-bit keys | the 4-byte
// sort's workspace ] overlapping the 8-byte sort's, the range in the last
// 256 bytes.  Only one of the two sorts does work; the other's launches
// (and its counter memsets, enqueued before or after the whole working
// path) touch nothing the working path still needs.
template <class K, bool PAIRS>
static msort_status sort_narrowed(const K* ik, const uint32_t* iv, K* keys, uint32_t* vals,
                                  size_t n, void* ws, cudaStream_t s) {
  const msort_dtype kd = K(-1) < K(0) ? MSORT_INT64 : MSORT_UINT64;
  const msort_dtype vd = PAIRS ? MSORT_UINT32 : MSORT_NONE;
  const size_t need = single_ws_bytes(n, kd, vd);
  char* w = static_cast<char*>(ws);
  auto* mm = reinterpret_cast<unsigned long long*>(w + need - 256);
  uint32_t* nk = reinterpret_cast<uint32_t*>(w);
  void* ws32 = w + align_up(n * 4, 256);
  const size_t ws32_bytes = single_ws_bytes(n, MSORT_UINT32, vd);
  int dev = 0, sms = 0;
  MSORT_CUDA_TRY(cudaGetDevice(&dev));
  MSORT_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const unsigned grid = (unsigned)std::max<int64_t>(
      1, std::min<int64_t>((int64_t)sms * 8, ((int64_t)n + 255) / 256));
  MSORT_CUDA_TRY(cudaMemsetAsync(mm, 0xff, 8, s));
  MSORT_CUDA_TRY(cudaMemsetAsync(mm + 1, 0, 8, s));
  {
    LaunchScope ls(KC_KEY_RANGE, s);
    k_key_range<K><<<grid, 256, 0, s>>>(ik, (int64_t)n, mm);
  }
  MSORT_CUDA_TRY(cudaGetLastError());
  // the 4-byte sort's K1 reads the 8-byte keys and narrows them as it loads
  // them (k1_in): no separate narrow pass
  MSORT_TRY((Kernels<uint32_t, PAIRS>::sort(nk, iv, nk, vals, n, ws32, ws32_bytes, s, mm, 1, ik,
                                            K(-1) < K(0) ? 1 : 2)));
  {
    LaunchScope ls(KC_KEY_RANGE, s);
    k_key_widen<K><<<grid, 256, 0, s>>>(nk, (int64_t)n, mm, keys);
  }
  MSORT_CUDA_TRY(cudaGetLastError());
  return Kernels<K, PAIRS>::sort(ik, iv, keys, vals, n, ws, need - 256, s, mm, 0);
}

template <class K>
static msort_status sort_k(const void* ik, const void* iv, void* keys, void* vals, size_t n,
                           void* ws, size_t ws_bytes, cudaStream_t s) {
#ifndef MSORT_K3_PERPASS
  if constexpr (sizeof(K) == 8) {
    if (n > (size_t)kK0MaxN && narrow_enabled()) {
      if (vals)
        return sort_narrowed<K, true>((const K*)ik, (const uint32_t*)iv, (K*)keys,
                                      (uint32_t*)vals, n, ws, s);
      return sort_narrowed<K, false>((const K*)ik, nullptr, (K*)keys, nullptr, n, ws, s);
    }
  }
#endif
  if (vals)
    return Kernels<K, true>::sort((const K*)ik, (const uint32_t*)iv, (K*)keys, (uint32_t*)vals,
                                  n, ws, ws_bytes, s);
  return Kernels<K, false>::sort((const K*)ik, nullptr, (K*)keys, nullptr, n, ws, ws_bytes, s);
}

msort_status sort_single_dispatch(const void* in_keys, const void* in_vals, void* keys,
                                  void* vals, size_t n, msort_dtype kd, msort_dtype vd, void* ws,
                                  size_t ws_bytes, cudaStream_t s) {
  if (vd == MSORT_NONE) vals = nullptr, in_vals = nullptr;
  switch (kd) {
    case MSORT_INT32: return sort_k<int32_t>(in_keys, in_vals, keys, vals, n, ws, ws_bytes, s);
    case MSORT_UINT32: return sort_k<uint32_t>(in_keys, in_vals, keys, vals, n, ws, ws_bytes, s);
    case MSORT_INT64: return sort_k<int64_t>(in_keys, in_vals, keys, vals, n, ws, ws_bytes, s);
    case MSORT_UINT64: return sort_k<uint64_t>(in_keys, in_vals, keys, vals, n, ws, ws_bytes, s);
    default: set_error("unknown key dtype"); return MSORT_ERROR_INVALID_VALUE;
  }
}

template <class K>
static msort_status seg_k(void* keys, void* vals, const int64_t* off, size_t nseg, bool dev_off,
                          int64_t n, void* ws, size_t ws_bytes, cudaStream_t s) {
  if (vals)
    return Kernels<K, true>::sort_segmented((K*)keys, (uint32_t*)vals, off, nseg, dev_off, n, ws,
                                            ws_bytes, s);
  return Kernels<K, false>::sort_segmented((K*)keys, nullptr, off, nseg, dev_off, n, ws, ws_bytes,
                                           s);
}

msort_status sort_segmented_dispatch(void* keys, void* vals, const int64_t* off, size_t nseg,
                                     bool dev_off, size_t n, msort_dtype kd, msort_dtype vd,
                                     void* ws, size_t ws_bytes, cudaStream_t s) {
  if (vd == MSORT_NONE) vals = nullptr;
  const int64_t nn = (int64_t)n;
  switch (kd) {
    case MSORT_INT32: return seg_k<int32_t>(keys, vals, off, nseg, dev_off, nn, ws, ws_bytes, s);
    case MSORT_UINT32: return seg_k<uint32_t>(keys, vals, off, nseg, dev_off, nn, ws, ws_bytes, s);
    case MSORT_INT64: return seg_k<int64_t>(keys, vals, off, nseg, dev_off, nn, ws, ws_bytes, s);
    case MSORT_UINT64: return seg_k<uint64_t>(keys, vals, off, nseg, dev_off, nn, ws, ws_bytes, s);
    default: set_error("unknown key dtype"); return MSORT_ERROR_INVALID_VALUE;
  }
}

template <class K>
static msort_status kway_k(void* sk, void* sv, void* tk, void* tv, void* dk, void* dv,
                           const int64_t* off, int runs, unsigned long long* ctr, cudaStream_t s) {
  if (sv)
    return Kernels<K, true>::kway((K*)sk, (uint32_t*)sv, (K*)tk, (uint32_t*)tv, (K*)dk,
                                  (uint32_t*)dv, off, runs, ctr, s);
  return Kernels<K, false>::kway((K*)sk, nullptr, (K*)tk, nullptr, (K*)dk, nullptr, off, runs,
                                 ctr, s);
}

msort_status kway_merge_dispatch(void* src_k, void* src_v, void* tmp_k, void* tmp_v,
                                 void* dst_k, void* dst_v, const int64_t* off_host, int runs,
                                 msort_dtype kd, msort_dtype vd, void* part_ws,
                                 cudaStream_t s) {
  auto* ctr = static_cast<unsigned long long*>(part_ws);  // scheduler counter
  if (vd == MSORT_NONE) src_v = tmp_v = dst_v = nullptr;
  switch (kd) {
    case MSORT_INT32:
      return kway_k<int32_t>(src_k, src_v, tmp_k, tmp_v, dst_k, dst_v, off_host, runs, ctr, s);
    case MSORT_UINT32:
      return kway_k<uint32_t>(src_k, src_v, tmp_k, tmp_v, dst_k, dst_v, off_host, runs, ctr, s);
    case MSORT_INT64:
      return kway_k<int64_t>(src_k, src_v, tmp_k, tmp_v, dst_k, dst_v, off_host, runs, ctr, s);
    case MSORT_UINT64:
      return kway_k<uint64_t>(src_k, src_v, tmp_k, tmp_v, dst_k, dst_v, off_host, runs, ctr, s);
    default: set_error("unknown key dtype"); return MSORT_ERROR_INVALID_VALUE;
  }
}

template <class K>
static msort_status pull_k(const PullRuns& pr, void* ok, void* ov, int64_t* off,
                           unsigned long long* ctr, cudaStream_t s) {
  if (ov) return Kernels<K, true>::pull(pr, (K*)ok, (uint32_t*)ov, off, ctr, s);
  return Kernels<K, false>::pull(pr, (K*)ok, nullptr, off, ctr, s);
}

msort_status pull_round_dispatch(const PullRuns& pr, void* out_k, void* out_v, int64_t* off_out,
                                 msort_dtype kd, msort_dtype vd, void* part_ws, cudaStream_t s) {
  auto* ctr = static_cast<unsigned long long*>(part_ws);
  if (vd == MSORT_NONE) out_v = nullptr;
  switch (kd) {
    case MSORT_INT32: return pull_k<int32_t>(pr, out_k, out_v, off_out, ctr, s);
    case MSORT_UINT32: return pull_k<uint32_t>(pr, out_k, out_v, off_out, ctr, s);
    case MSORT_INT64: return pull_k<int64_t>(pr, out_k, out_v, off_out, ctr, s);
    case MSORT_UINT64: return pull_k<uint64_t>(pr, out_k, out_v, off_out, ctr, s);
    default: set_error("unknown key dtype"); return MSORT_ERROR_INVALID_VALUE;
  }
}

template <class K>
static msort_status kway5_k(const PullRuns& pr, void* dst, void* scratch, size_t bytes,
                            cudaStream_t s) {
  K5Runs R{};
  R.p = pr.runs;
  for (int j = 0; j < pr.runs; ++j) R.k[j] = pr.k[j], R.n[j] = pr.n[j];
  return Kernels<K, false>::kway5(R, (K*)dst, (char*)scratch, bytes, s);
}

msort_status kway5_dispatch(const PullRuns& pr, void* dst, msort_dtype kd, void* scratch,
                            size_t scratch_bytes, cudaStream_t s) {
  if (pr.runs < 2 || pr.runs > kK5MaxRuns) {
    set_error("k5: run count out of range");
    return MSORT_ERROR_NOT_SUPPORTED;
  }
  switch (kd) {
    case MSORT_INT32: return kway5_k<int32_t>(pr, dst, scratch, scratch_bytes, s);
    case MSORT_UINT32: return kway5_k<uint32_t>(pr, dst, scratch, scratch_bytes, s);
    case MSORT_INT64: return kway5_k<int64_t>(pr, dst, scratch, scratch_bytes, s);
    case MSORT_UINT64: return kway5_k<uint64_t>(pr, dst, scratch, scratch_bytes, s);
    default: set_error("unknown key dtype"); return MSORT_ERROR_INVALID_VALUE;
  }
}

size_t kway5_dev_bytes(int64_t n_out, int p, msort_dtype kd) {
  return dtype_size(kd) == 4 ? Kernels<int32_t, false>::k5_dev_bytes(n_out, p)
                             : Kernels<int64_t, false>::k5_dev_bytes(n_out, p);
}

msort_status kway5_dev_dispatch(const int64_t* split, int me, int p, const void* const* bases,
                                void* dst, int64_t n_out, msort_dtype kd, void* scratch,
                                size_t scratch_bytes, cudaStream_t s) {
  switch (kd) {
#define K5D(T)                                                                                 \
  return Kernels<T, false>::kway5_dev(split, me, p, bases, (T*)dst, n_out, (char*)scratch,    \
                                      scratch_bytes, s)
    case MSORT_INT32: K5D(int32_t);
    case MSORT_UINT32: K5D(uint32_t);
    case MSORT_INT64: K5D(int64_t);
    case MSORT_UINT64: K5D(uint64_t);
#undef K5D
    default: set_error("unknown key dtype"); return MSORT_ERROR_INVALID_VALUE;
  }
}

template <class K>
static size_t kway5_bytes_k(const PullRuns& pr) {
  K5Runs R{};
  R.p = pr.runs;
  for (int j = 0; j < pr.runs; ++j) R.n[j] = pr.n[j];
  return Kernels<K, false>::k5_plan(R);
}

size_t kway5_scratch_bytes(const PullRuns& pr, msort_dtype kd) {
  // SIZE_MAX: K5 not applicable (run count) or disabled (MSORT_K5=0)
  if (pr.runs < 2 || pr.runs > Kernels<int32_t, false>::k5_max_runs()) return SIZE_MAX;
  return dtype_size(kd) == 4 ? kway5_bytes_k<int32_t>(pr) : kway5_bytes_k<int64_t>(pr);
}

// msort_merge_runs (include/msort.h): stable merge of p sorted runs of
// in_keys (run j = [off[j], off[j+1])), ties to the lower run, into keys_out.
// Keys only with 3..16 runs: one K5 pass; otherwise rounds of K3.
template <class K>
static size_t merge_runs_ws_k(size_t n, int p, bool pairs) {
  // K3 rounds: one ping-pong buffer (+ payloads) and the scheduler counters
  size_t b = align_up(n * sizeof(K), 256) + (pairs ? align_up(n * 4, 256) : 0) +
             align_up(kMaxLaunches * 8, 256);
  if (!pairs && p >= 3 && p <= kK5MaxRuns) {  // (any run count K5 may be asked for)
    // K5: the partition's sample arrays for the worst split of n over p runs
    K5Runs R{};
    R.p = p;
    for (int j = 0; j < p; ++j) R.n[j] = (int64_t)(n / p) + 1;
    size_t k5 = Kernels<K, false>::k5_plan(R);
    b = std::max(b, k5 + 4096);
  }
  return b;
}

size_t merge_runs_ws_bytes(size_t n, int p, msort_dtype kd, msort_dtype vd) {
  const bool pairs = vd != MSORT_NONE;
  return dtype_size(kd) == 4 ? merge_runs_ws_k<int32_t>(n, p, pairs)
                             : merge_runs_ws_k<int64_t>(n, p, pairs);
}

template <class K>
static msort_status merge_runs_k(const void* ik, const void* iv, const int64_t* off, int p,
                                 void* ok, void* ov, void* ws, size_t ws_bytes, cudaStream_t s) {
  const int64_t n = off[p] - off[0];
  if (!iv && p >= 3 && p <= Kernels<K, false>::k5_max_runs()) {
    K5Runs R{};
    R.p = p;
    for (int j = 0; j < p; ++j)
      R.k[j] = (const K*)ik + (off[j] - off[0]), R.n[j] = off[j + 1] - off[j];
    K5Runs Q = R;
    if (Kernels<K, false>::k5_plan(Q) <= ws_bytes)
      return Kernels<K, false>::kway5(R, (K*)ok, (char*)ws, ws_bytes, s);
  }
  char* w = (char*)ws;
  K* tk = (K*)w;
  w += align_up((size_t)n * sizeof(K), 256);
  uint32_t* tv = nullptr;
  if (iv) {
    tv = (uint32_t*)w;
    w += align_up((size_t)n * 4, 256);
  }
  auto* ctr = reinterpret_cast<unsigned long long*>(w);
  if (iv)
    return Kernels<K, true>::kway((K*)ik, (uint32_t*)iv, tk, tv, (K*)ok, (uint32_t*)ov, off, p,
                                  ctr, s);
  return Kernels<K, false>::kway((K*)ik, nullptr, tk, nullptr, (K*)ok, nullptr, off, p, ctr, s);
}

msort_status merge_runs_dispatch(const void* ik, const void* iv, const int64_t* off, int p,
                                 void* ok, void* ov, msort_dtype kd, msort_dtype vd, void* ws,
                                 size_t ws_bytes, cudaStream_t s) {
  if (vd == MSORT_NONE) iv = nullptr, ov = nullptr;
  switch (kd) {
    case MSORT_INT32: return merge_runs_k<int32_t>(ik, iv, off, p, ok, ov, ws, ws_bytes, s);
    case MSORT_UINT32: return merge_runs_k<uint32_t>(ik, iv, off, p, ok, ov, ws, ws_bytes, s);
    case MSORT_INT64: return merge_runs_k<int64_t>(ik, iv, off, p, ok, ov, ws, ws_bytes, s);
    case MSORT_UINT64: return merge_runs_k<uint64_t>(ik, iv, off, p, ok, ov, ws, ws_bytes, s);
    default: set_error("unknown key dtype"); return MSORT_ERROR_INVALID_VALUE;
  }
}

int tile_size_for(msort_dtype kd, msort_dtype vd) {
  bool p = vd != MSORT_NONE;
  switch (kd) {
    case MSORT_INT32:
    case MSORT_UINT32: return p ? Kernels<int32_t, true>::T : Kernels<int32_t, false>::T;
    case MSORT_INT64:
    case MSORT_UINT64: return p ? Kernels<int64_t, true>::T : Kernels<int64_t, false>::T;
    default: return 0;
  }
}

}  // namespace msort

extern "C" int msort_debug_set_quad(int mode) {
  msort::g_quad_mode.store(mode == 5 ? 5 : 0);
  return 0;
}
