// sort_single.cu -- single-GPU stable merge sort for sm_100a.
//
//   K1 k1_tile_sort     : each T-element tile sorted in registers + shared
//                         memory (the base case of the recursion, P:77-84;
//                         the chunk sort of the multiprocessing variant,
//                         P:270-285; `SMALLEST_ARRAY_SIZE` of P:121 = T).
//   K2 k2_partition     : merge-path co-rank of every output tile's first
//                         diagonal inside its run pair (global binary search).
//   K3 k3_merge_pass    : merges run pairs of length L into 2L (merge()),
//                         one output tile per CTA, staged through shared memory.
//   S4 placement        : K1's destination is picked from the parity of the
//                         merge-pass count so that the last pass lands in keys.
//
// "P:n" = /root/reference/PAPER.md line n.
#include <algorithm>
#include <cstdio>

#include "msort_device.cuh"
#include "msort_internal.h"

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
};

// ----------------------------------------------------------------- K1
template <class K, bool PAIRS, int NT, int VT>
__global__ void __launch_bounds__(NT)
    k1_tile_sort(const K* __restrict__ in_k, const uint32_t* __restrict__ in_v,
                 K* __restrict__ out_k, uint32_t* __restrict__ out_v, int64_t n) {
  constexpr int T = NT * VT;
  constexpr int TP = padded_len<K, T>();
  extern __shared__ __align__(16) unsigned char smem[];
  K* sk = reinterpret_cast<K*>(smem);
  int* si = reinterpret_cast<int*>(sk + TP);      // PAIRS: original in-tile index
  uint32_t* sv = reinterpret_cast<uint32_t*>(si + TP);  // PAIRS: payload staging

  const int tid = threadIdx.x;
  const int64_t base = (int64_t)blockIdx.x * T;
  const int cnt = (int)min((int64_t)T, n - base);

  // Load the tile; pad the partial last tile with the maximum key AFTER the
  // real elements, so the stable order keeps real keys first.
#pragma unroll 4
  for (int i = tid; i < T; i += NT) {
    sk[sidx<K, true>(i)] = i < cnt ? in_k[base + i] : KeyTraits<K>::max_key();
    if constexpr (PAIRS) {
      if (i < cnt) sv[i] = in_v[base + i];
    }
  }
  __syncthreads();

  K key[VT];
  int idx[VT];
#pragma unroll
  for (int k = 0; k < VT; ++k) {
    key[k] = sk[sidx<K, true>(tid * VT + k)];
    idx[k] = tid * VT + k;
  }
  // Per-thread register network.
  if constexpr (PAIRS) odd_even_transposition_sort<VT>(key, idx);
  else batcher_sort<VT>(key);

  // In-block merge rounds: runs of w -> 2w, merge path per thread.
#pragma unroll 1
  for (int w = VT; w < T; w *= 2) {
    __syncthreads();
#pragma unroll
    for (int k = 0; k < VT; ++k) {
      sk[sidx<K, true>(tid * VT + k)] = key[k];
      if constexpr (PAIRS) si[sidx<K, true>(tid * VT + k)] = idx[k];
    }
    __syncthreads();
    const int tpg = 2 * w / VT;  // threads per merge group
    const int g0 = (tid / tpg) * 2 * w;
    const int d = (tid % tpg) * VT;
    int i = merge_path<K, true>(sk, g0, w, g0 + w, w, d);
    serial_merge<K, true, PAIRS, VT>(sk, PAIRS ? si : nullptr, g0 + i, g0 + w, g0 + w + d - i,
                                     g0 + 2 * w, key, idx);
  }

  __syncthreads();
#pragma unroll
  for (int k = 0; k < VT; ++k) {
    sk[sidx<K, true>(tid * VT + k)] = key[k];
    if constexpr (PAIRS) si[sidx<K, true>(tid * VT + k)] = idx[k];
  }
  __syncthreads();
#pragma unroll 4
  for (int i = tid; i < cnt; i += NT) {
    out_k[base + i] = sk[sidx<K, true>(i)];
    if constexpr (PAIRS) out_v[base + i] = sv[si[sidx<K, true>(i)]];
  }
}

// ----------------------------------------------------------------- K2
template <class K, class PM>
__global__ void __launch_bounds__(256)
    k2_partition(const K* __restrict__ src, PM pm, int64_t ntiles, int T,
                 int64_t* __restrict__ part) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= ntiles) return;
  int64_t A0, na, nb, dl;
  pm.locate(q, T, A0, na, nb, dl);
  part[q] = merge_path_global(src + A0, na, src + A0 + na, nb, dl);
}

// ----------------------------------------------------------------- K3
template <class K, bool PAIRS, int NT, int VT, class PM>
__global__ void __launch_bounds__(NT)
    k3_merge_pass(const K* __restrict__ src_k, const uint32_t* __restrict__ src_v,
                  K* __restrict__ dst_k, uint32_t* __restrict__ dst_v, PM pm,
                  const int64_t* __restrict__ part) {
  constexpr int T = NT * VT;
  constexpr int TP = padded_len<K, T>();
  extern __shared__ __align__(16) unsigned char smem[];
  K* sin = reinterpret_cast<K*>(smem);              // staged A|B window (T)
  K* sout = sin + T;                                // padded output (TP)
  int* spos = reinterpret_cast<int*>(sout + TP);    // PAIRS: source position
  uint32_t* sv = reinterpret_cast<uint32_t*>(spos + TP);  // PAIRS: staged payload

  const int tid = threadIdx.x;
  const int64_t q = blockIdx.x;
  int64_t A0, na_all, nb_all, d0;
  pm.locate(q, T, A0, na_all, nb_all, d0);
  const int64_t tot_all = na_all + nb_all;
  const int64_t d1 = min(d0 + T, tot_all);
  const int64_t i0 = part[q];
  const int64_t i1 = d1 == tot_all ? na_all : part[q + 1];
  const int64_t j0 = d0 - i0, j1 = d1 - i1;
  const int na = (int)(i1 - i0), nb = (int)(j1 - j0), tot = na + nb;
  const K* a = src_k + A0 + i0;
  const K* b = src_k + A0 + na_all + j0;

#pragma unroll 4
  for (int i = tid; i < tot; i += NT) {
    sin[i] = i < na ? a[i] : b[i - na];
    if constexpr (PAIRS) sv[i] = i < na ? src_v[A0 + i0 + i] : src_v[A0 + na_all + j0 + i - na];
  }
  __syncthreads();

  K key[VT];
  int pos[VT];
  const int d = tid * VT;
  if (d < tot) {
    int i = merge_path<K, false>(sin, 0, na, na, nb, d);
    serial_merge<K, false, PAIRS, VT>(sin, nullptr, i, na, na + d - i, tot, key, pos);
  }
#pragma unroll
  for (int k = 0; k < VT; ++k) {
    if (d + k < tot) {
      sout[sidx<K, true>(d + k)] = key[k];
      if constexpr (PAIRS) spos[sidx<K, true>(d + k)] = pos[k];
    }
  }
  __syncthreads();
  K* out = dst_k + A0 + d0;
#pragma unroll 4
  for (int i = tid; i < tot; i += NT) {
    out[i] = sout[sidx<K, true>(i)];
    if constexpr (PAIRS) dst_v[A0 + d0 + i] = sv[spos[sidx<K, true>(i)]];
  }
}

// ------------------------------------------------------------ host driver
template <class K, bool PAIRS>
struct Kernels {
  using G = Geometry<K, PAIRS>;
  static constexpr int NT = G::NT, VT = G::VT, T = G::T;
  static constexpr int TP = padded_len<K, T>();
  static constexpr size_t k1_smem =
      TP * sizeof(K) + (PAIRS ? TP * sizeof(int) + T * sizeof(uint32_t) : 0);
  static constexpr size_t k3_smem =
      (T + TP) * sizeof(K) + (PAIRS ? TP * sizeof(int) + T * sizeof(uint32_t) : 0);

  static msort_status init() {
    static bool done = false;
    static msort_status st = MSORT_SUCCESS;
    if (done) return st;
    cudaError_t e = cudaFuncSetAttribute(k1_tile_sort<K, PAIRS, NT, VT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)k1_smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k3_merge_pass<K, PAIRS, NT, VT, UniformPairs>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k3_smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k3_merge_pass<K, PAIRS, NT, VT, ExplicitPairs>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k3_smem);
    st = e == cudaSuccess ? MSORT_SUCCESS : cuda_fail(e, "cudaFuncSetAttribute");
    done = true;
    return st;
  }

  template <class PM>
  static msort_status merge_pass(const K* sk, const uint32_t* sv, K* dk, uint32_t* dv,
                                 const PM& pm, int64_t ntiles, int64_t* part, cudaStream_t s,
                                 KernelClass kc) {
    {
      LaunchScope ls(KC_PARTITION, s);
      unsigned g = (unsigned)((ntiles + 255) / 256);
      k2_partition<K, PM><<<g, 256, 0, s>>>(sk, pm, ntiles, T, part);
    }
    {
      LaunchScope ls(kc, s);
      k3_merge_pass<K, PAIRS, NT, VT, PM>
          <<<(unsigned)ntiles, NT, k3_smem, s>>>(sk, sv, dk, dv, pm, part);
    }
    MSORT_CUDA_TRY(cudaGetLastError());
    return MSORT_SUCCESS;
  }

  // Sort in_k/in_v into out_k/out_v (in == out: in place; K1 reads a whole
  // tile into shared memory before writing it back, so that is safe).
  static msort_status sort(const K* in_k, const uint32_t* in_v, K* keys, uint32_t* vals,
                           size_t n, void* ws, size_t ws_bytes, cudaStream_t s) {
    MSORT_TRY(init());
    if (n < 2) {
      if (n == 1 && in_k != keys) {
        MSORT_CUDA_TRY(cudaMemcpyAsync(keys, in_k, sizeof(K), cudaMemcpyDeviceToDevice, s));
        if (PAIRS)
          MSORT_CUDA_TRY(cudaMemcpyAsync(vals, in_v, 4, cudaMemcpyDeviceToDevice, s));
      }
      return MSORT_SUCCESS;
    }
    const int64_t ntiles = (int64_t)((n + T - 1) / T);
    int passes = 0;
    while ((int64_t(1) << passes) < ntiles) ++passes;
    char* w = static_cast<char*>(ws);
    K* wk = reinterpret_cast<K*>(w);
    w += align_up(n * sizeof(K), 256);
    uint32_t* wv = nullptr;
    if (PAIRS) {
      wv = reinterpret_cast<uint32_t*>(w);
      w += align_up(n * sizeof(uint32_t), 256);
    }
    int64_t* part = reinterpret_cast<int64_t*>(w);
    (void)ws_bytes;

    K* bk[2] = {keys, wk};
    uint32_t* bv[2] = {vals, wv};
    int cur = passes % 2;  // S4: pick K1's destination so the last pass lands in keys
    {
      LaunchScope ls(KC_TILE_SORT, s);
      k1_tile_sort<K, PAIRS, NT, VT>
          <<<(unsigned)ntiles, NT, k1_smem, s>>>(in_k, in_v, bk[cur], bv[cur], (int64_t)n);
    }
    MSORT_CUDA_TRY(cudaGetLastError());
    for (int64_t L = T; L < (int64_t)n; L *= 2) {
      UniformPairs pm{(int64_t)n, L};
      MSORT_TRY(merge_pass(bk[cur], bv[cur], bk[cur ^ 1], bv[cur ^ 1], pm, ntiles, part, s,
                           KC_MERGE));
      cur ^= 1;
    }
    return MSORT_SUCCESS;
  }

  // Merge `runs` consecutive runs src[off[r], off[r+1]) into dst with rounds of
  // pairwise merges (ties to the lower run: merge() left-first at every
  // round keeps the lower run on the left).
  static msort_status kway(K* src_k, uint32_t* src_v, K* tmp_k, uint32_t* tmp_v, K* dst_k,
                           uint32_t* dst_v, const int64_t* off_in, int runs, int64_t* part,
                           cudaStream_t s) {
    MSORT_TRY(init());
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
    // Ping-pong src -> (tmp|dst) ... so that the last round writes dst.
    int64_t off[2 * kMaxPairs + 2];
    for (int r = 0; r <= runs; ++r) off[r] = off_in[r] - off_in[0];
    K* ck = src_k + off_in[0];
    uint32_t* cv = PAIRS ? src_v + off_in[0] : nullptr;
    for (int round = 0; round < rounds; ++round) {
      const bool last = round == rounds - 1;
      // rounds-1-round remaining after this one: alternate so the last hits dst
      const bool to_dst = ((rounds - 1 - round) % 2) == 0;
      K* nk = to_dst ? dst_k : tmp_k;
      uint32_t* nv = to_dst ? dst_v : tmp_v;
      ExplicitPairs pm{};
      pm.npairs = (runs + 1) / 2;
      int64_t tiles = 0;
      for (int m = 0; m < pm.npairs; ++m) {
        pm.first_tile[m] = tiles;
        int64_t a = off[2 * m], bmid = off[std::min(2 * m + 1, runs)],
                e = off[std::min(2 * m + 2, runs)];
        pm.off[2 * m] = a;
        pm.off[2 * m + 1] = bmid;
        pm.off[2 * m + 2] = e;
        tiles += (e - a + T - 1) / T;
      }
      pm.first_tile[pm.npairs] = tiles;
      // skip empty pairs in the tile map: first_tile is non-decreasing and
      // locate() takes the last pair whose first tile <= q, which is non-empty
      if (tiles > 0) MSORT_TRY(merge_pass(ck, cv, nk, nv, pm, tiles, part, s, KC_KWAY));
      // new runs: pair outputs
      int nr = pm.npairs;
      for (int m = 0; m <= nr; ++m) off[m] = off[std::min(2 * m, runs)];
      runs = nr;
      ck = nk;
      cv = nv;
      (void)last;
    }
    return MSORT_SUCCESS;
  }
};

template <class K>
static msort_status sort_k(const void* ik, const void* iv, void* keys, void* vals, size_t n,
                           void* ws, size_t ws_bytes, cudaStream_t s) {
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
static msort_status kway_k(void* sk, void* sv, void* tk, void* tv, void* dk, void* dv,
                           const int64_t* off, int runs, void* part, cudaStream_t s) {
  if (sv)
    return Kernels<K, true>::kway((K*)sk, (uint32_t*)sv, (K*)tk, (uint32_t*)tv, (K*)dk,
                                  (uint32_t*)dv, off, runs, (int64_t*)part, s);
  return Kernels<K, false>::kway((K*)sk, nullptr, (K*)tk, nullptr, (K*)dk, nullptr, off, runs,
                                 (int64_t*)part, s);
}

msort_status kway_merge_dispatch(void* src_k, void* src_v, void* tmp_k, void* tmp_v,
                                 void* dst_k, void* dst_v, const int64_t* off_host, int runs,
                                 msort_dtype kd, msort_dtype vd, void* part_ws,
                                 cudaStream_t s) {
  if (vd == MSORT_NONE) src_v = tmp_v = dst_v = nullptr;
  switch (kd) {
    case MSORT_INT32:
      return kway_k<int32_t>(src_k, src_v, tmp_k, tmp_v, dst_k, dst_v, off_host, runs, part_ws, s);
    case MSORT_UINT32:
      return kway_k<uint32_t>(src_k, src_v, tmp_k, tmp_v, dst_k, dst_v, off_host, runs, part_ws, s);
    case MSORT_INT64:
      return kway_k<int64_t>(src_k, src_v, tmp_k, tmp_v, dst_k, dst_v, off_host, runs, part_ws, s);
    case MSORT_UINT64:
      return kway_k<uint64_t>(src_k, src_v, tmp_k, tmp_v, dst_k, dst_v, off_host, runs, part_ws, s);
    default: set_error("unknown key dtype"); return MSORT_ERROR_INVALID_VALUE;
  }
}

int tile_size_for(msort_dtype kd, msort_dtype vd) {
  bool p = vd != MSORT_NONE;
  switch (kd) {
    case MSORT_INT32:
    case MSORT_UINT32: return p ? Geometry<int32_t, true>::T : Geometry<int32_t, false>::T;
    case MSORT_INT64:
    case MSORT_UINT64: return p ? Geometry<int64_t, true>::T : Geometry<int64_t, false>::T;
    default: return 0;
  }
}

}  // namespace msort
