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
// NT threads x VT items (VT odd: "blocked" shared accesses at stride VT are
// bank-conflict free without padding).
template <class K, bool PAIRS, int NT, int VT>
__global__ void __launch_bounds__(NT)
    k1_tile_sort(const K* __restrict__ in_k, const uint32_t* __restrict__ in_v,
                 K* __restrict__ out_k, uint32_t* __restrict__ out_v, int64_t n) {
  constexpr int T = NT * VT;
  extern __shared__ __align__(16) unsigned char smem[];
  K* sk = reinterpret_cast<K*>(smem);                 // T keys
  int* si = reinterpret_cast<int*>(sk + T);           // PAIRS: original in-tile index
  uint32_t* sv = reinterpret_cast<uint32_t*>(si + T);  // PAIRS: payload staging

  const int tid = threadIdx.x;
  const int64_t base = (int64_t)blockIdx.x * T;
  const int cnt = (int)min((int64_t)T, n - base);

  // Load the tile; pad the partial last tile with the maximum key AFTER the
  // real elements, so the stable order keeps real keys first.
#pragma unroll 4
  for (int i = tid; i < T; i += NT) {
    sk[i] = i < cnt ? in_k[base + i] : KeyTraits<K>::max_key();
    if constexpr (PAIRS) {
      if (i < cnt) sv[i] = in_v[base + i];
    }
  }
  __syncthreads();

  K key[VT];
  int idx[VT];
#pragma unroll
  for (int k = 0; k < VT; ++k) {
    key[k] = sk[tid * VT + k];
    idx[k] = tid * VT + k;
  }
  // Per-thread register network.
  if constexpr (PAIRS) odd_even_transposition_sort<VT>(key, idx);
  else keys_network<VT>(key);

  // In-block merge rounds: runs of w -> 2w, merge path per thread.
#pragma unroll 1
  for (int w = VT; w < T; w *= 2) {
    __syncthreads();
#pragma unroll
    for (int k = 0; k < VT; ++k) {
      sk[tid * VT + k] = key[k];
      if constexpr (PAIRS) si[tid * VT + k] = idx[k];
    }
    __syncthreads();
    const int tpg = 2 * w / VT;  // threads per merge group
    const int g0 = (tid / tpg) * 2 * w;
    const int d = (tid % tpg) * VT;
    int i = merge_path<K, false>(sk, g0, w, g0 + w, w, d);
    serial_merge<K, false, PAIRS, VT>(sk, PAIRS ? si : nullptr, g0 + i, g0 + w, g0 + w + d - i,
                                      g0 + 2 * w, T - 1, key, idx);
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

// ----------------------------------------------------------------- K3
struct TileMeta {
  int64_t out;  // global output index of the tile's first element
  int na, nb, offA, offB, offAv, offBv, tot, pad;
};

constexpr size_t align_up_c(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Shared memory of one K3 CTA: barriers, tile metadata, the co-rank ring and
// S stages.  A stage holds the staged A|B window of one output tile and is
// then overwritten in place by that tile's merged output, which leaves by a
// bulk store before the stage is handed back to the producer.
template <class K, bool PAIRS, int NC, int VT, int S>
struct K3Layout {
  static constexpr int Tm = NC * VT;
  static constexpr int EK = 16 / sizeof(K);
  static constexpr int R = 4;              // co-rank ring: R batches of 32
  static constexpr int SKE = Tm + 4 * EK;  // keys per stage (windows + phase slack)
  static constexpr int SVE = Tm + 16;      // payloads per stage
  static constexpr size_t bars = 0;        // full[S], empty[S], sfull[R], sempty[R]
  static constexpr size_t meta = 128;
  static constexpr size_t ring = meta + 48 * S;
  static constexpr size_t corank = ring + 8 * 32 * R;  // NC+1 ints: per-thread co-ranks
  static constexpr size_t stage_k = align_up_c(corank + 4 * (NC + 1), 128);
  static constexpr size_t stage_v = align_up_c(stage_k + (size_t)S * SKE * sizeof(K), 128);
  static constexpr size_t bytes = align_up_c(stage_v + (PAIRS ? (size_t)S * SVE * 4 : 0), 128);
};

// Persistent merge pass.  CTA c owns the contiguous tiles [t0, t0+cnt);
// warp 0 = TMA producer, warp 1 = co-rank searcher (K2), warps 2.. = mergers.
template <class K, bool PAIRS, int NC, int VT, int S, int MINB, class PM>
__global__ void __launch_bounds__(NC + 64, MINB)
    k3_merge_pass(const K* __restrict__ src_k, const uint32_t* __restrict__ src_v,
                  K* __restrict__ dst_k, uint32_t* __restrict__ dst_v, PM pm, int64_t ntiles) {
  using LY = K3Layout<K, PAIRS, NC, VT, S>;
  constexpr int Tm = LY::Tm, EK = LY::EK, R = LY::R;
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + LY::bars);
  uint64_t* empty = full + S;
  uint64_t* sfull = empty + S;
  uint64_t* sempty = sfull + R;
  TileMeta* meta = reinterpret_cast<TileMeta*>(smem + LY::meta);
  int64_t* ring = reinterpret_cast<int64_t*>(smem + LY::ring);
  K* stk = reinterpret_cast<K*>(smem + LY::stage_k);
  uint32_t* stv = reinterpret_cast<uint32_t*>(smem + LY::stage_v);
  int* corank = reinterpret_cast<int*>(smem + LY::corank);
  constexpr bool DUAL = (VT % 2) == 0;  // even: two chains per thread
  constexpr int H = VT / 2;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // contiguous tile range of this CTA
  const int64_t G = gridDim.x, per = ntiles / G, rem = ntiles % G, c = blockIdx.x;
  const int64_t t0 = c * per + min(c, rem);
  const int64_t cnt = per + (c < rem ? 1 : 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 32), mbar_init(&empty[s], 1);
    for (int r = 0; r < R; ++r) mbar_init(&sfull[r], 32), mbar_init(&sempty[r], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (cnt == 0) return;
  const int64_t nsplit = cnt + 1;  // co-ranks of local diagonals 0..cnt
  const int64_t nbatch = (nsplit + 31) / 32;

  if (warp == 1) {
    // ------------------------------------------------ co-rank searcher (K2)
    for (int64_t b = 0; b < nbatch; ++b) {
      const int r = (int)(b % R);
      const uint32_t u = (uint32_t)(b / R);
      mbar_wait(&sempty[r], (u & 1) ^ 1);
      const int64_t j = b * 32 + lane;
      int64_t v = 0;
      if (j < nsplit && t0 + j < ntiles) {
        int64_t A0, na, nb, dl;
        pm.locate(t0 + j, Tm, A0, na, nb, dl);
        v = merge_path_global(src_k + A0, na, src_k + A0 + na, nb, dl);
      }
      ring[r * 32 + lane] = v;
      mbar_arrive(&sfull[r]);
    }
  } else if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    for (int64_t k = 0; k < cnt; ++k) {
      const int64_t q = t0 + k;
      const int s = (int)(k % S);
      // co-ranks of diagonals k and k+1 (local), possibly in two batches
      const int64_t b0 = k / 32, b1 = (k + 1) / 32;
      mbar_wait(&sfull[b0 % R], (uint32_t)((b0 / R) & 1));
      if (b1 != b0) mbar_wait(&sfull[b1 % R], (uint32_t)((b1 / R) & 1));
      int64_t A0, na_all, nb_all, d0;
      pm.locate(q, Tm, A0, na_all, nb_all, d0);
      const int64_t tot_all = na_all + nb_all;
      const int64_t d1 = min(d0 + Tm, tot_all);
      const int64_t i0 = ring[(b0 % R) * 32 + (k % 32)];
      const int64_t i1 = d1 == tot_all ? na_all : ring[(b1 % R) * 32 + ((k + 1) % 32)];
      __syncwarp();
      if (k % 32 == 31 && lane == 0) mbar_arrive(&sempty[b0 % R]);  // batch b0 consumed
      const int64_t j0 = d0 - i0, j1 = d1 - i1;
      const int na = (int)(i1 - i0), nb = (int)(j1 - j0);
      const K* a = src_k + A0 + i0;
      const K* bp = src_k + A0 + na_all + j0;
      const int offA = stage_offset(a);
      const int offB = (offA + na + EK - 1) / EK * EK + stage_offset(bp);
      const uint32_t* av = nullptr;
      const uint32_t* bv = nullptr;
      int offAv = 0, offBv = 0;
      if constexpr (PAIRS) {
        av = src_v + A0 + i0;
        bv = src_v + A0 + na_all + j0;
        offAv = stage_offset(av);
        offBv = (offAv + na + 3) / 4 * 4 + stage_offset(bv);
      }
      mbar_wait(&empty[s], (uint32_t)(((k / S) & 1) ^ 1));
      K* sk = stk + (size_t)s * LY::SKE;
      uint32_t* sv = stv + (size_t)s * LY::SVE;
      if (lane == 0) {
        meta[s] = TileMeta{A0 + d0, na, nb, offA, offB, offAv, offBv, na + nb, 0};
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
  } else {
    // ------------------------------------------------------------ mergers
    const int ct = threadIdx.x - 64;  // 0..NC-1
    int prev_s = -1;
    for (int64_t k = 0; k < cnt; ++k) {
      const int s = (int)(k % S);
      mbar_wait(&full[s], (uint32_t)((k / S) & 1));
      const TileMeta m = meta[s];
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
      // everyone is done reading stage s (so it can be overwritten) and with
      // the previous tile's head/tail stores (so that stage can be recycled)
      named_bar_sync(1, NC);
      if (ct == 0 && prev_s >= 0) {
        bulk_wait_read<0>();         // the previous tile's bulk store has read it
        mbar_arrive(&empty[prev_s]);  // ... so it goes back to the producer
      }
      // The output keeps its global 16-byte phase so the aligned middle leaves
      // by one bulk store (TMA, cp.async.bulk.global.shared).
      K* gk = dst_k + m.out;
      const int phk = stage_offset(gk);
      uint32_t* gv = nullptr;
      int phv = 0;
      if constexpr (PAIRS) {
        gv = dst_v + m.out;
        phv = stage_offset(gv);
      }
#pragma unroll
      for (int t = 0; t < VT; ++t) {
        if (d + t < m.tot) {
          sk[phk + d + t] = key[t];
          if constexpr (PAIRS) sv[phv + d + t] = val[t];
        }
      }
      fence_proxy_async_smem();
      named_bar_sync(1, NC);  // output tile complete in shared memory
      int hk, mk;
      window_split(gk, m.tot, hk, mk);
      int hv = 0, mv = 0;
      if constexpr (PAIRS) window_split(gv, m.tot, hv, mv);
      if (ct == 0) {
        if (mk) bulk_s2g(gk + hk, sk + phk + hk, (uint32_t)(mk * sizeof(K)));
        if constexpr (PAIRS)
          if (mv) bulk_s2g(gv + hv, sv + phv + hv, (uint32_t)(mv * 4));
        bulk_commit();
      }
      for (int i = ct; i < m.tot - mk; i += NC) {
        const int j = i < hk ? i : i + mk;
        gk[j] = sk[phk + j];
      }
      if constexpr (PAIRS)
        for (int i = ct; i < m.tot - mv; i += NC) {
          const int j = i < hv ? i : i + mv;
          gv[j] = sv[phv + j];
        }
      prev_s = s;
    }
    if (ct == 0) bulk_wait_all();
  }
}

// ------------------------------------------------------------ host driver
#ifndef MSORT_K3_NC
#define MSORT_K3_NC 128  // merging threads per K3 CTA
#endif
#ifndef MSORT_K3_VT
#define MSORT_K3_VT 34  // outputs per merging thread (even: two chains)
#endif

template <class K, bool PAIRS>
struct Kernels {
  static constexpr int VT = 17;  // odd: conflict-free blocked shared accesses
  static constexpr int NT1 = 512;
  static constexpr int T = NT1 * VT;  // tile sort size
  static constexpr int NC = MSORT_K3_NC;
  static constexpr int VT3 = MSORT_K3_VT;
  static constexpr int Tm = NC * VT3;  // merge output tile (divides 2T)
  static constexpr int S = 3;
  using LY = K3Layout<K, PAIRS, NC, VT3, S>;
  // CTAs per SM the register budget is tuned for (shared memory allows 4 for
  // 4-byte keys without payload, 2-3 otherwise)
  static constexpr int MINB = (sizeof(K) == 4 && !PAIRS) ? 4 : 2;
  static constexpr size_t k1_smem = (size_t)T * sizeof(K) + (PAIRS ? (size_t)T * 8 : 0);
  static constexpr size_t k3_smem = LY::bytes;
  static_assert((2 * T) % Tm == 0, "pair boundaries must be tile boundaries");

  static int& grid3(int dev) {
    static int g[64] = {};
    return g[dev & 63];
  }

  static msort_status init() {
    int dev = 0;
    MSORT_CUDA_TRY(cudaGetDevice(&dev));
    if (grid3(dev)) return MSORT_SUCCESS;
    MSORT_CUDA_TRY(cudaFuncSetAttribute(k1_tile_sort<K, PAIRS, NT1, VT>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)k1_smem));
    auto ku = k3_merge_pass<K, PAIRS, NC, VT3, S, MINB, UniformPairs>;
    auto ke = k3_merge_pass<K, PAIRS, NC, VT3, S, MINB, ExplicitPairs>;
    MSORT_CUDA_TRY(cudaFuncSetAttribute(ku, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)k3_smem));
    MSORT_CUDA_TRY(cudaFuncSetAttribute(ke, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)k3_smem));
    int sms = 0, occ = 0;
    MSORT_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    MSORT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ku, NC + 64, k3_smem));
    if (occ < 1) {
      set_error("merge pass kernel does not fit on an SM");
      return MSORT_ERROR_NOT_SUPPORTED;
    }
    grid3(dev) = sms * occ;
    return MSORT_SUCCESS;
  }

  template <class PM>
  static msort_status merge_pass(const K* sk, const uint32_t* sv, K* dk, uint32_t* dv,
                                 const PM& pm, int64_t ntiles, cudaStream_t s, KernelClass kc) {
    int dev = 0;
    MSORT_CUDA_TRY(cudaGetDevice(&dev));
    const int64_t grid = std::min<int64_t>(grid3(dev), ntiles);
    {
      LaunchScope ls(kc, s);
      k3_merge_pass<K, PAIRS, NC, VT3, S, MINB, PM>
          <<<(unsigned)grid, NC + 64, k3_smem, s>>>(sk, sv, dk, dv, pm, ntiles);
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
    if (PAIRS) wv = reinterpret_cast<uint32_t*>(w);
    (void)ws_bytes;

    K* bk[2] = {keys, wk};
    uint32_t* bv[2] = {vals, wv};
    int cur = passes % 2;  // S4: pick K1's destination so the last pass lands in keys
    {
      LaunchScope ls(KC_TILE_SORT, s);
      k1_tile_sort<K, PAIRS, NT1, VT>
          <<<(unsigned)ntiles, NT1, k1_smem, s>>>(in_k, in_v, bk[cur], bv[cur], (int64_t)n);
    }
    MSORT_CUDA_TRY(cudaGetLastError());
    const int64_t mtiles = (int64_t)((n + Tm - 1) / Tm);
    for (int64_t L = T; L < (int64_t)n; L *= 2) {
      UniformPairs pm{(int64_t)n, L};
      MSORT_TRY(merge_pass(bk[cur], bv[cur], bk[cur ^ 1], bv[cur ^ 1], pm, mtiles, s, KC_MERGE));
      cur ^= 1;
    }
    return MSORT_SUCCESS;
  }

  // Merge `runs` consecutive runs src[off[r], off[r+1]) into dst with rounds of
  // pairwise merges (ties to the lower run: merge() left-first at every
  // round keeps the lower run on the left).
  static msort_status kway(K* src_k, uint32_t* src_v, K* tmp_k, uint32_t* tmp_v, K* dst_k,
                           uint32_t* dst_v, const int64_t* off_in, int runs, cudaStream_t s) {
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
        tiles += (e - a + Tm - 1) / Tm;
      }
      pm.first_tile[pm.npairs] = tiles;
      // empty pairs own no tiles; locate() picks the last pair whose first
      // tile <= q, which is never an empty one
      if (tiles > 0) MSORT_TRY(merge_pass(ck, cv, nk, nv, pm, tiles, s, KC_KWAY));
      int nr = pm.npairs;
      for (int m = 0; m <= nr; ++m) off[m] = off[std::min(2 * m, runs)];
      runs = nr;
      ck = nk;
      cv = nv;
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
                           const int64_t* off, int runs, cudaStream_t s) {
  if (sv)
    return Kernels<K, true>::kway((K*)sk, (uint32_t*)sv, (K*)tk, (uint32_t*)tv, (K*)dk,
                                  (uint32_t*)dv, off, runs, s);
  return Kernels<K, false>::kway((K*)sk, nullptr, (K*)tk, nullptr, (K*)dk, nullptr, off, runs, s);
}

msort_status kway_merge_dispatch(void* src_k, void* src_v, void* tmp_k, void* tmp_v,
                                 void* dst_k, void* dst_v, const int64_t* off_host, int runs,
                                 msort_dtype kd, msort_dtype vd, void* part_ws,
                                 cudaStream_t s) {
  (void)part_ws;
  if (vd == MSORT_NONE) src_v = tmp_v = dst_v = nullptr;
  switch (kd) {
    case MSORT_INT32:
      return kway_k<int32_t>(src_k, src_v, tmp_k, tmp_v, dst_k, dst_v, off_host, runs, s);
    case MSORT_UINT32:
      return kway_k<uint32_t>(src_k, src_v, tmp_k, tmp_v, dst_k, dst_v, off_host, runs, s);
    case MSORT_INT64:
      return kway_k<int64_t>(src_k, src_v, tmp_k, tmp_v, dst_k, dst_v, off_host, runs, s);
    case MSORT_UINT64:
      return kway_k<uint64_t>(src_k, src_v, tmp_k, tmp_v, dst_k, dst_v, off_host, runs, s);
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
