// block_sort.cuh -- H4 tile sort: a stable ascending sort of up to NT*VT items
// held in (padded) shared memory by one CTA.
//
// Paper anchor: §3(b) "If a run in the input is shorter than the minimal length
// for a run, insertion sort is called to create a longer run" (PAPER.md:94,
// Appendix A isort) and §4(a) the alpha cutoff.
// On the GPU the "minrun" is a whole CTA tile: each thread sorts VT keys in
// registers with odd-even transposition (swap only on strict '>', so it is
// stable), then log2(NT) merge-path levels in shared memory merge the
// per-thread runs; merges take from the left run on ties, so the
// whole tile sort is stable and pairs keep input order among equal keys.
#pragma once
#include "common.cuh"

namespace sr {

// Merge-path split ("binary search is used to locate the position
// in A where the current element in B should go"): the number of A elements
// among the first `diag` outputs of a stable merge of A and B (A wins ties).
template <typename K, typename LoadA, typename LoadB>
__device__ __forceinline__ int merge_path_search(LoadA a, int a_len, LoadB b, int b_len, int diag) {
  int lo = diag - b_len > 0 ? diag - b_len : 0;
  int hi = diag < a_len ? diag : a_len;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    K ak = a(mid), bk = b(diag - 1 - mid);
    if (!(bk < ak)) lo = mid + 1;  // A[mid] <= B[diag-1-mid]: A[mid] is among the first diag
    else hi = mid;
  }
  return lo;
}

template <typename K, bool HAS_V, int NT, int VT>
struct BlockSort {
  static constexpr int NV = NT * VT;
  static constexpr int KEYS_SMEM = padded_size<K>(NV);
  static constexpr int VALS_SMEM = HAS_V ? padded_size<uint32_t>(NV) : 1;

  // Stable in-register sort of VT items (odd-even transposition sort).
  __device__ __forceinline__ static void thread_sort(K (&k)[VT], uint32_t (&v)[VT]) {
#pragma unroll
    for (int r = 0; r < VT; r++) {
#pragma unroll
      for (int i = (r & 1); i + 1 < VT; i += 2) {
        if (k[i + 1] < k[i]) {  // strict: equal keys never swap
          K tk = k[i]; k[i] = k[i + 1]; k[i + 1] = tk;
          if (HAS_V) { uint32_t tv = v[i]; v[i] = v[i + 1]; v[i + 1] = tv; }
        }
      }
    }
  }

  __device__ __forceinline__ static void store_regs(K* ks, uint32_t* vs, const K (&k)[VT], const uint32_t (&v)[VT]) {
    const int t = threadIdx.x;
#pragma unroll
    for (int i = 0; i < VT; i++) {
      ks[pad_idx<K>(t * VT + i)] = k[i];
      if (HAS_V) vs[pad_idx<uint32_t>(t * VT + i)] = v[i];
    }
  }

  // Sort items [0, count) of ks (and vs) in place; count <= NV.  Only the
  // smallest power-of-two number of threads that covers count works, so a
  // short segment costs O(count log count).  All NT threads must call this.
  __device__ static void sort(K* ks, uint32_t* vs, int count) {
    const int t = threadIdx.x;
    const int need = (count + VT - 1) / VT;
    int nta = 1;
    while (nta < need) nta <<= 1;
    const bool act = t < nta;
    K k[VT];
    uint32_t v[VT];
    if (act) {
#pragma unroll
      for (int i = 0; i < VT; i++) {
        int p = t * VT + i;
        bool ok = p < count;
        k[i] = ok ? ks[pad_idx<K>(p)] : KeyTraits<K>::max_key();  // +inf padding stays last (stable)
        v[i] = (HAS_V && ok) ? vs[pad_idx<uint32_t>(p)] : 0u;
      }
      thread_sort(k, v);
    }
    __syncthreads();
    for (int coop = 2; coop <= nta; coop <<= 1) {
      if (act) store_regs(ks, vs, k, v);
      __syncthreads();
      if (act) {
        const int list = (coop >> 1) * VT;
        const int a0 = (t / coop) * coop * VT;
        const int b0 = a0 + list;
        const int diag = (t % coop) * VT;
        int mp = merge_path_search<K>([&](int i) { return ks[pad_idx<K>(a0 + i)]; }, list,
                                      [&](int i) { return ks[pad_idx<K>(b0 + i)]; }, list, diag);
        int ai = a0 + mp, bi = b0 + diag - mp;
        const int aend = a0 + list, bend = b0 + list;
        K ak = ai < aend ? ks[pad_idx<K>(ai)] : K(0);
        K bk = bi < bend ? ks[pad_idx<K>(bi)] : K(0);
        int src[VT];
#pragma unroll
        for (int i = 0; i < VT; i++) {
          bool take_a = (bi >= bend) || (ai < aend && !(bk < ak));
          k[i] = take_a ? ak : bk;
          src[i] = take_a ? ai : bi;
          if (take_a) {
            ++ai;
            if (ai < aend) ak = ks[pad_idx<K>(ai)];
          } else {
            ++bi;
            if (bi < bend) bk = ks[pad_idx<K>(bi)];
          }
        }
        if (HAS_V) {
#pragma unroll
          for (int i = 0; i < VT; i++) v[i] = vs[pad_idx<uint32_t>(src[i])];
        }
      }
      __syncthreads();
    }
    if (act) store_regs(ks, vs, k, v);
    __syncthreads();
  }
};

}  // namespace sr
