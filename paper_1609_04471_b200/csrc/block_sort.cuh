// block_sort.cuh -- H4 tile sort: a stable ascending sort of up to NT*VT items
// held in shared memory by one CTA.
//
// Paper anchor: §3(b) "If a run in the input is shorter than the minimal length
// for a run, insertion sort is called to create a longer run" (PAPER.md:94,
// Appendix A isort) and §4(a) the alpha cutoff.
// On the GPU the "minrun" is a whole CTA tile: each thread sorts VT keys in
// registers, then log2(NT) merge-path levels in shared memory merge the
// per-thread runs.  Merges take from the left run on ties.
//   keys only: the register sort is Batcher's odd-even merge network on
//              min/max (equal keys are indistinguishable, so stability is moot);
//   pairs:     odd-even transposition (swap only on strict '>'), stable, and
//              every merge tracks source positions to gather the payloads,
//   so the pair sort keeps input order among equal keys.
#pragma once
#include <utility>

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

// Batcher's odd-even merge sort network over N register slots, tabulated at
// compile time so every compare-exchange addresses registers by constants.
template <int N>
struct BatcherNet {
  static constexpr int count() {
    int c = 0;
    for (int p = 1; p < N; p += p)
      for (int k = p; k > 0; k /= 2)
        for (int j = k % p; j + k < N; j += k + k)
          for (int i = 0; i < k && i + j + k < N; i++)
            if ((i + j) / (p + p) == (i + j + k) / (p + p)) c++;
    return c;
  }
  static constexpr int C = count();
  struct Table {
    int a[C > 0 ? C : 1];
    int b[C > 0 ? C : 1];
  };
  static constexpr Table make() {
    Table t{};
    int c = 0;
    for (int p = 1; p < N; p += p)
      for (int k = p; k > 0; k /= 2)
        for (int j = k % p; j + k < N; j += k + k)
          for (int i = 0; i < k && i + j + k < N; i++)
            if ((i + j) / (p + p) == (i + j + k) / (p + p)) { t.a[c] = i + j; t.b[c] = i + j + k; c++; }
    return t;
  }
  static constexpr int a(int c) { return make().a[c]; }
  static constexpr int b(int c) { return make().b[c]; }
};

template <int N, typename CE, int... I>
__device__ __forceinline__ void batcher_apply(CE& ce, std::integer_sequence<int, I...>) {
  (ce(std::integral_constant<int, BatcherNet<N>::a(I)>::value, std::integral_constant<int, BatcherNet<N>::b(I)>::value),
   ...);
}

template <int N, typename CE>
__device__ __forceinline__ void batcher_network(CE&& ce) {
  batcher_apply<N>(ce, std::make_integer_sequence<int, BatcherNet<N>::C>{});
}

template <typename K, bool HAS_V, int NT, int VT>
struct BlockSort {
  static constexpr int NV = NT * VT;
  // slack after NV: the branch-free serial merge may read one element past a list
  static constexpr int KEYS_SMEM = NV + VT;
  static constexpr int VALS_SMEM = HAS_V ? NV + VT : 1;
  static_assert((VT & (VT - 1)) == 0, "VT must be a power of two");

  __device__ __forceinline__ static void thread_sort(K (&k)[VT], uint32_t (&v)[VT]) {
    if (!HAS_V) {
      batcher_network<VT>([&](int a, int b) {
        K x = k[a], y = k[b];
        k[a] = x < y ? x : y;
        k[b] = x < y ? y : x;
      });
    } else {
#pragma unroll
      for (int r = 0; r < VT; r++) {
#pragma unroll
        for (int i = (r & 1); i + 1 < VT; i += 2) {
          bool sw = k[i + 1] < k[i];  // strict: equal keys never swap (stable)
          K a = k[i], b = k[i + 1];
          uint32_t va = v[i], vb = v[i + 1];
          k[i] = sw ? b : a;
          k[i + 1] = sw ? a : b;
          v[i] = sw ? vb : va;
          v[i + 1] = sw ? va : vb;
        }
      }
    }
  }

  // Blocked store/load of VT consecutive elements as 16-byte vectors, built
  // element by element so the register arrays never need an address.
  __device__ __forceinline__ static uint32_t lo32(int32_t x) { return (uint32_t)x; }
  __device__ __forceinline__ static uint32_t lo32(uint32_t x) { return x; }
  template <typename T>
  __device__ __forceinline__ static void store_vec(T* base, const T (&x)[VT]) {
    static_assert((VT * sizeof(T)) % 16 == 0, "blocked vector I/O needs VT * sizeof(T) to be a multiple of 16");
    uint4* p = reinterpret_cast<uint4*>(base);
    if constexpr (sizeof(T) == 4) {
#pragma unroll
      for (int i = 0; i < VT / 4; i++)
        p[i] = make_uint4((uint32_t)x[4 * i], (uint32_t)x[4 * i + 1], (uint32_t)x[4 * i + 2], (uint32_t)x[4 * i + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < VT / 2; i++) {
        uint64_t a = (uint64_t)x[2 * i], b = (uint64_t)x[2 * i + 1];
        p[i] = make_uint4((uint32_t)a, (uint32_t)(a >> 32), (uint32_t)b, (uint32_t)(b >> 32));
      }
    }
  }
  template <typename T>
  __device__ __forceinline__ static void load_vec(const T* base, T (&x)[VT]) {
    static_assert((VT * sizeof(T)) % 16 == 0, "blocked vector I/O needs VT * sizeof(T) to be a multiple of 16");
    const uint4* p = reinterpret_cast<const uint4*>(base);
    if constexpr (sizeof(T) == 4) {
#pragma unroll
      for (int i = 0; i < VT / 4; i++) {
        uint4 q = p[i];
        x[4 * i] = (T)q.x; x[4 * i + 1] = (T)q.y; x[4 * i + 2] = (T)q.z; x[4 * i + 3] = (T)q.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < VT / 2; i++) {
        uint4 q = p[i];
        x[2 * i] = (T)(((uint64_t)q.y << 32) | q.x);
        x[2 * i + 1] = (T)(((uint64_t)q.w << 32) | q.z);
      }
    }
  }

  // One merge level: thread t of a cooperative group of `coop` threads merges
  // VT outputs of two adjacent sorted lists of (coop/2)*VT items.
  __device__ __forceinline__ static void merge_level(const K* ks, const uint32_t* vs, int coop, K (&k)[VT],
                                                     uint32_t (&v)[VT]) {
    const int t = threadIdx.x;
    const int list = (coop >> 1) * VT;
    const int a0 = (t & ~(coop - 1)) * VT;
    const int diag = (t & (coop - 1)) * VT;
    const K* A = ks + a0;
    const K* B = A + list;
    int lo = diag - list > 0 ? diag - list : 0;
    int hi = diag < list ? diag : list;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (!(B[diag - 1 - mid] < A[mid])) lo = mid + 1; else hi = mid;
    }
    int ai = lo, bi = diag - lo;
    K ak = A[ai], bk = B[bi];  // over-reads stay inside the slack
    int src[VT];
#pragma unroll
    for (int i = 0; i < VT; i++) {
      const bool p = (bi >= list) || (ai < list && !(bk < ak));
      k[i] = p ? ak : bk;
      if (HAS_V) src[i] = p ? a0 + ai : a0 + list + bi;
      ai += p;
      bi += !p;
      const K nx = *(p ? A + ai : B + bi);
      ak = p ? nx : ak;
      bk = p ? bk : nx;
    }
    if (HAS_V) {
#pragma unroll
      for (int i = 0; i < VT; i++) v[i] = vs[src[i]];
    }
  }

  // Sort items [0, count) of ks (and vs) in place; count <= NV.  Only the
  // smallest power-of-two number of threads covering count takes part, so a
  // short range costs O(count log count).  All NT threads must call this.
  __device__ static void sort(K* ks, uint32_t* vs, int count) {
    const int t = threadIdx.x;
    const int need = (count + VT - 1) / VT;
    int nta = 1;
    while (nta < need) nta <<= 1;
    const bool act = t < nta;
    K k[VT];
    uint32_t v[VT];
    if (act) {
      if ((t + 1) * VT <= count) {
        load_vec(ks + t * VT, k);
        if (HAS_V) load_vec(vs + t * VT, v);
      } else {
#pragma unroll
        for (int i = 0; i < VT; i++) {
          int p = t * VT + i;
          k[i] = p < count ? ks[p] : KeyTraits<K>::max_key();  // +inf padding stays last (stable)
          v[i] = (HAS_V && p < count) ? vs[p] : 0u;
        }
      }
      thread_sort(k, v);
    }
    __syncthreads();
    for (int coop = 2; coop <= nta; coop <<= 1) {
      if (act) {
        store_vec(ks + t * VT, k);
        if (HAS_V) store_vec(vs + t * VT, v);
      }
      __syncthreads();
      if (act) merge_level(ks, vs, coop, k, v);
      __syncthreads();
    }
    if (act) {
      store_vec(ks + t * VT, k);
      if (HAS_V) store_vec(vs + t * VT, v);
    }
    __syncthreads();
  }
};

}  // namespace sr
