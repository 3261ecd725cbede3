// bitonic.cuh -- H4 tile sort for keys only: a register / warp-shuffle bitonic
// network over up to NT*VT keys of one CTA.
//
// Same role as block_sort.cuh (the "minrun" tile sort of §3(b), PAPER.md:94;
// the alpha cutoff of §4(a)), but organised for sm_100a's
// latency profile: every stage is a set of VT independent compare-exchanges
// per thread (no dependent shared-memory chains as in a serial merge).
// Partners within a thread use registers, partners within a warp use
// __shfl_xor_sync, and only partners in another warp go through shared memory
// (double-buffered, one barrier per stage).  All runs are kept ascending: the
// first stage of every merge level compares mirrored positions ("flip"), the
// following half-cleaner stages compare i and i^j.  Equal keys are
// indistinguishable, so the missing stability is unobservable for keys-only
// sorts; pairs use the stable merge sort of block_sort.cuh.
#pragma once
#include "block_sort.cuh"
#include "common.cuh"

namespace sr {

template <typename K, int NT, int VT>
struct BitonicSort {
  static constexpr int NV = NT * VT;
  static constexpr int SMEM = 2 * NV;  // double buffer for cross-warp stages
  static_assert((VT & (VT - 1)) == 0 && VT >= 2, "VT must be a power of two");
  static_assert(NT % 32 == 0, "");

  __device__ __forceinline__ static K kmin(K a, K b) { return min(a, b); }
  __device__ __forceinline__ static K kmax(K a, K b) { return max(a, b); }
  // ascending compare-exchange.  int32: two IMNMX.  int64 has no 64-bit
  // min/max instruction, so compare once and select both outputs (6
  // instructions instead of two full min/max expansions, 8)
  __device__ __forceinline__ static void cex(K& x, K& y) {
    if constexpr (sizeof(K) == 8) {
      const bool sw = y < x;
      const K lo = sw ? y : x, hi = sw ? x : y;
      x = lo;
      y = hi;
    } else {
      const K lo = min(x, y), hi = max(x, y);
      x = lo;
      y = hi;
    }
  }
  // the half of a compare-exchange with partner value b that this side keeps
  // (min for the lower side, max for the upper one; ties are interchangeable)
  __device__ __forceinline__ static K keep(K k, K b, bool lower) {
    if constexpr (sizeof(K) == 8) return ((b < k) == lower) ? b : k;
    else return lower ? min(k, b) : max(k, b);
  }

  // partner values of a cross-thread stage are in b[]; flip pairs r with VT-1-r
  __device__ __forceinline__ static void combine(K (&k)[VT], const K (&b)[VT], bool lower, bool flip) {
#pragma unroll
    for (int r = 0; r < VT; r++) {
      K o = flip ? b[VT - 1 - r] : b[r];
      k[r] = keep(k[r], o, lower);
    }
  }

  // Register-frugal: partners are fetched pairwise (flip) or one at a time.
  __device__ __forceinline__ static void shfl_stage(K (&k)[VT], int mask, bool lower, bool flip) {
    if (flip) {
#pragma unroll
      for (int r = 0; r < VT / 2; r++) {
        const K b1 = __shfl_xor_sync(0xffffffffu, k[VT - 1 - r], mask);  // partner of k[r]
        const K b2 = __shfl_xor_sync(0xffffffffu, k[r], mask);           // partner of k[VT-1-r]
        k[r] = keep(k[r], b1, lower);
        k[VT - 1 - r] = keep(k[VT - 1 - r], b2, lower);
      }
    } else {
#pragma unroll
      for (int r = 0; r < VT; r++) {
        const K b = __shfl_xor_sync(0xffffffffu, k[r], mask);
        k[r] = keep(k[r], b, lower);
      }
    }
  }

  __device__ __forceinline__ static void reg_half_cleaners(K (&k)[VT]) {
#pragma unroll
    for (int j = VT / 2; j > 0; j >>= 1) {
#pragma unroll
      for (int r = 0; r < VT; r++) {
        if ((r & j) == 0) cex(k[r], k[r | j]);
      }
    }
  }

  // Sort ks[0, count) ascending in place (count <= NV); ks must hold SMEM
  // elements.  All NT threads must call.
  __device__ static void sort(K* ks, int count) {
    const int t = threadIdx.x;
    const int need = (count + VT - 1) / VT;
    int nta = 32;
    while (nta < need) nta <<= 1;
    const bool act = t < nta;
    K k[VT];
    if (act) {
#pragma unroll
      for (int i = 0; i < VT; i++) {
        int p = t * VT + i;
        k[i] = p < count ? ks[p] : KeyTraits<K>::max_key();
      }
      batcher_network<VT>([&](int a, int b) { cex(k[a], k[b]); });
    }
    int parity = 0;
    __syncthreads();  // everyone has read ks before the first cross-warp stage writes it
    for (int kk = 2 * VT; kk <= nta * VT; kk <<= 1) {
      const int tk = kk / VT;  // threads per merged run
      // flip stage: partner thread t ^ (tk-1), register VT-1-r
      {
        const int m = tk - 1;
        const bool lower = (t & (tk >> 1)) == 0;
        if (m < 32) {
          if (act) shfl_stage(k, m, lower, true);
        } else {
          K* buf = ks + parity * NV;
          if (act) BlockSort<K, false, NT, VT>::store_vec(buf + t * VT, k);
          __syncthreads();
          if (act) {
            K b[VT];
            BlockSort<K, false, NT, VT>::load_vec(buf + (t ^ m) * VT, b);
            combine(k, b, lower, true);
          }
          parity ^= 1;
        }
      }
      // half-cleaners across threads: j = kk/4 .. VT
      for (int jt = tk >> 2; jt >= 1; jt >>= 1) {
        const bool lower = (t & jt) == 0;
        if (jt < 32) {
          if (act) shfl_stage(k, jt, lower, false);
        } else {
          K* buf = ks + parity * NV;
          if (act) BlockSort<K, false, NT, VT>::store_vec(buf + t * VT, k);
          __syncthreads();
          if (act) {
            K b[VT];
            BlockSort<K, false, NT, VT>::load_vec(buf + (t ^ jt) * VT, b);
            combine(k, b, lower, false);
          }
          parity ^= 1;
        }
      }
      if (act) reg_half_cleaners(k);
    }
    __syncthreads();
    if (act) BlockSort<K, false, NT, VT>::store_vec(ks + t * VT, k);
    __syncthreads();
  }
};

}  // namespace sr

namespace sr {

// One warp sorts up to 32*VT keys held "blocked" in registers (lane l owns
// elements [l*VT, (l+1)*VT)): Batcher network inside the lane, then bitonic
// merge levels whose cross-lane stages are __shfl_xor_sync and whose in-lane
// stages are register compare-exchanges.  No shared memory, no barriers:
// used for the (bucket-sized) finishing items of the keys-only partition.
template <typename K, int VT>
struct WarpBitonic {
  static constexpr int CAP = 32 * VT;
  using BT = BitonicSort<K, 32, VT>;

  // ks: this warp's staging area (CAP elements), holding count keys.
  __device__ static void sort(K* ks, int count) {
    const int lane = threadIdx.x & 31;
    const int need = (count + VT - 1) / VT;
    int nl = 1;  // lanes taking part (power of two)
    while (nl < need) nl <<= 1;
    K k[VT];
    __syncwarp();
    // blocked 16-byte vector loads: a scalar load of ks[lane * VT + i] would
    // put all 32 lanes on one shared-memory bank for VT a multiple of 32 words
    BlockSort<K, false, 32, VT>::load_vec(ks + lane * VT, k);
#pragma unroll
    for (int i = 0; i < VT; i++)
      if (lane * VT + i >= count) k[i] = KeyTraits<K>::max_key();
    batcher_network<VT>([&](int a, int b) { BT::cex(k[a], k[b]); });
    for (int tk = 2; tk <= nl; tk <<= 1) {  // lanes per merged run
      BT::shfl_stage(k, tk - 1, (lane & (tk >> 1)) == 0, true);
      for (int jt = tk >> 2; jt >= 1; jt >>= 1) BT::shfl_stage(k, jt, (lane & jt) == 0, false);
      BT::reg_half_cleaners(k);
    }
    __syncwarp();
    if (lane < nl) BlockSort<K, false, 32, VT>::store_vec(ks + lane * VT, k);
    __syncwarp();
  }
};

}  // namespace sr
