// unit_sort.cuh -- H11 for one level-1 bucket held in shared memory: the
// quicksort recursion of Appendix B as one in-shared-memory
// 3-way sample partition followed by per-warp register networks.
//
//   is_sorted first -> the unit is copied out unchanged;
//   pivot choice from a sample: SB - 1 = 31 splitters, every
//     O2-th key of a regular sample of S2 = 256 keys ranked by counting;
//   3-way split: keys equal to a splitter that occurs more
//     than gamma = 2 times in the sample go to an equality bin,
//     which is final ("spared from the recursive calls") and written as a fill;
//   small pieces (the alpha cutoff) -> one warp's register
//     bitonic network over VT = 8 / 16 / 32 keys per lane (<= 1024 keys), or
//     two such networks and one warp merge-path merge (<= 2048 keys, the
//     mergesort level of §3, A wins ties PAPER.md:99); larger pieces (only
//     under extreme skew) -> a CTA-wide merge sort in shared memory.
//
// The code is deliberately compact (three network instantiations, loops over
// stages): the resident kernel runs every phase in one launch, and an
// unrolled-everything E phase blew the instruction cache (ncu r2_c2_res:
// 19% no_instruction stalls with 430 KB of SASS).
#pragma once
#include <type_traits>
#include "bitonic.cuh"
#include "block_sort.cuh"
#include "common.cuh"

namespace sr {

template <typename K, int CAP, int NT>
struct UnitSmem {
  static constexpr int SB = 32;            // sub-buckets: SB - 1 splitters
  static constexpr int NB = 2 * SB;        // 3-way bins: 2i range, 2i+1 equal to splitter i
  static constexpr int O2 = 8;             // oversampling
  static constexpr int S2 = SB * O2;       // sample
  static constexpr int NW = NT / 32;
  static constexpr int SLACK = 1024;       // a warp piece reads up to 2 * 32 * VT keys from a region start
  K x[CAP + SLACK];                        // the unit (the caller loads x[0, L))
  K y[CAP + 4 * NB + SLACK];               // bin regions (4-key aligned)
  uint8_t bin[CAP];
  K samp[S2];
  K srt[S2];
  K tree[SB];                              // Eytzinger [1, SB); the sorted splitters are in spl
  K spl[SB];
  uint8_t eqf[SB];
  uint32_t wcnt[NW][NB];                   // per-warp bin counts, then move cursors
  uint32_t ost[NB + 1];                    // bin starts in the output
  uint32_t reg[NB + 1];                    // bin regions in y
  uint32_t nbig;
  uint16_t big[NB];
};

// Sort ks[0, len) (16-byte aligned; 32*VT keys readable) in place by one warp:
// Batcher network inside the lane, bitonic merge levels whose cross-lane
// stages are shuffles (bitonic.cuh WarpBitonic), and exactly [0, len) written.
// (__noinline__: one copy of each network in the binary.  The networks are
// long straight-line code run a few times per SM; inlined at every call site
// they multiplied the code size and ran out of the instruction cache.)
template <typename K, int VT>
__device__ __noinline__ void unit_warp_net(K* ks, int len) {
  using BT = BitonicSort<K, 32, VT>;
  const int lane = threadIdx.x & 31;
  const int need = (len + VT - 1) / VT;
  int nl = 1;
  while (nl < need) nl <<= 1;
  K k[VT];
  BlockSort<K, false, 32, VT>::load_vec(ks + lane * VT, k);
#pragma unroll
  for (int i = 0; i < VT; i++)
    if (lane * VT + i >= len) k[i] = KeyTraits<K>::max_key();
  batcher_network<VT>([&](int a, int b) { BT::cex(k[a], k[b]); });
#pragma unroll 1
  for (int tk = 2; tk <= nl; tk <<= 1) {
    BT::shfl_stage(k, tk - 1, (lane & (tk >> 1)) == 0, true);
#pragma unroll 1
    for (int jt = tk >> 2; jt >= 1; jt >>= 1) BT::shfl_stage(k, jt, (lane & jt) == 0, false);
    BT::reg_half_cleaners(k);
  }
  __syncwarp();
  if ((lane + 1) * VT <= len) {
    BlockSort<K, false, 32, VT>::store_vec(ks + lane * VT, k);
  } else if (lane * VT < len) {
#pragma unroll
    for (int i = 0; i < VT; i++)
      if (lane * VT + i < len) ks[lane * VT + i] = k[i];
  }
  __syncwarp();
}

// Largest network: 32 keys per lane for int32, 16 for int64 (register budget
// of the 512-thread resident kernel); pieces up to twice that take two networks
// and a merge.
template <typename K>
struct UnitNet {
  static constexpr int VTMAX = sizeof(K) == 4 ? 32 : 16;
  static constexpr int NET = 32 * VTMAX;  // one network
  static constexpr int PIECE = 2 * NET;   // one warp
};

// ks[0, len) (len <= UnitNet<K>::NET) sorted in place by the narrowest network.
template <typename K>
__device__ __forceinline__ void unit_warp_sort(K* ks, int len) {
  if (len <= 1) return;
  if (len <= 256) unit_warp_net<K, 8>(ks, len);
  else if (UnitNet<K>::VTMAX == 16 || len <= 512) unit_warp_net<K, 16>(ks, len);
  else unit_warp_net<K, UnitNet<K>::VTMAX>(ks, len);
}

// One warp merges the sorted runs A[0, na) and B[0, nb) (shared memory) into
// dst[0, na + nb): each lane takes a contiguous slice of the output, finds its
// start by merge path and merges serially (A wins ties).  The
// slices are cut at 16-byte boundaries of dst and every lane stores groups of
// 16 / sizeof(K) outputs as one vector: a store instruction of the warp then
// touches 4x (int32) / 2x (int64) fewer sectors than one key per lane would
// (lane-strided slices are uncoalesced by construction).
template <typename K>
__device__ __noinline__ void unit_warp_merge(const K* A, int na, const K* B, int nb, K* __restrict__ dst) {
  constexpr int V = 16 / (int)sizeof(K);
  using Vec = typename std::conditional<sizeof(K) == 4, int4, longlong2>::type;
  const int lane = threadIdx.x & 31;
  const int len = na + nb;
  const int mis = (int)((reinterpret_cast<uintptr_t>(dst) & 15) / sizeof(K));
  const int head = min(len, mis ? V - mis : 0);  // keys before the first 16-byte boundary
  const int nvec = (len - head) / V;
  const int vper = (nvec + 31) / 32;
  const int vb = min(lane * vper, nvec), ve = min((lane + 1) * vper, nvec);
  const int d0 = lane == 0 ? 0 : head + vb * V;
  const int d1 = lane == 31 ? len : head + ve * V;
  if (d0 < d1) {
    int i = merge_path_search<K>([&](int q) { return A[q]; }, na, [&](int q) { return B[q]; }, nb, d0);
    int j = d0 - i;
    auto step = [&]() {
      const bool tA = j >= nb || (i < na && !(B[j] < A[i]));
      const K x = tA ? A[i] : B[j];
      i += tA;
      j += !tA;
      return x;
    };
    int d = d0;
    for (; d < d1 && d < head; d++) dst[d] = step();  // lane 0: the unaligned head
    const int vend = min(d1, head + nvec * V);
    for (; d + V <= vend; d += V) {
      union {
        Vec v;
        K k[V];
      } u;
#pragma unroll
      for (int q = 0; q < V; q++) u.k[q] = step();
      *reinterpret_cast<Vec*>(dst + d) = u.v;
    }
    for (; d < d1; d++) dst[d] = step();  // lane 31: the tail
  }
  __syncwarp();
}

// One warp sorts ks[0, len) (len <= UnitNet<K>::PIECE, 16-byte aligned, slack
// readable) and writes it to dst[0, len): one network, or two networks and a
// merge-path merge (A = the first NET keys wins ties).
template <typename K>
__device__ __forceinline__ void unit_warp_piece(K* ks, int len, K* __restrict__ dst) {
  constexpr int NET = UnitNet<K>::NET;
  const int lane = threadIdx.x & 31;
  if (len <= NET) {
    unit_warp_sort<K>(ks, len);
    for (int i = lane; i < len; i += 32) dst[i] = ks[i];
    __syncwarp();
    return;
  }
  unit_warp_net<K, UnitNet<K>::VTMAX>(ks, NET);
  unit_warp_net<K, UnitNet<K>::VTMAX>(ks + NET, len - NET);
  unit_warp_merge<K>(ks, NET, ks + NET, len - NET, dst);
}

// CTA-wide merge sort of a[0, L) (any L <= CAP) into dst, b as scratch: runs of
// 1024 sorted by the warps, then merge-path rounds (A wins ties).  Used only
// for pieces of more than 2048 keys after the partition (extreme skew).
template <typename K, int NT>
__device__ __noinline__ void unit_cta_merge_sort(K* a, K* b, int L, K* __restrict__ dst) {
  constexpr int R0 = UnitNet<K>::NET, VT = 8;
  const int w = threadIdx.x >> 5;
  for (int r = w * R0; r < L; r += (NT / 32) * R0) unit_warp_sort<K>(a + r, min(R0, L - r));
  __syncthreads();
  if (L <= R0) {
    for (int i = threadIdx.x; i < L; i += NT) dst[i] = a[i];
    __syncthreads();
    return;
  }
  K* src = a;
  K* out = b;
  for (int R = R0; R < L; R *= 2) {
    const bool last = 2 * R >= L;
    for (int o = threadIdx.x * VT; o < L; o += NT * VT) {
      const int p0 = (o / (2 * R)) * (2 * R);
      const int alen = min(R, L - p0);
      const int blen = min(R, L - p0 - alen);
      const K* A = src + p0;
      const K* B = A + alen;
      const int diag = o - p0;
      int i = merge_path_search<K>([&](int q) { return A[q]; }, alen, [&](int q) { return B[q]; }, blen, diag);
      int j = diag - i;
      K* op = last ? dst : out;
#pragma unroll
      for (int k = 0; k < VT; k++) {
        if (o + k < L && diag + k < alen + blen) {
          const bool tA = j >= blen || (i < alen && !(B[j] < A[i]));
          op[o + k] = tA ? A[i] : B[j];
          i += tA;
          j += !tA;
        }
      }
    }
    __syncthreads();
    K* t = src;
    src = out;
    out = t;
  }
}

// Sort e.x[0, L) (L <= CAP) into dst[0, L).  All NT threads call; returns
// with the shared buffers free (a trailing barrier).
#ifndef SR_UNIT_PROF
#define SR_UNIT_MARK(k)
#endif
template <typename K, int CAP, int NT>
__device__ __noinline__ void unit_sort(K* __restrict__ dst, int L, UnitSmem<K, CAP, NT>& e) {
  using U = UnitSmem<K, CAP, NT>;
  constexpr int SB = U::SB, NB = U::NB, O2 = U::O2, S2 = U::S2, NW = U::NW;
  constexpr int DEPTH = 5;
  static_assert((1 << DEPTH) == SB && S2 <= NT && NB <= 64, "");
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // is_sorted + the regular sample
  int unsorted = 0;
  for (int i = tid; i + 1 < L; i += NT) unsorted |= e.x[i + 1] < e.x[i];
  if (tid < S2) e.samp[tid] = e.x[(int)(((int64_t)(2 * tid + 1) * L) / (2 * S2))];
  for (int i = tid; i < NW * NB; i += NT) (&e.wcnt[0][0])[i] = 0u;
  if (tid == 0) e.nbig = 0;
  SR_UNIT_MARK(0);
  if (!__syncthreads_or(unsorted)) {
    for (int i = tid; i < L; i += NT) dst[i] = e.x[i];
    __syncthreads();
    return;
  }
  if (L <= UnitNet<K>::PIECE) {  // small unit: one warp
    if (w == 0) unit_warp_piece<K>(e.x, L, dst);
    __syncthreads();
    return;
  }
  {  // rank of sample q = its position in the stably sorted sample (two threads
     // per sample, each over half the sample read as 16-byte vectors)
    constexpr int KV = 16 / sizeof(K);  // keys per vector
    const int q = tid >> 1, h = tid & 1;
    const K v = q < S2 ? e.samp[q] : K(0);
    int r = 0;
    if (q < S2) {
      const uint4* sv = reinterpret_cast<const uint4*>(e.samp + h * (S2 / 2));
#pragma unroll 4
      for (int jv = 0; jv < S2 / 2 / KV; jv++) {
        const uint4 u4 = sv[jv];
        K u[KV];
        memcpy(u, &u4, 16);
#pragma unroll
        for (int t = 0; t < KV; t++) {
          const int j = h * (S2 / 2) + jv * KV + t;
          r += (u[t] < v) || (u[t] == v && j < q);
        }
      }
    }
    r += __shfl_xor_sync(0xffffffffu, r, 1);
    if (q < S2 && h == 0) e.srt[r] = v;
  }
  SR_UNIT_MARK(1);
  __syncthreads();
  if (tid < SB - 1) {  // splitter i = sorted sample O2 (i + 1) with its gamma flag (count > 2)
    const int r = O2 * (tid + 1);
    const K t = e.srt[r];
    const bool m1 = e.srt[r - 1] == t, m2 = e.srt[r - 2] == t;
    const bool p1 = r + 1 < S2 && e.srt[r + 1] == t, p2 = r + 2 < S2 && e.srt[r + 2] == t;
    e.spl[tid] = t;
    e.eqf[tid] = ((m1 && m2) || (m1 && p1) || (p1 && p2)) ? 1 : 0;
  }
  if (tid > 0 && tid < SB) {  // Eytzinger node tid <- splitter at in-order position pos
    const int d = 31 - __clz(tid);
    const int pos = ((2 * (tid - (1 << d)) + 1) << (DEPTH - 1 - d)) - 1;
    e.tree[tid] = e.srt[O2 * (pos + 1)];
  }
  SR_UNIT_MARK(2);
  __syncthreads();
  // classify (3-way ids) + per-warp counts; UC keys per thread in flight
  constexpr int UC = 4;
  for (int i0 = 0; i0 < L; i0 += NT * UC) {
    K x[UC];
    int j[UC];
#pragma unroll
    for (int u = 0; u < UC; u++) {
      const int i = i0 + u * NT + tid;
      x[u] = i < L ? e.x[i] : K(0);
      j[u] = 1;
    }
#pragma unroll
    for (int l = 0; l < DEPTH; l++)
#pragma unroll
      for (int u = 0; u < UC; u++) j[u] = 2 * j[u] + (e.tree[j[u]] < x[u] ? 1 : 0);
#pragma unroll
    for (int u = 0; u < UC; u++) {
      const int i = i0 + u * NT + tid;
      if (i < L) {
        const int sb = j[u] - SB;  // #splitters < x
        const int b = 2 * sb + ((sb < SB - 1 && e.spl[sb] == x[u] && e.eqf[sb]) ? 1 : 0);
        e.bin[i] = (uint8_t)b;
        atomicAdd(&e.wcnt[w][b], 1u);
      }
    }
  }
  SR_UNIT_MARK(3);
  __syncthreads();
  if (w == 0) {  // bin totals -> output starts, 4-key aligned regions, per-warp cursors; big pieces listed
    uint32_t c0 = 0, c1 = 0;
#pragma unroll
    for (int v = 0; v < NW; v++) { c0 += e.wcnt[v][2 * lane]; c1 += e.wcnt[v][2 * lane + 1]; }
    const uint32_t r0 = (c0 + 3u) & ~3u;  // equality bins take no region (filled, not moved)
    uint32_t oi = c0 + c1, ri = r0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t1 = __shfl_up_sync(0xffffffffu, oi, o), t2 = __shfl_up_sync(0xffffffffu, ri, o);
      if (lane >= o) { oi += t1; ri += t2; }
    }
    const uint32_t ob = oi - c0 - c1, rb = ri - r0;
    e.ost[2 * lane] = ob;
    e.ost[2 * lane + 1] = ob + c0;
    e.reg[2 * lane] = rb;
    e.reg[2 * lane + 1] = rb + r0;
    if (lane == 31) { e.ost[NB] = oi; e.reg[NB] = ri; }
    uint32_t run = rb;
#pragma unroll
    for (int v = 0; v < NW; v++) {
      const uint32_t cc = e.wcnt[v][2 * lane];
      e.wcnt[v][2 * lane] = run;
      run += cc;
    }
    if (c0 > (uint32_t)UnitNet<K>::PIECE) e.big[atomicAdd(&e.nbig, 1u)] = (uint16_t)(2 * lane);
  }
  SR_UNIT_MARK(4);
  __syncthreads();
  // move range keys to their bin regions (same key <-> warp map as the count)
  for (int i0 = 0; i0 < L; i0 += NT * UC) {
    K x[UC];
    int b[UC];
#pragma unroll
    for (int u = 0; u < UC; u++) {
      const int i = i0 + u * NT + tid;
      b[u] = i < L ? (int)e.bin[i] : 1;
      x[u] = i < L ? e.x[i] : K(0);
    }
#pragma unroll
    for (int u = 0; u < UC; u++)
      if (!(b[u] & 1)) e.y[atomicAdd(&e.wcnt[w][b[u]], 1u)] = x[u];
  }
  SR_UNIT_MARK(5);
  __syncthreads();
  // warps: sub-bucket s = range bin 2s (sorted) + equality bin 2s+1 (filled)
  for (int sb = w; sb < SB; sb += NW) {
    const int b = 2 * sb;
    const int o = (int)e.ost[b], len = (int)(e.ost[b + 1] - e.ost[b]);
    if (len > 0 && len <= UnitNet<K>::PIECE) unit_warp_piece<K>(e.y + e.reg[b], len, dst + o);
    const int oe = (int)e.ost[b + 1], le = (int)(e.ost[b + 2] - e.ost[b + 1]);
    if (le > 0) {
      const K key = e.spl[sb];
      for (int i = lane; i < le; i += 32) dst[oe + i] = key;
    }
  }
  SR_UNIT_MARK(6);
  __syncthreads();
  SR_UNIT_MARK(7);
  for (uint32_t k = 0; k < e.nbig; k++) {  // extreme skew: a piece above 2048 keys, CTA-wide
    const int b = e.big[k];
    const int o = (int)e.ost[b], len = (int)(e.ost[b + 1] - e.ost[b]);
    const int rg = (int)e.reg[b];
    for (int i = tid; i < len; i += NT) e.x[i] = e.y[rg + i];
    __syncthreads();
    unit_cta_merge_sort<K, NT>(e.x, e.y, len, dst + o);
  }
  __syncthreads();
}

}  // namespace sr
