// outlier.cuh -- the nearly-sorted route: k-exchange
// and similar inputs ("k-exchange ... k pairs of elements
// exchanged") are sorted by extracting their outliers instead of
// partitioning everything.
//
// One round: an element is an outlier when it is an endpoint of a descent
// (a[i-1] > a[i] or a[i] > a[i+1]).  Removing both endpoints of
// every descent leaves ascending stretches whose concatenation is sorted
// whenever the descents are isolated (a random exchange of positions p < q
// creates descents at p and q-1, and removing p, p+1, q-1, q leaves the
// ramp).  The kept keys are compacted in input order to dst[0, r) and the
// outliers to dst[r, n); the same kernel counts descents between kept keys so
// the host knows whether the remainder is sorted.  The outliers (about two per
// descent) are then sorted by the ordinary route and merged with the
// remainder (one merge-path pass, §3(g)); otherwise another round runs on the
// remainder, and after two rounds the route falls back to the partition.
#pragma once
#include "common.cuh"
#include "types.cuh"

namespace sr {

constexpr int kOutNT = 512;
template <typename K>
struct OutTile {  // keys per CTA: the tile state (OutSmem) fits the 48 KB static shared memory
  static constexpr int T = 16384 / (int)sizeof(K);
  static constexpr int VT = T / kOutNT;
};

// Shared state of one tile: the keys with a one-key halo on each side, the
// kept keys in order (and where they came from), and per-(u, warp) counts.
template <typename K, int NT, int TT = OutTile<K>::T>
struct OutSmem {
  static constexpr int T = TT, VT = TT / NT, NW = NT / 32;
  K s[T + 2];
  K sk[T];
  uint16_t si[T];
  uint8_t rm[T];
  int32_t gcnt[VT * NW + 1];
  int32_t flag;
};

// Loads tile [t0, t0 + len) with its halo and decides which keys are kept:
// first the endpoints of every descent are removed (using the neighbours
// outside the tile); then, inside the tile, the endpoints of every descent
// between consecutive kept keys, repeated until the kept keys are sorted (at
// most 4 times).  On return bal[u] holds the kept ballot of element u*NT+tid
// (striped), gcnt the exclusive kept counts of the (u, warp) groups and
// gcnt[VT*NW] the tile's kept total.  Returns true when the kept keys were
// found sorted (false: the iteration cap was hit first).
template <typename K, int NT, int TT = OutTile<K>::T>
__device__ __forceinline__ bool out_tile_flags(const K* __restrict__ src, int64_t n, int64_t t0, int len,
                                               OutSmem<K, NT, TT>& sm, unsigned (&bal)[TT / NT]) {
  constexpr int VT = TT / NT, NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  {
    K v[VT];
#pragma unroll
    for (int u = 0; u < VT; u++) {
      const int i = u * NT + tid;
      v[u] = i < len ? src[t0 + i] : K(0);
    }
#pragma unroll
    for (int u = 0; u < VT; u++) {
      const int i = u * NT + tid;
      if (i < len) { sm.s[1 + i] = v[u]; sm.rm[i] = 0; }
    }
    if (tid == 0) {
      if (t0 > 0) sm.s[0] = src[t0 - 1];
      if (t0 + len < n) sm.s[1 + len] = src[t0 + len];
    }
  }
  __syncthreads();
  bool keep[VT];
#pragma unroll
  for (int u = 0; u < VT; u++) {
    const int i = u * NT + tid;
    const int64_t gi = t0 + i;
    bool kp = false;
    if (i < len) {
      const K x = sm.s[1 + i];
      const bool dl = gi > 0 && sm.s[i] > x;
      const bool dr = gi + 1 < n && x > sm.s[2 + i];
      kp = !(dl || dr);
    }
    keep[u] = kp;
  }
  const unsigned lt = (1u << lane) - 1u;
  for (int iter = 0;; iter++) {
#pragma unroll
    for (int u = 0; u < VT; u++) {
      bal[u] = __ballot_sync(0xffffffffu, keep[u]);
      if (lane == 0) sm.gcnt[u * NW + w] = __popc(bal[u]);
    }
    __syncthreads();
    if (w == 0) {  // exclusive scan of the VT * NW group counts (element order: u major, warp minor)
      int carry = 0;
      for (int g0 = 0; g0 < VT * NW; g0 += 32) {
        const int v = g0 + lane < VT * NW ? sm.gcnt[g0 + lane] : 0;
        const int inc = warp_inclusive_sum(v);
        if (g0 + lane < VT * NW) sm.gcnt[g0 + lane] = carry + inc - v;
        carry += __shfl_sync(0xffffffffu, inc, 31);
      }
      if (lane == 0) { sm.gcnt[VT * NW] = carry; sm.flag = 0; }
    }
    __syncthreads();
    if (iter == 4) return false;
    const int tot = sm.gcnt[VT * NW];
#pragma unroll
    for (int u = 0; u < VT; u++) {
      const int i = u * NT + tid;
      if (keep[u]) {
        const int kr = sm.gcnt[u * NW + w] + __popc(bal[u] & lt);
        sm.sk[kr] = sm.s[1 + i];
        sm.si[kr] = (uint16_t)i;
      }
    }
    __syncthreads();
    int any = 0;
    for (int j = tid; j + 1 < tot; j += NT)
      if (sm.sk[j] > sm.sk[j + 1]) { sm.rm[sm.si[j]] = 1; sm.rm[sm.si[j + 1]] = 1; any = 1; }
    if (__syncthreads_or(any) == 0) return true;  // the kept keys are sorted
#pragma unroll
    for (int u = 0; u < VT; u++) {
      const int i = u * NT + tid;
      if (keep[u] && sm.rm[i]) keep[u] = false;
    }
    __syncthreads();
  }
}

// K-O1: kept keys per tile -> cnt[t] (cnt has G+1 entries, cnt[G] = 0, then
// an exclusive scan turns it into tile offsets with cnt[G] = r).
template <typename K, int NT>
__global__ void __launch_bounds__(NT) k_outlier_count(const K* __restrict__ src, int64_t n, uint32_t* __restrict__ cnt) {
  __shared__ OutSmem<K, NT> sm;
  constexpr int T = OutTile<K>::T, VT = OutTile<K>::VT, NW = NT / 32;
  const int64_t t0 = (int64_t)blockIdx.x * T;
  const int len = (int)(n - t0 < T ? n - t0 : T);
  unsigned bal[VT];
  out_tile_flags<K, NT>(src, n, t0, len, sm, bal);
  if (threadIdx.x == 0) cnt[blockIdx.x] = (uint32_t)sm.gcnt[VT * NW];
}

// K-O2: stable split of each tile: kept keys -> dst[cnt[t] + rank], outliers
// -> dst[r + (t*T - cnt[t]) + rank] (r = cnt[G]); counts the descents among
// kept keys inside the tile into *bad (zero after out_tile_flags unless its
// iteration cap was hit), and records the tile's first and last kept key
// (fl[2t], fl[2t+1]) with has[t] = 1 when the tile keeps any.
template <typename K, int NT>
__global__ void __launch_bounds__(NT) k_outlier_split(const K* __restrict__ src, int64_t n,
                                                      const uint32_t* __restrict__ cnt, int G, K* __restrict__ dst,
                                                      K* __restrict__ fl, uint8_t* __restrict__ has,
                                                      unsigned long long* __restrict__ bad) {
  __shared__ OutSmem<K, NT> sm;
  __shared__ int32_t red[NT / 32 + 1];
  constexpr int T = OutTile<K>::T, VT = OutTile<K>::VT, NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t t0 = (int64_t)blockIdx.x * T;
  const int len = (int)(n - t0 < T ? n - t0 : T);
  unsigned bal[VT];
  out_tile_flags<K, NT>(src, n, t0, len, sm, bal);
  const int tot = sm.gcnt[VT * NW];
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int u = 0; u < VT; u++) {
    const int i = u * NT + tid;
    if (i < len) {
      const int kr = sm.gcnt[u * NW + w] + __popc(bal[u] & lt);  // kept before element i
      if ((bal[u] >> lane) & 1u) sm.sk[kr] = sm.s[1 + i];
      else sm.sk[tot + (i - kr)] = sm.s[1 + i];
    }
  }
  __syncthreads();
  const uint32_t kbase = cnt[blockIdx.x];
  const uint32_t r = cnt[G];
  const int64_t obase = (int64_t)r + (t0 - kbase);
  SR_CHECK((int64_t)kbase + tot <= r && obase + (len - tot) <= n);
  for (int i = tid; i < tot; i += NT) dst[kbase + i] = sm.sk[i];
  for (int i = tid; i < len - tot; i += NT) dst[obase + i] = sm.sk[tot + i];
  int b = 0;
  for (int i = tid; i + 1 < tot; i += NT) b += sm.sk[i] > sm.sk[i + 1];
  b = block_reduce_sum<NT>(b, red);
  if (tid == 0) {
    if (b) atomicAdd(bad, (unsigned long long)b);
    has[blockIdx.x] = tot > 0;
    if (tot > 0) {
      fl[2 * blockIdx.x] = sm.sk[0];
      fl[2 * blockIdx.x + 1] = sm.sk[tot - 1];
    }
  }
}

// K-O3: descents between kept keys of consecutive tiles (tiles that keep
// nothing are skipped over).
template <typename K>
__global__ void k_outlier_check(const K* __restrict__ fl, const uint8_t* __restrict__ has, int G,
                                unsigned long long* __restrict__ bad) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= G || !has[t]) return;
  int u = t + 1;
  while (u < G && !has[u]) u++;
  if (u < G && fl[2 * t + 1] > fl[2 * u]) atomicAdd(bad, 1ull);
}

}  // namespace sr
