// distance.cuh -- the k-distance route (bounded
// displacement): inputs in which every key lies fewer than kDT = 2 kDSub
// positions from its place in the sorted output ("k-distance ...
// |rank(a_i) - i| <= k"; Table 1's "nearly sorted" class is 256-distance,
// PAPER.md:36).  The presortedness scan proves the bound from subtile minima
// and maxima (presort.cuh tile_mm_finish); the sort is then two passes:
//   A  every window [2j kDT, 2j kDT + 2 kDT) is sorted (one warp's register
//      network, unit_sort.cuh; is_sorted skip);
//   B  every window [(2j+1) kDT, (2j+1) kDT + 2 kDT) -- the upper half of one
//      A window and the lower half of the next, each sorted -- is merged
//      (merge path, A wins ties PAPER.md:99; ordered halves are "trimmed",
//      PAPER.md:99, and left alone).
// Why two passes suffice when every displacement is < kDT (keys-only; ties are
// ranked by position): the A window of tiles (P-1, P) (tiles of kDT keys)
// holds exactly kDT keys of rank < P kDT -- the keys of ranks in
// [(P-1) kDT, P kDT) that lie before it are as many as the keys of rank
// < (P-1) kDT that lie inside it, and no key moves further than one tile -- so
// after A tile P holds only ranks >= P kDT and tile P+1 only ranks < (P+2) kDT;
// the B window (P, P+1) therefore holds exactly ranks [P kDT, (P+2) kDT) and
// its merge puts them in place.  Tile 0 is final after A for the same reason.
// Traffic: the scan (1N) + A (2N) + B (2N, less where halves are trimmed).
#pragma once
#include "common.cuh"
#include "types.cuh"
#include "unit_sort.cuh"

namespace sr {

constexpr int kDT = 2 * kDSub;  // tile of the two passes: displacements < kDT
constexpr int kDistWarps = 4;   // warps per CTA (one window each)
static_assert(2 * kDT <= UnitNet<int64_t>::PIECE, "an A window is one warp's piece");

template <typename K>
__global__ void __launch_bounds__(32 * kDistWarps) k_window_sort(K* __restrict__ keys, int64_t n,
                                                                  const DevStats* __restrict__ gate) {
  if (gate && gate->route != kRouteDistance) return;
  constexpr int PIECE = UnitNet<K>::PIECE;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  K* stage = reinterpret_cast<K*>(smem_raw) + w * PIECE;
  constexpr int W = 2 * kDT;
  const int64_t nwin = (n + W - 1) / W;
  for (int64_t wi = (int64_t)blockIdx.x * kDistWarps + w; wi < nwin; wi += (int64_t)gridDim.x * kDistWarps) {
    const int64_t s = wi * W;
    const int len = (int)(n - s < W ? n - s : W);
    for (int i = lane; i < len; i += 32) stage[i] = keys[s + i];
    __syncwarp();
    int unsorted = 0;  // is_sorted
    for (int i = lane; i + 1 < len; i += 32) unsorted |= stage[i + 1] < stage[i];
    if (__any_sync(0xffffffffu, unsorted)) unit_warp_piece<K>(stage, len, keys + s);
    __syncwarp();
  }
}

template <typename K>
__global__ void __launch_bounds__(32 * kDistWarps) k_window_merge(K* __restrict__ keys, int64_t n,
                                                                   const DevStats* __restrict__ gate) {
  if (gate && gate->route != kRouteDistance) return;
  constexpr int PIECE = UnitNet<K>::PIECE;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  K* stage = reinterpret_cast<K*>(smem_raw) + w * PIECE;
  constexpr int W = 2 * kDT;
  const int64_t nwin = n > kDT ? (n - kDT + W - 1) / W : 0;
  for (int64_t wi = (int64_t)blockIdx.x * kDistWarps + w; wi < nwin; wi += (int64_t)gridDim.x * kDistWarps) {
    const int64_t s = kDT + wi * W;
    const int len = (int)(n - s < W ? n - s : W);
    if (len <= kDT) continue;                                        // one sorted half only
    if (!(keys[s + kDT] < keys[s + kDT - 1])) continue;              // trimmed: halves in order
    for (int i = lane; i < len; i += 32) stage[i] = keys[s + i];
    __syncwarp();
    unit_warp_merge<K>(stage, kDT, stage + kDT, len - kDT, keys + s);
  }
}

}  // namespace sr
