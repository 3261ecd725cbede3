// measures.cuh -- presortedness measures of the paper's input classes
// (SURVEY.md §8(f) NEXT #4), as a library call:
//   Run(A)  = #{i : a_i > a_{i+1}} + 1
//   Mono(A) = fewest contiguous pieces, each sorted or reversely sorted (:72)
//   Inv(A)  = #{(i, j) : i < j, a_i > a_j}                     (:64)
//   Dis(A)  = max_i |rank(a_i) - i|   (the k-distance class)   (:84)
//   Mis(A)  = #{i : rank(a_i) != i}   (<= 2k for k-exchange)   (:85)
// with rank = the stable rank.
//
// Mono: the greedy left-to-right partition (a piece is extended while it
// stays non-decreasing or non-increasing; its direction is fixed by its first
// strict step) is optimal for contiguous pieces.  Greedy is a 3-state
// automaton over the comparisons c_i of (a_i, a_{i+1}); the transition maps
// compose associatively, so every thread folds its chunk into one map, the
// CTA and then one final CTA compose the maps in order.  Inv is counted on
// the stable-rank permutation (ties never count) by log2(n) bottom-up merge
// levels in which every element finds its output slot by binary search in the
// other run and an element of a right run adds the number of left-run
// elements greater than it.
#pragma once
#include <cstdint>

#include "common.cuh"

namespace sr {

// transition map over the states U (direction undetermined) = 0, A (non-
// decreasing) = 1, D (non-increasing) = 2: next state per start state and the
// number of piece boundaries crossed
struct MonoMap {
  uint8_t next[3];
  uint8_t pad;
  uint32_t inc[3];
};

__device__ __forceinline__ MonoMap mono_identity() {
  MonoMap m;
  m.next[0] = 0; m.next[1] = 1; m.next[2] = 2; m.pad = 0;
  m.inc[0] = m.inc[1] = m.inc[2] = 0;
  return m;
}

// step: -1 (a_i > a_{i+1}), 0 (equal), +1 (a_i < a_{i+1})
__device__ __forceinline__ MonoMap mono_step(int step) {
  MonoMap m = mono_identity();
  if (step > 0) { m.next[0] = 1; m.next[2] = 0; m.inc[2] = 1; }       // U->A; D breaks
  else if (step < 0) { m.next[0] = 2; m.next[1] = 0; m.inc[1] = 1; }  // U->D; A breaks
  return m;
}

// f then g
__device__ __forceinline__ MonoMap mono_compose(const MonoMap& f, const MonoMap& g) {
  MonoMap h;
  h.pad = 0;
#pragma unroll
  for (int s = 0; s < 3; s++) {
    h.next[s] = g.next[f.next[s]];
    h.inc[s] = f.inc[s] + g.inc[f.next[s]];
  }
  return h;
}

// one map per CTA over the comparisons i in [b*CH, (b+1)*CH) (i + 1 < n), and
// the descents of those comparisons
template <typename K, int NT>
__global__ void __launch_bounds__(NT) k_mono_map(const K* __restrict__ keys, int64_t n, int64_t chunk,
                                                 MonoMap* __restrict__ maps, unsigned long long* __restrict__ descents) {
  __shared__ MonoMap s_m[NT];
  const int64_t c0 = (int64_t)blockIdx.x * chunk;
  const int64_t c1 = c0 + chunk < n - 1 ? c0 + chunk : n - 1;  // comparisons i in [c0, c1)
  const int64_t per = (chunk + NT - 1) / NT;
  const int64_t t0 = c0 + (int64_t)threadIdx.x * per;
  const int64_t t1 = t0 + per < c1 ? t0 + per : c1;
  MonoMap m = mono_identity();
  unsigned long long d = 0;
  for (int64_t i = t0; i < t1; i++) {
    const K x = keys[i], y = keys[i + 1];
    const int step = x < y ? 1 : (x > y ? -1 : 0);
    d += step < 0;
    m = mono_compose(m, mono_step(step));
  }
  s_m[threadIdx.x] = m;
  __syncthreads();
  for (int w = 1; w < NT; w *= 2) {  // ordered tree: s[i] = s[i] then s[i + w]
    MonoMap r;
    const bool act = (threadIdx.x % (2 * w)) == 0 && threadIdx.x + w < NT;
    if (act) r = mono_compose(s_m[threadIdx.x], s_m[threadIdx.x + w]);
    __syncthreads();
    if (act) s_m[threadIdx.x] = r;
    __syncthreads();
  }
  if (threadIdx.x == 0) maps[blockIdx.x] = s_m[0];
  __syncthreads();  // s_m is reused as the reduction scratch
  d = block_reduce_sum<NT>(d, reinterpret_cast<unsigned long long*>(s_m));
  if (threadIdx.x == 0 && d) atomicAdd(descents, d);
}

// compose the CTA maps in order (one thread; G is small) from state U
__global__ void k_mono_final(const MonoMap* __restrict__ maps, int G, unsigned long long* __restrict__ pieces) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  MonoMap m = mono_identity();
  for (int g = 0; g < G; g++) m = mono_compose(m, maps[g]);
  *pieces = 1ull + m.inc[0];
}

// idx = the stable-sorted order of the input positions: max |p - idx[p]| and #{p : idx[p] != p}
template <int NT>
__global__ void __launch_bounds__(NT) k_dis(const uint32_t* __restrict__ idx, int64_t n,
                                            unsigned long long* __restrict__ maxdis,
                                            unsigned long long* __restrict__ misplaced) {
  __shared__ unsigned long long s_red[NT / 32 + 1];
  unsigned long long mx = 0, mis = 0;
  for (int64_t p = (int64_t)blockIdx.x * NT + threadIdx.x; p < n; p += (int64_t)gridDim.x * NT) {
    const int64_t d = p - (int64_t)idx[p];
    const unsigned long long a = (unsigned long long)(d < 0 ? -d : d);
    mx = a > mx ? a : mx;
    mis += a != 0;
  }
  mis = block_reduce_sum<NT>(mis, s_red);
  mx = block_reduce_max<NT>(mx, s_red);
  if (threadIdx.x == 0) {
    if (mis) atomicAdd(misplaced, mis);
    atomicMax(maxdis, mx);
  }
}

// one merge level of width R over a permutation (distinct values): every
// element lands at (its index in its run) + (#smaller in the other run); an
// element of a right run contributes #greater in the left run to Inv
template <int NT>
__global__ void __launch_bounds__(NT) k_inv_level(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                                                  int64_t n, int64_t R, unsigned long long* __restrict__ inv) {
  __shared__ unsigned long long s_red[NT / 32 + 1];
  unsigned long long cnt = 0;
  for (int64_t g = (int64_t)blockIdx.x * NT + threadIdx.x; g < n; g += (int64_t)gridDim.x * NT) {
    const int64_t L0 = (g / (2 * R)) * (2 * R);
    const int64_t la = R < n - L0 ? R : n - L0;                 // left run length
    const int64_t lb = n - L0 - la < R ? n - L0 - la : R;       // right run length
    const uint32_t v = src[g];
    const bool left = g < L0 + la;
    const uint32_t* other = left ? src + L0 + la : src + L0;
    const int64_t lo_len = left ? lb : la;
    int64_t lo = 0, hi = lo_len;  // #elements of the other run smaller than v
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (other[mid] < v) lo = mid + 1; else hi = mid;
    }
    const int64_t own = left ? g - L0 : g - L0 - la;
    dst[L0 + own + lo] = v;
    if (!left) cnt += (unsigned long long)(la - lo);
  }
  cnt = block_reduce_sum<NT>(cnt, s_red);
  if (threadIdx.x == 0 && cnt) atomicAdd(inv, cnt);
}

__global__ void k_iota(uint32_t* __restrict__ idx, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    idx[i] = (uint32_t)i;
}

}  // namespace sr
