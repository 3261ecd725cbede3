// guide.cuh -- bucket classification (H8) through a guide table over the
// distinct splitters: the bucket id of a key is the 3-way id of the
// lower_bound i = #{t_j < x} among the level's sorted splitters t_0..t_{m-1}
// (2i for the range between t_{i-1} and t_i, 2i + 1 when
// x equals an equality splitter t_i, flagged by the gamma test of PAPER.md:168).
//
// The lower_bound is found by comparisons with the splitters, as the tree walk
// does (classify_keys); the table only narrows WHICH splitters to compare
// with.  The order-preserving unsigned images u(t) of the distinct splitter
// values ud_0 < ... < ud_{md-1} are covered by kGCells equal cells of width
// 2^shift starting at u(ud_0); cell c stores a = #{ud_k < start(c)} and the
// count of distinct splitters inside it, so #{ud_k < x} lies in [a, a + count]
// for every key of the cell.  A fixed, table-wide number of predicated
// bisection steps (enough for the fullest cell) closes that interval with no
// data-dependent branches; the splitter index is then i = first[k], the first
// occurrence of ud_k among the (possibly repeated) splitters, so the ids are
// exactly those of the tree walk.  Measured (tools/micro/classify.cu, 256M
// random int32, persistent CTAs): 0.40 ms at B = 512 and 0.52 ms at B = 2048,
// against 0.73 / 0.94 ms for the Eytzinger walk and 0.62 / 0.71 ms for the
// data-dependent guided search it replaces.
#pragma once
#include <cstdint>

#include "common.cuh"
#include "types.cuh"

namespace sr {

constexpr int kGCells = 4096;

template <typename K, int CELLS = kGCells, int BMAX = kMaxBuckets>
struct alignas(16) GuideTab {
  static constexpr int kCells = CELLS, kBMax = BMAX;  // cells; splitters (< BMAX)
  uint64_t u0, u1;                 // u(ud_0), u(ud_{md-1})
  int32_t shift, md, m, steps;     // cell width 2^shift; distinct / all splitters; bisection steps
  int32_t has_dup, any_eq, pad0, pad1;
  uint32_t cell[CELLS];            // a | count << 16
  K ud[BMAX];                      // distinct splitters, ascending
  uint16_t first[BMAX];            // index of ud_k's first occurrence among the splitters
  uint8_t eq[BMAX];                // equality flag of ud_k
};

template <typename K>
__device__ __forceinline__ uint64_t guide_u(K x) {  // order-preserving unsigned image
  return sizeof(K) == 4 ? (uint64_t)((uint32_t)x ^ 0x80000000u) : ((uint64_t)x ^ 0x8000000000000000ull);
}

// Build g from the m >= 1 sorted splitters spl[0, m) and their flags (all NT
// threads of the block; g may live in shared or global memory; red: NT/32 + 1
// ints of shared scratch).  O(m + kGCells) work and two block scans: the
// distinct splitters by a scan of "differs from its predecessor", then the
// cells by counting each distinct splitter into its cell and a scan of the
// counts (a = #{ud_k < start(c)} = #{k : cell(k) < c} because ud is sorted).
// Returns with g complete and visible to the block.
template <typename K, int NT, typename G>
__device__ __noinline__ void guide_build(const K* spl, const uint8_t* eqf, int m, G& g, int* red) {
  constexpr int kGCells = G::kCells;
  constexpr int PER = (G::kBMax + NT - 1) / NT;
  constexpr int CPT = kGCells / NT;
  static_assert(kGCells % NT == 0, "");
  const int tid = threadIdx.x;
  // 1. distinct values (ascending input: a value starts where it differs from its predecessor)
  int cnt = 0, dup = 0, aeq = 0;
  for (int r = 0; r < PER; r++) {
    const int j = tid * PER + r;
    if (j < m) {
      const bool f = j == 0 || spl[j] != spl[j - 1];
      cnt += f;
      dup |= !f;
      aeq |= eqf[j];
    }
  }
  int md;
  int ex = block_exclusive_sum<NT>(cnt, red, &md);
  for (int r = 0; r < PER; r++) {
    const int j = tid * PER + r;
    if (j < m && (j == 0 || spl[j] != spl[j - 1])) {
      g.ud[ex] = spl[j];
      g.first[ex] = (uint16_t)j;
      g.eq[ex] = eqf[j];
      ex++;
    }
  }
  for (int c = tid; c < kGCells; c += NT) g.cell[c] = 0u;
  dup = __syncthreads_or(dup);
  aeq = __syncthreads_or(aeq);
  // 2. cells of width 2^shift over [u(ud_0), u(ud_{md-1})]: counts, then prefixes
  const uint64_t u0 = guide_u<K>(g.ud[0]), u1 = guide_u<K>(g.ud[md - 1]);
  const uint64_t span = u1 - u0;
  int shift = 0;
  while (shift < 63 && (span >> shift) >= (uint64_t)kGCells) shift++;
  for (int k = tid; k < md; k += NT) atomicAdd(&g.cell[(int)((guide_u<K>(g.ud[k]) - u0) >> shift)], 1u);
  __syncthreads();
  uint32_t v[CPT], sum = 0, mx = 0;
#pragma unroll
  for (int r = 0; r < CPT; r++) {
    v[r] = g.cell[tid * CPT + r];
    sum += v[r];
    mx = max(mx, v[r]);
  }
  uint32_t total;
  uint32_t a = block_exclusive_sum<NT>(sum, reinterpret_cast<uint32_t*>(red), &total);
#pragma unroll
  for (int r = 0; r < CPT; r++) {
    g.cell[tid * CPT + r] = a | (v[r] << 16);
    a += v[r];
  }
  // block max of the cell counts -> bisection steps: an interval of length L
  // closes in ceil(log2(L + 1)) halvings
  mx = warp_reduce_max(mx);
  if ((tid & 31) == 0) red[tid >> 5] = (int)mx;
  __syncthreads();
  if (tid == 0) {
    int vm = 0;
    for (int w = 0; w < NT / 32; w++) vm = max(vm, red[w]);
    int st = 0;
    while ((1 << st) <= vm) st++;
    g.u0 = u0; g.u1 = u1; g.shift = shift; g.md = md; g.m = m; g.steps = st;
    g.has_dup = dup; g.any_eq = aeq; g.pad0 = 0; g.pad1 = 0;
  }
  __syncthreads();
}

// Copy a built table (global) into shared memory (all threads of the block; 16-byte words).
template <typename G>
__device__ __forceinline__ void guide_load(const G* __restrict__ src, G& dst) {
  static_assert(sizeof(G) % 16 == 0, "");
  const int4* s = reinterpret_cast<const int4*>(src);
  int4* d = reinterpret_cast<int4*>(&dst);
  for (int i = threadIdx.x; i < (int)(sizeof(G) / 16); i += blockDim.x) d[i] = __ldcg(s + i);
}

// 3-way bucket ids of U keys (lockstep, U-way ILP).
template <typename K, int U, typename G>
__device__ __forceinline__ void guide_classify(const K (&x)[U], int (&bin)[U], const G& g) {
  constexpr int kGCells = G::kCells;
  const int md = g.md, steps = g.steps, shift = g.shift;
  int lo[U], hi[U];
  if constexpr (sizeof(K) == 4) {
    const uint32_t u0 = (uint32_t)g.u0, u1 = (uint32_t)g.u1;
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint32_t v = (uint32_t)x[u] ^ 0x80000000u;
      const uint32_t c = min((v - u0) >> shift, (uint32_t)kGCells - 1);
      const uint32_t w = g.cell[c];
      const int a = (int)(w & 0xffffu), b = a + (int)(w >> 16);
      lo[u] = v <= u0 ? 0 : (v > u1 ? md : a);
      hi[u] = v <= u0 ? 0 : (v > u1 ? md : b);
    }
  } else {
    const uint64_t u0 = g.u0, u1 = g.u1;
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint64_t v = (uint64_t)x[u] ^ 0x8000000000000000ull;
      const uint64_t cc = (v - u0) >> shift;
      const uint32_t c = cc < (uint64_t)kGCells ? (uint32_t)cc : (uint32_t)kGCells - 1;
      const uint32_t w = g.cell[c];
      const int a = (int)(w & 0xffffu), b = a + (int)(w >> 16);
      lo[u] = v <= u0 ? 0 : (v > u1 ? md : a);
      hi[u] = v <= u0 ? 0 : (v > u1 ? md : b);
    }
  }
#pragma unroll 1
  for (int s = 0; s < steps; s++) {
#pragma unroll
    for (int u = 0; u < U; u++) {
      const bool act = lo[u] < hi[u];
      const int mid = (lo[u] + hi[u]) >> 1;
      const bool p = g.ud[mid] < x[u];
      lo[u] = (act && p) ? mid + 1 : lo[u];
      hi[u] = (act && !p) ? mid : hi[u];
    }
  }
  if (g.has_dup) {
    const int m = g.m;
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int k = lo[u];
      const int i = k < md ? (int)g.first[k] : m;
      bin[u] = 2 * i + ((g.any_eq && k < md && g.ud[k] == x[u] && g.eq[k]) ? 1 : 0);
    }
  } else if (g.any_eq) {
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int k = lo[u];
      bin[u] = 2 * k + ((k < md && g.ud[k] == x[u] && g.eq[k]) ? 1 : 0);
    }
  } else {
#pragma unroll
    for (int u = 0; u < U; u++) bin[u] = 2 * lo[u];
  }
}

// One CTA per segment: the guide table of segment blockIdx.x's splitters
// (spl_all / eq_all / m_all: kMaxBuckets-strided, as written by K7).
template <typename K, int NT>
__global__ void __launch_bounds__(NT) k_guide_build(const K* __restrict__ spl_all, const uint8_t* __restrict__ eq_all,
                                                    const int* __restrict__ m_all, GuideTab<K>* __restrict__ out,
                                                    const DevStats* __restrict__ gate) {
  if (gate && gate->route != kRoutePartition) return;  // speculative launch
  __shared__ int red[NT / 32 + 1];
  const int s = blockIdx.x;
  guide_build<K, NT>(spl_all + (int64_t)s * kMaxBuckets, eq_all + (int64_t)s * kMaxBuckets, m_all[s], out[s], red);
}

}  // namespace sr
