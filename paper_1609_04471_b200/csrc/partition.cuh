// partition.cuh -- the quicksort analogue (H7-H11): splitter sampling, bucket
// classification + histogram, count-matrix scan, bucket planning, stable
// 3-way scatter and bucket finishing.
//
// Paper anchors (§4; Appendix B):
//  (c) pseudo-median of 9 pivot "crucial" against O(n^2)
//      -> B-1 splitters from an oversampled, jittered, stratified sample (K7);
//  (d) 3-way splitting, equal keys "spared from the recursive calls"
//       -> equality buckets that are final after one scatter;
//  (e) "do not identify the position of the pivot ... presortedness of the
//      input is not disturbed" -> splitters are values and the
//      scatter is stable;
//  (g) "At first, use the 2-way splitting. If the array contains more than
//      gamma = 2 elements equal to the pivot, use the 3-way splitting"
//       -> a splitter becomes an equality splitter only when it
//      occurs more than twice in the sample;
//  (a)/(f) insertion sort below alpha and is_sorted at every call
//       -> buckets <= kCap are finished by the CTA tile
//      sort (K11) with an is_sorted skip.
#pragma once
#include "bitonic.cuh"
#include "block_sort.cuh"
#include "common.cuh"
#include "guide.cuh"
#include "presort.cuh"
#include "types.cuh"
#include "unit_sort.cuh"

namespace sr {

// Generic block exclusive scan with an associative op (scratch: NT/32+1).
template <int NT, typename T, typename Op>
__device__ __forceinline__ T block_exclusive_scan_op(T v, T identity, Op op, T* scratch, T* total) {
  constexpr int NW = NT / kWarp;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T inc = v;
#pragma unroll
  for (int o = 1; o < kWarp; o <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc = op(u, inc);
  }
  T ex = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane == 0) ex = identity;
  if (lane == 31) scratch[w] = inc;
  __syncthreads();
  if (w == 0) {
    T s = lane < NW ? scratch[lane] : identity;
    T si = s;
#pragma unroll
    for (int o = 1; o < kWarp; o <<= 1) {
      T u = __shfl_up_sync(0xffffffffu, si, o);
      if (lane >= o) si = op(u, si);
    }
    T se = __shfl_up_sync(0xffffffffu, si, 1);
    if (lane == 0) se = identity;
    if (lane < NW) scratch[lane] = se;
    if (lane == NW - 1) scratch[NW] = si;
  }
  __syncthreads();
  T r = op(scratch[w], ex);
  if (total) *total = scratch[NW];
  __syncthreads();
  return r;
}

// In-place scan of a shared array a[0, L) (L <= 4*NT).  exclusive / reverse
// (suffix) variants.  All NT threads must call.
template <int NT, typename T, typename Op>
__device__ void smem_scan(T* a, int L, T identity, Op op, bool exclusive, bool reverse, T* scratch) {
  const int ipt = (L + NT - 1) / NT;
  const int b0 = threadIdx.x * ipt;
  T agg = identity;
  for (int j = 0; j < ipt; j++) {
    int i = b0 + j;
    if (i < L) agg = op(agg, a[reverse ? L - 1 - i : i]);
  }
  T pre = block_exclusive_scan_op<NT>(agg, identity, op, scratch, (T*)nullptr);
  for (int j = 0; j < ipt; j++) {
    int i = b0 + j;
    if (i < L) {
      int idx = reverse ? L - 1 - i : i;
      T x = a[idx];
      T inc = op(pre, x);
      a[idx] = exclusive ? pre : inc;
      pre = inc;
    }
  }
  __syncthreads();
}

// Exclusive sum of a shared uint32 array in place (one out-of-line copy: the
// resident kernel calls it from several phases, and every inlined copy is
// instruction-cache footprint fetched cold after an L2 flush).
template <int NT>
__device__ __noinline__ void smem_exclusive_sum_u32(uint32_t* a, int L, uint32_t* scratch) {
  smem_scan<NT>(a, L, 0u, [](uint32_t x, uint32_t y) { return x + y; }, true, false, scratch);
}

// ---------------------------------------------------------------------------
// K7: splitters for every segment of a level, in two kernels.
//
// K7a ranks the S-key sample without sorting it: rank(i) = #{j : (s_j, j) <
// (s_i, i)}, the position of sample i in the stably sorted sample.  Grid =
// (S/NT) x J x segments; each CTA gathers one of J chunks of the sample into
// shared memory and every thread counts, for its own sample key, the chunk
// keys ordered before it (<= for j < i, < for j > i), then adds the partial
// count to rank[i].  O(S^2) compare+add pairs spread over the whole GPU, no
// serial merge levels.
template <typename K, int NT>
__global__ void __launch_bounds__(NT) k_sample_rank(const K* __restrict__ src, const SegDesc* __restrict__ segs,
                                                     int oversample, uint32_t* __restrict__ rank,
                                                     K* __restrict__ sample, const DevStats* __restrict__ gate) {
  if (gate && gate->route != kRoutePartition) return;  // speculative launch
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* s_chunk = reinterpret_cast<K*>(smem_raw);  // ceil(S_max / J) keys
  const int J = gridDim.y;
  const SegDesc seg = segs[blockIdx.z];
  int64_t S64 = (int64_t)seg.nbuckets * oversample;
  if (S64 > seg.len) S64 = seg.len;
  if (S64 > kMaxSample) S64 = kMaxSample;
  const int S = (int)S64;
  const int i0 = blockIdx.x * NT;
  if (i0 >= S) return;
  const int log2S = (S & (S - 1)) == 0 ? __ffs(S) - 1 : -1;
  const int cj = (S + J - 1) / J;
  const int j0 = blockIdx.y * cj;
  const int j1 = j0 + cj < S ? j0 + cj : S;
  if (j0 >= j1) return;
  const int len = j1 - j0;
  for (int base = 0; base < len; base += 8 * NT) {  // 8 gathers per thread in flight
    K y[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int jj = base + u * NT + threadIdx.x;
      y[u] = jj < len ? src[sample_position(seg.start, seg.len, S, j0 + jj, log2S)] : K(0);
    }
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int jj = base + u * NT + threadIdx.x;
      if (jj < len) s_chunk[jj] = y[u];
    }
  }
  const int i = i0 + threadIdx.x;
  K x = i < S ? src[sample_position(seg.start, seg.len, S, i, log2S)] : K(0);
  if (blockIdx.y == 0 && i < S) sample[seg.sample_base + i] = x;
  __syncthreads();
  if (i < S) {
    const int split = i - j0 < 0 ? 0 : (i - j0 > len ? len : i - j0);  // chunk keys before i: [0, split)
    uint32_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
    int jj = 0;
    for (; jj + 4 <= split; jj += 4) {
      r0 += s_chunk[jj] <= x; r1 += s_chunk[jj + 1] <= x; r2 += s_chunk[jj + 2] <= x; r3 += s_chunk[jj + 3] <= x;
    }
    for (; jj < split; jj++) r0 += s_chunk[jj] <= x;
    jj = (i >= j0 && i < j1) ? split + 1 : split;
    for (; jj + 4 <= len; jj += 4) {
      r0 += s_chunk[jj] < x; r1 += s_chunk[jj + 1] < x; r2 += s_chunk[jj + 2] < x; r3 += s_chunk[jj + 3] < x;
    }
    for (; jj < len; jj++) r0 += s_chunk[jj] < x;
    const uint32_t r = r0 + r1 + r2 + r3;
    atomicAdd(&rank[seg.sample_base + i], r);
  }
}

// K7b: one CTA per segment places the sample at its ranks (the sorted sample),
// then splitter t_j = sorted[((j+1)*S)/B], j = 0..B-2, with the equality flag
// set when t_j occurs more than gamma = 2 times in the sample,
// i.e. when three consecutive sorted samples around position r equal t_j.
template <typename K, int NT>
__global__ void __launch_bounds__(NT) k_select_splitters(const SegDesc* __restrict__ segs, int oversample,
                                                          const uint32_t* __restrict__ rank,
                                                          const K* __restrict__ sample, K* __restrict__ spl_out,
                                                          uint8_t* __restrict__ eq_out, int* __restrict__ m_out,
                                                          const DevStats* __restrict__ gate) {
  if (gate && gate->route != kRoutePartition) return;  // speculative launch
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* sorted = reinterpret_cast<K*>(smem_raw);
  const SegDesc seg = segs[blockIdx.x];
  const int B = seg.nbuckets;
  int64_t S64 = (int64_t)B * oversample;
  if (S64 > seg.len) S64 = seg.len;
  if (S64 > kMaxSample) S64 = kMaxSample;
  const int S = (int)S64;
  for (int i = threadIdx.x; i < S; i += NT) sorted[rank[seg.sample_base + i]] = sample[seg.sample_base + i];
  __syncthreads();
  K* out = spl_out + (int64_t)blockIdx.x * kMaxBuckets;
  uint8_t* eo = eq_out + (int64_t)blockIdx.x * kMaxBuckets;
  for (int j = threadIdx.x; j < B - 1; j += NT) {
    const int r = (int)(((int64_t)(j + 1) * S) / B);
    const K t = sorted[r];
    const bool m1 = r >= 1 && sorted[r - 1] == t, m2 = r >= 2 && sorted[r - 2] == t;
    const bool p1 = r + 1 < S && sorted[r + 1] == t, p2 = r + 2 < S && sorted[r + 2] == t;
    out[j] = t;
    eo[j] = ((m1 && m2) || (m1 && p1) || (p1 && p2)) ? 1 : 0;  // count > gamma = 2
  }
  if (threadIdx.x == 0) m_out[blockIdx.x] = B - 1;
}

// K7 (small samples, e.g. every level >= 2 segment): one CTA per segment
// gathers its S <= NT*VT samples, sorts them with the register/shuffle bitonic
// network and selects the splitters + gamma flags like K7b.
template <typename K, int NT, int VT>
__global__ void __launch_bounds__(NT) k_sample_sort(const K* __restrict__ src, const SegDesc* __restrict__ segs,
                                                     int oversample, K* __restrict__ spl_out,
                                                     uint8_t* __restrict__ eq_out, int* __restrict__ m_out,
                                                     const DevStats* __restrict__ gate) {
  if (gate && gate->route != kRoutePartition) return;  // speculative launch
  using BT = BitonicSort<K, NT, VT>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* sorted = reinterpret_cast<K*>(smem_raw);  // BT::SMEM keys
  const SegDesc seg = segs[blockIdx.x];
  const int B = seg.nbuckets;
  int64_t S64 = (int64_t)B * oversample;
  if (S64 > seg.len) S64 = seg.len;
  if (S64 > BT::NV) S64 = BT::NV;
  const int S = (int)S64;
  const int log2S = (S & (S - 1)) == 0 ? __ffs(S) - 1 : -1;
  {
    K y[VT];
#pragma unroll
    for (int u = 0; u < VT; u++) {
      const int k = u * NT + threadIdx.x;
      y[u] = k < S ? src[sample_position(seg.start, seg.len, S, k, log2S)] : K(0);
    }
#pragma unroll
    for (int u = 0; u < VT; u++) {
      const int k = u * NT + threadIdx.x;
      if (k < S) sorted[k] = y[u];
    }
  }
  __syncthreads();
  BT::sort(sorted, S);
  K* out = spl_out + (int64_t)blockIdx.x * kMaxBuckets;
  uint8_t* eo = eq_out + (int64_t)blockIdx.x * kMaxBuckets;
  for (int j = threadIdx.x; j < B - 1; j += NT) {
    const int r = (int)(((int64_t)(j + 1) * S) / B);
    const K t = sorted[r];
    const bool m1 = r >= 1 && sorted[r - 1] == t, m2 = r >= 2 && sorted[r - 2] == t;
    const bool p1 = r + 1 < S && sorted[r + 1] == t, p2 = r + 2 < S && sorted[r + 2] == t;
    out[j] = t;
    eo[j] = ((m1 && m2) || (m1 && p1) || (p1 && p2)) ? 1 : 0;  // count > gamma = 2
  }
  if (threadIdx.x == 0) m_out[blockIdx.x] = B - 1;
}

// ---------------------------------------------------------------------------
// Vectorised key loads for the count / scatter passes: thread t takes the
// G = U / 4 groups of 4 consecutive positions s0 + 4 (g NT + t) .. + 3, with
// s0 = sub rounded down to a multiple of 4 (16-byte int32 / 32-byte int64
// vectors when the base is aligned; scalar loads at the array end).
// Positions outside [lo, hi) are loaded as 0 and reported invalid.  The
// partition passes are order-agnostic within a sub-tile (keys only), so the
// position <-> thread map only has to be the same for the keys and their
// bucket ids.
template <typename K, int U, int NT>
__device__ __forceinline__ uint32_t load_keys_vec4(const K* __restrict__ src, int64_t s0, int64_t lo, int64_t hi,
                                                   K (&x)[U]) {
  static_assert(U % 4 == 0 && U <= 32, "");
  uint32_t valid = 0;
#pragma unroll
  for (int g = 0; g < U / 4; g++) {
    const int64_t p0 = s0 + 4 * ((int64_t)g * NT + threadIdx.x);
    if (p0 >= lo && p0 + 4 <= hi) {
      if (sizeof(K) == 4) {
        const int4 v = *reinterpret_cast<const int4*>(src + p0);
        memcpy(&x[4 * g], &v, 16);
      } else {
        const int4 v0 = reinterpret_cast<const int4*>(src + p0)[0], v1 = reinterpret_cast<const int4*>(src + p0)[1];
        memcpy(&x[4 * g], &v0, 16);
        memcpy(&x[4 * g + 2], &v1, 16);
      }
      valid |= 0xfu << (4 * g);
    } else {
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const bool ok = p0 + j >= lo && p0 + j < hi;
        x[4 * g + j] = ok ? src[p0 + j] : K(0);
        valid |= (uint32_t)ok << (4 * g + j);
      }
    }
  }
  return valid;
}
// position of slot u of load_keys_vec4
template <int NT>
__device__ __forceinline__ int64_t vec4_pos(int64_t s0, int u) {
  return s0 + 4 * ((int64_t)(u >> 2) * NT + threadIdx.x) + (u & 3);
}

// ---------------------------------------------------------------------------
// K8: bucket histogram of one chunk.  The segment's guide table (guide.cuh,
// built once per level by k_guide_build) is copied into shared memory; each
// key's 3-way bucket id is found by the table-narrowed,
// branch-free bisection over the distinct splitters.
template <typename K>
struct CountSmem {
  GuideTab<K> g;
  uint32_t hist[kMaxBins];
};

template <typename K, int NT>
__global__ void __launch_bounds__(NT) k_count(const K* __restrict__ src, const SegDesc* __restrict__ segs,
                                               const int* __restrict__ chunk_seg, int64_t chunk_size,
                                               const GuideTab<K>* __restrict__ guides, uint32_t* __restrict__ mat,
                                               uint32_t* __restrict__ tot, uint16_t* __restrict__ bins_out,
                                               const DevStats* __restrict__ gate) {
  if (gate && gate->route != kRoutePartition) return;  // speculative launch
  constexpr int U = 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CountSmem<K>& csm = *reinterpret_cast<CountSmem<K>*>(smem_raw);
  uint32_t* s_hist = csm.hist;
  const int c = blockIdx.x;
  const int s = chunk_seg[c];
  const SegDesc seg = segs[s];
  const int g = c - seg.chunk_base;
  guide_load(guides + s, csm.g);
  for (int b = threadIdx.x; b < seg.nbins; b += NT) s_hist[b] = 0;
  __syncthreads();
  const int64_t c0 = seg.start + (int64_t)g * chunk_size;
  const int64_t c1 = (c0 + chunk_size < seg.start + seg.len) ? c0 + chunk_size : seg.start + seg.len;
  const bool vec = (reinterpret_cast<uintptr_t>(src) & 15) == 0 && (reinterpret_cast<uintptr_t>(bins_out) & 7) == 0;
  for (int64_t base = vec ? (c0 & ~int64_t(3)) : c0; base < c1; base += NT * U) {
    K x[U];
    uint32_t valid = 0;
    if (vec) {
      valid = load_keys_vec4<K, U, NT>(src, base, c0, c1, x);
    } else {
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t i = base + u * NT + threadIdx.x;
        x[u] = i < c1 ? src[i] : K(0);
        valid |= (uint32_t)(i < c1) << u;
      }
    }
    int bin[U];
    guide_classify<K, U>(x, bin, csm.g);
#pragma unroll
    for (int u = 0; u < U; u++) hist_add(s_hist, bin[u], (valid >> u) & 1);
    if (bins_out) {  // reused by the scatter
      if (vec) {
#pragma unroll
        for (int g = 0; g < U / 4; g++) {
          const int64_t p0 = vec4_pos<NT>(base, 4 * g);
          if (((valid >> (4 * g)) & 0xf) == 0xf) {
            const uint2 w = make_uint2((uint32_t)bin[4 * g] | ((uint32_t)bin[4 * g + 1] << 16),
                                       (uint32_t)bin[4 * g + 2] | ((uint32_t)bin[4 * g + 3] << 16));
            *reinterpret_cast<uint2*>(bins_out + p0) = w;
          } else {
#pragma unroll
            for (int j = 0; j < 4; j++)
              if ((valid >> (4 * g + j)) & 1) bins_out[p0 + j] = (uint16_t)bin[4 * g + j];
          }
        }
      } else {
#pragma unroll
        for (int u = 0; u < U; u++)
          if ((valid >> u) & 1) bins_out[base + u * NT + threadIdx.x] = (uint16_t)bin[u];
      }
    }
  }
  __syncthreads();
  if (tot) {  // keys only: per-segment bucket totals at bin base seg.mat_base
    for (int b = threadIdx.x; b < seg.nbins; b += NT)
      if (s_hist[b]) atomicAdd(&tot[seg.mat_base + b], s_hist[b]);
  } else {
    for (int b = threadIdx.x; b < seg.nbins; b += NT) mat[seg.mat_base + (int64_t)b * seg.nchunks + g] = s_hist[b];
  }
}

// ---------------------------------------------------------------------------
// K9: single-pass exclusive scan of the count matrix (decoupled look-back).
// status[] and *tile_counter must be zero before launch.
template <int NT, int IPT>
__global__ void __launch_bounds__(NT) k_scan_u32(uint32_t* __restrict__ data, int64_t count,
                                                  unsigned long long* __restrict__ status, int* __restrict__ tile_counter,
                                                  const DevStats* __restrict__ gate) {
  if (gate && gate->route != kRoutePartition) return;  // speculative launch
  __shared__ int s_tile;
  __shared__ uint32_t s_red[NT / 32 + 1];
  __shared__ uint32_t s_stage[NT * IPT + NT * IPT / 32 + 1];
  __shared__ uint32_t s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1);
  __syncthreads();
  const int tile = s_tile;
  const int64_t base = (int64_t)tile * NT * IPT;
  for (int i = threadIdx.x; i < NT * IPT; i += NT) {
    int64_t p = base + i;
    s_stage[pad_idx<uint32_t>(i)] = p < count ? data[p] : 0u;
  }
  __syncthreads();
  uint32_t v[IPT];
  uint32_t sum = 0;
#pragma unroll
  for (int i = 0; i < IPT; i++) { v[i] = s_stage[pad_idx<uint32_t>(threadIdx.x * IPT + i)]; sum += v[i]; }
  uint32_t agg;
  uint32_t ex = block_exclusive_sum<NT>(sum, s_red, &agg);
  if (threadIdx.x < 32) {
    // warp-parallel look-back: lanes inspect 32 predecessors at a time
    volatile unsigned long long* vs = status;
    const int lane = threadIdx.x;
    if (lane == 0) vs[tile] = ((tile == 0 ? 2ull : 1ull) << 32) | agg;
    uint32_t prefix = 0;
    int j = tile - 1;
    while (j >= 0) {
      const int idx = j - lane;
      unsigned long long sv = idx >= 0 ? vs[idx] : (2ull << 32);
      unsigned flag = (unsigned)(sv >> 32);
      if (__any_sync(0xffffffffu, flag == 0)) continue;  // a predecessor has not published yet
      unsigned incl = __ballot_sync(0xffffffffu, flag == 2);
      int stop = incl ? __ffs(incl) - 1 : 31;
      uint32_t val = lane <= stop ? (uint32_t)sv : 0u;
      prefix += warp_reduce_sum(val);
      if (incl) break;
      j -= 32;
    }
    if (lane == 0) {
      if (tile > 0) vs[tile] = (2ull << 32) | (uint32_t)(prefix + agg);
      s_prefix = prefix;
    }
  }
  __syncthreads();
  uint32_t run = s_prefix + ex;
#pragma unroll
  for (int i = 0; i < IPT; i++) { s_stage[pad_idx<uint32_t>(threadIdx.x * IPT + i)] = run; run += v[i]; }
  __syncthreads();
  for (int i = threadIdx.x; i < NT * IPT; i += NT) {
    int64_t p = base + i;
    if (p < count) data[p] = s_stage[pad_idx<uint32_t>(i)];
  }
}

// ---------------------------------------------------------------------------
// K9b: bucket plan (one CTA per segment).  Turns the scanned count matrix into
// finishing items and next-level segments:
//   equality bucket (odd id, count > 0)  -> kItemFill (final)
//   range bucket > kCap                   -> next partition level (recursion,
//                                            Appendix B)
//   range bucket in (kCap/2, kCap]        -> its own kItemSort
//   range buckets <= kCap/2               -> packed with their neighbours into
//      kItemSort chunks < kCap (adjacent buckets are ordered, so sorting the
//      union of consecutive buckets equals sorting each one).
enum : uint8_t { kBinEmpty = 0, kBinFill = 1, kBinOvf = 2, kBinBig = 3, kBinSmall = 4 };

struct PlanSmem {
  int32_t p[kMaxBins + 1];
  int32_t epoch[kMaxBins];
  int32_t prev[kMaxBins];
  int32_t next[kMaxBins + 1];
  uint8_t type[kMaxBins];
};

// Per-thread slot reservation in one of the item lists: block scan + one
// global atomic per block.
template <int NT>
__device__ __forceinline__ int64_t reserve_slots(int mine, unsigned long long* counter, int32_t* s_red, long long* s_base) {
  int32_t tot;
  int32_t ex = block_exclusive_sum<NT>(mine, s_red, &tot);
  if (threadIdx.x == 0) *s_base = tot ? (long long)atomicAdd(counter, (unsigned long long)tot) : 0;
  __syncthreads();
  int64_t r = *s_base + ex;
  __syncthreads();
  return r;
}

template <typename K, int NT>
__global__ void __launch_bounds__(NT) k_plan(const SegDesc* __restrict__ segs, const uint32_t* __restrict__ mat,
                                              const K* __restrict__ spl_all, const int* __restrict__ m_all,
                                              int buf, Item* __restrict__ items, Item* __restrict__ items_big,
                                              OvfSeg* __restrict__ ovf, DevStats* __restrict__ st,
                                              const uint32_t* __restrict__ tot, uint32_t* __restrict__ cursor,
                                              const DevStats* __restrict__ gate, int small_max, int pack_h) {
  if (gate && gate->route != kRoutePartition) return;  // speculative launch
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PlanSmem& sm = *reinterpret_cast<PlanSmem*>(smem_raw);
  __shared__ int32_t s_red[NT / 32 + 1];
  __shared__ long long s_red64[NT / 32 + 1];
  __shared__ long long s_base;
  const SegDesc seg = segs[blockIdx.x];
  const int nb = seg.nbins;
  const int G = seg.nchunks;
  const int64_t send = seg.start + seg.len;
  // packing window: buckets <= H are packed with their neighbours into items < 2H
  // (adjacent buckets are ordered); larger buckets are items of their own
  const int H = pack_h;
  if (tot) {
    // keys only: bucket starts = seg.start + exclusive scan of the totals
    for (int b = threadIdx.x; b < nb; b += NT) sm.p[b] = (int32_t)tot[seg.mat_base + b];
    __syncthreads();
    smem_scan<NT>(sm.p, nb, 0, [](int32_t a, int32_t b) { return a + b; }, true, false, s_red);
    for (int b = threadIdx.x; b < nb; b += NT) {
      sm.p[b] += (int32_t)seg.start;
      cursor[seg.mat_base + b] = (uint32_t)sm.p[b];
    }
  } else {
    for (int b = threadIdx.x; b < nb; b += NT)
      sm.p[b] = (int32_t)(seg.start + ((int64_t)mat[seg.mat_base + (int64_t)b * G] - seg.len_prefix));
  }
  if (threadIdx.x == 0) sm.p[nb] = (int32_t)send;
  __syncthreads();
  long long noneq = 0, eqk = 0, ovk = 0;
  for (int b = threadIdx.x; b < nb; b += NT) {
    int c = sm.p[b + 1] - sm.p[b];
    uint8_t ty;
    if (b & 1) ty = c > 0 ? kBinFill : kBinEmpty;
    else if (c == 0) ty = kBinEmpty;
    else if (c > kCap) ty = kBinOvf;
    else if (c > H) ty = kBinBig;
    else ty = kBinSmall;
    sm.type[b] = ty;
    sm.epoch[b] = (ty == kBinFill || ty == kBinOvf || ty == kBinBig) ? 1 : 0;
    sm.prev[b] = ty == kBinSmall ? b : -1;
    if (b & 1) eqk += c; else noneq += c;
    if (ty == kBinOvf) ovk += c;
  }
  __syncthreads();
  auto add = [](int32_t a, int32_t b) { return a + b; };
  auto mx = [](int32_t a, int32_t b) { return a > b ? a : b; };
  auto mn = [](int32_t a, int32_t b) { return a < b ? a : b; };
  smem_scan<NT>(sm.epoch, nb, 0, add, true, false, s_red);   // separators before b
  smem_scan<NT>(sm.prev, nb, -1, mx, true, false, s_red);    // last small bin before b
  // chunk heads and boundaries
  for (int b = threadIdx.x; b < nb; b += NT) {
    bool head = false;
    if (sm.type[b] == kBinSmall) {
      int pv = sm.prev[b];
      head = pv < 0 || sm.epoch[pv] != sm.epoch[b] ||
             (sm.p[pv] - (int32_t)seg.start) / H != (sm.p[b] - (int32_t)seg.start) / H;
    }
    uint8_t ty = sm.type[b];
    bool bound = head || ty == kBinFill || ty == kBinOvf || ty == kBinBig;
    sm.next[b] = bound ? sm.p[b] : (int32_t)send;
    if (head) sm.type[b] = kBinSmall | 0x80;
  }
  __syncthreads();
  smem_scan<NT>(sm.next, nb, (int32_t)send, mn, false, true, s_red);  // suffix min
  // item lengths per bin (0 = no item); fills split into kFillChunk pieces
  constexpr int IPT = (kMaxBins + NT - 1) / NT;
  int n_small = 0, n_big = 0, n_ovf = 0;
  long long bigk = 0;
  for (int k = 0; k < IPT; k++) {
    int b = threadIdx.x + k * NT;
    if (b >= nb) break;
    uint8_t ty = sm.type[b];
    int c = sm.p[b + 1] - sm.p[b];
    int len = ty == (kBinSmall | 0x80) ? ((b + 1 < nb ? sm.next[b + 1] : (int32_t)send) - sm.p[b])
                                       : (ty == kBinBig ? c : 0);
    if (len) (len <= small_max ? n_small : n_big)++;
    if (len > small_max) bigk += len;
    if (ty == kBinFill) n_small += (c + kFillChunk - 1) / kFillChunk;
    if (ty == kBinOvf) n_ovf++;
  }
  int64_t o_small = reserve_slots<NT>(n_small, (unsigned long long*)&st->n_items, s_red, &s_base);
  int64_t o_big = reserve_slots<NT>(n_big, (unsigned long long*)&st->n_items_big, s_red, &s_base);
  int64_t o_ovf = reserve_slots<NT>(n_ovf, (unsigned long long*)&st->n_ovf, s_red, &s_base);
  const int m = m_all[blockIdx.x];
  const K* spl = spl_all + (int64_t)blockIdx.x * kMaxBuckets;
  for (int k = 0; k < IPT; k++) {
    int b = threadIdx.x + k * NT;
    if (b >= nb) break;
    uint8_t ty = sm.type[b];
    int c = sm.p[b + 1] - sm.p[b];
    int len = ty == (kBinSmall | 0x80) ? ((b + 1 < nb ? sm.next[b + 1] : (int32_t)send) - sm.p[b])
                                       : (ty == kBinBig ? c : 0);
    if (len) {
      Item it;
      it.start = sm.p[b]; it.len = len; it.kind = kItemSort | (buf << 4); it.key = 0;
      if (len <= small_max) items[o_small++] = it; else items_big[o_big++] = it;
    } else if (ty == kBinFill) {
      int i = (b - 1) / 2;
      if (i >= m) atomicAdd((unsigned long long*)&st->error, 1ull);
      for (int f = 0; f < c; f += kFillChunk) {
        Item it;
        it.start = sm.p[b] + f; it.len = min(kFillChunk, c - f); it.kind = kItemFill | (buf << 4);
        it.key = i < m ? (int64_t)spl[i] : 0;
        items[o_small++] = it;
      }
    } else if (ty == kBinOvf) {
      OvfSeg o; o.start = sm.p[b]; o.len = c;
      ovf[o_ovf++] = o;
    }
  }
  noneq = block_reduce_sum<NT>(noneq, s_red64);
  eqk = block_reduce_sum<NT>(eqk, s_red64);
  ovk = block_reduce_sum<NT>(ovk, s_red64);
  bigk = block_reduce_sum<NT>(bigk, s_red64);
  if (threadIdx.x == 0) {
    if (bigk) atomicAdd((unsigned long long*)&st->big_keys, (unsigned long long)bigk);
    atomicAdd((unsigned long long*)&st->noneq_total, (unsigned long long)noneq);
    atomicAdd((unsigned long long*)&st->eq_keys, (unsigned long long)eqk);
    atomicAdd((unsigned long long*)&st->ovf_keys, (unsigned long long)ovk);
  }
}

// ---------------------------------------------------------------------------
// K10: stable 3-way scatter of one chunk (H10).  The chunk is processed in
// sub-tiles of NT*VTS keys in input order; within a sub-tile each key's rank
// among equal-bucket keys comes from per-warp counters (lanes with the same
// bucket found by one ballot per id bit, popc of the lower lanes), so the
// scatter is stable.  Keys are staged in shared memory in bucket order and
// written out contiguously per bucket.  Keys of equality buckets are not
// written (the finishing fill writes them; "spared"); their
// payloads are.
//
// NBMAX < kMaxBins: the COMPACT variant for levels whose splitters take few
// distinct values (few-unique inputs, e.g. configs[3]: 100 values among 2047
// splitters): bucket id b = 2i + e (i = a first-occurrence index of the
// guide table, guide.cuh) is renumbered 2k + e over the md distinct splitters,
// so the per-sub-tile bucket tables shrink from 2 B + 1 to 2 md + 2 entries
// and shared memory from ~190 KB to ~60 KB (three CTAs per SM instead of one).
// Each instance serves the segments of its size class and exits on the others.
constexpr int kBinBits = 13;  // bucket ids 0 .. kMaxBins (invalid) < 2^13
static_assert(kMaxBins < (1 << kBinBits), "");
constexpr int bits_for(int v) { return v <= 1 ? 1 : 1 + bits_for(v >> 1); }  // bits of 0..v

template <typename K, bool HAS_V, int NT, int VTS, int NBMAX>
struct ScatterSmem {
  static constexpr int NW = NT / 32;
  static constexpr int ST = NT * VTS;
  static constexpr bool COMPACT = NBMAX < kMaxBins;
  K stk[ST];
  uint32_t stv[HAS_V ? ST : 1];
  uint32_t cur[NBMAX];
  uint32_t lstart[NBMAX];
  uint32_t tot[NBMAX];
  uint16_t stb[ST];
  uint16_t wcnt[NW][NBMAX + 1];
  uint16_t inv[COMPACT ? kMaxBuckets + 1 : 1];  // splitter index i -> distinct index k
  uint32_t red[NT / 32 + 1];
};

constexpr int kCompactBins = 512;  // compact variant: 2 md + 2 <= 512 bucket ids

template <typename K, bool HAS_V, int NT, int VTS, int NBMAX>
__global__ void __launch_bounds__(NT) k_scatter(const K* __restrict__ src_k, const uint32_t* __restrict__ src_v,
                                                 K* __restrict__ dst_k, uint32_t* __restrict__ dst_v,
                                                 const SegDesc* __restrict__ segs, const int* __restrict__ chunk_seg,
                                                 int64_t chunk_size, const GuideTab<K>* __restrict__ guides,
                                                 const uint32_t* __restrict__ mat, const uint16_t* __restrict__ bins_in,
                                                 const DevStats* __restrict__ gate) {
  using SM = ScatterSmem<K, HAS_V, NT, VTS, NBMAX>;
  constexpr bool COMPACT = SM::COMPACT;
  // speculative launch: only on the partition route, and keys-only with every
  // key in an equality bucket needs no scatter at all
  if (gate && (gate->route != kRoutePartition || (!HAS_V && gate->noneq_total == 0))) return;
  constexpr int NW = SM::NW;
  constexpr int ST = SM::ST;
  constexpr int BITS = COMPACT ? bits_for(NBMAX) : kBinBits;  // ids 0 .. NBMAX (invalid)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int c = blockIdx.x;
  const int s = chunk_seg[c];
  const GuideTab<K>& gd = guides[s];
  const int md = gd.md;
  if (COMPACT != (2 * md + 2 <= kCompactBins)) return;  // the other instance's segment
  const SegDesc seg = segs[s];
  const int g = c - seg.chunk_base;
  const int m = gd.m;
  const int nb = COMPACT ? 2 * md + 2 : seg.nbins;
  if (COMPACT) {
    // occurring splitter indices are first occurrences (and m); any other index
    // would need t_{i-1} < x <= t_i with t_{i-1} = t_i
    for (int k = tid; k < md; k += NT) sm.inv[gd.first[k]] = (uint16_t)k;
    if (tid == 0) sm.inv[m] = (uint16_t)md;
  }
  for (int b = tid; b < nb; b += NT) {
    const int ob = COMPACT ? 2 * ((b >> 1) < md ? (int)gd.first[b >> 1] : m) + (b & 1) : b;
    sm.cur[b] = (uint32_t)(seg.start + ((int64_t)mat[seg.mat_base + (int64_t)ob * seg.nchunks + g] - seg.len_prefix));
  }
  __syncthreads();
  const int64_t c0 = seg.start + (int64_t)g * chunk_size;
  const int64_t c1 = (c0 + chunk_size < seg.start + seg.len) ? c0 + chunk_size : seg.start + seg.len;
  const unsigned lt = lanemask_lt();
  for (int64_t sub = c0; sub < c1; sub += ST) {
    for (int b = lane; b < nb; b += 32) sm.wcnt[w][b] = 0;
    __syncwarp();
    K x[VTS];
    uint32_t v[VTS];
    uint16_t bi[VTS];
#pragma unroll
    for (int i = 0; i < VTS; i++) {
      const int64_t pos = sub + (int64_t)w * 32 * VTS + i * 32 + lane;
      x[i] = pos < c1 ? src_k[pos] : K(0);
      if (HAS_V) v[i] = pos < c1 ? src_v[pos] : 0u;
      bi[i] = pos < c1 ? bins_in[pos] : (uint16_t)0;
    }
    uint16_t rk[VTS];
#pragma unroll
    for (int i = 0; i < VTS; i++) {
      const int64_t pos = sub + (int64_t)w * 32 * VTS + i * 32 + lane;
      const bool valid = pos < c1;
      const int b0 = (int)bi[i];
      const int b = !valid ? NBMAX : (COMPACT ? 2 * (int)sm.inv[b0 >> 1] + (b0 & 1) : b0);
      // lanes with the same bucket: one ballot per bit of the id (cheaper than
      // MATCH.ANY, which dominated this kernel's stalls)
      unsigned peers = 0xffffffffu;
#pragma unroll
      for (int bit = 0; bit < BITS; bit++) {
        const unsigned bal = __ballot_sync(0xffffffffu, (b >> bit) & 1);
        peers &= ((b >> bit) & 1) ? bal : ~bal;
      }
      const int base = sm.wcnt[w][b];
      rk[i] = (uint16_t)(base + __popc(peers & lt));
      __syncwarp();
      if (lane == __ffs(peers) - 1) sm.wcnt[w][b] = (uint16_t)(base + __popc(peers));
      __syncwarp();
      bi[i] = (uint16_t)b;
    }
    __syncthreads();
    for (int b = tid; b < nb; b += NT) {
      uint32_t run = 0;
#pragma unroll
      for (int w2 = 0; w2 < NW; w2++) {
        uint32_t cc = sm.wcnt[w2][b];
        sm.wcnt[w2][b] = (uint16_t)run;
        run += cc;
      }
      sm.tot[b] = run;
      sm.lstart[b] = run;
    }
    __syncthreads();
    smem_scan<NT>(sm.lstart, nb, 0u, [](uint32_t a, uint32_t b) { return a + b; }, true, false, sm.red);
#pragma unroll
    for (int i = 0; i < VTS; i++) {
      const int b = bi[i];
      if (b < NBMAX) {
        const int lp = sm.lstart[b] + sm.wcnt[w][b] + rk[i];
        SR_CHECK(lp < (uint32_t)ST);
        sm.stk[lp] = x[i];
        sm.stb[lp] = (uint16_t)b;
        if (HAS_V) sm.stv[lp] = v[i];
      }
    }
    __syncthreads();
    const int cnt = (int)((c1 - sub) < ST ? (c1 - sub) : ST);
    for (int p = tid; p < cnt; p += NT) {
      const int b = sm.stb[p];
      const int64_t d = (int64_t)sm.cur[b] + (p - (int)sm.lstart[b]);
      if (!(b & 1)) dst_k[d] = sm.stk[p];
      if (HAS_V) dst_v[d] = sm.stv[p];
    }
    __syncthreads();
    for (int b = tid; b < nb; b += NT) sm.cur[b] += sm.tot[b];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K10 (keys only): 3-way scatter with atomic bucket reservation.  Equal keys
// are indistinguishable, so the order inside a range bucket is irrelevant (the
// finishing sort fixes it) and keys of equality buckets are not written at all
// (the fill writes them; "spared from the recursive calls").  Per
// sub-tile: classify, rank inside the CTA with shared-memory atomics, reserve
// each bucket's slice with one global atomic on its cursor, stage in bucket
// order, write contiguous slices.
template <typename K, int NT, int VTS>
struct ScatterKeysSmem {
  static constexpr int ST = NT * VTS;
  K spl[2 * kMaxBuckets];
  K stk[ST];
  uint32_t cnt[kMaxBins];
  uint32_t lstart[kMaxBins];
  uint32_t base[kMaxBins];
  uint32_t run[kMaxBins];  // matrix mode: running destination of each bucket in this chunk
  uint16_t stb[ST];
  uint8_t eq[kMaxBuckets];
  uint32_t red[NT / 32 + 1];
  uint32_t total;
};

template <typename K, int NT, int VTS>
__global__ void __launch_bounds__(NT) k_scatter_keys(const K* __restrict__ src, K* __restrict__ dst,
                                                      const SegDesc* __restrict__ segs,
                                                      const int* __restrict__ chunk_seg, int64_t chunk_size,
                                                      const K* __restrict__ spl_all, const uint8_t* __restrict__ eq_all,
                                                      const int* __restrict__ m_all, uint32_t* __restrict__ cursor,
                                                      const uint16_t* __restrict__ bins_in,
                                                      const uint32_t* __restrict__ mat,
                                                      const DevStats* __restrict__ gate) {
  if (gate && (gate->route != kRoutePartition || gate->noneq_total == 0)) return;
  using SM = ScatterKeysSmem<K, NT, VTS>;
  constexpr int ST = SM::ST;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  const int tid = threadIdx.x;
  const int c = blockIdx.x;
  const int s = chunk_seg[c];
  const SegDesc seg = segs[s];
  const int g = c - seg.chunk_base;
  const int nb = seg.nbins;
  const int m = m_all[s];
  const int depth = tree_depth(m);
  uint32_t* cur = mat ? nullptr : cursor + seg.mat_base;
  if (mat)  // matrix mode (large levels): this chunk's slice of every bucket, no global atomics
    for (int b = tid; b < nb; b += NT)
      sm.run[b] = (uint32_t)(seg.start + ((int64_t)mat[seg.mat_base + (int64_t)b * seg.nchunks + g] - seg.len_prefix));
  if (!bins_in) load_splitters_smem(spl_all + (int64_t)s * kMaxBuckets, eq_all + (int64_t)s * kMaxBuckets, m, sm.spl, sm.eq);
  const int64_t c0 = seg.start + (int64_t)g * chunk_size;
  const int64_t c1 = (c0 + chunk_size < seg.start + seg.len) ? c0 + chunk_size : seg.start + seg.len;
  // (scalar loads: 16-byte vector loads and evict-first hints measured slower here)
  for (int64_t sub = c0; sub < c1; sub += ST) {
    for (int b = tid; b < nb; b += NT) sm.cnt[b] = 0;
    __syncthreads();
    K x[VTS];
    int bin[VTS];
    uint32_t rk[VTS];
    uint32_t valid = 0;
#pragma unroll
    for (int i = 0; i < VTS; i++) {
      const int64_t p = sub + i * NT + tid;
      x[i] = p < c1 ? src[p] : K(0);
      if (bins_in) bin[i] = p < c1 ? (int)bins_in[p] : 0;
      valid |= (uint32_t)(p < c1) << i;
    }
    if (!bins_in) classify_keys<K, VTS>(x, bin, sm.spl, sm.eq, m, depth);
#pragma unroll
    for (int i = 0; i < VTS; i++) {
      // range buckets only; equality buckets are filled later
      if (!((valid >> i) & 1) || (bin[i] & 1)) bin[i] = -1;
      else rk[i] = atomicAdd(&sm.cnt[bin[i]], 1u);
    }
    __syncthreads();
    for (int b = tid; b < nb; b += NT) {
      uint32_t cb = sm.cnt[b];
      sm.lstart[b] = cb;
      if (mat) {
        sm.base[b] = sm.run[b];
        sm.run[b] += cb;
      } else if (cb) {
        sm.base[b] = atomicAdd(&cur[b], cb);
      }
    }
    __syncthreads();
    smem_scan<NT>(sm.lstart, nb, 0u, [](uint32_t a, uint32_t b) { return a + b; }, true, false, sm.red);
    if (tid == 0) sm.total = sm.lstart[nb - 1] + sm.cnt[nb - 1];
#pragma unroll
    for (int i = 0; i < VTS; i++) {
      if (bin[i] >= 0) {
        uint32_t lp = sm.lstart[bin[i]] + rk[i];
        SR_CHECK(lp < (uint32_t)ST);
        sm.stk[lp] = x[i];
        sm.stb[lp] = (uint16_t)bin[i];
      }
    }
    __syncthreads();
    const int tot = (int)sm.total;
    for (int p = tid; p < tot; p += NT) {
      int b = sm.stb[p];
      SR_CHECK((int64_t)sm.base[b] + (p - (int)sm.lstart[b]) >= seg.start &&
               (int64_t)sm.base[b] + (p - (int)sm.lstart[b]) < seg.start + seg.len);
      dst[(int64_t)sm.base[b] + (p - (int)sm.lstart[b])] = sm.stk[p];
    }
    __syncthreads();
  }
}

// K10k2 (keys only, bucket ids from the count pass): the same per-sub-tile
// counting sort as k_scatter_keys with NT = 512 threads, 8K-key sub-tiles and
// tables sized for NBC bins, so that two CTAs share an SM and one's loads
// overlap the other's stores (k_scatter_keys: one 1024-thread CTA per SM whose
// phases are serialised by its barriers).
template <typename K, int NT, int VTS, int NBC>
struct ScatterKeys2Smem {
  static constexpr int ST = NT * VTS;
  K stk[ST];
  uint32_t cnt[NBC];
  uint32_t base[NBC];
  uint32_t run[NBC];
  uint16_t lstart[NBC];
  uint16_t stb[ST];
  uint32_t red[NT / 32 + 1];
  uint32_t total;
};

template <typename K, int NT, int VTS, int NBC>
__global__ void __launch_bounds__(NT, 2) k_scatter_keys2(const K* __restrict__ src, K* __restrict__ dst,
                                                          const SegDesc* __restrict__ segs,
                                                          const int* __restrict__ chunk_seg, int64_t chunk_size,
                                                          uint32_t* __restrict__ cursor,
                                                          const uint16_t* __restrict__ bins_in,
                                                          const uint32_t* __restrict__ mat,
                                                          const DevStats* __restrict__ gate) {
  if (gate && (gate->route != kRoutePartition || gate->noneq_total == 0)) return;
  using SM = ScatterKeys2Smem<K, NT, VTS, NBC>;
  constexpr int ST = SM::ST;
  static_assert(ST <= 65535, "16-bit local offsets");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  const int tid = threadIdx.x;
  const int c = blockIdx.x;
  const int s = chunk_seg[c];
  const SegDesc seg = segs[s];
  const int g = c - seg.chunk_base;
  const int nb = seg.nbins;
  uint32_t* cur = mat ? nullptr : cursor + seg.mat_base;
  if (mat)
    for (int b = tid; b < nb; b += NT)
      sm.run[b] = (uint32_t)(seg.start + ((int64_t)mat[seg.mat_base + (int64_t)b * seg.nchunks + g] - seg.len_prefix));
  const int64_t c0 = seg.start + (int64_t)g * chunk_size;
  const int64_t c1 = (c0 + chunk_size < seg.start + seg.len) ? c0 + chunk_size : seg.start + seg.len;
  for (int64_t sub = c0; sub < c1; sub += ST) {
    for (int b = tid; b < nb; b += NT) sm.cnt[b] = 0;
    __syncthreads();
    K x[VTS];
    int bin[VTS];
    uint32_t rk[VTS];
#pragma unroll
    for (int i = 0; i < VTS; i++) {
      const int64_t p = sub + i * NT + tid;
      x[i] = p < c1 ? src[p] : K(0);
      bin[i] = p < c1 ? (int)bins_in[p] : -1;
    }
#pragma unroll
    for (int i = 0; i < VTS; i++) {
      if (bin[i] & 1) bin[i] = -1;  // (also the positions past c1) equality buckets are filled later
      else rk[i] = atomicAdd(&sm.cnt[bin[i]], 1u);
    }
    __syncthreads();
    {  // local starts (exclusive scan of cnt) and this chunk's slices of the buckets
      constexpr int BPT = (NBC + NT - 1) / NT;
      uint32_t v[BPT], sum = 0;
#pragma unroll
      for (int r = 0; r < BPT; r++) {
        const int b = tid * BPT + r;
        v[r] = b < nb ? sm.cnt[b] : 0u;
        sum += v[r];
      }
      uint32_t tot;
      uint32_t pre = block_exclusive_sum<NT>(sum, sm.red, &tot);
#pragma unroll
      for (int r = 0; r < BPT; r++) {
        const int b = tid * BPT + r;
        if (b < nb) {
          sm.lstart[b] = (uint16_t)pre;
          if (mat) {
            sm.base[b] = sm.run[b];
            sm.run[b] += v[r];
          } else if (v[r]) {
            sm.base[b] = atomicAdd(&cur[b], v[r]);
          }
        }
        pre += v[r];
      }
      if (tid == 0) sm.total = tot;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < VTS; i++) {
      if (bin[i] >= 0) {
        const uint32_t lp = sm.lstart[bin[i]] + rk[i];
        SR_CHECK(lp < (uint32_t)ST);
        sm.stk[lp] = x[i];
        sm.stb[lp] = (uint16_t)bin[i];
      }
    }
    __syncthreads();
    const int tot = (int)sm.total;
    for (int p = tid; p < tot; p += NT) {
      const int b = sm.stb[p];
      SR_CHECK((int64_t)sm.base[b] + (p - (int)sm.lstart[b]) >= seg.start &&
               (int64_t)sm.base[b] + (p - (int)sm.lstart[b]) < seg.start + seg.len);
      dst[(int64_t)sm.base[b] + (p - (int)sm.lstart[b])] = sm.stk[p];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K11w (keys only): every warp finishes whole items of (min_len, 32*VT] keys with
// the warp-register bitonic sort: coalesced load into the warp's staging
// area, is_sorted check, sort, coalesced store into the
// caller's keys.  Fills (equality buckets) are written here too.
template <typename K, int VT, int WARPS>
__global__ void __launch_bounds__(32 * WARPS) k_finish_warp(const Item* __restrict__ items,
                                                             const int64_t* __restrict__ count_ptr, K* __restrict__ keys,
                                                             const K* __restrict__ ws_k,
                                                             const DevStats* __restrict__ gate, int64_t gate_route,
                                                             int min_len, int fills) {
  if (gate && gate->route != gate_route) return;  // speculative launch on another route
  using WB = WarpBitonic<K, VT>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  K* ks = reinterpret_cast<K*>(smem_raw) + w * WB::CAP;
  const int64_t count = *count_ptr;
  for (int64_t it = (int64_t)blockIdx.x * WARPS + w; it < count; it += (int64_t)gridDim.x * WARPS) {
    const Item item = items[it];
    const bool from_ws = (item.kind >> 4) & 1;
    const int64_t s = item.start;
    const int len = item.len;
    K* dk = keys + s;
    if ((item.kind & 0xf) == kItemFill) {
      if (!fills) continue;
      const K key = (K)item.key;
      for (int i = lane; i < len; i += 32) dk[i] = key;
      continue;
    }
    // size class of this launch: (min_len, 32 VT] (narrow networks use fewer
    // registers, so the common small items run at a higher occupancy)
    if (len <= min_len || len > 32 * VT) continue;
    const K* sk = (from_ws ? ws_k : keys) + s;
    // all loads in flight at once (striped, coalesced), then stage in smem
    {
      K x[VT];
#pragma unroll
      for (int r = 0; r < VT; r++) {
        const int i = r * 32 + lane;
        x[r] = i < len ? sk[i] : KeyTraits<K>::max_key();
      }
#pragma unroll
      for (int r = 0; r < VT; r++) ks[r * 32 + lane] = x[r];
    }
    __syncwarp();
    int unsorted = 0;
    for (int i = lane; i + 1 < len; i += 32) unsorted |= ks[i + 1] < ks[i];
    unsorted = __any_sync(0xffffffffu, unsorted);
    if (unsorted) {  // the narrowest register network that holds the item
      if (VT >= 4 && len <= 128) WarpBitonic<K, 4>::sort(ks, len);
      else if (VT >= 8 && len <= 256) WarpBitonic<K, (VT >= 8 ? 8 : VT)>::sort(ks, len);
      else if (VT >= 16 && len <= 512) WarpBitonic<K, (VT >= 16 ? 16 : VT)>::sort(ks, len);
      else if (VT >= 32 && len <= 1024) WarpBitonic<K, (VT >= 32 ? 32 : VT)>::sort(ks, len);
      else WB::sort(ks, len);
    }
    if (unsorted || from_ws) {
      __syncwarp();
      for (int i = lane; i < len; i += 32) dk[i] = ks[i];
    }
    __syncwarp();
  }
}

// K11w2 (keys only): items of (min_len, 64 VH] keys as two halves sorted by the
// VH-key-per-lane network and one warp merge-path merge straight into the
// caller's keys (A = the first half wins ties).  Against one
// 2 VH network: fewer instructions per key and half the registers (the wide
// network's 128 registers held the SM at 16 warps).
template <typename K, int VH, int WARPS>
__global__ void __launch_bounds__(32 * WARPS) k_finish_warp_split(const Item* __restrict__ items,
                                                                   const int64_t* __restrict__ count_ptr,
                                                                   K* __restrict__ keys, const K* __restrict__ ws_k,
                                                                   const DevStats* __restrict__ gate, int64_t gate_route,
                                                                   int min_len) {
  if (gate && gate->route != gate_route) return;  // speculative launch on another route
  constexpr int H = 32 * VH;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  K* ks = reinterpret_cast<K*>(smem_raw) + w * 2 * H;
  const int64_t count = *count_ptr;
  for (int64_t it = (int64_t)blockIdx.x * WARPS + w; it < count; it += (int64_t)gridDim.x * WARPS) {
    const Item item = items[it];
    if ((item.kind & 0xf) == kItemFill) continue;  // (fills: the 16-key launch)
    const int len = item.len;
    if (len <= min_len || len > 2 * H) continue;
    const bool from_ws = (item.kind >> 4) & 1;
    const int64_t s = item.start;
    K* dk = keys + s;
    const K* sk = (from_ws ? ws_k : keys) + s;
#pragma unroll
    for (int h = 0; h < 2; h++) {  // striped, coalesced loads, VH in flight per half
      K x[VH];
#pragma unroll
      for (int r = 0; r < VH; r++) {
        const int i = h * H + r * 32 + lane;
        x[r] = i < len ? sk[i] : KeyTraits<K>::max_key();
      }
#pragma unroll
      for (int r = 0; r < VH; r++) ks[h * H + r * 32 + lane] = x[r];
    }
    __syncwarp();
    int unsorted = 0;
    for (int i = lane; i + 1 < len; i += 32) unsorted |= ks[i + 1] < ks[i];
    if (__any_sync(0xffffffffu, unsorted)) {
      WarpBitonic<K, VH>::sort(ks, H);
      WarpBitonic<K, VH>::sort(ks + H, len - H);
      unit_warp_merge<K>(ks, H, ks + H, len - H, dk);
    } else if (from_ws) {
      for (int i = lane; i < len; i += 32) dk[i] = ks[i];
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// K11: finishing (H11 + H4 segmented).  Persistent CTAs walk the item list:
// fills write the equality value (and move payloads); sorts load the range
// into shared memory, skip the sort when it is already ordered (is_sorted at
// every call) and otherwise run the stable tile sort, then
// write into the caller's buffers.  Items of up to 2*NV keys sort both halves
// in shared memory and merge them straight into global memory.
template <typename K, bool HAS_V, int NT, int VT>
struct FinishSmem {
  static constexpr int NV = NT * VT;
  // keys only: two bitonic halves, the second one's double buffer above the first;
  // pairs: two stable merge-sorted halves plus payloads
  static constexpr int KEYS = HAS_V ? 2 * NV + VT : 3 * NV + VT;
  static constexpr int VALS = HAS_V ? 2 * NV + VT : 1;
  static constexpr size_t bytes() { return sizeof(K) * KEYS + 4 * VALS; }
};

template <typename K, bool HAS_V, int NT, int VT>
__device__ __forceinline__ void finish_sort_smem(K* ks, uint32_t* vs, int len) {
  if (HAS_V) BlockSort<K, HAS_V, NT, VT>::sort(ks, vs, len);
  else BitonicSort<K, NT, VT>::sort(ks, len);
}

template <typename K, bool HAS_V, int NT, int VT, bool TWO_HALVES>
__global__ void __launch_bounds__(NT) k_finish(const Item* __restrict__ items, const int64_t* __restrict__ count_ptr,
                                                int64_t item_begin, K* __restrict__ keys, uint32_t* __restrict__ vals,
                                                const K* __restrict__ ws_k, const uint32_t* __restrict__ ws_v,
                                                const DevStats* __restrict__ gate, int64_t gate_route) {
  if (gate && gate->route != gate_route) return;  // speculative launch on another route
  using FS = FinishSmem<K, HAS_V, NT, VT>;
  constexpr int NV = NT * VT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* ks = reinterpret_cast<K*>(smem_raw);
  uint32_t* vs = reinterpret_cast<uint32_t*>(smem_raw + sizeof(K) * FS::KEYS);
  const int64_t count = *count_ptr - item_begin;
  for (int64_t it = blockIdx.x; it < count; it += gridDim.x) {
    const Item item = items[item_begin + it];
    const int kind = item.kind & 0xf;
    const bool from_ws = (item.kind >> 4) & 1;
    const int64_t s = item.start;
    const int len = item.len;
    if (kind == kItemFill) {
      const K key = (K)item.key;
      constexpr int UF = 8;  // payload loads in flight per thread
      for (int i0 = 0; i0 < len; i0 += NT * UF) {
        uint32_t pv[UF];
        if (HAS_V && from_ws) {
#pragma unroll
          for (int u = 0; u < UF; u++) {
            const int i = i0 + u * NT + threadIdx.x;
            pv[u] = i < len ? ws_v[s + i] : 0u;
          }
        }
#pragma unroll
        for (int u = 0; u < UF; u++) {
          const int i = i0 + u * NT + threadIdx.x;
          if (i < len) {
            keys[s + i] = key;
            if (HAS_V && from_ws) vals[s + i] = pv[u];
          }
        }
      }
      continue;
    }
    const K* sk = (from_ws ? ws_k : keys) + s;
    const uint32_t* sv = (from_ws ? ws_v : vals) + s;
    K* dk = keys + s;
    uint32_t* dv = vals + s;
    const int first = (!TWO_HALVES || len <= NV) ? len : NV;
    {  // VT loads per thread in flight at once (striped, coalesced)
      K x[VT];
      uint32_t y[VT];
#pragma unroll
      for (int r = 0; r < VT; r++) {
        const int i = r * NT + threadIdx.x;
        x[r] = i < first ? sk[i] : K(0);
        if (HAS_V) y[r] = i < first ? sv[i] : 0u;
      }
#pragma unroll
      for (int r = 0; r < VT; r++) {
        const int i = r * NT + threadIdx.x;
        if (i < first) {
          ks[i] = x[r];
          if (HAS_V) vs[i] = y[r];
        }
      }
    }
    // is_sorted
    int unsorted = 0;
    __syncthreads();
    for (int i = threadIdx.x; i + 1 < first; i += NT) unsorted |= ks[i + 1] < ks[i];
    for (int i = first - 1 + threadIdx.x; i + 1 < len; i += NT) unsorted |= sk[i + 1] < sk[i];
    unsorted = __syncthreads_or(unsorted);
    if (!unsorted) {
      if (from_ws)
        for (int i = threadIdx.x; i < len; i += NT) {
          dk[i] = sk[i];
          if (HAS_V) dv[i] = sv[i];
        }
      __syncthreads();
      continue;
    }
    if (!TWO_HALVES || len <= NV) {  // small-item kernels never see len > NV
      finish_sort_smem<K, HAS_V, NT, VT>(ks, vs, len);
      for (int i = threadIdx.x; i < len; i += NT) {
        dk[i] = ks[i];
        if (HAS_V) dv[i] = vs[i];
      }
    } else {
      // two halves sorted in shared memory, then one merge level written
      // straight to global memory
      finish_sort_smem<K, HAS_V, NT, VT>(ks, vs, NV);
      const int nb = len - NV;
      for (int i = threadIdx.x; i < nb; i += NT) {
        ks[NV + i] = sk[NV + i];
        if (HAS_V) vs[NV + i] = sv[NV + i];
      }
      __syncthreads();
      finish_sort_smem<K, HAS_V, NT, VT>(ks + NV, vs + NV, nb);
      for (int d0 = threadIdx.x * VT; d0 < len; d0 += NT * VT) {
        int mp = merge_path_search<K>([&](int i) { return ks[i]; }, NV, [&](int i) { return ks[NV + i]; }, nb, d0);
        int ai = mp, bi = d0 - mp;
#pragma unroll
        for (int i = 0; i < VT; i++) {
          if (d0 + i < len) {
            const bool p = (bi >= nb) || (ai < NV && !(ks[NV + bi] < ks[ai]));
            dk[d0 + i] = p ? ks[ai] : ks[NV + bi];
            if (HAS_V) dv[d0 + i] = p ? vs[ai] : vs[NV + bi];
            ai += p;
            bi += !p;
          }
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace sr
