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
#include "block_sort.cuh"
#include "common.cuh"
#include "presort.cuh"
#include "types.cuh"

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

// ---------------------------------------------------------------------------
// K7: splitters for every segment of a level (one CTA per segment).
template <typename K, int NT, int VT>
__global__ void __launch_bounds__(NT) k_splitters(const K* __restrict__ src, const SegDesc* __restrict__ segs,
                                                   int oversample, K* __restrict__ spl_out,
                                                   uint8_t* __restrict__ eq_out, int* __restrict__ m_out) {
  using BS = BlockSort<K, false, NT, VT>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* ks = reinterpret_cast<K*>(smem_raw);
  __shared__ int32_t s_red[NT / 32 + 1];
  __shared__ int s_m;
  const SegDesc seg = segs[blockIdx.x];
  const int B = seg.nbuckets;
  int64_t S64 = (int64_t)B * oversample;
  if (S64 > seg.len) S64 = seg.len;
  if (S64 > BS::NV) S64 = BS::NV;
  const int S = (int)S64;
  for (int k = threadIdx.x; k < S; k += NT) ks[pad_idx<K>(k)] = src[sample_position(seg.start, seg.len, S, k)];
  __syncthreads();
  BS::sort(ks, nullptr, S);
  // candidates c_j = sample[((j+1)*S)/B], j = 0..B-2; keep the first of equal runs
  const int ncand = B - 1;
  const int j0 = threadIdx.x * 2;
  K c[2];
  int f[2];
#pragma unroll
  for (int u = 0; u < 2; u++) {
    int j = j0 + u;
    f[u] = 0;
    if (j < ncand) {
      c[u] = ks[pad_idx<K>((int)(((int64_t)(j + 1) * S) / B))];
      f[u] = (j == 0) ? 1 : (ks[pad_idx<K>((int)(((int64_t)j * S) / B))] != c[u]);
    }
  }
  int32_t tot;
  int32_t ex = block_exclusive_sum<NT>(f[0] + f[1], s_red, &tot);
  K* out = spl_out + (int64_t)blockIdx.x * kMaxBuckets;
  uint8_t* eo = eq_out + (int64_t)blockIdx.x * kMaxBuckets;
#pragma unroll
  for (int u = 0; u < 2; u++) {
    if (f[u]) {
      // occurrences of c in the sorted sample: upper_bound - lower_bound
      int lo = 0, hi = S;
      while (lo < hi) { int mid = (lo + hi) >> 1; if (ks[pad_idx<K>(mid)] < c[u]) lo = mid + 1; else hi = mid; }
      int lb = lo;
      hi = S;
      while (lo < hi) { int mid = (lo + hi) >> 1; if (c[u] < ks[pad_idx<K>(mid)]) hi = mid; else lo = mid + 1; }
      out[ex] = c[u];
      eo[ex] = (lo - lb) > 2 ? 1 : 0;  // gamma = 2
      ex++;
    }
  }
  if (threadIdx.x == 0) s_m = tot;
  __syncthreads();
  if (threadIdx.x == 0) m_out[blockIdx.x] = s_m;
}

// ---------------------------------------------------------------------------
// K8: bucket histogram of one chunk (levels >= 2; level 1 fuses it into K1).
template <typename K, int NT>
__global__ void __launch_bounds__(NT) k_count(const K* __restrict__ src, const SegDesc* __restrict__ segs,
                                               const int* __restrict__ chunk_seg, int64_t chunk_size,
                                               const K* __restrict__ spl_all, const uint8_t* __restrict__ eq_all,
                                               const int* __restrict__ m_all, uint32_t* __restrict__ mat) {
  constexpr int U = 4;
  __shared__ K s_spl[kMaxBuckets];
  __shared__ uint8_t s_eq[kMaxBuckets];
  __shared__ uint32_t s_hist[kMaxBins];
  const int c = blockIdx.x;
  const int s = chunk_seg[c];
  const SegDesc seg = segs[s];
  const int g = c - seg.chunk_base;
  const int m = m_all[s];
  int P2;
  load_splitters_smem(spl_all + (int64_t)s * kMaxBuckets, eq_all + (int64_t)s * kMaxBuckets, m, s_spl, s_eq, P2);
  for (int b = threadIdx.x; b < seg.nbins; b += NT) s_hist[b] = 0;
  __syncthreads();
  const int64_t c0 = seg.start + (int64_t)g * chunk_size;
  const int64_t c1 = (c0 + chunk_size < seg.start + seg.len) ? c0 + chunk_size : seg.start + seg.len;
  for (int64_t base = c0; base < c1; base += NT * U) {
    K x[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      int64_t i = base + u * NT + threadIdx.x;
      x[u] = i < c1 ? src[i] : K(0);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      int64_t i = base + u * NT + threadIdx.x;
      bool valid = i < c1;
      int bin = valid ? classify_key<K>(x[u], s_spl, s_eq, m, P2) : 0;
      hist_add(s_hist, bin, valid);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < seg.nbins; b += NT) mat[seg.mat_base + (int64_t)b * seg.nchunks + g] = s_hist[b];
}

// ---------------------------------------------------------------------------
// K9: single-pass exclusive scan of the count matrix (decoupled look-back).
// status[] and *tile_counter must be zero before launch.
template <int NT, int IPT>
__global__ void __launch_bounds__(NT) k_scan_u32(uint32_t* __restrict__ data, int64_t count,
                                                  unsigned long long* __restrict__ status, int* __restrict__ tile_counter) {
  __shared__ int s_tile;
  __shared__ uint32_t s_red[NT / 32 + 1];
  __shared__ uint32_t s_stage[NT * IPT];
  __shared__ uint32_t s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1);
  __syncthreads();
  const int tile = s_tile;
  const int64_t base = (int64_t)tile * NT * IPT;
  for (int i = threadIdx.x; i < NT * IPT; i += NT) {
    int64_t p = base + i;
    s_stage[i] = p < count ? data[p] : 0u;
  }
  __syncthreads();
  uint32_t v[IPT];
  uint32_t sum = 0;
#pragma unroll
  for (int i = 0; i < IPT; i++) { v[i] = s_stage[threadIdx.x * IPT + i]; sum += v[i]; }
  uint32_t agg;
  uint32_t ex = block_exclusive_sum<NT>(sum, s_red, &agg);
  if (threadIdx.x == 0) {
    volatile unsigned long long* vs = status;
    uint32_t prefix = 0;
    if (tile == 0) {
      vs[0] = (2ull << 32) | agg;
    } else {
      vs[tile] = (1ull << 32) | agg;
      int j = tile - 1;
      while (true) {
        unsigned long long sv = vs[j];
        unsigned flag = (unsigned)(sv >> 32);
        if (flag == 0) continue;
        prefix += (uint32_t)sv;
        if (flag == 2) break;
        j--;
      }
      __threadfence();
      vs[tile] = (2ull << 32) | (uint32_t)(prefix + agg);
    }
    s_prefix = prefix;
  }
  __syncthreads();
  uint32_t run = s_prefix + ex;
#pragma unroll
  for (int i = 0; i < IPT; i++) { s_stage[threadIdx.x * IPT + i] = run; run += v[i]; }
  __syncthreads();
  for (int i = threadIdx.x; i < NT * IPT; i += NT) {
    int64_t p = base + i;
    if (p < count) data[p] = s_stage[i];
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

template <typename K, int NT>
__global__ void __launch_bounds__(NT) k_plan(const SegDesc* __restrict__ segs, const uint32_t* __restrict__ mat,
                                              const K* __restrict__ spl_all, const int* __restrict__ m_all,
                                              int buf, Item* __restrict__ items, OvfSeg* __restrict__ ovf,
                                              DevStats* __restrict__ st) {
  __shared__ int32_t s_p[kMaxBins + 1];
  __shared__ uint8_t s_type[kMaxBins];
  __shared__ int32_t s_epoch[kMaxBins];
  __shared__ int32_t s_prev[kMaxBins];
  __shared__ int32_t s_next[kMaxBins + 1];
  __shared__ int32_t s_red[NT / 32 + 1];
  __shared__ long long s_red64[NT / 32 + 1];
  const SegDesc seg = segs[blockIdx.x];
  const int nb = seg.nbins;
  const int G = seg.nchunks;
  const int64_t send = seg.start + seg.len;
  constexpr int H = kCap / 2;
  for (int b = threadIdx.x; b < nb; b += NT)
    s_p[b] = (int32_t)(seg.start + ((int64_t)mat[seg.mat_base + (int64_t)b * G] - seg.len_prefix));
  if (threadIdx.x == 0) s_p[nb] = (int32_t)send;
  __syncthreads();
  long long noneq = 0, eqk = 0, ovk = 0;
  for (int b = threadIdx.x; b < nb; b += NT) {
    int c = s_p[b + 1] - s_p[b];
    uint8_t ty;
    if (b & 1) ty = c > 0 ? kBinFill : kBinEmpty;
    else if (c == 0) ty = kBinEmpty;
    else if (c > kCap) ty = kBinOvf;
    else if (c > H) ty = kBinBig;
    else ty = kBinSmall;
    s_type[b] = ty;
    s_epoch[b] = (ty == kBinFill || ty == kBinOvf || ty == kBinBig) ? 1 : 0;
    s_prev[b] = ty == kBinSmall ? b : -1;
    if (b & 1) eqk += c; else noneq += c;
    if (ty == kBinOvf) ovk += c;
  }
  __syncthreads();
  auto add = [](int32_t a, int32_t b) { return a + b; };
  auto mx = [](int32_t a, int32_t b) { return a > b ? a : b; };
  auto mn = [](int32_t a, int32_t b) { return a < b ? a : b; };
  smem_scan<NT>(s_epoch, nb, 0, add, true, false, s_red);   // separators before b
  smem_scan<NT>(s_prev, nb, -1, mx, true, false, s_red);    // last small bin before b
  // chunk heads and boundaries
  for (int b = threadIdx.x; b < nb; b += NT) {
    bool head = false;
    if (s_type[b] == kBinSmall) {
      int pv = s_prev[b];
      head = pv < 0 || s_epoch[pv] != s_epoch[b] ||
             (s_p[pv] - (int32_t)seg.start) / H != (s_p[b] - (int32_t)seg.start) / H;
    }
    uint8_t ty = s_type[b];
    bool bound = head || ty == kBinFill || ty == kBinOvf || ty == kBinBig;
    s_next[b] = bound ? s_p[b] : (int32_t)send;
    if (head) s_type[b] = kBinSmall | 0x80;
  }
  __syncthreads();
  smem_scan<NT>(s_next, nb, (int32_t)send, mn, false, true, s_red);  // suffix min
  const int m = m_all[blockIdx.x];
  const K* spl = spl_all + (int64_t)blockIdx.x * kMaxBuckets;
  for (int b = threadIdx.x; b < nb; b += NT) {
    uint8_t ty = s_type[b];
    int c = s_p[b + 1] - s_p[b];
    if (ty == (kBinSmall | 0x80)) {
      int end = b + 1 < nb ? s_next[b + 1] : (int32_t)send;
      unsigned long long slot = atomicAdd((unsigned long long*)&st->n_items, 1ull);
      Item it; it.start = s_p[b]; it.len = end - s_p[b]; it.kind = kItemSort | (buf << 4); it.key = 0;
      items[slot] = it;
    } else if (ty == kBinBig) {
      unsigned long long slot = atomicAdd((unsigned long long*)&st->n_items, 1ull);
      Item it; it.start = s_p[b]; it.len = c; it.kind = kItemSort | (buf << 4); it.key = 0;
      items[slot] = it;
    } else if (ty == kBinFill) {
      unsigned long long slot = atomicAdd((unsigned long long*)&st->n_items, 1ull);
      int i = (b - 1) / 2;
      Item it; it.start = s_p[b]; it.len = c; it.kind = kItemFill | (buf << 4);
      it.key = i < m ? (int64_t)spl[i] : 0;
      if (i >= m) atomicAdd((unsigned long long*)&st->error, 1ull);
      items[slot] = it;
    } else if (ty == kBinOvf) {
      unsigned long long slot = atomicAdd((unsigned long long*)&st->n_ovf, 1ull);
      OvfSeg o; o.start = s_p[b]; o.len = c;
      ovf[slot] = o;
    }
  }
  noneq = block_reduce_sum<NT>(noneq, s_red64);
  eqk = block_reduce_sum<NT>(eqk, s_red64);
  ovk = block_reduce_sum<NT>(ovk, s_red64);
  if (threadIdx.x == 0) {
    atomicAdd((unsigned long long*)&st->noneq_total, (unsigned long long)noneq);
    atomicAdd((unsigned long long*)&st->eq_keys, (unsigned long long)eqk);
    atomicAdd((unsigned long long*)&st->ovf_keys, (unsigned long long)ovk);
  }
}

// ---------------------------------------------------------------------------
// K10: stable 3-way scatter of one chunk (H10).  The chunk is processed in
// sub-tiles of NT*VTS keys in input order; within a sub-tile each key's rank
// among equal-bucket keys comes from per-warp counters (match-any + popc),
// so the scatter is stable.  Keys are staged in shared memory in bucket order
// and written out contiguously per bucket.  Keys of equality buckets are not
// written (the finishing fill writes them; "spared"); their
// payloads are.
template <typename K, bool HAS_V, int NT, int VTS>
struct ScatterSmem {
  static constexpr int NW = NT / 32;
  static constexpr int ST = NT * VTS;
  K spl[kMaxBuckets];
  K stk[ST];
  uint32_t stv[HAS_V ? ST : 1];
  uint32_t cur[kMaxBins];
  uint32_t lstart[kMaxBins];
  uint32_t tot[kMaxBins];
  uint16_t stb[ST];
  uint16_t wcnt[NW][kMaxBins + 1];
  uint8_t eq[kMaxBuckets];
  uint32_t red[NT / 32 + 1];
};

template <typename K, bool HAS_V, int NT, int VTS>
__global__ void __launch_bounds__(NT) k_scatter(const K* __restrict__ src_k, const uint32_t* __restrict__ src_v,
                                                 K* __restrict__ dst_k, uint32_t* __restrict__ dst_v,
                                                 const SegDesc* __restrict__ segs, const int* __restrict__ chunk_seg,
                                                 int64_t chunk_size, const K* __restrict__ spl_all,
                                                 const uint8_t* __restrict__ eq_all, const int* __restrict__ m_all,
                                                 const uint32_t* __restrict__ mat) {
  using SM = ScatterSmem<K, HAS_V, NT, VTS>;
  constexpr int NW = SM::NW;
  constexpr int ST = SM::ST;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int c = blockIdx.x;
  const int s = chunk_seg[c];
  const SegDesc seg = segs[s];
  const int g = c - seg.chunk_base;
  const int nb = seg.nbins;
  const int m = m_all[s];
  int P2;
  load_splitters_smem(spl_all + (int64_t)s * kMaxBuckets, eq_all + (int64_t)s * kMaxBuckets, m, sm.spl, sm.eq, P2);
  for (int b = tid; b < nb; b += NT)
    sm.cur[b] = (uint32_t)(seg.start + ((int64_t)mat[seg.mat_base + (int64_t)b * seg.nchunks + g] - seg.len_prefix));
  __syncthreads();
  const int64_t c0 = seg.start + (int64_t)g * chunk_size;
  const int64_t c1 = (c0 + chunk_size < seg.start + seg.len) ? c0 + chunk_size : seg.start + seg.len;
  const unsigned lt = lanemask_lt();
  for (int64_t sub = c0; sub < c1; sub += ST) {
    for (int b = lane; b < nb; b += 32) sm.wcnt[w][b] = 0;
    __syncwarp();
    K x[VTS];
    uint32_t v[VTS];
    int bin[VTS];
    int rk[VTS];
#pragma unroll
    for (int i = 0; i < VTS; i++) {
      int64_t pos = sub + (int64_t)w * 32 * VTS + i * 32 + lane;
      x[i] = pos < c1 ? src_k[pos] : K(0);
      if (HAS_V) v[i] = pos < c1 ? src_v[pos] : 0u;
    }
#pragma unroll
    for (int i = 0; i < VTS; i++) {
      int64_t pos = sub + (int64_t)w * 32 * VTS + i * 32 + lane;
      bool valid = pos < c1;
      int b = valid ? classify_key<K>(x[i], sm.spl, sm.eq, m, P2) : kMaxBins;
      unsigned peers = __match_any_sync(0xffffffffu, b);
      int base = sm.wcnt[w][b];
      rk[i] = base + __popc(peers & lt);
      bin[i] = b;
      __syncwarp();
      if (lane == __ffs(peers) - 1) sm.wcnt[w][b] = (uint16_t)(base + __popc(peers));
      __syncwarp();
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
      int b = bin[i];
      if (b < kMaxBins) {
        int lp = sm.lstart[b] + sm.wcnt[w][b] + rk[i];
        sm.stk[lp] = x[i];
        sm.stb[lp] = (uint16_t)b;
        if (HAS_V) sm.stv[lp] = v[i];
      }
    }
    __syncthreads();
    const int cnt = (int)((c1 - sub) < ST ? (c1 - sub) : ST);
    for (int p = tid; p < cnt; p += NT) {
      int b = sm.stb[p];
      int64_t d = (int64_t)sm.cur[b] + (p - (int)sm.lstart[b]);
      if (!(b & 1)) dst_k[d] = sm.stk[p];
      if (HAS_V) dst_v[d] = sm.stv[p];
    }
    __syncthreads();
    for (int b = tid; b < nb; b += NT) sm.cur[b] += sm.tot[b];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K11: finishing (H11 + H4 segmented).  Persistent CTAs walk the item list:
// fills write the equality value (and move payloads); sorts load the range
// into shared memory, skip the sort when it is already ordered (is_sorted at
// every call) and otherwise run the stable tile sort, then
// write into the caller's buffers.
template <typename K, bool HAS_V, int NT, int VT>
__global__ void __launch_bounds__(NT) k_finish(const Item* __restrict__ items, const int64_t* __restrict__ count_ptr,
                                                int64_t item_begin, K* __restrict__ keys, uint32_t* __restrict__ vals,
                                                const K* __restrict__ ws_k, const uint32_t* __restrict__ ws_v) {
  using BS = BlockSort<K, HAS_V, NT, VT>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* ks = reinterpret_cast<K*>(smem_raw);
  uint32_t* vs = reinterpret_cast<uint32_t*>(smem_raw + sizeof(K) * BS::KEYS_SMEM);
  const int64_t count = *count_ptr - item_begin;
  for (int64_t it = blockIdx.x; it < count; it += gridDim.x) {
    const Item item = items[item_begin + it];
    const int kind = item.kind & 0xf;
    const bool from_ws = (item.kind >> 4) & 1;
    const int64_t s = item.start;
    const int len = item.len;
    if (kind == kItemFill) {
      const K key = (K)item.key;
      for (int i = threadIdx.x; i < len; i += NT) {
        keys[s + i] = key;
        if (HAS_V && from_ws) vals[s + i] = ws_v[s + i];
      }
      continue;
    }
    const K* sk = from_ws ? ws_k : keys;
    const uint32_t* sv = from_ws ? ws_v : vals;
    for (int i = threadIdx.x; i < len; i += NT) {
      ks[pad_idx<K>(i)] = sk[s + i];
      if (HAS_V) vs[pad_idx<uint32_t>(i)] = sv[s + i];
    }
    __syncthreads();
    int unsorted = 0;
    for (int i = threadIdx.x; i + 1 < len; i += NT) unsorted |= ks[pad_idx<K>(i + 1)] < ks[pad_idx<K>(i)];
    unsorted = __syncthreads_or(unsorted);
    if (unsorted) BS::sort(ks, vs, len);
    if (unsorted || from_ws) {
      for (int i = threadIdx.x; i < len; i += NT) {
        keys[s + i] = ks[pad_idx<K>(i)];
        if (HAS_V) vals[s + i] = vs[pad_idx<uint32_t>(i)];
      }
    }
    __syncthreads();
  }
}

}  // namespace sr
