// presort.cuh -- H1 presortedness scan (K1), run resolve (K2), H2 run reversal (K3).
//
// H1 follows §4(f) "If n >= alpha, test if the array is already sorted; if
// yes, exit" (Appendix B is_sorted PAPER.md:385) and §3(a)
// scanning for runs (Appendix A).  One read of
// the keys yields D = |{i : a_i > a_{i+1}}| = Run(A) - 1, the
// descending-run breaks, and the long (>= L_min) natural runs of either
// direction.  With L_min >= tile size a long run always touches a tile edge,
// so per-tile first/last break positions are enough to recover every long run.
#pragma once
#include "common.cuh"
#include "types.cuh"

namespace sr {

// Splitter search structure in shared memory (H8).  tree[1..kMaxBuckets-1]
// holds the splitters padded with +inf to 2^L - 1 = kMaxBuckets - 1 entries in
// level (Eytzinger) order; tree[kMaxBuckets + i] holds the i-th splitter in
// sorted order for the equality test, eqf[i] its equality flag.  A binary
// search over a plain sorted array sends every lane of a warp to the same
// bank at the deep levels (addresses = step-1 mod 2*step); in level order each
// level is contiguous, so the lanes spread over the banks.
constexpr int kTreeLevels = 11;  // log2(kMaxBuckets)
static_assert((1 << kTreeLevels) == kMaxBuckets, "");

// Bucket id of x: i = #{t_j < x} (lower_bound); 2i+1 when x equals an
// equality splitter (3-way split, switched on per splitter
// by the gamma test of PAPER.md:168), else 2i.
template <typename K>
__device__ __forceinline__ int classify_key(K x, const K* tree, const uint8_t* eqf, int m, int depth) {
  int j = 1;
  for (int l = 0; l < depth; l++) j = 2 * j + (tree[j] < x ? 1 : 0);
  const int i = j - (1 << depth);
  return 2 * i + ((i < m && tree[kMaxBuckets + i] == x && eqf[i]) ? 1 : 0);
}

// Batched classification: the U searches advance in lockstep so their
// shared-memory loads are independent and overlap (U-way ILP).  depth =
// log2(padded bucket count) of this segment (<= kTreeLevels).
template <typename K, int U>
__device__ __forceinline__ void classify_keys(const K (&x)[U], int (&bin)[U], const K* tree, const uint8_t* eqf, int m,
                                              int depth) {
  int j[U];
#pragma unroll
  for (int u = 0; u < U; u++) j[u] = 1;
#pragma unroll 1
  for (int l = 0; l < depth; l++) {
#pragma unroll
    for (int u = 0; u < U; u++) j[u] = 2 * j[u] + (tree[j[u]] < x[u] ? 1 : 0);
  }
#pragma unroll
  for (int u = 0; u < U; u++) {
    const int i = j[u] - (1 << depth);
    bin[u] = 2 * i + ((i < m && tree[kMaxBuckets + i] == x[u] && eqf[i]) ? 1 : 0);
  }
}

// Build the search structure from the m sorted splitters: tree[1..2^depth)
// in level order (splitters padded with +inf to 2^depth - 1), the sorted
// splitters at tree[kMaxBuckets..), flags eqf[0..m).  depth = tree_depth(m).
__host__ __device__ __forceinline__ int tree_depth(int m) {  // smallest d >= 1 with 2^d - 1 >= m
#ifdef __CUDA_ARCH__
  return m <= 1 ? 1 : 32 - __clz(m);
#else
  int d = 1;
  while ((1 << d) - 1 < m) d++;
  return d;
#endif
}
template <typename K>
__device__ __forceinline__ void load_splitters_smem(const K* spl, const uint8_t* eqf, int m, K* s_tree,
                                                    uint8_t* s_eq) {
  const int depth = tree_depth(m);
  const int nodes = 1 << depth;
  for (int i = threadIdx.x; i < kMaxBuckets; i += blockDim.x) {
    if (i < nodes) {
      const K v = i < m ? spl[i] : KeyTraits<K>::max_key();
      s_tree[kMaxBuckets + i] = v;
      s_eq[i] = i < m ? eqf[i] : 0;
      if (i >= 1) {  // node i of the level-order tree <- sorted position pos(i)
        const int d = 31 - __clz(i);
        const int pos = ((2 * (i - (1 << d)) + 1) << (depth - 1 - d)) - 1;
        s_tree[i] = pos < m ? spl[pos] : KeyTraits<K>::max_key();
      }
    }
  }
}

// Guide table for the classification: the sorted splitters' order-preserving
// unsigned images u(t) are covered by kGuideCells equal cells of width
// 2^shift starting at u(t_0); tab[c] = #{t_j : u(t_j) < u(t_0) + c 2^shift}.
// A key's bucket #{t_j < x} then lies in [tab[c], tab[c+1]] for its cell c and
// is found by bisecting that (usually tiny) range of the sorted splitters --
// the same lower_bound as the tree walk, with a few shared-memory loads
// instead of depth ones.
constexpr int kGuideCells = 4096;
struct Guide {
  uint64_t u0, u1;  // u(t_0), u(t_{m-1})
  int shift, m;
  uint16_t tab[kGuideCells + 1];
};

template <typename K>
__device__ __forceinline__ uint64_t key_u(K x) {  // order-preserving unsigned image
  return sizeof(K) == 4 ? (uint64_t)((uint32_t)x ^ 0x80000000u) : ((uint64_t)x ^ 0x8000000000000000ull);
}

// All threads: the guide of the m sorted splitters spl[0, m) (shared memory).
template <typename K>
__device__ __forceinline__ void build_guide(const K* spl, int m, Guide& g) {
  if (m <= 0) {
    if (threadIdx.x == 0) { g.m = 0; g.shift = 0; g.u0 = 0; g.u1 = 0; }
    return;
  }
  const uint64_t u0 = key_u<K>(spl[0]), u1 = key_u<K>(spl[m - 1]);
  const uint64_t span = u1 - u0;
  int shift = 0;
  while (shift < 64 && (span >> shift) >= (uint64_t)kGuideCells) shift++;
  for (int c = threadIdx.x; c <= kGuideCells; c += blockDim.x) {
    int r;
    if (c == 0) r = 0;
    else if (c == kGuideCells || (uint64_t)c > (span >> shift)) r = m;  // the cell start lies beyond u1
    else {
      const uint64_t v = u0 + ((uint64_t)c << shift);
      int lo = 0, hi = m;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (key_u<K>(spl[mid]) < v) lo = mid + 1; else hi = mid;
      }
      r = lo;
    }
    g.tab[c] = (uint16_t)r;
  }
  if (threadIdx.x == 0) { g.u0 = u0; g.u1 = u1; g.shift = shift; g.m = m; }
}

// Bucket ids of U keys through the guide (sorted splitters at spl): lockstep
// bisection over the per-key ranges, then the 3-way id 2 i + [x equals an
// equality splitter].  Same result as classify_keys.
template <typename K, int U>
__device__ __forceinline__ void classify_keys_guided(const K (&x)[U], int (&bin)[U], const K* spl, const uint8_t* eqf,
                                                     const Guide& g) {
  const int m = g.m;
  const uint64_t u0 = g.u0, u1 = g.u1;
  const int shift = g.shift;
  int lo[U], hi[U];
  int span = 0;
#pragma unroll
  for (int u = 0; u < U; u++) {
    const uint64_t v = key_u<K>(x[u]);
    if (v <= u0) { lo[u] = 0; hi[u] = 0; }          // x <= t_0
    else if (v > u1) { lo[u] = m; hi[u] = m; }      // x > t_{m-1}
    else {
      const int c = (int)((v - u0) >> shift);
      lo[u] = g.tab[c];
      hi[u] = g.tab[c + 1];
    }
    span = max(span, hi[u] - lo[u]);
  }
  while (span > 0) {  // interval lengths at least halve every step
#pragma unroll
    for (int u = 0; u < U; u++) {
      if (lo[u] < hi[u]) {
        const int mid = (lo[u] + hi[u]) >> 1;
        if (spl[mid] < x[u]) lo[u] = mid + 1; else hi[u] = mid;
      }
    }
    span >>= 1;
  }
#pragma unroll
  for (int u = 0; u < U; u++) {
    const int i = lo[u];
    bin[u] = 2 * i + ((i < m && spl[i] == x[u] && eqf[i]) ? 1 : 0);
  }
}

// Shared memory of the histogram passes (K1 fused, K8): dynamic, > 48 KB for int64.
template <typename K>
struct ClassifySmem {
  K tree[2 * kMaxBuckets];
  uint32_t hist[kMaxBins];
  uint8_t eq[kMaxBuckets];
  Guide guide;
};

// Shared-memory histogram increment (hardware-serialised on conflicts).
__device__ __forceinline__ void hist_add(uint32_t* hist, int bin, bool valid) {
  if (valid) atomicAdd(&hist[bin], 1u);
}

// Descent at i (a[i] > a[i+1]) whose outer neighbours are out of order,
// a[i-1] > a[i+2]: removing the descent's two endpoints would not leave the
// neighbourhood sorted.  Counted for the outlier route's choice (isolated
// exchanges, have none; shuffled runs or a random tail have many).
// a[i-1] and a[i+2] come from the warp's shuffles and a halo loaded together
// with the keys (no dependent loads).
template <typename K>
__device__ __forceinline__ int straddle_regs(int64_t n, int64_t i, K am1, K ap2) {
  return (i >= 1 && i + 2 < n && am1 > ap2) ? 1 : 0;
}

// Halo of a warp's 32 consecutive keys starting at i - lane: lane 0 loads
// a[i-1], lane 31 loads a[i+1] and a[i+2], all issued with the keys.
template <typename K>
__device__ __forceinline__ void load_halo(const K* __restrict__ keys, int64_t n, int64_t i, int lane, K& h1, K& h2) {
  h1 = K(0);
  h2 = K(0);
  if (lane == 0 && i >= 1 && i - 1 < n) h1 = keys[i - 1];
  if (lane == 31 && i + 1 < n) h1 = keys[i + 1];
  if (lane == 31 && i + 2 < n) h2 = keys[i + 2];
}

// Neighbours of x = a[i] from the warp: next a[i+1], prev a[i-1], next2 a[i+2].
template <typename K>
__device__ __forceinline__ void warp_neighbours(K x, K h1, K h2, int lane, K& next, K& prev, K& next2) {
  next = __shfl_down_sync(0xffffffffu, x, 1);
  prev = __shfl_up_sync(0xffffffffu, x, 1);
  next2 = __shfl_down_sync(0xffffffffu, x, 2);
  const K h1n = __shfl_down_sync(0xffffffffu, h1, 1);  // lane 30: lane 31's a[i+1] = its own a[i+2]
  if (lane == 31) { next = h1; next2 = h2; }
  if (lane == 30) next2 = h1n;
  if (lane == 0) prev = h1;
}

// Running H1 statistics of one thread (reduced over the CTA by the caller).
struct ScanAcc {
  int cd = 0, ca = 0, cv = 0;                       // descents, descending-run breaks, straddle violations
  int fd = INT32_MAX, ld = -1, fa = INT32_MAX, la = -1;  // first / last descent, first / last break
};

// H1 over the pairs (i, i+1), i in [t0, t1), with 16-byte vector loads: each
// thread owns V = 16 / sizeof(K) consecutive keys per vector, so V - 1 of its
// pairs are in registers and only three shuffles per vector reach the
// neighbours (lane 0 / lane 31 load the halo across warps).  The per-pair
// flags become bit masks; counts are popcounts and first / last positions
// come from ffs / clz once per vector.  Requires keys 16-byte aligned and
// t0 a multiple of V; keys beyond n are never read.
// With smn / smx (shared, one entry per kDSub-key subtile of [t0, t1), set to
// +inf / -inf by the caller; t0 a multiple of kDSub) the pass also records
// every subtile's min and max for the k-distance test (tile_mm_finish): a
// warp's 32 vectors of a round lie in one subtile, so one warp reduction and
// one shared atomic per round and warp.
template <typename K, bool STRICT, int NT, int R>
__device__ __forceinline__ void scan_range_vec(const K* __restrict__ keys, int64_t n, int64_t t0, int64_t t1,
                                               ScanAcc& acc, K* smn = nullptr, K* smx = nullptr) {
  constexpr int V = 16 / (int)sizeof(K);
  static_assert(kDSub % (32 * V) == 0, "a warp's round lies in one subtile");
  const int tid = threadIdx.x & (NT - 1), lane = threadIdx.x & 31;
  for (int64_t vb = t0 / V; vb * V < t1; vb += (int64_t)NT * R) {
    K x[R][V], hp[R], hn0[R], hn1[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
      const int64_t i0 = (vb + (int64_t)r * NT + tid) * V;
      if (i0 + V <= n) {
        const int4 v = __ldg(reinterpret_cast<const int4*>(keys + i0));
        memcpy(&x[r][0], &v, 16);
      } else {
#pragma unroll
        for (int j = 0; j < V; j++) x[r][j] = i0 + j < n ? keys[i0 + j] : K(0);
      }
      hp[r] = (lane == 0 && i0 >= 1 && i0 - 1 < n) ? keys[i0 - 1] : K(0);
      hn0[r] = (lane == 31 && i0 + V < n) ? keys[i0 + V] : K(0);
      hn1[r] = (lane == 31 && i0 + V + 1 < n) ? keys[i0 + V + 1] : K(0);
    }
#pragma unroll
    for (int r = 0; r < R; r++) {
      const int64_t i0 = (vb + (int64_t)r * NT + tid) * V;
      K e[V + 3];  // e[0] = a[i0-1], e[1 .. V] = the vector, e[V+1], e[V+2] = a[i0+V], a[i0+V+1]
      e[0] = __shfl_up_sync(0xffffffffu, x[r][V - 1], 1);
      e[V + 1] = __shfl_down_sync(0xffffffffu, x[r][0], 1);
      e[V + 2] = __shfl_down_sync(0xffffffffu, x[r][1], 1);
      if (lane == 0) e[0] = hp[r];
      if (lane == 31) { e[V + 1] = hn0[r]; e[V + 2] = hn1[r]; }
#pragma unroll
      for (int j = 0; j < V; j++) e[j + 1] = x[r][j];
      // valid pairs: i < t1 and i + 1 < n
      const int64_t lim64 = (t1 < n - 1 ? t1 : n - 1) - i0;
      const int lim = lim64 <= 0 ? 0 : (lim64 >= V ? V : (int)lim64);
      const unsigned valid = (1u << lim) - 1u;
      unsigned dm = 0, am = 0, sm = 0;
#pragma unroll
      for (int j = 0; j < V; j++) {
        const K a = e[j + 1], b = e[j + 2];
        dm |= (unsigned)(b < a) << j;
        am |= (unsigned)(STRICT ? !(b < a) : (a < b)) << j;
        // straddle: a[i-1] > a[i+2], defined for 1 <= i and i + 2 < n
        const bool inr = (j > 0 || i0 >= 1) && (i0 + j + 2 < n);
        sm |= (unsigned)(inr && e[j] > e[j + 3]) << j;
      }
      dm &= valid;
      am &= valid;
      sm &= dm;
      if (smn) {  // subtile min / max over the keys of [t0, t1)
        K mn = KeyTraits<K>::max_key(), mx = KeyTraits<K>::min_key();
        if (i0 + V <= t1 && i0 + V <= n) {  // (every vector but the last of a range)
#pragma unroll
          for (int j = 0; j < V; j++) { mn = min(mn, x[r][j]); mx = max(mx, x[r][j]); }
        } else {
#pragma unroll
          for (int j = 0; j < V; j++)
            if (i0 + j < t1 && i0 + j < n) { mn = min(mn, x[r][j]); mx = max(mx, x[r][j]); }
        }
        mn = warp_reduce_min(mn);
        mx = warp_reduce_max(mx);
        if (lane == 0 && i0 < t1) {
          const int q = (int)((i0 - t0) / kDSub);
          atomicMin(reinterpret_cast<typename KeyTraits<K>::AtomicT*>(smn + q), (typename KeyTraits<K>::AtomicT)mn);
          atomicMax(reinterpret_cast<typename KeyTraits<K>::AtomicT*>(smx + q), (typename KeyTraits<K>::AtomicT)mx);
        }
      }
      acc.cd += __popc(dm);
      acc.ca += __popc(am);
      acc.cv += __popc(sm);
      if (dm) {
        acc.fd = min(acc.fd, (int)i0 + __ffs(dm) - 1);
        acc.ld = max(acc.ld, (int)i0 + 31 - __clz(dm));
      }
      if (am) {
        acc.fa = min(acc.fa, (int)i0 + __ffs(am) - 1);
        acc.la = max(acc.la, (int)i0 + 31 - __clz(am));
      }
    }
  }
}

// k-distance test of one tile (all threads of the block; smn / smx filled by
// scan_range_vec): ok = max(subtile q) <= min(subtile q + 2) for every q with
// both subtiles inside [t0, t1) -- with such pairs on every tile boundary too
// (checked by the resolve), every key lies less than 2 kDSub positions from its
// place in the sorted output (PAPER.md:84 k-distance, k < 2 kDSub): the keys of
// subtiles <= q-2 are <= x and those of subtiles >= q+2 are >= x for every x in
// subtile q.  valid = 0 (no subtile statistics) makes the tile fail.
template <typename K>
__device__ __forceinline__ void tile_mm_init(K* smn, K* smx, int nsub) {
  for (int q = threadIdx.x; q < nsub; q += blockDim.x) {
    smn[q] = KeyTraits<K>::max_key();
    smx[q] = KeyTraits<K>::min_key();
  }
}
template <typename K>
__device__ __forceinline__ int tile_mm_finish(const K* smn, const K* smx, int nsub, int valid, TileMM* out) {
  int bad = !valid;
  for (int q = threadIdx.x; q + 2 < nsub; q += blockDim.x) bad |= smx[q] > smn[q + 2];
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    TileMM t;
    t.mn0 = (int64_t)smn[0];
    t.mn1 = nsub > 1 ? (int64_t)smn[1] : INT64_MAX;
    t.mx0 = nsub > 1 ? (int64_t)smx[nsub - 2] : INT64_MIN;
    t.mx1 = (int64_t)smx[nsub - 1];
    t.ok = !bad;
    t.nsub = nsub;
    *out = t;
  }
  return !bad;  // (every thread)
}

// K1: one CTA per tile of `tile` keys.  STRICT selects the descending-run
// break rule: a_i <= a_{i+1} (pairs: only strictly descending runs may be
// reversed, "the reversely sorted subsequence cannot contain equal
// elements") or a_i < a_{i+1} (keys-only: non-increasing runs).
// FUSE additionally classifies every key against the level-1 splitters and
// writes the tile's bucket histogram (H8 fused into the H1 read).
template <typename K, bool STRICT, bool FUSE, int NT>
__global__ void __launch_bounds__(NT) k_presort_scan(const K* __restrict__ keys, int64_t n, int tile,
                                                      TileSummary* __restrict__ sums, const K* __restrict__ spl,
                                                      const uint8_t* __restrict__ eqf, const int* __restrict__ mcount,
                                                      uint32_t* __restrict__ mat, int nbins, int G,
                                                      uint32_t* __restrict__ tot, uint16_t* __restrict__ bins_out,
                                                      TileMM* __restrict__ mm) {
  constexpr int U = 8;
  __shared__ K s_mn[65536 / kDSub], s_mx[65536 / kDSub];  // tile <= 65536 keys
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ClassifySmem<K>& csm = *reinterpret_cast<ClassifySmem<K>*>(smem_raw);  // FUSE only (dynamic)
  K* s_spl = csm.tree;
  uint8_t* s_eq = csm.eq;
  uint32_t* s_hist = csm.hist;
  __shared__ int32_t s_red[NT / 32 + 1];
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t t0 = (int64_t)blockIdx.x * tile;
  const int64_t t1 = t0 + tile < n ? t0 + tile : n;
  int m = 0, depth = 1;
  if (FUSE) {
    m = mcount[0];
    depth = tree_depth(m);
    load_splitters_smem(spl, eqf, m, s_spl, s_eq);
    for (int b = tid; b < nbins; b += NT) s_hist[b] = 0;
    __syncthreads();
  }
  int cd = 0, ca = 0, cv = 0;
  int fd = INT32_MAX, ld = -1, fa = INT32_MAX, la = -1;
  const int nsub = (int)((t1 - t0 + kDSub - 1) / kDSub);
  const bool vec = !FUSE && (reinterpret_cast<uintptr_t>(keys) & 15) == 0 && t0 % (16 / (int)sizeof(K)) == 0;
  if (mm) {
    tile_mm_init<K>(s_mn, s_mx, nsub);
    __syncthreads();
  }
  if (vec) {
    ScanAcc acc;
    scan_range_vec<K, STRICT, NT, (sizeof(K) == 4 ? 2 : 4)>(keys, n, t0, t1, acc, mm ? s_mn : nullptr,
                                                            mm ? s_mx : nullptr);
    cd = acc.cd; ca = acc.ca; cv = acc.cv; fd = acc.fd; ld = acc.ld; fa = acc.fa; la = acc.la;
  } else
  for (int64_t base = t0; base < t1; base += NT * U) {
    K x[U], h1[U], h2[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      int64_t i = base + u * NT + tid;
      x[u] = i < n ? keys[i] : K(0);
      load_halo<K>(keys, n, i, lane, h1[u], h2[u]);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      int64_t i = base + u * NT + tid;
      K y, pv, n2;
      warp_neighbours<K>(x[u], h1[u], h2[u], lane, y, pv, n2);
      if (i < t1 && i + 1 < n) {
        if (y < x[u]) {
          cd++; fd = min(fd, (int)i); ld = max(ld, (int)i);
          cv += straddle_regs<K>(n, i, pv, n2);
        }
        bool brk = STRICT ? !(y < x[u]) : (x[u] < y);
        if (brk) { ca++; fa = min(fa, (int)i); la = max(la, (int)i); }
      }
    }
    if (FUSE) {
      int bin[U];
      classify_keys<K, U>(x, bin, s_spl, s_eq, m, depth);
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t i = base + u * NT + tid;
        hist_add(s_hist, bin[u], i < t1);
        if (bins_out && i < t1) bins_out[i] = (uint16_t)bin[u];  // reused by the scatter
      }
    }
  }
  if (mm) {
    __syncthreads();
    tile_mm_finish<K>(s_mn, s_mx, nsub, vec ? 1 : 0, mm + blockIdx.x);
  }
  cd = block_reduce_sum<NT>(cd, s_red);
  ca = block_reduce_sum<NT>(ca, s_red);
  fd = block_reduce_min<NT>(fd, s_red);
  ld = block_reduce_max<NT>(ld, s_red);
  fa = block_reduce_min<NT>(fa, s_red);
  la = block_reduce_max<NT>(la, s_red);
  cv = block_reduce_sum<NT>(cv, s_red);
  if (tid == 0) {
    TileSummary s;
    s.ndesc = cd; s.nab = ca; s.fdesc = fd; s.ldesc = ld; s.fab = fa; s.lab = la; s.nviol = cv; s.tok = 0;
    sums[blockIdx.x] = s;
  }
  if (FUSE) {
    __syncthreads();
    if (tot) {  // keys only: bucket totals (no count matrix)
      for (int b = tid; b < nbins; b += NT)
        if (s_hist[b]) atomicAdd(&tot[b], s_hist[b]);
    } else {
      for (int b = tid; b < nbins; b += NT) mat[(int64_t)b * G + blockIdx.x] = s_hist[b];
    }
  }
}

// Device-side route (H3 first stage) from the resolved statistics;
// kRouteUndecided hands the merge-vs-partition cost comparison to the host planner.
__device__ __forceinline__ int64_t resolve_route(int64_t n, int64_t D, int64_t A, int64_t V, int64_t covA, int64_t covD,
                                                 int force, int merge_ok, int dist_ok = 0) {
  if (D == 0) return kRouteSorted;
  if (A == 0 && force == 0) return kRouteReversed;
  if (force == kRouteMerge) return kRouteMerge;
  if (n <= kCap) return kRouteTile;
  if (force == kRoutePartition) return kRoutePartition;
  if (force == kRouteOutlier) return kRouteOutlier;
  // few, isolated descents (k-exchange-like): extract the outliers
  if ((merge_ok & kAllowOutlier) && A > 0 && kViolRatio * V <= D &&
      ((merge_ok & kOutlierStrict) ? kOutlierRatioStrict : kOutlierRatio) * D <= n)
    return kRouteOutlier;
  // bounded displacement (k-distance): two passes of window sorts
  if (dist_ok && (merge_ok & kAllowDistance)) return kRouteDistance;
  if ((merge_ok & kAllowMerge) && 2 * (covA + covD) >= n) return kRouteUndecided;
  return kRoutePartition;
}

// The k-distance test over all tiles: every tile passed its own test and the
// subtile pairs that straddle a tile boundary (the last two subtiles of tile
// t against the first two of tile t+1) are ordered too.  mm == nullptr: no.
__device__ __forceinline__ int tile_mm_pair_ok(const TileMM* __restrict__ mm, int t, int G) {
  const int64_t* q = reinterpret_cast<const int64_t*>(mm + t);
  if (!__ldcg(reinterpret_cast<const int*>(q + 4))) return 0;  // ok
  if (t + 1 >= G) return 1;
  const int64_t mx0 = __ldcg(q + 2), mx1 = __ldcg(q + 3);
  const int64_t* r = reinterpret_cast<const int64_t*>(mm + t + 1);
  const int64_t mn0 = __ldcg(r + 0), mn1 = __ldcg(r + 1);
  return mx0 <= mn0 && mx1 <= mn1;
}

// K2: resolve tile summaries into D, the long runs of both directions and
// their covers (single CTA; loops over the tiles with a carried prefix).
// Block-level body of K2 (all NT threads of one CTA call it); also run by CTA 0
// of the resident kernel (resident.cuh).  Cross-CTA inputs are read with
// __ldcg so a caller that produced them in an earlier grid-sync phase sees them.
// Returns the device route to every thread; WRITE = false computes the route
// only (the resident kernel's CTAs other than 0 resolve redundantly instead of
// waiting for a grid barrier).
template <typename K, int NT, bool WRITE = true>
__device__ __forceinline__ int64_t presort_resolve_block(const K* __restrict__ keys, int64_t n,
                                                      const TileSummary* __restrict__ sums, int G, int64_t lmin,
                                                      RunDesc* __restrict__ asc, RunDesc* __restrict__ desc,
                                                      DevStats* __restrict__ st, int force, int merge_ok,
                                                      const TileMM* __restrict__ mm = nullptr) {
  __shared__ int32_t s_incl[2][NT];
  __shared__ int64_t s_red64[NT / 32 + 1];
  __shared__ int32_t s_red[NT / 32 + 1];
  __shared__ int64_t s_route;
  const int tid = threadIdx.x;
  int32_t carryD = -1, carryA = -1;
  int64_t D = 0, A = 0, V = 0, nasc = 0, ndsc = 0, covA = 0, covD = 0;
  for (int c0 = 0; c0 < G; c0 += NT) {
    const int t = c0 + tid;
    TileSummary s;
    if (t < G) {
      const int4* p = reinterpret_cast<const int4*>(sums + t);
      int4 a = __ldcg(p), b = __ldcg(p + 1);
      s.ndesc = a.x; s.nab = a.y; s.fdesc = a.z; s.ldesc = a.w; s.fab = b.x; s.lab = b.y; s.nviol = b.z; s.tok = 0;
    } else { s.ndesc = 0; s.nab = 0; s.fdesc = 0; s.ldesc = -1; s.fab = 0; s.lab = -1; s.nviol = 0; }
    D += s.ndesc;
    A += s.nab;
    V += s.nviol;
    int32_t iD = block_inclusive_max<NT>(s.ldesc, s_red, -1);
    int32_t iA = block_inclusive_max<NT>(s.lab, s_red, -1);
    s_incl[0][tid] = iD;
    s_incl[1][tid] = iA;
    __syncthreads();
    int32_t prevD = tid > 0 ? s_incl[0][tid - 1] : -1;
    int32_t prevA = tid > 0 ? s_incl[1][tid - 1] : -1;
    prevD = max(prevD, carryD);
    prevA = max(prevA, carryA);
    // ascending run ending at this tile's first descent
    int64_t lenA = (s.ndesc > 0) ? (int64_t)s.fdesc - prevD : 0;
    int fA = (t < G && s.ndesc > 0 && lenA >= lmin) ? 1 : 0;
    int64_t lenDd = (s.nab > 0) ? (int64_t)s.fab - prevA : 0;
    int fDd = (t < G && s.nab > 0 && lenDd >= lmin) ? 1 : 0;
    int32_t totA, totD;
    int32_t exA = block_exclusive_sum<NT>(fA, s_red, &totA);
    int32_t exD = block_exclusive_sum<NT>(fDd, s_red, &totD);
    if (WRITE && fA) {
      RunDesc r;
      r.start = prevD + 1; r.len = lenA;
      r.kfirst = (int64_t)keys[r.start]; r.klast = (int64_t)keys[r.start + r.len - 1];
      asc[nasc + exA] = r;
    }
    if (WRITE && fDd) {
      RunDesc r;
      r.start = prevA + 1; r.len = lenDd;
      r.kfirst = (int64_t)keys[r.start]; r.klast = (int64_t)keys[r.start + r.len - 1];
      desc[ndsc + exD] = r;
    }
    covA += fA ? lenA : 0;
    covD += fDd ? lenDd : 0;
    nasc += totA;
    ndsc += totD;
    carryD = max(carryD, s_incl[0][NT - 1]);
    carryA = max(carryA, s_incl[1][NT - 1]);
    __syncthreads();
  }
  D = block_reduce_sum<NT>(D, s_red64);
  A = block_reduce_sum<NT>(A, s_red64);
  V = block_reduce_sum<NT>(V, s_red64);
  covA = block_reduce_sum<NT>(covA, s_red64);
  covD = block_reduce_sum<NT>(covD, s_red64);
  int dok = mm != nullptr;
  if (mm)
    for (int t = tid; t < G; t += NT) dok &= tile_mm_pair_ok(mm, t, G);
  dok = __syncthreads_and(dok);
  if (tid == 0) {
    // final runs after the last break
    int64_t lastLen = n - 1 - (int64_t)carryD;
    if (n > 0 && lastLen >= lmin) {
      if (WRITE) {
        RunDesc r;
        r.start = carryD + 1; r.len = lastLen;
        r.kfirst = (int64_t)keys[r.start]; r.klast = (int64_t)keys[n - 1];
        asc[nasc] = r;
      }
      nasc++;
      covA += lastLen;
    }
    int64_t lastLenD = n - 1 - (int64_t)carryA;
    if (n > 0 && lastLenD >= lmin) {
      if (WRITE) {
        RunDesc r;
        r.start = carryA + 1; r.len = lastLenD;
        r.kfirst = (int64_t)keys[r.start]; r.klast = (int64_t)keys[n - 1];
        desc[ndsc] = r;
      }
      ndsc++;
      covD += lastLenD;
    }
    const int64_t route = resolve_route(n, D, A, V, covA, covD, force, merge_ok, dok);
    if (WRITE) {
      st->dist_ok = dok;
      st->n = n;
      st->descents = D;
      st->asc_breaks = A;
      st->n_asc_runs = nasc;
      st->n_desc_runs = ndsc;
      st->asc_cover = covA;
      st->desc_cover = covD;
      st->route = route;
    }
    s_route = route;
  }
  __syncthreads();
  const int64_t route = s_route;
  __syncthreads();
  return route;
}

// K2 for one warp (the resident kernel, G <= 32 * 32 tiles): the same
// statistics, run descriptors and route as presort_resolve_block, from tile
// summaries already in shared memory, without block barriers.  Lane l owns the
// contiguous tiles [l TPL, (l+1) TPL); the last break before its chunk comes
// from a warp max-scan, the run descriptors' slots from a warp prefix sum.
// All 32 lanes of the warp call; every lane returns the route.
template <typename K, bool WRITE>
__device__ int64_t presort_resolve_warp(const K* __restrict__ keys, int64_t n, const TileSummary* ts, int G,
                                        int64_t lmin, RunDesc* __restrict__ asc, RunDesc* __restrict__ desc,
                                        DevStats* __restrict__ st, int force, int merge_ok,
                                        const TileMM* __restrict__ mm = nullptr) {
  const int lane = threadIdx.x & 31;
  const int TPL = (G + 31) / 32;
  const int t0 = lane * TPL < G ? lane * TPL : G, t1 = t0 + TPL < G ? t0 + TPL : G;
  int64_t D = 0, A = 0, V = 0;
  int32_t lastD = -1, lastA = -1;
  for (int t = t0; t < t1; t++) {
    D += ts[t].ndesc;
    A += ts[t].nab;
    V += ts[t].nviol;
    lastD = max(lastD, ts[t].ldesc);
    lastA = max(lastA, ts[t].lab);
  }
  int32_t carryD = lastD, carryA = lastA;  // inclusive max-scan, then shifted to exclusive
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t u = __shfl_up_sync(0xffffffffu, carryD, o), v = __shfl_up_sync(0xffffffffu, carryA, o);
    if (lane >= o) { carryD = max(carryD, u); carryA = max(carryA, v); }
  }
  const int32_t endD = __shfl_sync(0xffffffffu, carryD, 31), endA = __shfl_sync(0xffffffffu, carryA, 31);
  carryD = __shfl_up_sync(0xffffffffu, carryD, 1);
  carryA = __shfl_up_sync(0xffffffffu, carryA, 1);
  if (lane == 0) { carryD = -1; carryA = -1; }
  // runs ending inside this lane's tiles
  int nA = 0, nD = 0;
  int64_t covA = 0, covD = 0;
  {
    int32_t pD = carryD, pA = carryA;
    for (int t = t0; t < t1; t++) {
      const TileSummary s = ts[t];
      if (s.ndesc > 0 && (int64_t)s.fdesc - pD >= lmin) { nA++; covA += (int64_t)s.fdesc - pD; }
      if (s.nab > 0 && (int64_t)s.fab - pA >= lmin) { nD++; covD += (int64_t)s.fab - pA; }
      pD = max(pD, s.ldesc);
      pA = max(pA, s.lab);
    }
  }
  int exA = nA, exD = nD;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, exA, o), v = __shfl_up_sync(0xffffffffu, exD, o);
    if (lane >= o) { exA += u; exD += v; }
  }
  const int totA = __shfl_sync(0xffffffffu, exA, 31), totD = __shfl_sync(0xffffffffu, exD, 31);
  exA -= nA;
  exD -= nD;
  if (WRITE) {
    int32_t pD = carryD, pA = carryA;
    for (int t = t0; t < t1; t++) {
      const TileSummary s = ts[t];
      if (s.ndesc > 0 && (int64_t)s.fdesc - pD >= lmin) {
        RunDesc r;
        r.start = pD + 1; r.len = (int64_t)s.fdesc - pD;
        r.kfirst = (int64_t)keys[r.start]; r.klast = (int64_t)keys[r.start + r.len - 1];
        asc[exA++] = r;
      }
      if (s.nab > 0 && (int64_t)s.fab - pA >= lmin) {
        RunDesc r;
        r.start = pA + 1; r.len = (int64_t)s.fab - pA;
        r.kfirst = (int64_t)keys[r.start]; r.klast = (int64_t)keys[r.start + r.len - 1];
        desc[exD++] = r;
      }
      pD = max(pD, s.ldesc);
      pA = max(pA, s.lab);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    D += __shfl_xor_sync(0xffffffffu, D, o);
    A += __shfl_xor_sync(0xffffffffu, A, o);
    V += __shfl_xor_sync(0xffffffffu, V, o);
    covA += __shfl_xor_sync(0xffffffffu, covA, o);
    covD += __shfl_xor_sync(0xffffffffu, covD, o);
  }
  int64_t nasc = totA, ndsc = totD;
  // final runs after the last break
  const int64_t lastLen = n - 1 - (int64_t)endD, lastLenD = n - 1 - (int64_t)endA;
  if (n > 0 && lastLen >= lmin) {
    if (WRITE && lane == 0) {
      RunDesc r;
      r.start = endD + 1; r.len = lastLen;
      r.kfirst = (int64_t)keys[r.start]; r.klast = (int64_t)keys[n - 1];
      asc[nasc] = r;
    }
    nasc++;
    covA += lastLen;
  }
  if (n > 0 && lastLenD >= lmin) {
    if (WRITE && lane == 0) {
      RunDesc r;
      r.start = endA + 1; r.len = lastLenD;
      r.kfirst = (int64_t)keys[r.start]; r.klast = (int64_t)keys[n - 1];
      desc[ndsc] = r;
    }
    ndsc++;
    covD += lastLenD;
  }
  // the k-distance test only where it can change the route (every route before
  // it in resolve_route is independent of dist_ok); the tiles' own verdicts are
  // in ts[t].tok, so the straddle pairs in global memory are read only when
  // every tile passed
  int64_t route = resolve_route(n, D, A, V, covA, covD, force, merge_ok, 0);
  int dok = 0;
  if (mm && (merge_ok & kAllowDistance) && (route == kRoutePartition || route == kRouteUndecided)) {
    dok = 1;
    for (int t = t0; t < t1; t++) dok &= ts[t].tok != 0;
    dok = __all_sync(0xffffffffu, dok);
    if (dok) {
      for (int t = t0; t < t1; t++) dok &= tile_mm_pair_ok(mm, t, G);
      dok = __all_sync(0xffffffffu, dok);
    }
    if (dok) route = resolve_route(n, D, A, V, covA, covD, force, merge_ok, dok);
  }
  if (WRITE && lane == 0) {
    st->dist_ok = dok;
    st->n = n;
    st->descents = D;
    st->asc_breaks = A;
    st->n_asc_runs = nasc;
    st->n_desc_runs = ndsc;
    st->asc_cover = covA;
    st->desc_cover = covD;
    st->route = route;
  }
  return route;
}

template <typename K, int NT>
__global__ void __launch_bounds__(NT) k_presort_resolve(const K* __restrict__ keys, int64_t n,
                                                         const TileSummary* __restrict__ sums, int G, int64_t lmin,
                                                         RunDesc* __restrict__ asc, RunDesc* __restrict__ desc,
                                                         DevStats* __restrict__ st, int force, int merge_ok,
                                                         const TileMM* __restrict__ mm) {
  presort_resolve_block<K, NT>(keys, n, sums, G, lmin, asc, desc, st, force, merge_ok, mm);
}

// K3: in-place reversal of ranges [start, start+len) (H2; PAPER.md:93 and
// Appendix A reverse()).  Block b maps to (range, chunk)
// through the host-built chunk prefix; each chunk swaps NT*U mirrored pairs
// with coalesced front and back accesses.
template <typename K, bool HAS_V, int NT>
__global__ void __launch_bounds__(NT) k_reverse(K* __restrict__ keys, uint32_t* __restrict__ vals,
                                                 const RunDesc* __restrict__ ranges,
                                                 const int64_t* __restrict__ chunk_prefix, int nranges,
                                                 const DevStats* __restrict__ gate, int64_t whole_len) {
  if (gate && gate->route != kRouteReversed) return;  // speculative launch
  constexpr int U = 8;
  constexpr int CH = NT * U;
  int64_t s, len, c0;
  if (!ranges) {  // the whole array [0, whole_len)
    s = 0;
    len = whole_len;
    c0 = (int64_t)blockIdx.x * CH;
  } else {
    __shared__ int s_r;
    if (threadIdx.x == 0) {
      int lo = 0, hi = nranges - 1;
      while (lo < hi) {  // last r with chunk_prefix[r] <= blockIdx.x
        int mid = (lo + hi + 1) >> 1;
        if (chunk_prefix[mid] <= (int64_t)blockIdx.x) lo = mid; else hi = mid - 1;
      }
      s_r = lo;
    }
    __syncthreads();
    const int r = s_r;
    s = ranges[r].start;
    len = ranges[r].len;
    c0 = ((int64_t)blockIdx.x - chunk_prefix[r]) * CH;
  }
  const int64_t half = len / 2;
  // the whole-array launch is grid-strided (a bounded grid keeps the gated,
  // speculative launch cheap when another route is taken)
  const int64_t stride = ranges ? INT64_MAX : (int64_t)gridDim.x * CH;
  for (; c0 < half; c0 += stride) {
    K a[U], b[U];
    uint32_t va[U], vb[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      int64_t p = c0 + u * NT + threadIdx.x;
      if (p < half) {
        a[u] = keys[s + p];
        b[u] = keys[s + len - 1 - p];
        if (HAS_V) { va[u] = vals[s + p]; vb[u] = vals[s + len - 1 - p]; }
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      int64_t p = c0 + u * NT + threadIdx.x;
      if (p < half) {
        keys[s + p] = b[u];
        keys[s + len - 1 - p] = a[u];
        if (HAS_V) { vals[s + p] = vb[u]; vals[s + len - 1 - p] = va[u]; }
      }
    }
    if (stride == INT64_MAX) break;
  }
}

}  // namespace sr
