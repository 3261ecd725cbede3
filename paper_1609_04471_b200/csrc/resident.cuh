// resident.cuh -- the resident path: the whole keys-only sort of an L2-resident
// array (kCap < n <= kResMaxN) as ONE cooperative launch of one CTA per SM.
//
// The multi-kernel path (presort.cuh, partition.cuh) pays a launch plus a
// drain per step and a one-CTA bookkeeping kernel per level; at the paper's
// Table 1 size (n = 2,000,000) a full pass over the keys is
// ~1.2 us of HBM time, so those fixed costs dominated.  Here the steps run as
// three phases of one persistent kernel separated by two grid-wide barriers,
// and the quicksort recursion (Appendix B) is two levels of
// splitter partitioning: a global one over <= 1024 buckets, then each bucket
// is sorted by one CTA in shared memory.
//   A  H1 scan of every presort tile (same tiles and TileSummary as K1).
//      Meanwhile the last two CTAs (they scan the fewest tiles) each gather
//      and sort one half of the level-1 sample (S1 = 8 B1 jittered
//      positions, R8).
//   -- grid sync --
//   C  every CTA resolves the tile summaries into the device route (K2's
//      logic; CTA 0 also writes the statistics and run lists).  SORTED exits
//      (PAPER.md:167); REVERSED reverses in place; MERGE /
//      undecided return to the host planner.  PARTITION: splitters t_j =
//      element 8(j+1) of the two merged halves (merge-path selection), with
//      their gamma flags (count > gamma = 2 in the sample; R9)
//      -> Eytzinger tree; each tile is classified
//      (3-way ids) and written to the same span of the
//      workspace grouped by bucket (a tile-local counting sort: contiguous,
//      coalesced writes), with its per-bucket counts and local starts; the
//      bucket totals are accumulated with atomics.
//   -- grid sync --
//   E  bucket starts = exclusive scan of the totals (every CTA).  Units:
//      equality buckets are filled ("spared from the recursive calls",
//      PAPER.md:158); a range bucket is gathered from its per-tile pieces
//      into shared memory by one CTA, checked with is_sorted,
//      and sorted there: 128-key runs by 16-lane register bitonic networks
//      (the insertion-sort-below-alpha step), then merge-path
//      merge rounds (the mergesort levels of §3, A wins ties),
//      the last one writing the output.  Buckets beyond CAPB keys are
//      gathered unsorted into their final range and listed for the host,
//      which runs further partition levels on them.
#pragma once
#include <cooperative_groups.h>
#include <cstddef>

#include "bitonic.cuh"
#include "common.cuh"
#include "partition.cuh"
#include "presort.cuh"
#include "types.cuh"

namespace sr {

constexpr int kResNT = 512;
constexpr int kResCtasPerSM = 1;
constexpr int kResWarps = kResNT / 32;
constexpr int kResTile = 8192;          // presort tile in the resident range (choose_tile)
constexpr int kResGrp = 8192;           // phase C grouping unit: one tile-local counting sort
constexpr int kResO1 = 8;               // level-1 oversampling
constexpr int kResFill = 32768;         // equality fill per unit
constexpr int kResMaxNG = 512;          // grouping units (n <= kResMaxNG * kResGrp)

template <typename K> struct ResCfg;
template <> struct ResCfg<int32_t> {
  static constexpr int CAPB = 16384;    // largest level-1 bucket sorted by one CTA
  static constexpr int B1MAX = 1024;    // level-1 buckets
  static constexpr int64_t MAXN = int64_t(4) << 20;
};
template <> struct ResCfg<int64_t> {
  static constexpr int CAPB = 8192;
  static constexpr int B1MAX = 1024;
  static constexpr int64_t MAXN = int64_t(4) << 20;
};
constexpr int64_t kResMaxN = ResCfg<int32_t>::MAXN;  // largest resident n over the key types
static_assert(kResMaxN <= (int64_t)kResMaxNG * kResGrp, "");

template <typename K>
struct ResArgs {
  K* keys;
  K* ws;
  int64_t n;
  int tile, G;              // presort tiles (K1's tiling)
  TileSummary* sums;
  RunDesc* asc;
  RunDesc* desc;
  DevStats* st;             // route, statistics; n_ovf counts the host list
  int S1, B1;               // level-1 sample size, buckets (power of two <= B1MAX)
  int NG;                   // grouping units of kResGrp keys
  K* samp;                  // S1 keys: the two sorted halves of the level-1 sample
  uint32_t* tot;            // 2 B1 + 1 bucket totals (zeroed by the host)
  uint32_t* mcnt;           // NG x nbins: per-group bucket counts
  uint32_t* mlst;           // NG x nbins: per-group bucket starts inside the group's span of ws
  OvfSeg* ovf;              // ranges of keys left unsorted for the host's next level
  int64_t lmin;
  int force, merge_ok;
  int capb;                 // largest level-1 bucket sorted in-kernel (CAPB; lowered by tests)
  unsigned long long* tstamp;  // optional: %globaltimer, [0..8) CTA 0 phase starts, then 8 per CTA
  uint32_t* unit_counter;   // phase E work counter (zeroed by the host)
};

#define SR_RES_STAMP(k)                                                                \
  do {                                                                                 \
    if (a.tstamp && tid == 0) a.tstamp[8 + (size_t)blockIdx.x * 8 + (k)] = res_now(); \
  } while (0)

__device__ __forceinline__ unsigned long long res_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Shared memory: the persistent bucket table + phase-local buffers in a union.
template <typename K>
struct ResSmem {
  static constexpr int CAPB = ResCfg<K>::CAPB;
  static constexpr int B1MAX = ResCfg<K>::B1MAX;
  static constexpr int NB1 = 2 * B1MAX + 1;
  static constexpr int S1MAX = kResO1 * B1MAX;
  struct alignas(16) CT {          // C: one group's counting sort
    uint32_t cnt[NB1];
    uint32_t lst[NB1];
    K stk[kResGrp];
  };
  struct alignas(16) E {
    K x[CAPB];                     // the gathered bucket (padded to whole runs)
    K y[CAPB];                     // merge ping-pong buffer
    uint32_t piece[kResMaxNG + 1]; // gather offsets of the bucket's per-group pieces
    uint32_t pbase[kResMaxNG];     // ws position of each piece
  };
  uint32_t start[NB1 + 1];         // level-1 bucket starts, start[nbins] = n
  uint32_t upre[NB1 + 1];          // exclusive prefix of E units per bin
  K tree1[2 * B1MAX];              // level-1 Eytzinger tree [1, B1) + sorted splitters at [B1MAX, ...)
  uint8_t eq1[B1MAX];
  union alignas(16) {
    K samp1[S1MAX];                // A: half of the level-1 sample + BitonicSort scratch
    CT ct;
    E e;
  } u;
  int32_t red[kResNT / 32 + 1];
  int64_t red64[kResNT / 32 + 1];
  int32_t agg[kResWarps][7];
};

// Level-order (Eytzinger) part of a splitter tree whose sorted copy is at tree[BMAX + i].
template <typename K, int BMAX>
__device__ __forceinline__ void res_build_tree(int depth, K* tree) {
  const int nodes = 1 << depth;
  for (int i = threadIdx.x + 1; i < nodes; i += blockDim.x) {
    const int d = 31 - __clz(i);
    const int pos = ((2 * (i - (1 << d)) + 1) << (depth - 1 - d)) - 1;
    tree[i] = tree[BMAX + pos];  // +inf padding beyond the splitters
  }
}

// Bucket id: i = #{t_j < x} (lower_bound), 2i+1 if x equals an equality
// splitter, else 2i (3-way split).
template <typename K, int BMAX, int U>
__device__ __forceinline__ void res_classify(const K (&x)[U], int (&bin)[U], const K* tree, const uint8_t* eq, int m,
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
    bin[u] = 2 * i + ((i < m && tree[BMAX + i] == x[u] && eq[i]) ? 1 : 0);
  }
}

// Rank of sample q in s[0, S): #{s_j < x} + #{s_j == x, j < q} (its position in
// the stably sorted sample), computed by GL lanes over strided j and reduced.
template <typename K, int GL>
__device__ __forceinline__ int res_rank(const K* s, int S, int q, int gl) {
  const K x = s[q];
  int r = 0;
  for (int j = gl; j < S; j += GL) {
    const K y = s[j];
    r += (y < x) || (y == x && j < q);
  }
#pragma unroll
  for (int o = GL / 2; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  return r;
}

// Splitter j = sorted[(j+1) o] with the gamma flag (the value occurs more than
// gamma = 2 times in the sample); LD reads one sorted element.
template <typename K, typename LD>
__device__ __forceinline__ void res_pick(LD ld, int S, int o, int j, K& t, uint8_t& f) {
  const int r = (j + 1) * o;
  t = ld(r);
  const bool m1 = r >= 1 && ld(r - 1) == t, m2 = r >= 2 && ld(r - 2) == t;
  const bool p1 = r + 1 < S && ld(r + 1) == t, p2 = r + 2 < S && ld(r + 2) == t;
  f = ((m1 && m2) || (m1 && p1) || (p1 && p2)) ? 1 : 0;
}

// Register bitonic sort of `count` keys by a group of GL lanes holding VT keys
// each (blocked: lane l owns [l VT, (l+1) VT)), loaded from the 16-byte
// aligned `src` (GL * VT readable keys; slots >= count are ignored) and written
// to dst[0, count).  All lanes of the warp call with the same VT and GL.
template <typename K, int VT, int GL>
__device__ __forceinline__ void res_group_sort(const K* src, int count, K* __restrict__ dst) {
  using BT = BitonicSort<K, 32, VT>;
  const int gl = threadIdx.x & (GL - 1);
  K k[VT];
  BlockSort<K, false, 32, VT>::load_vec(src + gl * VT, k);
#pragma unroll
  for (int i = 0; i < VT; i++)
    if (gl * VT + i >= count) k[i] = KeyTraits<K>::max_key();
  batcher_network<VT>([&](int a, int b) {
    K x = k[a], y = k[b];
    k[a] = BT::kmin(x, y);
    k[b] = BT::kmax(x, y);
  });
#pragma unroll
  for (int tk = 2; tk <= GL; tk <<= 1) {  // lanes per merged run
    BT::shfl_stage(k, tk - 1, (gl & (tk >> 1)) == 0, true);
#pragma unroll
    for (int jt = tk >> 2; jt >= 1; jt >>= 1) BT::shfl_stage(k, jt, (gl & jt) == 0, false);
    BT::reg_half_cleaners(k);
  }
#pragma unroll
  for (int i = 0; i < VT; i++)
    if (gl * VT + i < count) dst[gl * VT + i] = k[i];
}

// One CTA sorts x[0, L) (L <= CAPB, already gathered in shared memory) into
// dst: H11 for one level-1 bucket.  is_sorted first;
// then runs of 128 keys sorted by 16-lane register bitonic networks (the
// insertion-sort-below-alpha step), then merge-path merge rounds
// in shared memory (the paper's mergesort levels, §3; A wins ties,
// PAPER.md:99), the last round writing straight into dst.  The tail up to a
// whole run is padded with +inf, which sorts last and is not written.
template <typename K, int NT>
__device__ void res_bucket_sort(K* __restrict__ dst, int L, typename ResSmem<K>::E& e,
                                unsigned long long* prof = nullptr) {
  constexpr int VT = 8;  // merge outputs per thread
  constexpr int RVT = 8, RGL = 16;  // runs: 16-lane groups of VT 8 (128 keys), two per warp
  constexpr int kResRun = RGL * RVT;
  const int tid = threadIdx.x;
  unsigned long long tprev = (prof && tid == 0) ? res_now() : 0;
  auto mark = [&](int k) {  // optional per-step time accumulation (thread 0 of one CTA)
    if (prof && tid == 0) {
      const unsigned long long t = res_now();
      prof[k] += t - tprev;
      tprev = t;
    }
  };
  int unsorted = 0;
  for (int i = tid; i + 1 < L; i += NT) unsorted |= e.x[i + 1] < e.x[i];
  if (!__syncthreads_or(unsorted)) {
    for (int i = tid; i < L; i += NT) dst[i] = e.x[i];
    return;
  }
  const int nruns = (L + kResRun - 1) / kResRun;
  const int Lp = nruns * kResRun;
  for (int i = L + tid; i < Lp; i += NT) e.x[i] = KeyTraits<K>::max_key();
  __syncthreads();
  mark(0);
  {  // both halves of a warp always take part (the shuffles span the warp); a
     // half without a run sorts nothing
    const int half = (tid >> 4) & 1, w = tid >> 5;
    for (int r0 = 2 * w; r0 < nruns; r0 += NT / RGL) {
      const int r = r0 + half < nruns ? r0 + half : r0;
      const int cnt = r0 + half < nruns ? (nruns == 1 ? L : kResRun) : 0;
      res_group_sort<K, RVT, RGL>(e.x + r * kResRun, cnt, nruns == 1 ? dst : e.y + r * kResRun);
    }
  }
  __syncthreads();
  mark(1);
  if (nruns == 1) return;
  K* src = e.y;
  K* out = e.x;
  for (int R = kResRun; R < Lp; R *= 2) {
    const bool last = 2 * R >= Lp;
    for (int o = tid * VT; o < Lp; o += NT * VT) {
      const int p0 = (o / (2 * R)) * (2 * R);
      const int alen = R < Lp - p0 ? R : Lp - p0;
      const int blen = Lp - p0 - alen < R ? Lp - p0 - alen : R;
      const K* A = src + p0;
      const K* B = A + alen;
      const int diag = o - p0;
      const int i = merge_path_search<K>([&](int q) { return A[q]; }, alen, [&](int q) { return B[q]; }, blen, diag);
      const int j = diag - i;
      // the VT outputs are the VT smallest of A[i, i+VT) and B[j, j+VT): all
      // loads issued together, then a half-cleaner against the reversed B
      // window (a bitonic sequence of the VT smallest) and a bitonic merge in
      // registers -- no dependent load chain (equal keys are interchangeable)
      K res[VT], bw[VT];
#pragma unroll
      for (int k = 0; k < VT; k++) {
        res[k] = i + k < alen ? A[i + k] : KeyTraits<K>::max_key();
        bw[k] = j + k < blen ? B[j + k] : KeyTraits<K>::max_key();
      }
#pragma unroll
      for (int k = 0; k < VT; k++) res[k] = min(res[k], bw[VT - 1 - k]);
#pragma unroll
      for (int h = VT / 2; h > 0; h >>= 1) {
#pragma unroll
        for (int k = 0; k < VT; k++) {
          if ((k & h) == 0) {
            const K x = res[k], y = res[k | h];
            res[k] = min(x, y);
            res[k | h] = max(x, y);
          }
        }
      }
      if (last) {
#pragma unroll
        for (int k = 0; k < VT; k++)
          if (o + k < L) dst[o + k] = res[k];
      } else {
        BlockSort<K, false, 32, VT>::store_vec(out + o, res);
      }
    }
    __syncthreads();
    K* t = src;
    src = out;
    out = t;
  }
  mark(2);
}

static_assert(offsetof(ResSmem<int32_t>, u) % 16 == 0 && offsetof(ResSmem<int64_t>, u) % 16 == 0,
              "vectorised sort buffers need 16-byte alignment");

template <typename K>
__global__ void __launch_bounds__(kResNT, kResCtasPerSM) k_resident(ResArgs<K> a) {
  namespace cg = cooperative_groups;
  using SM = ResSmem<K>;
  constexpr int NT = kResNT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int P = gridDim.x, c = blockIdx.x;
  const int64_t n = a.n;
  const int nbins = 2 * a.B1 + 1;
  auto add = [](uint32_t x, uint32_t y) { return x + y; };

  // ================= A: H1 tile scan; level-1 sample ranked by every CTA =================
  if (a.tstamp && c == 0 && tid == 0) a.tstamp[0] = res_now();
  // level-1 sample: two halves of S1/2, each gathered and sorted by one of the
  // last two CTAs (they scan the fewest tiles); every CTA later picks the
  // splitters from the two sorted halves by merge-path selection
  const int S1 = a.S1, H1 = S1 / 2;
  constexpr int B1MAX = SM::B1MAX;
  constexpr int SG = SM::S1MAX / 2 / NT;
  const int half1 = P - 1 - c;
  const bool sampler = half1 < 2;
  K sx[SG];
  if (sampler) {  // gathers issued first, so they overlap the scan
    const int log2S = __ffs(S1) - 1;
#pragma unroll
    for (int r = 0; r < SG; r++) {
      const int q = r * NT + tid;
      sx[r] = q < H1 ? a.keys[sample_position(0, n, S1, (int64_t)half1 * H1 + q, log2S)] : K(0);
    }
  }
  constexpr int UA = 16;  // keys per thread per load round
  for (int t = c; t < a.G; t += P) {
    const int64_t t0 = (int64_t)t * a.tile;
    const int64_t t1 = t0 + a.tile < n ? t0 + a.tile : n;
    int cd = 0, ca = 0, cv = 0;
    int fd = INT32_MAX, ld = -1, fa = INT32_MAX, la = -1;
    for (int64_t base = t0; base < t1; base += NT * UA) {
      K x[UA], nx[UA];
#pragma unroll
      for (int u = 0; u < UA; u++) {
        const int64_t i = base + u * NT + tid;
        x[u] = i < n ? a.keys[i] : K(0);
        nx[u] = (lane == 31 && i + 1 < n) ? a.keys[i + 1] : K(0);  // next warp's first key
      }
#pragma unroll
      for (int u = 0; u < UA; u++) {
        const int64_t i = base + u * NT + tid;
        K y = __shfl_down_sync(0xffffffffu, x[u], 1);
        const K pv = __shfl_up_sync(0xffffffffu, x[u], 1), n2 = __shfl_down_sync(0xffffffffu, x[u], 2);
        if (lane == 31) y = nx[u];
        if (i < t1 && i + 1 < n) {
          if (y < x[u]) {
            cd++; fd = min(fd, (int)i); ld = max(ld, (int)i);
            cv += straddle_violation<K>(a.keys, n, i, lane, pv, n2);
          }
          if (x[u] < y) { ca++; fa = min(fa, (int)i); la = max(la, (int)i); }  // keys only: non-increasing runs
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {  // one combined block reduction of the six tile statistics
      cd += __shfl_xor_sync(0xffffffffu, cd, o);
      ca += __shfl_xor_sync(0xffffffffu, ca, o);
      fd = min(fd, __shfl_xor_sync(0xffffffffu, fd, o));
      ld = max(ld, __shfl_xor_sync(0xffffffffu, ld, o));
      fa = min(fa, __shfl_xor_sync(0xffffffffu, fa, o));
      la = max(la, __shfl_xor_sync(0xffffffffu, la, o));
      cv += __shfl_xor_sync(0xffffffffu, cv, o);
    }
    if (lane == 0) {
      sm.agg[w][0] = cd; sm.agg[w][1] = ca; sm.agg[w][2] = fd; sm.agg[w][3] = ld; sm.agg[w][4] = fa; sm.agg[w][5] = la;
      sm.agg[w][6] = cv;
    }
    __syncthreads();
    if (tid == 0) {
      for (int v = 1; v < kResWarps; v++) {
        cd += sm.agg[v][0]; ca += sm.agg[v][1];
        fd = min(fd, sm.agg[v][2]); ld = max(ld, sm.agg[v][3]); fa = min(fa, sm.agg[v][4]); la = max(la, sm.agg[v][5]);
        cv += sm.agg[v][6];
      }
      TileSummary ts;
      ts.ndesc = cd; ts.nab = ca; ts.fdesc = fd; ts.ldesc = ld; ts.fab = fa; ts.lab = la; ts.nviol = cv; ts.pad1 = 0;
      a.sums[t] = ts;
    }
    __syncthreads();
  }
  SR_RES_STAMP(0);
  if (sampler) {
#pragma unroll
    for (int r = 0; r < SG; r++) {
      const int q = r * NT + tid;
      if (q < H1) sm.u.samp1[q] = sx[r];
    }
    __syncthreads();
    BitonicSort<K, NT, SM::S1MAX / 2 / NT>::sort(sm.u.samp1, H1);
    for (int q = tid; q < H1; q += NT) a.samp[(int64_t)half1 * H1 + q] = sm.u.samp1[q];
  }
  SR_RES_STAMP(1);
  grid.sync();

  // ================= C: route (every CTA); splitters; tile-local bucket grouping =================
  if (a.tstamp && c == 0 && tid == 0) a.tstamp[1] = res_now();
  int64_t route;
  if (c == 0)
    route = presort_resolve_block<K, NT, true>(a.keys, n, a.sums, a.G, a.lmin, a.asc, a.desc, a.st, a.force,
                                                a.merge_ok);
  else
    route = presort_resolve_block<K, NT, false>(a.keys, n, a.sums, a.G, a.lmin, a.asc, a.desc, a.st, a.force,
                                                 a.merge_ok);
  SR_RES_STAMP(2);
  if (route == kRouteSorted) return;
  if (route == kRouteReversed) {
    const int64_t half = n / 2;
    for (int64_t p = (int64_t)c * NT + tid; p < half; p += (int64_t)P * NT) {
      const K x = a.keys[p], y = a.keys[n - 1 - p];
      a.keys[p] = y;
      a.keys[n - 1 - p] = x;
    }
    return;
  }
  if (route != kRoutePartition) return;  // MERGE / undecided: the host planner continues
  const int m1 = a.B1 - 1;
  const int depth1 = tree_depth(m1);
  {  // splitter j = element 8(j+1) of the merged halves (R9), with its gamma flag
    K* hs = sm.u.samp1;  // [0, H1) half 0, [H1, S1) half 1
    {
      constexpr int SI = SM::S1MAX / NT;
      K v[SI];
#pragma unroll
      for (int r = 0; r < SI; r++) v[r] = r * NT + tid < S1 ? __ldcg(a.samp + r * NT + tid) : K(0);
#pragma unroll
      for (int r = 0; r < SI; r++)
        if (r * NT + tid < S1) hs[r * NT + tid] = v[r];
    }
    __syncthreads();
    const K* A0 = hs;
    const K* A1 = hs + H1;
    for (int j = tid; j < B1MAX; j += NT) {
      K t = KeyTraits<K>::max_key();
      uint8_t f = 0;
      if (j < m1) {
        const int r = (j + 1) * kResO1;
        const int d0 = r - 2 > 0 ? r - 2 : 0;
        int i0 = merge_path_search<K>([&](int i) { return A0[i]; }, H1, [&](int i) { return A1[i]; }, H1, d0);
        int i1 = d0 - i0;
        K win[5];  // merged elements d0 .. d0+4 (A0 wins ties)
#pragma unroll
        for (int q = 0; q < 5; q++) {
          const bool take0 = i1 >= H1 || (i0 < H1 && !(A1[i1] < A0[i0]));
          win[q] = (i0 >= H1 && i1 >= H1) ? KeyTraits<K>::max_key() : (take0 ? A0[i0] : A1[i1]);
          i0 += take0;
          i1 += !take0;
        }
        const int k = r - d0;
        t = win[k];
        const bool m1e = k >= 1 && win[k - 1] == t, m2e = k >= 2 && win[k - 2] == t;
        const bool p1e = r + 1 < S1 && win[k + 1] == t, p2e = r + 2 < S1 && win[k + 2] == t;
        f = ((m1e && m2e) || (m1e && p1e) || (p1e && p2e)) ? 1 : 0;  // count > gamma = 2
      }
      sm.tree1[B1MAX + j] = t;
      sm.eq1[j] = f;
    }
  }
  __syncthreads();
  res_build_tree<K, B1MAX>(depth1, sm.tree1);
  __syncthreads();
  SR_RES_STAMP(3);
  {
    typename SM::CT& ct = sm.u.ct;
    constexpr int U = kResGrp / NT;
    for (int t = c; t < a.NG; t += P) {
      const int64_t t0 = (int64_t)t * kResGrp;
      const int64_t t1 = t0 + kResGrp < n ? t0 + kResGrp : n;
      for (int b = tid; b < nbins; b += NT) ct.cnt[b] = 0;
      K x[U];
      int bin[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t i = t0 + u * NT + tid;
        x[u] = i < t1 ? a.keys[i] : K(0);
      }
      res_classify<K, B1MAX, U>(x, bin, sm.tree1, sm.eq1, m1, depth1);
      __syncthreads();
      uint32_t rk[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t i = t0 + u * NT + tid;
        const bool valid = i < t1;
        rk[u] = 0;
        if (__any_sync(0xffffffffu, valid && (bin[u] & 1))) {
          // equality ids: warp-aggregated increments, ranks from the peer mask
          const unsigned peers = __match_any_sync(0xffffffffu, valid ? bin[u] : -1);
          const int leader = __ffs(peers) - 1;
          uint32_t base = 0;
          if (valid && lane == leader) base = atomicAdd(&ct.cnt[bin[u]], (uint32_t)__popc(peers));
          base = __shfl_sync(0xffffffffu, base, leader);
          rk[u] = base + __popc(peers & lanemask_lt());
        } else if (valid) {
          rk[u] = atomicAdd(&ct.cnt[bin[u]], 1u);
        }
        if (!valid) bin[u] = -1;
      }
      __syncthreads();
      for (int b = tid; b < nbins; b += NT) ct.lst[b] = ct.cnt[b];
      __syncthreads();
      smem_scan<NT>(ct.lst, nbins, 0u, add, true, false, reinterpret_cast<uint32_t*>(sm.red));
#pragma unroll
      for (int u = 0; u < U; u++)
        if (bin[u] >= 0) ct.stk[ct.lst[bin[u]] + rk[u]] = x[u];
      for (int b = tid; b < nbins; b += NT) {  // this tile's bucket table + the global totals
        const uint32_t cb = ct.cnt[b];
        a.mcnt[(size_t)t * nbins + b] = cb;
        a.mlst[(size_t)t * nbins + b] = ct.lst[b];
        if (cb) atomicAdd(&a.tot[b], cb);
      }
      __syncthreads();
      for (int i = tid; i < (int)(t1 - t0); i += NT) a.ws[t0 + i] = ct.stk[i];  // contiguous, coalesced
      __syncthreads();
    }
  }
  SR_RES_STAMP(4);
  grid.sync();

  // ================= E: bucket starts; fills and per-CTA bucket sorts =================
  if (a.tstamp && c == 0 && tid == 0) a.tstamp[2] = res_now();
  uint32_t* start = sm.start;
  {
    constexpr int BI = (SM::NB1 + NT - 1) / NT;
    uint32_t v[BI];
#pragma unroll
    for (int r = 0; r < BI; r++) v[r] = r * NT + tid < nbins ? __ldcg(a.tot + r * NT + tid) : 0u;
#pragma unroll
    for (int r = 0; r < BI; r++)
      if (r * NT + tid < nbins) start[r * NT + tid] = v[r];
  }
  __syncthreads();
  smem_scan<NT>(start, nbins, 0u, add, true, false, reinterpret_cast<uint32_t*>(sm.red));
  if (tid == 0) start[nbins] = (uint32_t)n;
  __syncthreads();
  for (int b = tid; b < nbins; b += NT) {
    const uint32_t cnt = start[b + 1] - start[b];
    sm.upre[b] = (b & 1) ? (cnt + kResFill - 1) / kResFill : (cnt > 0 ? 1u : 0u);
  }
  if (tid == 0) sm.upre[nbins] = 0;
  __syncthreads();
  smem_scan<NT>(sm.upre, nbins + 1, 0u, add, true, false, reinterpret_cast<uint32_t*>(sm.red));
  if (c == 0) {  // statistics
    long long noneq = 0, eqk = 0;
    for (int b = tid; b < nbins; b += NT) {
      const uint32_t cnt = start[b + 1] - start[b];
      if (b & 1) eqk += cnt; else noneq += cnt;
    }
    noneq = block_reduce_sum<NT>(noneq, reinterpret_cast<long long*>(sm.red64));
    eqk = block_reduce_sum<NT>(eqk, reinterpret_cast<long long*>(sm.red64));
    if (tid == 0) {
      a.st->noneq_total = noneq;
      a.st->eq_keys = eqk;
      a.st->n_items = sm.upre[nbins];
    }
  }
  SR_RES_STAMP(5);
  const uint32_t UE = sm.upre[nbins];
  __shared__ uint32_t s_unit;
  for (;;) {  // units handed out dynamically (bucket sizes vary)
    if (tid == 0) s_unit = atomicAdd(a.unit_counter, 1u);
    __syncthreads();
    const uint32_t u = s_unit;
    __syncthreads();
    if (u >= UE) break;
    int lo = 0, hi = nbins - 1;  // last bin with upre <= u
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (sm.upre[mid] <= u) lo = mid; else hi = mid - 1;
    }
    const int b = lo;
    const int s = (int)start[b], len = (int)(start[b + 1] - start[b]);
    if (b & 1) {  // equality bucket: fill
      const K key = sm.tree1[B1MAX + (b - 1) / 2];
      const int f0 = (int)(u - sm.upre[b]) * kResFill;
      const int f1 = f0 + kResFill < len ? f0 + kResFill : len;
      for (int i = f0 + tid; i < f1; i += NT) a.keys[s + i] = key;
      continue;
    }
    // gather the bucket's per-tile pieces (tile t: ws[t*T + mlst[t][b], + mcnt[t][b])):
    // piece metadata in shared memory, then each warp copies every 16th piece
    // with all of its lanes' loads issued before the stores
    typename SM::E& e = sm.u.e;
    const unsigned long long tg0 = (a.tstamp && c == 0 && tid == 0) ? res_now() : 0;
    const bool fits = len <= a.capb;
    for (int t = tid; t < a.NG; t += NT) {
      e.piece[t] = __ldcg(a.mcnt + (size_t)t * nbins + b);
      e.pbase[t] = (uint32_t)t * (uint32_t)kResGrp + __ldcg(a.mlst + (size_t)t * nbins + b);
    }
    if (tid == 0) e.piece[a.NG] = 0;
    __syncthreads();
    smem_scan<NT>(e.piece, a.NG + 1, 0u, add, true, false, reinterpret_cast<uint32_t*>(sm.red));
    K* gdst = fits ? e.x : a.keys + s;  // too large for one CTA: gathered unsorted into its final range
    {
      constexpr int PB = 8;  // pieces per warp in flight
      for (int t0 = w; t0 < a.NG; t0 += kResWarps * PB) {
        K v[PB];
        int dpos[PB];
#pragma unroll
        for (int k = 0; k < PB; k++) {
          const int t = t0 + k * kResWarps;
          dpos[k] = -1;
          if (t < a.NG) {
            const int po = (int)e.piece[t], pl = (int)(e.piece[t + 1] - e.piece[t]);
            if (lane < pl) {
              v[k] = __ldcg(a.ws + e.pbase[t] + lane);
              dpos[k] = po + lane;
            }
          }
        }
#pragma unroll
        for (int k = 0; k < PB; k++)
          if (dpos[k] >= 0) gdst[dpos[k]] = v[k];
      }
      for (int t = w; t < a.NG; t += kResWarps) {  // pieces longer than a warp (presorted inputs)
        const int po = (int)e.piece[t], pl = (int)(e.piece[t + 1] - e.piece[t]);
        for (int i0 = 32; i0 < pl; i0 += 32 * PB) {
          K v[PB];
#pragma unroll
          for (int k = 0; k < PB; k++) {
            const int i = i0 + k * 32 + lane;
            v[k] = i < pl ? __ldcg(a.ws + e.pbase[t] + i) : K(0);
          }
#pragma unroll
          for (int k = 0; k < PB; k++) {
            const int i = i0 + k * 32 + lane;
            if (i < pl) gdst[po + i] = v[k];
          }
        }
      }
    }
    __syncthreads();
    if (!fits) {
      if (tid == 0) {
        const unsigned long long k = atomicAdd((unsigned long long*)&a.st->n_ovf, 1ull);
        OvfSeg o;
        o.start = s;
        o.len = len;
        a.ovf[k] = o;
        atomicAdd((unsigned long long*)&a.st->ovf_keys, (unsigned long long)len);
      }
      continue;
    }
    unsigned long long* prof = (a.tstamp && c == 0) ? a.tstamp + 8 + 8 * (size_t)P : nullptr;
    if (prof && tid == 0) { prof[5] += res_now() - tg0; prof[7] += 1; }
    res_bucket_sort<K, NT>(a.keys + s, len, e, prof);
    __syncthreads();
  }
  if (a.tstamp && c == 0 && tid == 0) a.tstamp[3] = res_now();
  SR_RES_STAMP(6);
}

}  // namespace sr
