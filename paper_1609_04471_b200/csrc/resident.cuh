// resident.cuh -- the resident path: the whole keys-only sort of an L2-resident
// array (kCap < n <= (GPC * 148 - 4) * kResGrp) as ONE cooperative launch of
// one CTA per SM.
//
// The multi-kernel path (presort.cuh, partition.cuh) pays a launch plus a
// drain per step and a one-CTA bookkeeping kernel per level; at the paper's
// Table 1 size (n = 2,000,000) a full pass over the keys is
// ~1.2 us of HBM time, so those fixed costs dominated.  Here the steps run as
// four phases of one persistent kernel separated by three grid-wide barriers,
// and the quicksort recursion (Appendix B) is a global
// splitter partition into <= 2048 buckets followed by per-warp (or, for big
// buckets, per-CTA) sorts of the buckets.
//   A  H1 scan of every tile (vectorised, presort.cuh scan_range_vec); CTA 0
//      zeroes the control block.  The last four CTAs (no tile) gather and
//      sort one quarter each of the level-1 sample (S1 = O1 B1 jittered
//      positions, R8), merge the quarters pairwise, select the
//      splitters (R14) and build the guide table (sampler 0) -- speculatively,
//      before the route is known, so the splitters are ready when it is.
//   -- grid sync --
//   C  warp 0 resolves the tile summaries into the device route (K2's logic;
//      CTA 0 also writes the statistics and run lists).  SORTED exits;
//      REVERSED reverses in place; MERGE / undecided
//      return to the host planner.  PARTITION: splitter j = element O1 (j+1)
//      of the merged halves (merge-path selection, R14) with its gamma flag
//      (count > gamma = 2 in the sample) -> guide table; each
//      held tile is classified (3-way ids) and its range
//      keys counting-sorted by bucket in shared memory (equality keys are only
//      counted); its piece offset inside every bucket comes from one atomicAdd
//      on the bucket total.
//   -- grid sync --
//   D  bucket starts (exclusive scan of the totals, every CTA); every held
//      key goes to start[b] + offset + rank in the workspace, so each bucket
//      is contiguous; equality keys are not written.
//   -- grid sync --
//   E  CTA units: range buckets above WCAP, one CTA each (unit_sort.cuh: an
//      in-shared-memory 3-way sample partition into 32 sub-buckets that the
//      warps sort, R17); then warp units, largest first: range buckets <=
//      WCAP sorted by one warp's register bitonic network, two networks and a
//      merge above half of WCAP (R15), and equality fills ("spared from the
//      recursive calls").  Every bucket is checked with
//      is_sorted first.  Buckets beyond the in-kernel cap are
//      copied unsorted into their final range and listed for the host, which
//      runs further partition levels on them.
//   CTA 0 publishes the outcome to a host-mapped record as soon as it is known
//   (after the route step, or on the partition route once the bucket sizes are
//   known at the start of D), so the host call returns while the kernel runs.
#pragma once
#include <cooperative_groups.h>
#include <cstddef>

#include "bitonic.cuh"
#include "common.cuh"
#include "guide.cuh"
#include "outlier.cuh"
#include "partition.cuh"
#include "presort.cuh"
#include "types.cuh"
#include "unit_sort.cuh"

namespace sr {

constexpr int kResNT = 512;
constexpr int kResCtasPerSM = 1;
constexpr int kResWarps = kResNT / 32;
constexpr int kResGrp = 8192;           // largest tile: H1 scan unit and phase C grouping unit (one
                                        // tile-local counting sort); the host picks the tile so that
                                        // every CTA gets <= GPC tiles and the samplers one
constexpr int kResWarpFill = 4096;      // equality fill per warp unit
constexpr int kResSamplers = 4;         // CTAs that sort one quarter of the level-1 sample each
constexpr int kResMaxG = 512;           // tiles (G <= GPC * gridDim.x - kResSamplers)

template <typename K> struct ResCfg;
template <> struct ResCfg<int32_t> {
  static constexpr int CAPB = 16384;    // largest level-1 bucket sorted by one CTA
  static constexpr int B1MAX = 2048;    // level-1 buckets
  static constexpr int O1 = 4;          // level-1 oversampling (S1 = O1 B1 <= 8192: four 2048-key sampler sorts)
  static constexpr int GPC = 2;         // grouping units held per CTA across the scatter barrier
  static constexpr int WCAP = 2048;     // level-1 buckets up to this size are sorted by one warp
  static constexpr int TARGET = 1024;   // mean level-1 bucket the host aims for
  static constexpr int64_t MAXN = int64_t(4) << 20;
};
template <> struct ResCfg<int64_t> {
  static constexpr int CAPB = 8192;
  static constexpr int B1MAX = 1024;
  static constexpr int O1 = 8;
  static constexpr int GPC = 2;
  static constexpr int WCAP = 1024;
  static constexpr int TARGET = 4096;
  static constexpr int64_t MAXN = int64_t(4) << 20;
};
constexpr int64_t kResMaxN = ResCfg<int32_t>::MAXN;  // largest resident n over the key types

// In-kernel outlier route (nearly sorted inputs, k-exchange PAPER.md:85; the
// multi-kernel rounds of outlier.cuh in one launch):
//   OA  tiles of TO keys: the endpoints of every descent are outliers (then,
//       inside the tile, until the kept keys are sorted); kept keys in order
//       then the outliers are written to ws[t0, t1)
//   --  kept keys R (the tiles' kept prefixes, in order) must be sorted across
//       tiles: a boundary out of order loses both endpoints until it is in
//       order; splitter j = R[(j+1) OL - 1]; every outlier goes to bucket
//       #{splitters < x} (at most OCAP per bucket)
//   OD  bucket j = R[j OL, (j+1) OL) merged with its sorted outliers in one
//       warp's shared staging area, then copied to keys[j OL + outliers of the
//       buckets before j, ...) (R wins ties).  A tile boundary out of order or a full bucket leaves the
//       keys untouched and hands the sort to the host's outlier route.
template <typename K>
struct ResOut {
  static constexpr int TO = sizeof(K) == 4 ? 8192 : 4096;  // OA tile
  static constexpr int OL = ResCfg<K>::WCAP * 3 / 8;       // kept keys per bucket
  static constexpr int OCAP = ResCfg<K>::WCAP / 8;         // outliers per bucket (one warp network)
  static_assert(OL + OCAP + OL + OCAP <= ResCfg<K>::WCAP, "R, O and the merged bucket fit one warp's staging");
  static constexpr int OBMAX = 2 * ResCfg<K>::B1MAX;       // buckets (their starts live in ResSmem::start)
  static constexpr int MAXG = (int)(ResCfg<K>::MAXN / TO);
  static constexpr int64_t MAXN = (int64_t)OL * OBMAX;     // n this route accepts
};

struct ResDone;

template <typename K>
struct ResArgs {
  K* keys;
  K* ws;
  int64_t n;
  int tile, G;              // presort tiles (K1's tiling)
  TileSummary* sums;
  TileMM* mm;               // per tile: the k-distance test (presort.cuh tile_mm_finish)
  RunDesc* asc;
  RunDesc* desc;
  DevStats* st;             // route, statistics; n_ovf counts the host list
  int S1, B1;               // level-1 sample size, buckets (power of two <= B1MAX)
  int NG;                   // grouping units = the scan tiles (NG = G)
  K* samp;                  // S1 keys: the sorted pieces of the level-1 sample
  K* mrg;                   // S1 keys: the sample pieces merged pairwise (each sampler writes half a merge)
  K* spl;                   // B1MAX level-1 splitters (+inf padded), written by the samplers
  uint8_t* spf;             // B1MAX equality flags of the splitters
  uint32_t* tot;            // 2 B1 + 1 bucket totals (zeroed in phase A)
  uint32_t* goff;           // NG x nbins: offset of group t's piece inside bucket b
  OvfSeg* ovf;              // ranges of keys left unsorted for the host's next level
  int64_t lmin;
  int force, merge_ok;
  int capb;                 // largest level-1 bucket sorted in-kernel (CAPB; lowered by tests)
  unsigned long long* tstamp;  // optional: %globaltimer, [0..8) CTA 0 phase starts, then 8 per CTA
  uint32_t* unit_counter;   // [0] CTA units, [2] warp units, [3] sampler steps (zeroed by CTA 0 in phase A)
  uint32_t* pairc;          // B1MAX: halves done per class-A warp unit (zeroed with the control block)
  uint32_t* arrive;         // persistent arrival counter of the route step (never reset)
  uint32_t arrive_base;     // its value before this launch (every launch adds gridDim.x + 1)
  uint32_t* scount;         // persistent sampler-step counter (never reset; every launch adds 3 kResSamplers)
  uint32_t scount_base;     // its value before this launch
  GuideTab<K, 2048, ResCfg<K>::B1MAX>* guide;  // level-1 classification table (built by sampler 0)
  int ctrl_words;           // 32-bit words of the control block st | unit_counter | tot (zeroed in phase A)
  ResDone* done;            // host-mapped completion record (CTA 0 writes it once the outcome is known)
  uint32_t seq;             // this call's completion sequence number
  // in-kernel outlier route (ResOut): out_res = 1 when this launch runs it
  int out_res, GO;          // GO tiles of ResOut::TO keys
  uint32_t* okc;            // GO: kept keys per tile
  K* ofl;                   // 2 GO: first / last kept key per tile
  uint32_t* ocnt;           // OBMAX bucket counts, [OBMAX] unsorted tile, [OBMAX + 1] full bucket (control block)
  K* obuf;                  // buckets x OCAP: the outliers of each bucket
};

// Host-mapped completion record: the statistics the planner needs and whether
// the launch finishes the sort by itself, then the sequence number.  CTA 0
// writes it ONCE, as soon as the route (and, on the partition route, every
// bucket size) is known -- long before the kernel ends -- so the host returns
// from the call while the kernel is still running (the result is valid when
// the stream reaches the end of the kernel).  The host spins on `seq` instead
// of a device->host copy + stream synchronisation (tools/micro/api.cu).
struct ResDone {
  DevStats st;
  int32_t in_kernel;        // 1: nothing left for the host; 0: the host continues after the kernel
  volatile uint32_t seq;
  uint32_t pad[30];
};
// phase C sub-steps of CTA 0's first group (SR_TIMING diagnostics)
#define SR_RES_SUB(kk)                                                                              \
  do {                                                                                              \
    if (a.tstamp && c == 0 && k == 0 && tid == 0) a.tstamp[8 + 8 * (size_t)gridDim.x + 8 + (kk)] = res_now(); \
  } while (0)

// splitter sub-steps of sampler 0, the last CTA (SR_TIMING diagnostics)
#define SR_RES_CSUB(kk)                                                                             \
  do {                                                                                              \
    if (a.tstamp && c == (int)gridDim.x - 1 && tid == 0) a.tstamp[8 + 8 * (size_t)gridDim.x + 16 + (kk)] = res_now(); \
  } while (0)

#define SR_RES_STAMP(k)                                                                \
  do {                                                                                 \
    if (a.tstamp && tid == 0) a.tstamp[8 + (size_t)blockIdx.x * 8 + (k)] = res_now(); \
  } while (0)

__device__ __forceinline__ unsigned long long res_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Publish the early completion record (one thread of CTA 0, after this CTA
// wrote the statistics in a.st).
template <typename K>
__device__ __forceinline__ void res_publish(const ResArgs<K>& a, int in_kernel) {
  if (!a.done) return;
  __threadfence();
  const unsigned long long* s = reinterpret_cast<const unsigned long long*>(a.st);
  unsigned long long* d = reinterpret_cast<unsigned long long*>(&a.done->st);
  for (int i = 0; i < (int)(sizeof(DevStats) / 8); i++) d[i] = __ldcg(s + i);
  a.done->in_kernel = in_kernel;
  __threadfence_system();
  a.done->seq = a.seq;
}

// The same by a whole warp (all 32 lanes call): the statistics words are copied
// in parallel (one L2 round trip instead of one per word by a single thread).
template <typename K>
__device__ __forceinline__ void res_publish_warp(const ResArgs<K>& a, int in_kernel) {
  if (!a.done) return;
  const int lane = threadIdx.x & 31;
  __threadfence();  // (the lane that wrote a.st)
  __syncwarp();
  const unsigned long long* s = reinterpret_cast<const unsigned long long*>(a.st);
  unsigned long long* d = reinterpret_cast<unsigned long long*>(&a.done->st);
  for (int i = lane; i < (int)(sizeof(DevStats) / 8); i += 32) d[i] = __ldcg(s + i);
  if (lane == 0) a.done->in_kernel = in_kernel;
  __threadfence_system();
  __syncwarp();
  if (lane == 0) a.done->seq = a.seq;
}

// Shared memory: the persistent bucket table + phase-local buffers in a union.
template <typename K>
struct ResSmem {
  static constexpr int CAPB = ResCfg<K>::CAPB;
  static constexpr int B1MAX = ResCfg<K>::B1MAX;
  static constexpr int NB1 = 2 * B1MAX + 1;
  static constexpr int S1MAX = ResCfg<K>::O1 * B1MAX;
  static constexpr int WCAP = ResCfg<K>::WCAP;
  static constexpr int GPC = ResCfg<K>::GPC;
  static_assert(ResOut<K>::OBMAX <= NB1, "outlier bucket starts live in start[]");
  struct alignas(16) CT {          // C: tile-local counting sorts of this CTA's groups
    uint32_t cnt[NB1];             // current group's bucket counts; in D its piece offsets (goff)
    uint32_t lst[GPC][NB1 + 1];    // per held group: bucket starts inside stk, lst[nbins] = group length
    K stk[GPC][kResGrp];           // per held group: its keys grouped by bucket
    uint16_t stb[GPC][kResGrp];    // per held group: the bucket of stk[i]
  };
  struct alignas(16) SP {          // route step: tile summaries; samplers: sample pieces, merged halves
    K q[S1MAX];
    TileSummary ts[kResMaxG];
  };
  using E = UnitSmem<K, CAPB, kResNT>;  // E: the CTA units (unit_sort.cuh); warp-unit staging spans x and y
  static_assert(kResWarps * WCAP <= 2 * CAPB, "warp-unit staging areas live in x and y");
  uint32_t start[NB1 + 1];         // level-1 bucket starts, start[nbins] = n
  struct EU {                      // E: unit lists
    uint16_t upa[NB1 + 1];         // exclusive prefix of E warp units, class A (WCAP/2 < range bucket <= WCAP)
    uint16_t upb[NB1 + 1];         // exclusive prefix of E warp units, class B (smaller range buckets, fills)
    uint16_t cbin[B1MAX + 8];      // E CTA units: range buckets above WCAP
  };
  union alignas(16) {
    GuideTab<K, 2048, B1MAX> guide1;  // C: level-1 classification table (guide.cuh)
    EU eu;                         // E
    struct {                       // outlier route: per tile, kept keys [ks, ke) and their offset in R
      uint32_t koff[ResOut<K>::MAXG + 1];
      uint16_t ks[ResOut<K>::MAXG], ke[ResOut<K>::MAXG];
    } ot;
  } v;
  union alignas(16) {
    K samp1[S1MAX];                // A: the sampler's piece of the sample + BitonicSort scratch
    SP sp;
    CT ct;
    E e;  // (UnitSmem: aligned x / y buffers)
    OutSmem<K, kResNT, ResOut<K>::TO> ot;  // outlier route OA
    K ospl[ResOut<K>::OBMAX];      // outlier route: bucket splitters
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

static_assert(sizeof(ResSmem<int32_t>) <= 227 * 1024 && sizeof(ResSmem<int64_t>) <= 227 * 1024,
              "one CTA per SM: the shared-memory layout must fit the 227 KB opt-in limit");
static_assert(offsetof(ResSmem<int32_t>, u) % 16 == 0 && offsetof(ResSmem<int64_t>, u) % 16 == 0,
              "vectorised sort buffers need 16-byte alignment");

// Block sort of x[0, L) (L a power of two, 128 <= L <= 4 NT; x and y hold L
// keys each): every warp sorts 128-key chunks with its register network, then
// log2(L / 128) merge-path rounds (4 outputs per thread, one barrier each)
// ping-pong between x and y.  Returns the buffer holding the sorted keys.
// (Used for the samplers' quarters: the block bitonic network with a barrier
// per cross-warp stage took 5.5 us for 2048 keys.)
template <typename K, int NT>
__device__ __forceinline__ K* res_block_sort(K* x, K* y, int L) {
  const int tid = threadIdx.x, w = tid >> 5;
  for (int c0 = w * 128; c0 < L; c0 += NT * 4) WarpBitonic<K, 4>::sort(x + c0, 128);
  __syncthreads();
  K* src = x;
  K* dst = y;
  for (int W = 128; W < L; W *= 2) {
    for (int o0 = tid * 4; o0 < L; o0 += NT * 4) {
      const int p0 = (o0 / (2 * W)) * (2 * W);
      const K* A = src + p0;
      const K* B = A + W;
      const int diag = o0 - p0;
      int i = merge_path_search<K>([&](int q) { return A[q]; }, W, [&](int q) { return B[q]; }, W, diag);
      int j = diag - i;
#pragma unroll
      for (int d = 0; d < 4; d++) {
        const bool tA = j >= W || (i < W && !(B[j] < A[i]));
        dst[o0 + d] = tA ? A[i] : B[j];
        i += tA;
        j += !tA;
      }
    }
    __syncthreads();
    K* t = src;
    src = dst;
    dst = t;
  }
  return src;
}

// outlier-route sub-steps of CTA 0 (SR_TIMING diagnostics)
#define SR_RES_OSUB(kk)                                                                             \
  do {                                                                                              \
    if (a.tstamp && c == 0 && tid == 0) a.tstamp[8 + 8 * (size_t)gridDim.x + 40 + (kk)] = res_now(); \
  } while (0)

// Coalesced copy of cnt keys from global (L2) to a warp's shared staging area.
template <typename K>
__device__ __forceinline__ void res_warp_copy(K* __restrict__ dst, const K* __restrict__ src, int cnt) {
  const int lane = threadIdx.x & 31;
  constexpr int UL = 16;
  for (int i0 = 0; i0 < cnt; i0 += 32 * UL) {
    K v[UL];
#pragma unroll
    for (int u = 0; u < UL; u++) {
      const int i = i0 + u * 32 + lane;
      v[u] = i < cnt ? __ldcg(src + i) : K(0);
    }
#pragma unroll
    for (int u = 0; u < UL; u++) {
      const int i = i0 + u * 32 + lane;
      if (i < cnt) dst[i] = v[u];
    }
  }
}

// ks[0, len) (len <= 64) sorted in place by one warp: each lane ranks its
// (up to two) keys against all of them (ties by position) and stores them at
// their ranks.
template <typename K>
__device__ __forceinline__ void res_warp_rank_sort(K* ks, int len) {
  const int lane = threadIdx.x & 31;
  const K x0 = lane < len ? ks[lane] : K(0);
  const K x1 = lane + 32 < len ? ks[lane + 32] : K(0);
  int r0 = 0, r1 = 0;
  for (int k = 0; k < len; k++) {
    const K y = ks[k];
    r0 += (y < x0) || (y == x0 && k < lane);
    r1 += (y < x1) || (y == x1 && k < lane + 32);
  }
  __syncwarp();
  if (lane < len) ks[r0] = x0;
  if (lane + 32 < len) ks[r1] = x1;
  __syncwarp();
}

// The in-kernel outlier route (ResOut above).  Called by every CTA after the
// route step chose kRouteOutlier; CTA 0 publishes the outcome.
template <typename K, typename SM>
__device__ __forceinline__ void res_outlier(const ResArgs<K>& a, SM& sm) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  using RO = ResOut<K>;
  constexpr int NT = kResNT, TO = RO::TO, OL = RO::OL, OCAP = RO::OCAP, OBMAX = RO::OBMAX;
  constexpr int VT = TO / NT, NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int P = gridDim.x, c = blockIdx.x;
  const int64_t n = a.n;
  const int GO = a.GO;
  // ---- OA: outliers of every tile; ws[t0, t1) = kept keys in order, then the outliers
  {
    OutSmem<K, NT, TO>& os = sm.u.ot;
    const unsigned lt = (1u << lane) - 1u;
    for (int t = c; t < GO; t += P) {
      const int64_t t0 = (int64_t)t * TO;
      const int len = (int)(n - t0 < TO ? n - t0 : TO);
      unsigned bal[VT];
      if (t == c) SR_RES_OSUB(0);
      const bool sorted = out_tile_flags<K, NT, TO>(a.keys, n, t0, len, os, bal);
      if (t == c) SR_RES_OSUB(1);
      const int tot = os.gcnt[VT * NW];
#pragma unroll
      for (int u = 0; u < VT; u++) {
        const int i = u * NT + tid;
        if (i < len) {
          const int kr = os.gcnt[u * NW + w] + __popc(bal[u] & lt);  // kept before element i
          if ((bal[u] >> lane) & 1u) os.sk[kr] = os.s[1 + i];
          else os.sk[tot + (i - kr)] = os.s[1 + i];
        }
      }
      __syncthreads();
      SR_CHECK(t0 + len <= n);
      for (int i = tid; i < len; i += NT) a.ws[t0 + i] = os.sk[i];
      if (tid == 0) {
        a.okc[t] = (uint32_t)tot;
        if (tot > 0) {
          a.ofl[2 * t] = os.sk[0];
          a.ofl[2 * t + 1] = os.sk[tot - 1];
        }
        if (!sorted) atomicOr(a.ocnt + OBMAX, 1u);
      }
      __syncthreads();
      if (t == c) SR_RES_OSUB(2);
    }
  }
  if (a.tstamp && tid == 0) a.tstamp[8 + (size_t)c * 8 + 4] = res_now();
  grid.sync();
  // ---- tile boundaries, tile offsets of the kept keys R, splitters, outlier buckets
  // A boundary whose kept keys are out of order (a descent between the last
  // kept key of tile t and the first of t+1) loses both endpoints until it is
  // in order, as inside the tiles: tile t keeps ws[t0 + oks[t], t0 + oke[t]).
  // (Every CTA resolves every boundary itself, so no further grid barrier.)
  uint32_t* koff = sm.v.ot.koff;
  uint16_t* oks = sm.v.ot.ks;
  uint16_t* oke = sm.v.ot.ke;
  int bad = 0;
  if (tid == 0 && __ldcg(a.ocnt + OBMAX)) bad = 1;  // a tile's kept keys were not sorted
  for (int t = tid; t < GO; t += NT) {
    const int kc = (int)__ldcg(a.okc + t);
    if (kc == 0) bad = 1;
    if (t == 0) oks[0] = 0;
    if (t == GO - 1) oke[t] = (uint16_t)kc;
    if (t + 1 < GO && kc > 0) {
      const int kn = (int)__ldcg(a.okc + t + 1);
      const K* wt = a.ws + (int64_t)t * TO;
      const K* wu = wt + TO;
      int ia = kc - 1, ib = 0;
      K x = __ldcg(a.ofl + 2 * t + 1), y = __ldcg(a.ofl + 2 * t + 2);
      while (x > y) {
        ia--;
        ib++;
        if (ia < 0 || ib >= kn || ib > 64) { bad = 1; break; }
        x = __ldcg(wt + ia);
        y = __ldcg(wu + ib);
      }
      oke[t] = (uint16_t)(ia + 1);
      oks[t + 1] = (uint16_t)ib;
    }
  }
  bad = __syncthreads_or(bad);
  for (int t = tid; t < GO && !bad; t += NT) {
    if (oks[t] >= oke[t]) bad = 1;
    koff[t] = (uint32_t)(oke[t] - oks[t]);
  }
  if (tid == 0) koff[GO] = 0u;
  bad = __syncthreads_or(bad);
  if (!bad) smem_exclusive_sum_u32<NT>(koff, GO + 1, reinterpret_cast<uint32_t*>(sm.red));
  SR_RES_OSUB(3);
  const uint32_t r = bad ? 0u : koff[GO];
  const int nbo = (int)((r + OL - 1) / OL);
  if (__syncthreads_or(bad || r == 0 || nbo > OBMAX)) {  // not a few-outlier input: the host's rounds take over (keys untouched)
    if (c == 0 && tid == 0) res_publish(a, 0);
    return;
  }
  SR_RES_OSUB(4);
  auto tile_of = [&](uint32_t g) {  // tile holding R[g]: the last t with koff[t] <= g
    int lo = 0, hi = GO - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (koff[mid] <= g) lo = mid; else hi = mid - 1;
    }
    return lo;
  };
  K* ospl = sm.u.ospl;
  {  // (every thread's gathers issued together)
    constexpr int SPT = (RO::OBMAX + NT - 1) / NT;
    K v[SPT];
#pragma unroll
    for (int q = 0; q < SPT; q++) {
      const int j = q * NT + tid;
      if (j < nbo - 1) {
        const uint32_t g = (uint32_t)(j + 1) * OL - 1u;
        const int t = tile_of(g);
        v[q] = __ldcg(a.ws + (int64_t)t * TO + oks[t] + (g - koff[t]));
      }
    }
#pragma unroll
    for (int q = 0; q < SPT; q++)
      if (q * NT + tid < nbo - 1) ospl[q * NT + tid] = v[q];
  }
  __syncthreads();
  SR_RES_OSUB(5);
  {  // this CTA's outliers (its tiles t = c + k P hold them at ws[t0 + kept, t1)), two per thread in flight
    int total = 0;
    for (int t = c; t < GO; t += P) total += (int)(min((int64_t)TO, n - (int64_t)t * TO) - (koff[t + 1] - koff[t]));
    auto at = [&](int f) {  // flat index -> position in ws (a tile's outliers: [0, oks) and [oke, len))
      for (int t = c;; t += P) {
        const int64_t t0 = (int64_t)t * TO;
        const int ks = oks[t], ke = oke[t];
        const int oc_t = (int)(min((int64_t)TO, n - t0) - (ke - ks));
        if (f < oc_t) return t0 + (f < ks ? f : ke + (f - ks));
        f -= oc_t;
      }
    };
    for (int f0 = tid; f0 < total; f0 += 2 * NT) {
      K x[2];
      int lo[2] = {0, 0}, hi[2];
#pragma unroll
      for (int q = 0; q < 2; q++) {
        const int f = f0 + q * NT;
        x[q] = f < total ? a.ws[at(f)] : K(0);  // (written by this CTA)
        hi[q] = f < total ? nbo - 1 : 0;  // bucket = #{splitters < x}
      }
      while (lo[0] < hi[0] || lo[1] < hi[1]) {
#pragma unroll
        for (int q = 0; q < 2; q++)
          if (lo[q] < hi[q]) {
            const int mid = (lo[q] + hi[q]) >> 1;
            if (ospl[mid] < x[q]) lo[q] = mid + 1; else hi[q] = mid;
          }
      }
      uint32_t slot[2];
#pragma unroll
      for (int q = 0; q < 2; q++) slot[q] = f0 + q * NT < total ? atomicAdd(a.ocnt + lo[q], 1u) : 0u;
#pragma unroll
      for (int q = 0; q < 2; q++)
        if (f0 + q * NT < total) {
          if (slot[q] < (uint32_t)OCAP) a.obuf[(int64_t)lo[q] * OCAP + slot[q]] = x[q];
          else atomicOr(a.ocnt + OBMAX + 1, 1u);
        }
    }
  }
  __syncthreads();
  SR_RES_OSUB(6);
  if (a.tstamp && tid == 0) a.tstamp[8 + (size_t)c * 8 + 5] = res_now();
  grid.sync();
  // ---- OD: bucket starts; each bucket merged by one warp into its final range
  if (a.tstamp && c == 0 && tid == 0) a.tstamp[2] = res_now();
  if (__ldcg(a.ocnt + OBMAX + 1)) {  // a bucket overflowed: the host's rounds take over (keys untouched)
    if (c == 0 && tid == 0) res_publish(a, 0);
    return;
  }
  uint32_t* obase = sm.start;
  for (int j = tid; j < nbo; j += NT) obase[j] = __ldcg(a.ocnt + j);
  if (tid == 0) obase[nbo] = 0u;
  __syncthreads();
  smem_exclusive_sum_u32<NT>(obase, nbo + 1, reinterpret_cast<uint32_t*>(sm.red));
  if (c == 0 && tid == 0) {
    a.st->n_items = nbo;
    a.st->noneq_total = (long long)(n - r);  // (the outliers)
    res_publish(a, 1);
  }
  K* stage = sm.u.e.x + w * SM::WCAP;
  SR_RES_OSUB(7);
  for (;;) {
    uint32_t u = 0;
    if (lane == 0) u = atomicAdd(a.unit_counter + 2, 1u);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u >= (uint32_t)nbo) break;
    const int j = (int)u;
    const bool first = a.tstamp && u == 0 && lane == 0;  // SR_TIMING: the first unit's steps
    if (first) a.tstamp[8 + 8 * (size_t)P + 50] = res_now();
    const uint32_t g0 = (uint32_t)j * OL;
    const int len = (int)min((uint32_t)OL, r - g0);
    const int oc = (int)(obase[j + 1] - obase[j]);
    int t = tile_of(g0);
    for (int done = 0; done < len; t++) {  // R[g0, g0 + len) from the tiles' kept prefixes
      const uint32_t off = g0 + (uint32_t)done - koff[t];
      const int take = min((int)(koff[t + 1] - koff[t] - off), len - done);
      if (take > 0) res_warp_copy<K>(stage + done, a.ws + (int64_t)t * TO + oks[t] + off, take);
      done += take > 0 ? take : 0;
    }
    res_warp_copy<K>(stage + OL, a.obuf + (int64_t)j * OCAP, oc);
    __syncwarp();
    if (first) a.tstamp[8 + 8 * (size_t)P + 51] = res_now();
    // bucket j = R[g0, g0 + len) merged with its sorted outliers O[0, oc) (R
    // wins ties) into the staging area's last half, then copied
    // out coalesced
    SR_CHECK((int64_t)g0 + obase[j] + len + oc <= n && oc <= OCAP && len <= OL);
    K* dst = a.keys + g0 + obase[j];
    K* O = stage + OL;
    K* out = stage + OL + OCAP;
    if (oc > 1) {
      if (oc <= 64) res_warp_rank_sort<K>(O, oc);
      else unit_warp_sort<K>(O, oc);
    }
    if (first) a.tstamp[8 + 8 * (size_t)P + 52] = res_now();
    const K* src = stage;
    if (oc > 0) {
      unit_warp_merge<K>(stage, len, O, oc, out);
      src = out;
    }
    for (int i = lane; i < len + oc; i += 32) dst[i] = src[i];
    __syncwarp();
    if (first) a.tstamp[8 + 8 * (size_t)P + 53] = res_now();
  }
  if (a.tstamp && c == 0 && tid == 0) a.tstamp[3] = res_now();
  if (a.tstamp && tid == 0) a.tstamp[8 + (size_t)c * 8 + 6] = res_now();
}

// Phase C for one held group (tile [t0, t1) of src, slot k): 3-way bucket ids
// from the guide table, a counting sort of the group by bucket in shared
// memory, and the group's piece offset inside every bucket (one atomicAdd on
// the bucket total).
template <typename K, typename SM>
__device__ __noinline__ void res_group(const ResArgs<K>& a, SM& sm, const K* __restrict__ src, int64_t t0, int64_t t1,
                                       int k, int nbins, uint32_t* __restrict__ tot, uint32_t* __restrict__ goff_row) {
  constexpr int NT = kResNT;
  constexpr int U = kResGrp / NT;
  const int tid = threadIdx.x, lane = tid & 31;
  const int c = blockIdx.x;
  typename SM::CT& ct = sm.u.ct;
  SR_RES_SUB(0);
  for (int b = tid; b < nbins; b += NT) ct.cnt[b] = 0;
  K x[U];
  int bin[U];
#pragma unroll
  for (int u = 0; u < U; u++) {
    const int64_t i = t0 + u * NT + tid;
    x[u] = i < t1 ? src[i] : K(0);
  }
  guide_classify<K, U>(x, bin, sm.v.guide1);
  SR_RES_SUB(1);
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
  SR_RES_SUB(2);
  __syncthreads();
  uint32_t* lst = ct.lst[k];
  int ranged = 0;  // any range key in this group (else nothing is placed: no scan)
  {  // unrolled: all of a thread's atomics in flight together
    constexpr int BI = (SM::NB1 + NT - 1) / NT;
    uint32_t go[BI];
#pragma unroll
    for (int r = 0; r < BI; r++) {
      const int b = r * NT + tid;
      const uint32_t cb = b < nbins ? ct.cnt[b] : 0u;
      // only range keys are placed (equality keys are never moved: their
      // buckets are filled in phase E)
      if (b < nbins) lst[b] = (b & 1) ? 0u : cb;
      ranged |= !(b & 1) && cb;
      // this group's piece of bucket b starts at offset goff inside the bucket
      // (pieces of different groups in arbitrary order: the bucket is sorted later)
      go[r] = cb ? atomicAdd(&tot[b], cb) : 0u;
    }
#pragma unroll
    for (int r = 0; r < BI; r++)
      if (r * NT + tid < nbins) goff_row[r * NT + tid] = go[r];
  }
  SR_RES_SUB(3);
  if (__syncthreads_or(ranged)) {
    smem_exclusive_sum_u32<NT>(lst, nbins, reinterpret_cast<uint32_t*>(sm.red));
    if (tid == 0) lst[nbins] = lst[nbins - 1] + ct.cnt[nbins - 1];  // placed (range) keys; bin nbins-1 is a range bin
  } else if (tid == 0) {
    lst[nbins] = 0;  // every key of the group is in an equality bucket (few-unique inputs)
  }
  SR_RES_SUB(4);
#pragma unroll
  for (int u = 0; u < U; u++)
    if (bin[u] >= 0 && !(bin[u] & 1)) {
      SR_CHECK(bin[u] < nbins && lst[bin[u]] + rk[u] < (uint32_t)kResGrp);
      ct.stk[k][lst[bin[u]] + rk[u]] = x[u];
      ct.stb[k][lst[bin[u]] + rk[u]] = (uint16_t)bin[u];
    }
  __syncthreads();
  SR_RES_SUB(5);
}

template <typename K>
__global__ void __launch_bounds__(kResNT, kResCtasPerSM) k_resident(const __grid_constant__ ResArgs<K> a) {
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

  // ================= A: H1 tile scan; level-1 sample ranked by every CTA =================
  if (a.tstamp && c == 0 && tid == 0) a.tstamp[0] = res_now();
  if (c == 0) {  // control block (statistics, counters, bucket totals): first used after the grid sync
    uint32_t* z = reinterpret_cast<uint32_t*>(a.st);
    for (int i = tid; i < a.ctrl_words; i += NT) z[i] = 0u;
  }
  // level-1 sample: kResSamplers pieces, each gathered and sorted by one of the
  // last CTAs (they scan one tile); every CTA merges them pairwise into two
  // halves and picks the splitters by merge-path selection (R14)
  const int S1 = a.S1, QS = S1 / kResSamplers, H1 = S1 / 2;
  constexpr int B1MAX = SM::B1MAX;
  constexpr int SG = SM::S1MAX / kResSamplers / NT;
  const int quarter = P - 1 - c;  // this sampler's piece of the sample
  const bool sampler = quarter < kResSamplers;
  K sx[SG];
  if (sampler) {  // gathers issued first, so they overlap the scan
    const int log2S = __ffs(S1) - 1;
#pragma unroll
    for (int r = 0; r < SG; r++) {
      const int q = r * NT + tid;
      sx[r] = q < QS ? a.keys[sample_position(0, n, S1, (int64_t)quarter * QS + q, log2S)] : K(0);
    }
  }
  constexpr int UA = 16;  // keys per thread per load round
  // tiles t = c + k PS go to the CTAs c < PS = P - kResSamplers; the samplers
  // scan none, so their sample sorts start at once
  const int PS = P - kResSamplers;
  for (int t = c; c < PS && t < a.G; t += PS) {
    const int64_t t0 = (int64_t)t * a.tile;
    const int64_t t1 = t0 + a.tile < n ? t0 + a.tile : n;
    int cd = 0, ca = 0, cv = 0;
    int fd = INT32_MAX, ld = -1, fa = INT32_MAX, la = -1;
    // subtile minima / maxima for the k-distance test (scratch: the route
    // step's sample area, unused by the scanning CTAs until then)
    K* mmn = sm.u.sp.q;
    K* mmx = sm.u.sp.q + kResGrp / kDSub;
    const int nsub = (int)((t1 - t0 + kDSub - 1) / kDSub);
    const bool vec = (reinterpret_cast<uintptr_t>(a.keys) & 15) == 0 && t0 % (16 / (int)sizeof(K)) == 0;
    tile_mm_init<K>(mmn, mmx, nsub);
    __syncthreads();
    if (vec) {
      ScanAcc acc;
      scan_range_vec<K, false, NT, (sizeof(K) == 4 ? 4 : 8)>(a.keys, n, t0, t1, acc, mmn, mmx);
      cd = acc.cd; ca = acc.ca; cv = acc.cv; fd = acc.fd; ld = acc.ld; fa = acc.fa; la = acc.la;
    } else
    for (int64_t base = t0; base < t1; base += NT * UA) {
      K x[UA], h1[UA], h2[UA];
#pragma unroll
      for (int u = 0; u < UA; u++) {
        const int64_t i = base + u * NT + tid;
        x[u] = i < n ? a.keys[i] : K(0);
        load_halo<K>(a.keys, n, i, lane, h1[u], h2[u]);
      }
#pragma unroll
      for (int u = 0; u < UA; u++) {
        const int64_t i = base + u * NT + tid;
        K y, pv, n2;
        warp_neighbours<K>(x[u], h1[u], h2[u], lane, y, pv, n2);
        if (i < t1 && i + 1 < n) {
          if (y < x[u]) {
            cd++; fd = min(fd, (int)i); ld = max(ld, (int)i);
            cv += straddle_regs<K>(n, i, pv, n2);
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
    // (tile_mm_finish's barrier orders the agg writes above and the next tile's init)
    const int tok = tile_mm_finish<K>(mmn, mmx, nsub, vec ? 1 : 0, a.mm + t);
    if (tid == 0) {
      for (int v = 1; v < kResWarps; v++) {
        cd += sm.agg[v][0]; ca += sm.agg[v][1];
        fd = min(fd, sm.agg[v][2]); ld = max(ld, sm.agg[v][3]); fa = min(fa, sm.agg[v][4]); la = max(la, sm.agg[v][5]);
        cv += sm.agg[v][6];
      }
      TileSummary ts;
      ts.ndesc = cd; ts.nab = ca; ts.fdesc = fd; ts.ldesc = ld; ts.fab = fa; ts.lab = la; ts.nviol = cv; ts.tok = tok;
      a.sums[t] = ts;
    }
    __syncthreads();
  }
  SR_RES_STAMP(0);
  // ================= route: every CTA announces its tiles and waits for all ==============
  // (a counter, not a grid barrier: the samplers arrive before sorting their
  // sample quarter, so sorted / reversed inputs do not wait for the sorts)
  if (tid == 0) {  // arrive as soon as this CTA's tiles are published
    __threadfence();
    atomicAdd(a.arrive, 1u);
  }
  // the samplers sort their sample quarter meanwhile (wasted only on the
  // sorted / reversed routes, which the other CTAs finish without them)
  if (sampler) {  // the quarter, sorted and written to a.samp
    typename SM::E& e = sm.u.e;
#pragma unroll
    for (int r = 0; r < SG; r++) {
      const int q = r * NT + tid;
      if (q < QS) e.x[q] = sx[r];
    }
    __syncthreads();
    SR_RES_CSUB(5);
    const K* sq = QS >= 128 ? res_block_sort<K, NT>(e.x, e.y, QS) : e.x;
    if (QS < 128) BitonicSort<K, NT, SG>::sort(e.x, QS);
    SR_RES_CSUB(6);
    for (int q = tid; q < QS; q += NT) a.samp[(int64_t)quarter * QS + q] = sq[q];
  }
  __shared__ int s_skip;              // (samplers) another route was published: the speculative work stops
  __shared__ long long s_skip_route;  // ... and this is it
  if (sampler) {  // the samplers turn their sorted pieces into the level-1 splitters (R14)
    static_assert(kResSamplers == 4, "four sorted sample pieces");
    // speculatively, before the route is known (the splitters are ready when it
    // is; wasted only on the sorted / reversed / outlier routes, which the
    // other CTAs finish without the samplers).  Sampler steps are counted on a
    // persistent counter that every launch advances by 3 kResSamplers.
    const int m1 = a.B1 - 1;
    typename SM::SP& sp = sm.u.sp;
    // (every sampler takes every step, so the counter advances by the same
    // amount in every launch; once CTA 0 has published a route other than
    // PARTITION the remaining work is skipped)
    if (tid == 0) s_skip = 0;
    __syncthreads();  // (step() reads it first)
    int steps_done = 0;  // (thread 0) this sampler's increments of the step counter in this launch
    bool part_known = false;  // (thread 0) the published route is PARTITION: nothing more to watch
    // a route other than PARTITION, published by CTA 0 (one more arrival), ends the samplers'
    // work at once, also while waiting for the others; this sampler's remaining increments
    // are added then, so that the counter still advances by 3 kResSamplers per launch, and
    // the route is kept for the route step below
    auto step = [&](uint32_t target) {  // publish this CTA's writes, wait for the other samplers'
      if (s_skip) return true;  // (uniform: written before the barrier that ended the last step)
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        atomicAdd(a.scount, 1u);
        steps_done++;
        for (;;) {
          uint32_t v, arr;  // both counters in flight together (relaxed loads, fenced below)
          asm volatile("ld.relaxed.gpu.global.u32 %0, [%2];\n\tld.relaxed.gpu.global.u32 %1, [%3];"
                       : "=r"(v), "=r"(arr) : "l"(a.scount), "l"(a.arrive) : "memory");
          if (!part_known && (uint32_t)(arr - a.arrive_base) >= (uint32_t)P + 1u) {  // CTA 0 has published the route
            __threadfence();
            const long long r = __ldcg(reinterpret_cast<const long long*>(&a.st->route));
            if (r != kRoutePartition) {
              if (steps_done < 3) atomicAdd(a.scount, (uint32_t)(3 - steps_done));
              steps_done = 3;
              s_skip_route = r;
              s_skip = 1;
              break;
            }
            part_known = true;
          }
          if ((uint32_t)(v - a.scount_base) >= target) break;
        }
        __threadfence();  // (acquire: the other samplers' writes, published before their increments)
      }
      __syncthreads();
      return s_skip != 0;
    };
    const bool skip1 = step(kResSamplers);
    SR_RES_CSUB(0);
    if (!skip1) {  // half h = quarter / 2 of the pairwise merges (pieces 2h, 2h+1), this sampler's
       // part of it: merged positions [part R, (part + 1) R), written to mrg[h 2R + ...]
      const int R = QS, h = quarter >> 1, part = quarter & 1;
      for (int i = tid; i < 2 * R; i += NT) sp.q[i] = __ldcg(a.samp + (int64_t)h * 2 * R + i);
      __syncthreads();
      SR_RES_CSUB(1);
      const K* A = sp.q;
      const K* B = sp.q + R;
      const int per = (R + NT - 1) / NT, d0 = part * R + tid * per, d1 = min(d0 + per, (part + 1) * R);
      if (d0 < d1) {
        int i = merge_path_search<K>([&](int x) { return A[x]; }, R, [&](int x) { return B[x]; }, R, d0);
        int j = d0 - i;
        for (int d = d0; d < d1; d++) {
          const bool tA = j >= R || (i < R && !(B[j] < A[i]));
          a.mrg[(int64_t)h * 2 * R + d] = tA ? A[i] : B[j];
          i += tA;
          j += !tA;
        }
      }
    }
    SR_RES_CSUB(4);
    const bool skip2 = step(2 * kResSamplers);
    SR_RES_CSUB(2);
    // splitter j = element O1 (j+1) of the merged halves (R9, R14),
    // with its gamma flag (more than gamma = 2 of the elements r-2 .. r+2 equal
    // to it); this sampler's quarter of the j range, +inf padded
    if (!skip2) {
    for (int i = tid; i < S1; i += NT) sp.q[i] = __ldcg(a.mrg + i);
    __syncthreads();
    const K* A0 = sp.q;
    const K* A1 = sp.q + H1;
    constexpr int JQ = B1MAX / kResSamplers;
    for (int j = quarter * JQ + tid; j < (quarter + 1) * JQ; j += NT) {
      K t = KeyTraits<K>::max_key();
      uint8_t f = 0;
      if (j < m1) {
        const int r = (j + 1) * ResCfg<K>::O1;
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
      a.spl[j] = t;
      a.spf[j] = f;
    }
    }
    SR_RES_CSUB(3);
    const bool skip3 = step(3 * kResSamplers);
    if (quarter == 0 && !skip3) {  // one guide table (guide.cuh) for every CTA: built once, loaded in phase C
      K* s_spl = sm.u.ct.stk[0];
      uint8_t* s_eq = reinterpret_cast<uint8_t*>(sm.u.ct.stb[0]);
      for (int j = tid; j < m1; j += NT) {
        s_spl[j] = __ldcg(a.spl + j);
        s_eq[j] = __ldcg(a.spf + j);
      }
      __syncthreads();
      guide_build<K, NT>(s_spl, s_eq, m1, sm.v.guide1, sm.red);
      const int4* gs = reinterpret_cast<const int4*>(&sm.v.guide1);
      int4* gd = reinterpret_cast<int4*>(a.guide);
      for (int i = tid; i < (int)(sizeof(sm.v.guide1) / 16); i += NT) gd[i] = gs[i];
      SR_RES_CSUB(7);
    }
  }
  SR_RES_STAMP(1);
  // samplers take the route CTA 0 publishes (one more arrival) instead of
  // resolving it themselves; the others wait for every CTA's tiles
  const uint32_t need = sampler ? (uint32_t)P + 1u : (uint32_t)P;
  const bool have_route = sampler && s_skip;  // (uniform: s_skip is final after the sampler block's barriers)
  if (tid == 0 && !have_route) {
    uint32_t v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.arrive) : "memory");
    } while ((uint32_t)(v - a.arrive_base) < need);
  }
  __syncthreads();
  if (a.tstamp && c == 0 && tid == 0) a.tstamp[1] = res_now();
  typename SM::SP& sp = sm.u.sp;
  if (!sampler) {  // tile summaries into shared memory (the samplers read the published route)
    const int4* src = reinterpret_cast<const int4*>(a.sums);
    int4* dst = reinterpret_cast<int4*>(sp.ts);
    for (int i = tid; i < 2 * a.G; i += NT) dst[i] = __ldcg(src + i);
  }
  __syncthreads();
  if (a.tstamp && c == 0 && tid == 0) a.tstamp[8 + 8 * (size_t)P + 32] = res_now();
  __shared__ int64_t s_route;
  if (sampler) {
    if (tid == 0) s_route = have_route ? s_skip_route : __ldcg(reinterpret_cast<const long long*>(&a.st->route));
  } else if (w == 0) {  // H1 resolve by one warp (CTA 0 also writes the statistics and run lists)
    const int64_t r = c == 0 ? presort_resolve_warp<K, true>(a.keys, n, sp.ts, a.G, a.lmin, a.asc, a.desc, a.st,
                                                             a.force, a.merge_ok, a.mm)
                             : presort_resolve_warp<K, false>(a.keys, n, sp.ts, a.G, a.lmin, a.asc, a.desc, a.st,
                                                              a.force, a.merge_ok, a.mm);
    if (a.tstamp && c == 0 && lane == 0) a.tstamp[8 + 8 * (size_t)P + 33] = res_now();
    if (lane == 0) {
      s_route = r;
      if (c == 0) {  // the route is in a.st: tell the samplers
        __threadfence();
        atomicAdd(a.arrive, 1u);
      }
    }
    // every route but the partition is decided here: sorted / reversed finish
    // in this launch, merge / outlier / undecided continue on the host
    if (c == 0 && r != kRoutePartition && !(r == kRouteOutlier && a.out_res))
      res_publish_warp(a, (r == kRouteSorted || r == kRouteReversed) ? 1 : 0);
  }
  __syncthreads();
  const int64_t route = s_route;
  SR_RES_STAMP(2);
  if (route == kRouteSorted) return;
  if (route == kRouteReversed) {
    // UR pairs per thread in flight (a dependent load/store pair per thread
    // and round would leave the reversal latency-bound)
    constexpr int UR = 8;
    const int64_t half = n / 2, stride = (int64_t)P * NT;
    constexpr int V = 16 / (int)sizeof(K);
    if ((reinterpret_cast<uintptr_t>(a.keys) & 15) == 0 && n % V == 0) {
      // 16-byte vectors: vector p swaps with vector nv-1-p, both reversed inside
      // (a quarter of the scalar loop's memory instructions)
      constexpr int UV = 4;
      const int64_t nv = n / V, halfv = nv / 2;
      int4* kv = reinterpret_cast<int4*>(a.keys);
      auto rev = [](int4 v) { return sizeof(K) == 4 ? make_int4(v.w, v.z, v.y, v.x) : make_int4(v.z, v.w, v.x, v.y); };
      for (int64_t p0 = (int64_t)c * NT + tid; p0 < halfv; p0 += UV * stride) {
        int4 x[UV], y[UV];
#pragma unroll
        for (int u = 0; u < UV; u++) {
          const int64_t p = p0 + u * stride;
          if (p < halfv) { x[u] = kv[p]; y[u] = kv[nv - 1 - p]; }
        }
#pragma unroll
        for (int u = 0; u < UV; u++) {
          const int64_t p = p0 + u * stride;
          if (p < halfv) { kv[p] = rev(y[u]); kv[nv - 1 - p] = rev(x[u]); }
        }
      }
      if ((nv & 1) && c == 0 && tid == 0) kv[halfv] = rev(kv[halfv]);  // the middle vector
      __syncthreads();
      SR_RES_STAMP(3);  // (SR_TIMING: printed as "C.tree" on this route)
      return;
    }
    for (int64_t p0 = (int64_t)c * NT + tid; p0 < half; p0 += UR * stride) {
      K x[UR], y[UR];
#pragma unroll
      for (int u = 0; u < UR; u++) {
        const int64_t p = p0 + u * stride;
        if (p < half) { x[u] = a.keys[p]; y[u] = a.keys[n - 1 - p]; }
      }
#pragma unroll
      for (int u = 0; u < UR; u++) {
        const int64_t p = p0 + u * stride;
        if (p < half) { a.keys[p] = y[u]; a.keys[n - 1 - p] = x[u]; }
      }
    }
    return;
  }
  if (route == kRouteOutlier && a.out_res) {
    res_outlier<K, SM>(a, sm);
    return;
  }
  if (route != kRoutePartition) return;  // MERGE / undecided: the host planner continues
  grid.sync();

  // ================= C: splitter tree; tile-local bucket grouping =================
  guide_load(a.guide, sm.v.guide1);  // (built once by sampler 0)
  __syncthreads();
  SR_RES_STAMP(3);
  const int ngm = (c < PS && a.NG > c) ? (a.NG - 1 - c) / PS + 1 : 0;  // groups of this CTA: t = c + k PS, k < ngm <= GPC
  {
    for (int k = 0; k < ngm; k++) {
      const int t = c + k * PS;
      const int64_t t0 = (int64_t)t * a.tile;
      const int64_t t1 = t0 + a.tile < n ? t0 + a.tile : n;
      res_group<K, SM>(a, sm, a.keys, t0, t1, k, nbins, a.tot, a.goff + (size_t)t * nbins);
    }
  }
  SR_RES_STAMP(4);
  grid.sync();

  // ================= D: bucket starts; pieces written to their buckets in ws =================
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
  smem_exclusive_sum_u32<NT>(start, nbins, reinterpret_cast<uint32_t*>(sm.red));
  if (tid == 0) start[nbins] = (uint32_t)n;
  __syncthreads();
  if (c == 0) {  // statistics; every bucket size is known: publish the outcome early
    long long noneq = 0, eqk = 0;
    int over = 0;
    for (int b = tid; b < nbins; b += NT) {
      const uint32_t cnt = start[b + 1] - start[b];
      if (b & 1) eqk += cnt; else noneq += cnt;
      over |= !(b & 1) && cnt > (uint32_t)a.capb;  // listed for the host's next level
    }
    noneq = block_reduce_sum<NT>(noneq, reinterpret_cast<long long*>(sm.red64));
    eqk = block_reduce_sum<NT>(eqk, reinterpret_cast<long long*>(sm.red64));
    over = __syncthreads_or(over);
    if (tid == 0) {
      a.st->noneq_total = noneq;
      a.st->eq_keys = eqk;
      res_publish(a, over ? 0 : 1);
    }
  }
  {  // every key of a held group to its bucket in ws (runs of the same bucket are
     // consecutive, so the stores coalesce per piece); equality buckets are
     // filled in E
    typename SM::CT& ct = sm.u.ct;
    for (int k = 0; k < ngm; k++) {
      const int t = c + k * PS;
      if (ct.lst[k][nbins] == 0) continue;  // nothing placed (every key in an equality bucket)
      {
        constexpr int BI = (SM::NB1 + NT - 1) / NT;
        uint32_t go[BI];
#pragma unroll
        for (int r = 0; r < BI; r++)
          go[r] = r * NT + tid < nbins ? __ldcg(a.goff + (size_t)t * nbins + r * NT + tid) : 0u;
#pragma unroll
        for (int r = 0; r < BI; r++)
          if (r * NT + tid < nbins) ct.cnt[r * NT + tid] = start[r * NT + tid] + go[r];
      }
      __syncthreads();
      const uint32_t* lst = ct.lst[k];
      const int len = (int)lst[nbins];
      constexpr int UD = kResGrp / NT;
#pragma unroll
      for (int u = 0; u < UD; u++) {
        const int i = u * NT + tid;
        if (i < len) {
          const int b = ct.stb[k][i];
          SR_CHECK(b < nbins && (int64_t)ct.cnt[b] + i - lst[b] < n);
          if (!(b & 1)) a.ws[ct.cnt[b] + (uint32_t)i - lst[b]] = ct.stk[k][i];
        }
      }
      __syncthreads();
    }
  }
  SR_RES_STAMP(5);
  grid.sync();

  // ================= E: bucket sorts and equality fills =================
  // Units: CTA units first (range buckets above WCAP: one CTA each, in-shared-
  // memory partition + warp sorts), then warp units (range buckets <= WCAP:
  // one warp's register network; equality fills of kResWarpFill keys).  Every
  // CTA derives both lists from the bucket starts, so no hand-off is needed.
  if (a.tstamp && c == 0 && tid == 0) a.tstamp[2] = res_now();
  constexpr int WCAP = SM::WCAP;
  int nbig = 0;
  {  // unit counts per bin -> exclusive prefixes (each thread scans BPT consecutive bins)
    constexpr int BPT = (SM::NB1 + 1 + NT - 1) / NT;
    uint32_t ca[BPT], cb[BPT], sa = 0, sb = 0;
#pragma unroll
    for (int r = 0; r < BPT; r++) {
      const int b = tid * BPT + r;
      const uint32_t cnt = b < nbins ? start[b + 1] - start[b] : 0u;
      const bool rng = b < nbins && !(b & 1);
      ca[r] = rng && cnt > (uint32_t)(WCAP / 2) && cnt <= (uint32_t)WCAP;
      cb[r] = b >= nbins ? 0u : (b & 1) ? (cnt + kResWarpFill - 1) / kResWarpFill : (cnt > 0 && cnt <= (uint32_t)(WCAP / 2));
      nbig += rng && cnt > (uint32_t)WCAP;
      sa += ca[r];
      sb += cb[r];
    }
    uint32_t ta, tb;
    uint32_t* red = reinterpret_cast<uint32_t*>(sm.red);
    uint32_t pa = block_exclusive_sum<NT>(sa, red, &ta);
    uint32_t pb = block_exclusive_sum<NT>(sb, red, &tb);
#pragma unroll
    for (int r = 0; r < BPT; r++) {
      const int b = tid * BPT + r;
      if (b <= nbins) {
        sm.v.eu.upa[b] = (uint16_t)pa;
        sm.v.eu.upb[b] = (uint16_t)pb;
      }
      pa += ca[r];
      pb += cb[r];
    }
  }
  __syncthreads();
  int NC = 0;
  if (__syncthreads_or(nbig)) {  // compact the big buckets (bucket order) into cbin
    constexpr int BPT = (SM::NB1 + NT - 1) / NT;
    int f = 0;
    for (int r = 0; r < BPT; r++) {
      const int b = tid * BPT + r;
      f += b < nbins && !(b & 1) && start[b + 1] - start[b] > (uint32_t)WCAP;
    }
    int tot;
    int o = block_exclusive_sum<NT>(f, sm.red, &tot);
    for (int r = 0; r < BPT; r++) {
      const int b = tid * BPT + r;
      if (b < nbins && !(b & 1) && start[b + 1] - start[b] > (uint32_t)WCAP) {
        sm.v.eu.cbin[o] = (uint16_t)b;
        o++;
      }
    }
    NC = tot;
    __syncthreads();
  }
  if (c == 0 && tid == 0) a.st->n_items = (int64_t)sm.v.eu.upa[nbins] + sm.v.eu.upb[nbins] + NC;
  __shared__ uint32_t s_unit;
  typename SM::E& e = sm.u.e;
  if (NC > 0) {
    for (;;) {  // CTA units, handed out dynamically
      if (tid == 0) s_unit = atomicAdd(a.unit_counter, 1u);
      __syncthreads();
      const uint32_t u = s_unit;
      __syncthreads();
      if (u >= (uint32_t)NC) break;
      // a big bucket beyond the in-kernel cap: copied unsorted into its final
      // range and listed for the host's next level
      const int b = (int)sm.v.eu.cbin[u];
      const int s = (int)start[b], len = (int)(start[b + 1] - start[b]);
      const unsigned long long tg0 = (a.tstamp && c == 0 && tid == 0) ? res_now() : 0;
      const unsigned long long tg1 = a.tstamp ? res_now() : 0;
      const bool fits = len <= a.capb;
      K* gdst = fits ? e.x : a.keys + s;
      {
        constexpr int UL = 8;
        for (int i0 = 0; i0 < len; i0 += NT * UL) {
          K v[UL];
#pragma unroll
          for (int uu = 0; uu < UL; uu++) {
            const int i = i0 + uu * NT + tid;
            v[uu] = i < len ? __ldcg(a.ws + s + i) : K(0);
          }
#pragma unroll
          for (int uu = 0; uu < UL; uu++) {
            const int i = i0 + uu * NT + tid;
            if (i < len) gdst[i] = v[uu];
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
      SR_CHECK((int64_t)s + len <= n && len <= SM::CAPB);
      unit_sort<K, SM::CAPB, NT>(a.keys + s, len, e);
      if (a.tstamp && tid == 0) {  // SR_TIMING: longest CTA unit, count
        unsigned long long* q = a.tstamp + 8 + 8 * (size_t)P + 24;
        atomicMax(q + 0, res_now() - tg1);
        atomicAdd(q + 1, 1ull);
      }
    }
  }
  {  // warp units, largest first: the halves of the class-A buckets (two warps
     // each, the second to finish merges), then class B (one warp each), so
     // that the last units handed out are short
    const uint32_t UA = sm.v.eu.upa[nbins], UW = 2 * UA + sm.v.eu.upb[nbins];
    K* stage = e.x + w * WCAP;  // x and y are adjacent: kResWarps * WCAP keys
    constexpr int NET = UnitNet<K>::NET;
    static_assert(2 * NET == WCAP, "a class-A bucket is two networks");
    for (;;) {
      uint32_t u = 0;
      if (lane == 0) u = atomicAdd(a.unit_counter + 2, 1u);
      u = __shfl_sync(0xffffffffu, u, 0);
      if (u >= UW) break;
      const unsigned long long ti0 = a.tstamp ? res_now() : 0;
      if (u < 2 * UA) {  // half h of class-A bucket v (WCAP/2 < len <= WCAP): sort it in ws
        const uint32_t v = u >> 1;
        const int h = (int)(u & 1);
        const uint16_t* up = sm.v.eu.upa;
        int lo = 0, hi = nbins - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (up[mid] <= v) lo = mid; else hi = mid - 1;
        }
        const int s = (int)start[lo], len = (int)(start[lo + 1] - start[lo]);
        const int h0 = h ? NET : 0, hl = h ? len - NET : NET;
        SR_CHECK((int64_t)s + len <= n && len <= WCAP && h0 + hl <= len);
        K* hw = a.ws + s + h0;
        for (int i = lane; i < hl; i += 32) stage[i] = __ldcg(hw + i);
        __syncwarp();
        int unsorted = 0;  // is_sorted
        for (int i = lane; i + 1 < hl; i += 32) unsorted |= stage[i + 1] < stage[i];
        if (__any_sync(0xffffffffu, unsorted)) {
          unit_warp_sort<K>(stage, hl);
          for (int i = lane; i < hl; i += 32) hw[i] = stage[i];
        }
        __threadfence();  // this half is in ws before the pair counter says so
        __syncwarp();
        uint32_t prev = 0;
        if (lane == 0) prev = atomicAdd(a.pairc + v, 1u);
        prev = __shfl_sync(0xffffffffu, prev, 0);
        if (prev == 1) {  // the other half is done too: merge both into keys (A wins ties)
          __threadfence();
          for (int i = lane; i < len; i += 32) stage[i] = __ldcg(a.ws + s + i);
          __syncwarp();
          if (stage[NET - 1] <= stage[NET]) {  // trimmed: already in order
            for (int i = lane; i < len; i += 32) a.keys[s + i] = stage[i];
            __syncwarp();
          } else {
            unit_warp_merge<K>(stage, NET, stage + NET, len - NET, a.keys + s);
          }
        }
        if (a.tstamp && lane == 0)  // SR_TIMING: longest warp item
          atomicMax(a.tstamp + 8 + 8 * (size_t)P + 26, res_now() - ti0);
        continue;
      }
      const uint16_t* up = sm.v.eu.upb;
      const uint32_t v = u - 2 * UA;
      int lo = 0, hi = nbins - 1;  // last bin with up <= v
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (up[mid] <= v) lo = mid; else hi = mid - 1;
      }
      const int b = lo;
      const int s = (int)start[b], len = (int)(start[b + 1] - start[b]);
      if (b & 1) {  // equality bucket: fill
        const K key = __ldcg(a.spl + (b - 1) / 2);
        const int f0 = (int)(v - up[b]) * kResWarpFill;
        const int f1 = f0 + kResWarpFill < len ? f0 + kResWarpFill : len;
        SR_CHECK((int64_t)s + f1 <= n);
        for (int i = f0 + lane; i < f1; i += 32) a.keys[s + i] = key;
        continue;
      }
      {  // coalesced load into the warp's staging area
        constexpr int UL = 8;
        for (int i0 = 0; i0 < len; i0 += 32 * UL) {
          K v[UL];
#pragma unroll
          for (int uu = 0; uu < UL; uu++) {
            const int i = i0 + uu * 32 + lane;
            v[uu] = i < len ? __ldcg(a.ws + s + i) : K(0);
          }
#pragma unroll
          for (int uu = 0; uu < UL; uu++) {
            const int i = i0 + uu * 32 + lane;
            if (i < len) stage[i] = v[uu];
          }
        }
      }
      __syncwarp();
      int unsorted = 0;  // is_sorted
      for (int i = lane; i + 1 < len; i += 32) unsorted |= stage[i + 1] < stage[i];
      if (__any_sync(0xffffffffu, unsorted)) {
        SR_CHECK((int64_t)s + len <= n && len <= WCAP);
        unit_warp_piece<K>(stage, len, a.keys + s);  // <= WCAP keys: one network, or two and a merge
      } else {
        for (int i = lane; i < len; i += 32) a.keys[s + i] = stage[i];
      }
      __syncwarp();
      if (a.tstamp && lane == 0)  // SR_TIMING: longest warp item
        atomicMax(a.tstamp + 8 + 8 * (size_t)P + 26, res_now() - ti0);
    }
  }
  if (a.tstamp && c == 0 && tid == 0) a.tstamp[3] = res_now();
  SR_RES_STAMP(6);
}

}  // namespace sr
