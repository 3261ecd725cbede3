// resident.cuh -- the resident path: the whole keys-only sort of an L2-resident
// array (kCap < n <= kResMaxN) as ONE cooperative launch of one CTA per SM.
//
// The multi-kernel path (presort.cuh, partition.cuh) pays a launch plus a
// drain per step; at the paper's Table 1 size (n = 2,000,000)
// the steps themselves move ~8 MB each (~1.2 us of HBM time), so launches and
// single-CTA bookkeeping kernels dominated.  Here the same steps (H1, H2, H3's
// device stage, H7-H11) run as phases of one persistent kernel separated by
// grid-wide barriers, every CTA computing the small bookkeeping (bucket starts,
// finishing work list) redundantly in its own shared memory instead of a
// one-CTA kernel:
//   A  H1 scan of the CTA's presort tiles (same tiles and TileSummary as K1) +
//      H7 sample gather: CTA c gathers sample slice c and sorts it locally;
//   -- grid sync --
//   B  CTA 0: K2 resolve (D, long runs, device route).
//      all:   ranks of the CTA's own slice in the whole sample by binary
//             searches in every sorted slice; the sample at rank
//             floor((j+1)S/B) writes splitter j and its gamma flag
//             (count > gamma = 2) -- R8/R9 of DESIGN.md;
//   -- grid sync --
//   C  route: SORTED exits; REVERSED reverses in place and exits;
//      MERGE / undecided exit to the host planner.  PARTITION: classify the
//      CTA's keys (Eytzinger tree, 3-way ids), histogram,
//      one atomicAdd per (CTA, bucket) on the global totals -> this CTA's
//      offset inside every bucket (keys only: the order of equal keys is
//      unobservable);
//   -- grid sync --
//   D  bucket starts = exclusive scan of the totals (every CTA); scatter of
//      the range-bucket keys into the workspace (equality keys are not moved:
//      "spared from the recursive calls"); finishing work list;
//   -- grid sync --
//   E  finishing (H11): buckets of (kResWarpCap, kResCtaCap] keys by one CTA
//      (BitonicSort), buckets <= kResWarpCap by one warp (register bitonic),
//      equality buckets filled; each with the is_sorted skip.
//      Range buckets > kResCtaCap stay in the workspace and are listed for the
//      host, which runs the next partition level on them (Appendix B
//      recursion).
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
constexpr int kResWarps = kResNT / 32;
constexpr int kResWarpCap = 1024;  // range buckets <= this: one warp
constexpr int kResCtaCap = 4096;   // (kResWarpCap, kResCtaCap]: one CTA; larger: next level (host)
constexpr int kResFill = 8192;     // equality fills per warp unit
constexpr int kResU = 8;           // keys per thread per pass
constexpr int kResSlice = 1024;    // sample slice sorted by one CTA in phase A (<= 16 slices)
constexpr int kResTarget = 512;    // mean bucket size aimed for
constexpr int64_t kResMaxN = int64_t(4) << 20;

template <typename K> struct ResCfg;
template <> struct ResCfg<int32_t> { static constexpr int BMAX = 4096; };
template <> struct ResCfg<int64_t> { static constexpr int BMAX = 2048; };

template <typename K>
struct ResArgs {
  K* keys;
  K* ws;
  int64_t n;
  int tile, G;              // presort tiles (K1's tiling)
  TileSummary* sums;
  RunDesc* asc;
  RunDesc* desc;
  DevStats* st;
  K* sample;                // S keys, sorted per slice in phase A
  int S, B;                 // sample size, buckets (power of two <= BMAX)
  K* spl;                   // B-1 splitters
  uint8_t* eqf;             // B-1 equality flags
  uint32_t* tot;            // 2B+1 bucket totals (zeroed by CTA 0 in phase A)
  uint16_t* bins;           // n bucket ids
  OvfSeg* ovf;              // range buckets > kResCtaCap (host: next level)
  int64_t lmin;
  int force, merge_ok;
  int warp_cap, cta_cap;    // finishing caps (kResWarpCap, kResCtaCap; lowered by tests)
  unsigned long long* tstamp;  // optional: %globaltimer, [0..8) CTA 0 phase starts, then 8 per CTA
};

#define SR_RES_STAMP(k)                                                         \
  do {                                                                          \
    if (a.tstamp && tid == 0) a.tstamp[8 + (size_t)blockIdx.x * 8 + (k)] = res_now(); \
  } while (0)

__device__ __forceinline__ unsigned long long res_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Shared memory of the resident kernel.  Phase B's sample copy overlays the
// phase C-E arrays; phase E's sort buffers overlay phase C/D's offsets.
template <typename K>
struct ResSmem {
  static constexpr int BMAX = ResCfg<K>::BMAX;
  static constexpr int NB = 2 * BMAX + 1;  // bins
  struct alignas(16) CE {
    K tree[2 * BMAX];
    uint32_t start[NB + 1];  // bucket starts (global positions), start[nbins] = n
    uint32_t wpre[NB + 1];   // exclusive prefix of warp units per bin
    uint32_t cpre[NB + 1];   // exclusive prefix of CTA units per bin
    uint8_t eq[BMAX];
    union alignas(16) {
      struct {
        uint32_t off[NB];  // C: this CTA's offset inside each bucket, D: + start
        uint32_t run[NB];  // D: running rank per bucket
      } cd;
      K stage[kResWarps * kResWarpCap];  // E: warp staging
      K cta[2 * kResCtaCap];             // E: CTA bitonic buffer
    } u;
  };
  struct alignas(16) PB {
    K samp[BMAX * kOversample + 16];  // B: the whole sample, slice j at j * (SL + 1) (bank padding)
  };
  union {
    CE ce;
    PB pb;  // phase B only
  };
  int32_t red[kResNT / 32 + 1];
  int64_t red64[kResNT / 32 + 1];
  int32_t agg[kResNT / 32][6];  // tile-scan partials per warp
};

// Eytzinger tree + sorted copy of the m = B-1 splitters (as load_splitters_smem,
// for a BMAX-sized layout); cross-CTA data read with __ldcg.
template <typename K, int BMAX, int NT>
__device__ __forceinline__ void res_load_tree(const K* spl, const uint8_t* eqf, int m, int depth, K* tree,
                                              uint8_t* eq) {
  const int nodes = 1 << depth;
  constexpr int TI = (BMAX + NT - 1) / NT;
  K v[TI];
  uint8_t e[TI];
#pragma unroll
  for (int r = 0; r < TI; r++) {  // all loads in flight before the first store
    const int i = r * NT + threadIdx.x;
    v[r] = i < m ? __ldcg(spl + i) : KeyTraits<K>::max_key();
    e[r] = i < m ? __ldcg(eqf + i) : (uint8_t)0;
  }
#pragma unroll
  for (int r = 0; r < TI; r++) {
    const int i = r * NT + threadIdx.x;
    if (i < nodes) {
      tree[BMAX + i] = v[r];
      eq[i] = e[r];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x + 1; i < nodes; i += NT) {  // node i of the level-order tree <- sorted position pos(i)
    const int d = 31 - __clz(i);
    const int pos = ((2 * (i - (1 << d)) + 1) << (depth - 1 - d)) - 1;
    tree[i] = tree[BMAX + pos];  // +inf padding beyond m
  }
}

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

// Q independent lower_bound / upper_bound searches of x[q] in s[s0[q], s0[q] +
// len[q]), advanced in lockstep so their dependent shared-memory loads overlap.
template <typename K, int Q>
__device__ __forceinline__ void res_bounds(const K* s, const int (&s0)[Q], const int (&len)[Q], const K (&x)[Q],
                                           int (&lt)[Q], int (&le)[Q]) {
  int lo[Q], n1[Q], lo2[Q], n2[Q];
#pragma unroll
  for (int q = 0; q < Q; q++) { lo[q] = s0[q]; n1[q] = len[q]; lo2[q] = s0[q]; n2[q] = len[q]; }
  bool more = true;
  while (more) {
    more = false;
#pragma unroll
    for (int q = 0; q < Q; q++) {
      if (n1[q] > 0) {
        const int h = n1[q] >> 1;
        if (s[lo[q] + h] < x[q]) { lo[q] += h + 1; n1[q] -= h + 1; } else n1[q] = h;
        more = true;
      }
      if (n2[q] > 0) {
        const int h = n2[q] >> 1;
        if (!(x[q] < s[lo2[q] + h])) { lo2[q] += h + 1; n2[q] -= h + 1; } else n2[q] = h;
        more = true;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < Q; q++) { lt[q] = lo[q] - s0[q]; le[q] = lo2[q] - s0[q]; }
}

// Warp finishing of one range bucket [s, s+len) of ws into keys (len <= 32*VT).
template <typename K, int VT>
__device__ __forceinline__ void res_warp_sort(const K* __restrict__ src, K* __restrict__ dst, int len, K* stage) {
  const int lane = threadIdx.x & 31;
  {
    K x[VT];
#pragma unroll
    for (int r = 0; r < VT; r++) {
      const int i = r * 32 + lane;
      x[r] = i < len ? __ldcg(src + i) : KeyTraits<K>::max_key();
    }
#pragma unroll
    for (int r = 0; r < VT; r++) stage[r * 32 + lane] = x[r];
  }
  __syncwarp();
  int unsorted = 0;
  for (int i = lane; i + 1 < len; i += 32) unsorted |= stage[i + 1] < stage[i];
  if (__any_sync(0xffffffffu, unsorted)) WarpBitonic<K, VT>::sort(stage, len);
  __syncwarp();
  for (int i = lane; i < len; i += 32) dst[i] = stage[i];
  __syncwarp();
}

static_assert(offsetof(ResSmem<int32_t>::CE, u) % 16 == 0 && offsetof(ResSmem<int64_t>::CE, u) % 16 == 0,
              "vectorised sort buffers need 16-byte alignment");

template <typename K>
__global__ void __launch_bounds__(kResNT, 1) k_resident(ResArgs<K> a) {
  namespace cg = cooperative_groups;
  using SM = ResSmem<K>;
  constexpr int BMAX = SM::BMAX;
  constexpr int NT = kResNT;
  constexpr int U = kResU;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int P = gridDim.x, c = blockIdx.x;
  const int64_t n = a.n;
  const int nbins = 2 * a.B + 1;

  // ================= A: H1 tile scan + sample slice =================
  if (a.tstamp && c == 0 && tid == 0) a.tstamp[0] = res_now();
  if (c == 0) {
    for (int b = tid; b < nbins; b += NT) a.tot[b] = 0;
    if (tid == 0) {
      DevStats* st = a.st;
      st->noneq_total = 0; st->n_items = 0; st->n_items_big = 0; st->n_ovf = 0;
      st->ovf_keys = 0; st->eq_keys = 0; st->error = 0; st->big_keys = 0;
    }
  }
  // sample: S = B*o jittered positions (R8) in NSL slices of
  // SL = min(S, kResSlice) keys; slice j is gathered and sorted by CTA P-1-j
  // (the last CTAs scan the fewest tiles); its gathers are issued first so
  // they overlap the scan
  const int S = a.S;
  const int log2S = (S & (S - 1)) == 0 ? __ffs(S) - 1 : -1;
  const int SL = S < kResSlice ? S : kResSlice;
  const int NSL = S / SL;
  const int slice = P - 1 - c;
  constexpr int SG = kResSlice / NT;
  K sx[SG];
  if (slice < NSL) {
#pragma unroll
    for (int r = 0; r < SG; r++) {
      const int q = r * NT + tid;
      sx[r] = q < SL ? a.keys[sample_position(0, n, S, (int64_t)slice * SL + q, log2S)] : K(0);
    }
  }
  constexpr int UA = 16;  // one load round per 8192-key tile
  for (int t = c; t < a.G; t += P) {
    const int64_t t0 = (int64_t)t * a.tile;
    const int64_t t1 = t0 + a.tile < n ? t0 + a.tile : n;
    int cd = 0, ca = 0;
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
        if (lane == 31) y = nx[u];
        if (i < t1 && i + 1 < n) {
          if (y < x[u]) { cd++; fd = min(fd, (int)i); ld = max(ld, (int)i); }
          if (x[u] < y) { ca++; fa = min(fa, (int)i); la = max(la, (int)i); }  // keys only: non-increasing runs
        }
      }
    }
    // one combined block reduction of the six tile statistics
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      cd += __shfl_xor_sync(0xffffffffu, cd, o);
      ca += __shfl_xor_sync(0xffffffffu, ca, o);
      fd = min(fd, __shfl_xor_sync(0xffffffffu, fd, o));
      ld = max(ld, __shfl_xor_sync(0xffffffffu, ld, o));
      fa = min(fa, __shfl_xor_sync(0xffffffffu, fa, o));
      la = max(la, __shfl_xor_sync(0xffffffffu, la, o));
    }
    if (lane == 0) {
      sm.agg[w][0] = cd; sm.agg[w][1] = ca; sm.agg[w][2] = fd; sm.agg[w][3] = ld; sm.agg[w][4] = fa; sm.agg[w][5] = la;
    }
    __syncthreads();
    if (tid == 0) {
      for (int v = 1; v < kResWarps; v++) {
        cd += sm.agg[v][0]; ca += sm.agg[v][1];
        fd = min(fd, sm.agg[v][2]); ld = max(ld, sm.agg[v][3]); fa = min(fa, sm.agg[v][4]); la = max(la, sm.agg[v][5]);
      }
      TileSummary ts;
      ts.ndesc = cd; ts.nab = ca; ts.fdesc = fd; ts.ldesc = ld; ts.fab = fa; ts.lab = la; ts.pad0 = 0; ts.pad1 = 0;
      a.sums[t] = ts;
    }
    __syncthreads();
  }
  SR_RES_STAMP(0);
  if (slice < NSL) {
    K* buf = reinterpret_cast<K*>(&sm.ce.u);  // BitonicSort scratch: 2 * kResSlice keys
#pragma unroll
    for (int r = 0; r < SG; r++) {
      const int q = r * NT + tid;
      if (q < SL) buf[q] = sx[r];
    }
    __syncthreads();
    BitonicSort<K, kResSlice / 4, 4>::sort(buf, SL);  // threads >= 256 idle
    for (int q = tid; q < SL; q += NT) a.sample[(int64_t)slice * SL + q] = buf[q];
  }
  SR_RES_STAMP(1);
  grid.sync();

  // ================= B: resolve (CTA 0) + splitters by ranking =================
  if (a.tstamp && c == 0 && tid == 0) a.tstamp[1] = res_now();
  if (c == 0)
    presort_resolve_block<K, NT>(a.keys, n, a.sums, a.G, a.lmin, a.asc, a.desc, a.st, a.force, a.merge_ok);
  {
    // rank of every sample g of this CTA's share in the whole sample: lower /
    // upper bounds in each sorted slice (16 lanes per sample, one slice per
    // lane); the sample at rank floor((j+1) S / B) writes splitter j
    typename SM::PB& pb = sm.pb;
    const int g0 = (int)(((int64_t)c * S) / P), g1 = (int)(((int64_t)(c + 1) * S) / P);
    {
      constexpr int SI = (ResCfg<K>::BMAX * kOversample + NT - 1) / NT;
      K v[SI];
#pragma unroll
      for (int r = 0; r < SI; r++) {
        const int q = r * NT + tid;
        v[r] = q < S ? __ldcg(a.sample + q) : K(0);
      }
#pragma unroll
      for (int r = 0; r < SI; r++) {
        const int q = r * NT + tid;
        if (q < S) pb.samp[q + q / SL] = v[r];
      }
    }
    __syncthreads();
    SR_RES_STAMP(2);
    const int half = lane >> 4, sl = lane & 15;
    for (int g = g0 + 2 * w + half; g - half < g1; g += 2 * kResWarps) {
      const bool valid = g < g1;
      const int gg = valid ? g : g1 - 1;
      const int own = gg / SL;
      const K x = pb.samp[gg + own];
      int lt = 0, le = 0;
      if (valid && sl < NSL) {
        int l[1], e[1];
        const int s0[1] = {sl * (SL + 1)}, ln[1] = {SL};
        const K xx[1] = {x};
        res_bounds<K, 1>(pb.samp, s0, ln, xx, l, e);
        lt = l[0];
        le = e[0];
      }
      const int eqb = sl < own ? le - lt : 0;
      const int own_lt = sl == own ? lt : 0;
      int t_lt = lt, t_le = le, t_eqb = eqb, t_own = own_lt;
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {  // reduce within the 16-lane half
        t_lt += __shfl_xor_sync(0xffffffffu, t_lt, o);
        t_le += __shfl_xor_sync(0xffffffffu, t_le, o);
        t_eqb += __shfl_xor_sync(0xffffffffu, t_eqb, o);
        t_own += __shfl_xor_sync(0xffffffffu, t_own, o);
      }
      if (valid && sl == 0) {
        const int pos = t_lt + t_eqb + (gg - own * SL - t_own);  // position in the stably sorted sample
        const int mult = t_le - t_lt;
        const int j1 = (int)(((int64_t)pos * a.B + S - 1) / S);  // smallest j+1 with floor((j+1)S/B) >= pos
        if (j1 >= 1 && j1 <= a.B - 1 && (int)(((int64_t)j1 * S) / a.B) == pos) {
          a.spl[j1 - 1] = x;
          a.eqf[j1 - 1] = mult > 2 ? 1 : 0;  // count > gamma = 2
        }
      }
    }
  }
  SR_RES_STAMP(3);
  grid.sync();

  // ================= C: route; classify + histogram =================
  if (a.tstamp && c == 0 && tid == 0) a.tstamp[2] = res_now();
  const int64_t route = __ldcg(&a.st->route);
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
  const int m = a.B - 1;
  const int depth = tree_depth(m);
  res_load_tree<K, BMAX, NT>(a.spl, a.eqf, m, depth, sm.ce.tree, sm.ce.eq);
  uint32_t* hist = sm.ce.u.cd.off;
  for (int b = tid; b < nbins; b += NT) hist[b] = 0;
  __syncthreads();
  SR_RES_STAMP(4);
  for (int t = c; t < a.G; t += P) {
    const int64_t t0 = (int64_t)t * a.tile;
    const int64_t t1 = t0 + a.tile < n ? t0 + a.tile : n;
    for (int64_t base = t0; base < t1; base += NT * U) {
      K x[U];
      int bin[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t i = base + u * NT + tid;
        x[u] = i < t1 ? a.keys[i] : K(0);
      }
      res_classify<K, BMAX, U>(x, bin, sm.ce.tree, sm.ce.eq, m, depth);
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t i = base + u * NT + tid;
        const bool valid = i < t1;
        if (__any_sync(0xffffffffu, valid && (bin[u] & 1))) {
          // equality bins collect many equal ids: warp-aggregated increments
          const unsigned peers = __match_any_sync(0xffffffffu, valid ? bin[u] : -1);
          if (valid && lane == __ffs(peers) - 1) atomicAdd(&hist[bin[u]], (uint32_t)__popc(peers));
        } else if (valid) {
          atomicAdd(&hist[bin[u]], 1u);
        }
        if (valid) a.bins[i] = (uint16_t)bin[u];
      }
    }
  }
  __syncthreads();
  {  // this CTA's offset inside every bucket: one atomicAdd per non-empty bin, all
     // in flight at once; CTAs start at different bins so that the same total
     // is not hit by every CTA at the same time
    constexpr int BI = (SM::NB + NT - 1) / NT;
    const int rot = (int)(((int64_t)c * nbins) / P);
    uint32_t h[BI];
#pragma unroll
    for (int r = 0; r < BI; r++) {
      const int i = r * NT + tid;
      const int b = i + rot < nbins ? i + rot : i + rot - nbins;
      h[r] = i < nbins ? hist[b] : 0u;
    }
#pragma unroll
    for (int r = 0; r < BI; r++) {
      const int i = r * NT + tid;
      const int b = i + rot < nbins ? i + rot : i + rot - nbins;
      h[r] = h[r] ? atomicAdd(&a.tot[b], h[r]) : 0u;
    }
#pragma unroll
    for (int r = 0; r < BI; r++) {
      const int i = r * NT + tid;
      const int b = i + rot < nbins ? i + rot : i + rot - nbins;
      if (i < nbins) hist[b] = h[r];
    }
  }
  SR_RES_STAMP(5);
  grid.sync();

  // ================= D: bucket starts, scatter, finishing work list =================
  if (a.tstamp && c == 0 && tid == 0) a.tstamp[3] = res_now();
  uint32_t* start = sm.ce.start;
  {
    constexpr int BI = (SM::NB + NT - 1) / NT;
    uint32_t v[BI];
#pragma unroll
    for (int r = 0; r < BI; r++) v[r] = r * NT + tid < nbins ? __ldcg(a.tot + r * NT + tid) : 0u;
#pragma unroll
    for (int r = 0; r < BI; r++)
      if (r * NT + tid < nbins) start[r * NT + tid] = v[r];
  }
  __syncthreads();
  auto add = [](uint32_t x, uint32_t y) { return x + y; };
  smem_scan<NT>(start, nbins, 0u, add, true, false, reinterpret_cast<uint32_t*>(sm.red));
  if (tid == 0) start[nbins] = (uint32_t)n;
  __syncthreads();
  uint32_t* off = sm.ce.u.cd.off;
  uint32_t* run = sm.ce.u.cd.run;
  for (int b = tid; b < nbins; b += NT) {
    off[b] += start[b];
    run[b] = 0;
    const uint32_t cnt = start[b + 1] - start[b];
    uint32_t wu = 0, cu = 0;
    if (b & 1) wu = (cnt + kResFill - 1) / kResFill;
    else if (cnt > 0 && cnt <= (uint32_t)a.warp_cap) wu = 1;
    else if (cnt > (uint32_t)a.warp_cap && cnt <= (uint32_t)a.cta_cap) cu = 1;
    sm.ce.wpre[b] = wu;
    sm.ce.cpre[b] = cu;
  }
  if (tid == 0) { sm.ce.wpre[nbins] = 0; sm.ce.cpre[nbins] = 0; }
  __syncthreads();
  smem_scan<NT>(sm.ce.wpre, nbins + 1, 0u, add, true, false, reinterpret_cast<uint32_t*>(sm.red));
  smem_scan<NT>(sm.ce.cpre, nbins + 1, 0u, add, true, false, reinterpret_cast<uint32_t*>(sm.red));
  for (int t = c; t < a.G; t += P) {
    const int64_t t0 = (int64_t)t * a.tile;
    const int64_t t1 = t0 + a.tile < n ? t0 + a.tile : n;
    for (int64_t base = t0; base < t1; base += NT * U) {
      K x[U];
      int bin[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t i = base + u * NT + tid;
        x[u] = i < t1 ? a.keys[i] : K(0);
        bin[u] = i < t1 ? (int)a.bins[i] : 1;
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        if (!(bin[u] & 1)) {
          const uint32_t r = atomicAdd(&run[bin[u]], 1u);
          a.ws[off[bin[u]] + r] = x[u];
        }
      }
    }
  }
  if (c == 0) {  // statistics + oversized buckets for the host
    long long noneq = 0, eqk = 0, ovk = 0;
    for (int b = tid; b < nbins; b += NT) {
      const uint32_t cnt = start[b + 1] - start[b];
      if (b & 1) eqk += cnt;
      else {
        noneq += cnt;
        if (cnt > (uint32_t)a.cta_cap) {
          ovk += cnt;
          const unsigned long long k = atomicAdd((unsigned long long*)&a.st->n_ovf, 1ull);
          OvfSeg o;
          o.start = start[b];
          o.len = cnt;
          a.ovf[k] = o;
        }
      }
    }
    noneq = block_reduce_sum<NT>(noneq, reinterpret_cast<long long*>(sm.red64));
    eqk = block_reduce_sum<NT>(eqk, reinterpret_cast<long long*>(sm.red64));
    ovk = block_reduce_sum<NT>(ovk, reinterpret_cast<long long*>(sm.red64));
    if (tid == 0) {
      a.st->noneq_total = noneq;
      a.st->eq_keys = eqk;
      a.st->ovf_keys = ovk;
      a.st->n_items = sm.ce.wpre[nbins];
      a.st->n_items_big = sm.ce.cpre[nbins];
    }
  }
  SR_RES_STAMP(6);
  grid.sync();

  // ================= E: finishing =================
  if (a.tstamp && c == 0 && tid == 0) a.tstamp[4] = res_now();
  const uint32_t UW = sm.ce.wpre[nbins], UC = sm.ce.cpre[nbins];
  auto find_bin = [&](const uint32_t* pre, uint32_t u) {  // last b with pre[b] <= u
    int lo = 0, hi = nbins - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (pre[mid] <= u) lo = mid; else hi = mid - 1;
    }
    return lo;
  };
  for (uint32_t u = c; u < UC; u += P) {
    const int b = find_bin(sm.ce.cpre, u);
    const int s = (int)start[b], len = (int)(start[b + 1] - start[b]);
    K* buf = sm.ce.u.cta;
    for (int i = tid; i < len; i += NT) buf[i] = __ldcg(a.ws + s + i);
    __syncthreads();
    int unsorted = 0;
    for (int i = tid; i + 1 < len; i += NT) unsorted |= buf[i + 1] < buf[i];
    if (__syncthreads_or(unsorted)) BitonicSort<K, NT, kResCtaCap / NT>::sort(buf, len);
    for (int i = tid; i < len; i += NT) a.keys[s + i] = buf[i];
    __syncthreads();
  }
  K* stage = sm.ce.u.stage + w * kResWarpCap;
  for (uint32_t u = (uint32_t)c * kResWarps + w; u < UW; u += (uint32_t)P * kResWarps) {
    const int b = find_bin(sm.ce.wpre, u);
    const int s = (int)start[b], len = (int)(start[b + 1] - start[b]);
    if (b & 1) {  // equality bucket: fill chunk
      const K key = sm.ce.tree[BMAX + (b - 1) / 2];
      const int f0 = (int)(u - sm.ce.wpre[b]) * kResFill;
      const int f1 = f0 + kResFill < len ? f0 + kResFill : len;
      for (int i = f0 + lane; i < f1; i += 32) a.keys[s + i] = key;
      continue;
    }
    const K* src = a.ws + s;
    K* dst = a.keys + s;
    if (len <= 128) res_warp_sort<K, 4>(src, dst, len, stage);
    else if (len <= 256) res_warp_sort<K, 8>(src, dst, len, stage);
    else if (len <= 512) res_warp_sort<K, 16>(src, dst, len, stage);
    else res_warp_sort<K, 32>(src, dst, len, stage);
  }
  if (a.tstamp && c == 0 && tid == 0) a.tstamp[5] = res_now();
  SR_RES_STAMP(7);
}

}  // namespace sr
