// bucket_sort.cuh -- the large keys-only path's second partition level fused
// with the bucket finishing (H7-H11 on one level-1 bucket per CTA, DESIGN.md
// §6.3).
//
// Above the resident range the level-1 scatter leaves B1 buckets of ~n/B1 keys
// in the workspace.  The multi-kernel recursion (partition.cuh) then ran a
// whole second level -- count (HBM read, bucket-id write), scan, plan, a host
// round trip, scatter (HBM read of keys and ids, HBM write), finishing (HBM
// read + write) -- i.e. ~5N more traffic and five launches with their tails.
// Here ONE persistent kernel takes the level-1 buckets one per CTA (a
// level-1 bucket of <= 512 KB stays in L2 while its CTA works on it):
//   1. the bucket's sub-splitters (sampled by k_sample_sort, PAPER.md:157,
//      gamma flags PAPER.md:168) -> an Eytzinger tree in shared memory;
//   2. count: every key classified into 2 B2 bins (3-way ids, PAPER.md:158,
//      :163), shared-memory histogram (the bucket's only HBM read);
//   3. scatter: the bucket read again (L2), classified again, counting-sorted
//      per sub-tile in shared memory and written bin-contiguously into its
//      final range of `keys` (L2); equality keys are not moved ("spared from
//      the recursive calls");
//   4. finishing: every range bin <= PIECE keys is loaded by one warp (L2),
//      checked with is_sorted and sorted by the warp's register
//      network (two networks and a merge above NET keys, unit_sort.cuh) in
//      place; equality bins are filled with their splitter.  Range bins above
//      PIECE (skew only) are listed for k_finish (<= kCap) or for the host's
//      next partition level (> kCap), so every input is sorted correctly.
// HBM traffic of the step: one read of the workspace, one write of `keys`.
#pragma once
#include "common.cuh"
#include "partition.cuh"
#include "types.cuh"
#include "unit_sort.cuh"

namespace sr {

template <typename K>
struct BsCfg {
  static constexpr int NT = 512;                    // one CTA per SM
  static constexpr int NW = NT / 32;
  static constexpr int U = sizeof(K) == 4 ? 16 : 8; // keys per thread per sub-tile
  static constexpr int ST = NT * U;                 // sub-tile keys
  static constexpr int B2MAX = 512;                 // sub-buckets per level-1 bucket
  static constexpr int NB = 2 * B2MAX + 1;          // 3-way bins (+1 unused)
  static constexpr int PIECE = UnitNet<K>::PIECE;   // largest bin one warp sorts
  static constexpr int TARGET = 256;                // mean sub-bucket the host aims for
};

template <typename K>
struct BsSmem {
  using C = BsCfg<K>;
  K tree[2 * C::B2MAX];           // Eytzinger [1, B2) + the sorted splitters at [B2MAX, B2MAX + m)
  uint8_t eq[C::B2MAX];
  uint32_t bst[C::NB + 1];        // bin starts inside the bucket; bst[nb] = len
  uint32_t cur[C::NB];            // next output offset of each bin (scatter)
  uint32_t lcnt[C::NB];           // sub-tile counts
  uint32_t lst[C::NB];            // sub-tile starts inside the staging area
  union alignas(16) {
    struct {
      K stk[C::ST];
      uint16_t stb[C::ST];
    } s;
    K stage[C::NW][C::PIECE];     // finishing: one staging area per warp
  } u;
  uint32_t red[C::NW + 1];
  int seg;
};

// Bucket ids of U keys (lockstep Eytzinger descent, U-way ILP): i = #{t_j < x},
// id 2i + [x equals an equality splitter].
template <typename K, int BMAX, int U>
__device__ __forceinline__ void bs_classify(const K (&x)[U], int (&bin)[U], const K* tree, const uint8_t* eq, int m,
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

// Exclusive scan of cnt[0, nb) into out[0, nb); returns the total.  Each
// thread scans BPT consecutive bins.  All NT threads call (barriers inside;
// out[] is visible to every thread on return).
template <int NT, int NB>
__device__ __forceinline__ uint32_t bs_scan_bins(const uint32_t* cnt, uint32_t* out, int nb, uint32_t* red) {
  constexpr int BPT = (NB + NT - 1) / NT;
  uint32_t v[BPT], s = 0;
#pragma unroll
  for (int r = 0; r < BPT; r++) {
    const int b = threadIdx.x * BPT + r;
    v[r] = b < nb ? cnt[b] : 0u;
    s += v[r];
  }
  uint32_t tot;
  uint32_t p = block_exclusive_sum<NT>(s, red, &tot);
#pragma unroll
  for (int r = 0; r < BPT; r++) {
    const int b = threadIdx.x * BPT + r;
    if (b < nb) out[b] = p;
    p += v[r];
  }
  __syncthreads();
  return tot;
}

template <typename K>
__global__ void __launch_bounds__(BsCfg<K>::NT, 1)
    k_bucket_sort(const K* __restrict__ src, K* __restrict__ dst, const SegDesc* __restrict__ segs, int nseg,
                  const K* __restrict__ spl_all, const uint8_t* __restrict__ eq_all, const int* __restrict__ m_all,
                  uint32_t* __restrict__ counter, Item* __restrict__ big, OvfSeg* __restrict__ ovf,
                  DevStats* __restrict__ st, int skip) {
  using C = BsCfg<K>;
  using SM = BsSmem<K>;
  constexpr int NT = C::NT, U = C::U, ST = C::ST, BMAX = C::B2MAX, NW = C::NW;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (;;) {
    if (tid == 0) sm.seg = (int)atomicAdd(counter, 1u);
    __syncthreads();
    const int s = sm.seg;
    if (s >= nseg) break;
    const SegDesc sd = segs[s];
    const int64_t start = sd.start;
    const int len = (int)sd.len;
    const int m = m_all[s];
    const int depth = tree_depth(m);
    const int nb = 2 * (1 << depth);  // ids 0 .. 2 (2^depth - 1) + 1
    const K* sk = src + start;
    K* dk = dst + start;
    // 1. splitters -> tree (sorted copy at [BMAX, ...), +inf padded)
    {
      const K* spl = spl_all + (int64_t)s * kMaxBuckets;
      const uint8_t* eqs = eq_all + (int64_t)s * kMaxBuckets;
      const int nodes = 1 << depth;
      for (int i = tid; i < nodes; i += NT) {
        sm.tree[BMAX + i] = i < m ? spl[i] : KeyTraits<K>::max_key();
        sm.eq[i] = i < m ? eqs[i] : 0;
        if (i >= 1) {
          const int d = 31 - __clz(i);
          const int pos = ((2 * (i - (1 << d)) + 1) << (depth - 1 - d)) - 1;
          sm.tree[i] = pos < m ? spl[pos] : KeyTraits<K>::max_key();
        }
      }
      for (int b = tid; b < nb; b += NT) sm.lcnt[b] = 0u;
    }
    __syncthreads();
    // 2. count (the bucket's HBM read; U loads per thread in flight)
    for (int i0 = 0; i0 < len; i0 += ST) {
      K x[U];
      int bin[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int i = i0 + u * NT + tid;
        x[u] = i < len ? sk[i] : K(0);
      }
      bs_classify<K, BMAX, U>(x, bin, sm.tree, sm.eq, m, depth);
#pragma unroll
      for (int u = 0; u < U; u++)
        if (i0 + u * NT + tid < len) atomicAdd(&sm.lcnt[bin[u]], 1u);
    }
    __syncthreads();
    bs_scan_bins<NT, C::NB>(sm.lcnt, sm.bst, nb, sm.red);
    for (int b = tid; b < nb; b += NT) sm.cur[b] = sm.bst[b];
    if (tid == 0) sm.bst[nb] = (uint32_t)len;
    __syncthreads();
    // 3. scatter, sub-tile by sub-tile (the second read hits L2)
    for (int i0 = 0; i0 < ((skip & 2) ? 0 : len); i0 += ST) {
      for (int b = tid; b < nb; b += NT) sm.lcnt[b] = 0u;
      K x[U];
      int bin[U];
      uint32_t rk[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int i = i0 + u * NT + tid;
        x[u] = i < len ? sk[i] : K(0);
      }
      bs_classify<K, BMAX, U>(x, bin, sm.tree, sm.eq, m, depth);
      __syncthreads();  // lcnt zeroed
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int i = i0 + u * NT + tid;
        // range bins only: equality keys are filled later
        if (i >= len || (bin[u] & 1)) bin[u] = -1;
        else rk[u] = atomicAdd(&sm.lcnt[bin[u]], 1u);
      }
      __syncthreads();
      const uint32_t tot = bs_scan_bins<NT, C::NB>(sm.lcnt, sm.lst, nb, sm.red);
#pragma unroll
      for (int u = 0; u < U; u++) {
        if (bin[u] >= 0) {
          const uint32_t p = sm.lst[bin[u]] + rk[u];
          sm.u.s.stk[p] = x[u];
          sm.u.s.stb[p] = (uint16_t)bin[u];
        }
      }
      __syncthreads();
      for (int p = tid; p < (int)tot; p += NT) {
        const int b = sm.u.s.stb[p];
        dk[sm.cur[b] + (uint32_t)p - sm.lst[b]] = sm.u.s.stk[p];
      }
      __syncthreads();
      for (int b = tid; b < nb; b += NT) sm.cur[b] += sm.lcnt[b];
    }
    __syncthreads();  // every bin of this bucket is in place in dst (visible to the CTA)
    // 4. finishing: warp w takes sub-buckets r = w, w + NW, ...: range bin 2r, equality bin 2r + 1
    K* stage = sm.u.stage[w];
    for (int r = w; 2 * r < ((skip & 1) ? 0 : nb); r += NW) {
      const int b = 2 * r;
      const int o = (int)sm.bst[b], c = (int)(sm.bst[b + 1] - sm.bst[b]);
      if (c > C::PIECE) {  // skew: a CTA item (<= kCap) or the host's next level
        if (lane == 0) {
          if (c <= kCap) {
            Item it;
            it.start = start + o; it.len = c; it.kind = kItemSort; it.key = 0;
            big[atomicAdd((unsigned long long*)&st->n_items_big, 1ull)] = it;
            atomicAdd((unsigned long long*)&st->big_keys, (unsigned long long)c);
          } else {
            OvfSeg q;
            q.start = start + o; q.len = c;
            ovf[atomicAdd((unsigned long long*)&st->n_ovf, 1ull)] = q;
            atomicAdd((unsigned long long*)&st->ovf_keys, (unsigned long long)c);
          }
        }
      } else if (c > 1) {
        constexpr int UL = 8;
        for (int j0 = 0; j0 < c; j0 += 32 * UL) {
          K v[UL];
#pragma unroll
          for (int q = 0; q < UL; q++) {
            const int j = j0 + q * 32 + lane;
            v[q] = j < c ? __ldcg(dk + o + j) : K(0);
          }
#pragma unroll
          for (int q = 0; q < UL; q++) {
            const int j = j0 + q * 32 + lane;
            if (j < c) stage[j] = v[q];
          }
        }
        __syncwarp();
        int unsorted = 0;  // is_sorted
        for (int j = lane; j + 1 < c; j += 32) unsorted |= stage[j + 1] < stage[j];
        if (__any_sync(0xffffffffu, unsorted)) unit_warp_piece<K>(stage, c, dk + o);
        __syncwarp();
      }
      const int oe = (int)sm.bst[b + 1], ce = (int)(sm.bst[b + 2] - sm.bst[b + 1]);
      if (ce > 0) {  // equality bin: fill
        const K key = sm.tree[BMAX + r];
        for (int j = lane; j < ce; j += 32) dk[oe + j] = key;
      }
    }
    __syncthreads();  // shared memory reused by the next bucket
  }
}

}  // namespace sr
