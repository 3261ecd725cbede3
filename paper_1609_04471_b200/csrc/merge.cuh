// merge.cuh -- natural-mergesort analogue (H5 merge-path partition, H6 merge
// round, run-boundary check, bulk copy).
//
// Paper anchors (§3; Appendix A):
//  (f) "Merge is always done among two consecutive sorted subarrays, say A and
//      B. Any element in A no bigger than the first element of B is removed
//      from the merge process. Similarly, any element of B bigger than the
//      last element of A is also removed" -> a CTA whose output
//      range is fed by one side only is a pure copy; a boundary that is
//      already ordered costs nothing (runs are coalesced before merging);
//  (g) galloping: "the binary search is used to locate the position in A where
//      the current element in B should go" -> the merge-path
//      diagonal search (K5), which splits every merge evenly across CTAs;
//  (e2) the half-down list (Appendix A) is the
//      host-side merge schedule; each level of that merge tree is one K6 launch.
#pragma once
#include "block_sort.cuh"
#include "common.cuh"

namespace sr {

// One stable merge A=[start, start+na) from abuf, B=[start+na, start+na+nb)
// from bbuf (same buffer after host-side harmonisation) into the other buffer.
struct MergeJob {
  int64_t start, na, nb;
  int64_t cta_begin;  // prefix of CTA counts over jobs
  int32_t src;        // 0 = primary (caller's arrays), 1 = workspace
  int32_t pad;
};

__device__ __forceinline__ int find_job(const MergeJob* jobs, int njobs, int64_t cta) {
  int lo = 0, hi = njobs - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].cta_begin <= cta) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Merge-path split in global memory: #A among the first d outputs of the
// stable merge of a[0..na) and b[0..nb) (A wins ties).  A trimmed pair
// (A.last <= B.first) needs no search.
template <typename K>
__device__ __forceinline__ int64_t merge_path_global(const K* a, int64_t na, const K* b, int64_t nb, int64_t d) {
  int64_t lo = d - nb > 0 ? d - nb : 0;
  int64_t hi = d < na ? d : na;
  if (nb == 0 || na == 0 || !(b[0] < a[na - 1])) return hi;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (!(b[d - 1 - mid] < a[mid])) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// K5: merge-path split for the first output of every CTA (one thread each).
template <typename K, int NV>
__global__ void k_merge_partition(const K* __restrict__ primary, const K* __restrict__ ws,
                                  const MergeJob* __restrict__ jobs, int njobs, int64_t total_ctas,
                                  int64_t* __restrict__ splits) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= total_ctas) return;
  const int j = find_job(jobs, njobs, c);
  const MergeJob jb = jobs[j];
  const K* a = (jb.src ? ws : primary) + jb.start;
  splits[c] = merge_path_global(a, jb.na, a + jb.na, jb.nb, (c - jb.cta_begin) * NV);
}

// Merge-path splits at arbitrary diagonals (step-level entry point for H5).
template <typename K>
__global__ void k_merge_path_diags(const K* __restrict__ a, int64_t na, const K* __restrict__ b, int64_t nb,
                                   const int64_t* __restrict__ diags, int64_t nd, int64_t* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nd) out[i] = merge_path_global(a, na, b, nb, diags[i]);
}

// K6: one merge level.  Each CTA produces NV = NT*VT outputs of one job.
template <typename K, bool HAS_V, int NT, int VT>
__global__ void __launch_bounds__(NT) k_merge(K* __restrict__ pk, uint32_t* __restrict__ pv, K* __restrict__ wk,
                                               uint32_t* __restrict__ wv, const MergeJob* __restrict__ jobs,
                                               int njobs, const int64_t* __restrict__ splits) {
  constexpr int NV = NT * VT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K* ks = reinterpret_cast<K*>(smem_raw);
  uint32_t* vs = reinterpret_cast<uint32_t*>(smem_raw + sizeof(K) * padded_size<K>(NV));
  __shared__ int s_j;
  const int64_t c = blockIdx.x;
  if (threadIdx.x == 0) s_j = find_job(jobs, njobs, c);
  __syncthreads();
  const MergeJob jb = jobs[s_j];
  const K* sk = jb.src ? wk : pk;
  const uint32_t* sv = jb.src ? wv : pv;
  K* dk = jb.src ? pk : wk;
  uint32_t* dv = jb.src ? pv : wv;
  const int64_t total = jb.na + jb.nb;
  const int64_t d0 = (c - jb.cta_begin) * NV;
  const int64_t d1 = d0 + NV < total ? d0 + NV : total;
  const bool last = (c + 1 == jb.cta_begin + (total + NV - 1) / NV);
  const int64_t i0 = splits[c];
  const int64_t i1 = last ? jb.na : splits[c + 1];
  const int64_t j0 = d0 - i0, j1 = d1 - i1;
  const int na = (int)(i1 - i0), nb = (int)(j1 - j0);
  const int cnt = na + nb;
  const K* A = sk + jb.start + i0;
  const K* B = sk + jb.start + jb.na + j0;
  K* out = dk + jb.start + d0;
  if (na == 0 || nb == 0) {  // one side only: pure copy (trimmed merge)
    const K* from = na ? A : B;
    const uint32_t* fv = sv + (na ? jb.start + i0 : jb.start + jb.na + j0);
    for (int i = threadIdx.x; i < cnt; i += NT) {
      out[i] = from[i];
      if (HAS_V) dv[jb.start + d0 + i] = fv[i];
    }
    return;
  }
  for (int i = threadIdx.x; i < cnt; i += NT) {
    K x = i < na ? A[i] : B[i - na];
    ks[pad_idx<K>(i)] = x;
    if (HAS_V) vs[pad_idx<uint32_t>(i)] = i < na ? sv[jb.start + i0 + i] : sv[jb.start + jb.na + j0 + i - na];
  }
  __syncthreads();
  const int diag = threadIdx.x * VT;
  K k[VT];
  int src[VT];
  if (diag < cnt) {
    int mp = merge_path_search<K>([&](int i) { return ks[pad_idx<K>(i)]; }, na,
                                  [&](int i) { return ks[pad_idx<K>(na + i)]; }, nb, diag);
    int ai = mp, bi = na + diag - mp;
    const int aend = na, bend = cnt;
    K ak = ai < aend ? ks[pad_idx<K>(ai)] : K(0);
    K bk = bi < bend ? ks[pad_idx<K>(bi)] : K(0);
#pragma unroll
    for (int i = 0; i < VT; i++) {
      bool take_a = (bi >= bend) || (ai < aend && !(bk < ak));
      k[i] = take_a ? ak : bk;
      src[i] = take_a ? ai : bi;
      if (take_a) { ++ai; if (ai < aend) ak = ks[pad_idx<K>(ai)]; }
      else { ++bi; if (bi < bend) bk = ks[pad_idx<K>(bi)]; }
    }
  }
  uint32_t v[VT];
  if (HAS_V && diag < cnt) {
#pragma unroll
    for (int i = 0; i < VT; i++) v[i] = vs[pad_idx<uint32_t>(src[i] < cnt ? src[i] : 0)];
  }
  __syncthreads();
  if (diag < cnt) {
#pragma unroll
    for (int i = 0; i < VT; i++) {
      if (diag + i < cnt) {
        ks[pad_idx<K>(diag + i)] = k[i];
        if (HAS_V) vs[pad_idx<uint32_t>(diag + i)] = v[i];
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < cnt; i += NT) {
    out[i] = ks[pad_idx<K>(i)];
    if (HAS_V) dv[jb.start + d0 + i] = vs[pad_idx<uint32_t>(i)];
  }
}

// Run-boundary check (H2 post-reversal check): flag[r] = 1 when the boundary
// in front of position pos[r] is out of order (a_{p-1} > a_p).
template <typename K>
__global__ void k_boundary_check(const K* __restrict__ keys, const int64_t* __restrict__ pos, int64_t count,
                                 uint8_t* __restrict__ flags, unsigned long long* __restrict__ nbad) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool bad = false;
  if (r < count) {
    int64_t p = pos[r];
    bad = keys[p] < keys[p - 1];
    flags[r] = bad ? 1 : 0;
  }
  unsigned b = __ballot_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(nbad, (unsigned long long)__popc(b));
}

// Copy ranges between the primary arrays and the workspace (dir 0: primary ->
// workspace, 1: workspace -> primary).  Used for result placement (H12).
struct CopyJob {
  int64_t start, len;
  int64_t cta_begin;
  int32_t dir, pad;
};

template <typename K, bool HAS_V, int NT>
__global__ void __launch_bounds__(NT) k_copy(K* __restrict__ pk, uint32_t* __restrict__ pv, K* __restrict__ wk,
                                              uint32_t* __restrict__ wv, const CopyJob* __restrict__ jobs, int njobs) {
  constexpr int U = 8;
  constexpr int CH = NT * U;
  __shared__ int s_j;
  if (threadIdx.x == 0) {
    int lo = 0, hi = njobs - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (jobs[mid].cta_begin <= (int64_t)blockIdx.x) lo = mid; else hi = mid - 1;
    }
    s_j = lo;
  }
  __syncthreads();
  const CopyJob jb = jobs[s_j];
  const K* sk = jb.dir ? wk : pk;
  K* dk = jb.dir ? pk : wk;
  const uint32_t* sv = jb.dir ? wv : pv;
  uint32_t* dv = jb.dir ? pv : wv;
  const int64_t c0 = ((int64_t)blockIdx.x - jb.cta_begin) * CH;
#pragma unroll
  for (int u = 0; u < U; u++) {
    int64_t p = c0 + u * NT + threadIdx.x;
    if (p < jb.len) {
      dk[jb.start + p] = sk[jb.start + p];
      if (HAS_V) dv[jb.start + p] = sv[jb.start + p];
    }
  }
}

}  // namespace sr
