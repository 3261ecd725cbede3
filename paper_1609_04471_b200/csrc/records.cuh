// records.cuh -- record keys: the paper's "random
// 16-/64-/256-list" classes, lists of int32 compared lexicographically
// (Table 2).
//
// A record is `words` consecutive signed int32 values; the order is the
// lexicographic one.  The sort refines an index permutation: round 0 sorts
// (idx) by the 64-bit key (w0, w1) (w0 in the high half, w1 biased into the
// unsigned low half, so signed int64 order is the lexicographic order of the
// pair); every later round r sorts by (segment id, word r + 1), where the
// segment id numbers the runs of records equal in all words so far.  The pair
// sort is stable, so records equal in every word keep their input order (they
// are bit-identical, so the output is unique).  Rounds stop when every
// segment is a single record or the words are exhausted; a final gather
// permutes the records.
#pragma once
#include <cstdint>

namespace sr {

// round 0: key = (w0, w1) or w0 alone; idx = identity
__global__ void k_rec_init(const int32_t* __restrict__ recs, int64_t n, int words, int64_t* __restrict__ key,
                           uint32_t* __restrict__ idx) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int32_t* r = recs + i * words;
    key[i] = words >= 2 ? (int64_t)(((uint64_t)(uint32_t)r[0] << 32) | (uint32_t)(r[1] ^ INT32_MIN)) : (int64_t)r[0];
    idx[i] = (uint32_t)i;
  }
}

// boundary flags of the sorted keys (flag[i] = key[i] != key[i-1], flag[0] = 0)
// and whether any two adjacent keys are equal (a further round is needed)
__global__ void k_rec_flags(const int64_t* __restrict__ key, int64_t n, uint32_t* __restrict__ flag,
                            uint32_t* __restrict__ any_tie) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool tie = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const bool b = i > 0 && key[i] != key[i - 1];
    flag[i] = b ? 1u : 0u;
    tie |= i > 0 && !b;
  }
  if (__any_sync(0xffffffffu, tie) && (threadIdx.x & 31) == 0) atomicOr(any_tie, 1u);
}

// round r >= 1: key = (segment id, word w of the record); ex = exclusive scan of the flags
__global__ void k_rec_next(const int32_t* __restrict__ recs, int64_t n, int words, int w,
                           const uint32_t* __restrict__ ex, const int64_t* __restrict__ key_in,
                           int64_t* __restrict__ key_out, const uint32_t* __restrict__ idx) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const bool b = i > 0 && key_in[i] != key_in[i - 1];  // the flag, recomputed (the scan overwrote it)
    const uint64_t seg = (uint64_t)ex[i] + (b ? 1u : 0u);
    key_out[i] = (int64_t)((seg << 32) | (uint32_t)(recs[(int64_t)idx[i] * words + w] ^ INT32_MIN));
  }
}

// out[i] = recs[idx[i]] (words int32 each)
__global__ void k_rec_gather(const int32_t* __restrict__ recs, int64_t n, int words, const uint32_t* __restrict__ idx,
                             int32_t* __restrict__ out) {
  const int64_t total = n * words;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
    const int64_t i = t / words;
    const int j = (int)(t - i * words);
    out[t] = recs[(int64_t)idx[i] * words + j];
  }
}

}  // namespace sr
