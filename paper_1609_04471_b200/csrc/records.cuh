// records.cuh -- record keys: the paper's "random
// 16-/64-/256-list" classes, lists of int32 compared lexicographically
// (Table 2).
//
// A record is `words` consecutive signed int32 values; the order is the
// lexicographic one.  The sort refines an index permutation by rounds of the
// stable int64 pair sort (key, idx).  Word j's values are first reduced to
// their range [min_j, max_j]; its field is (w_j - min_j) in b_j = bits(max_j -
// min_j) bits (0 for a constant word, which is skipped), so comparing fields
// compares the words.  A round's 64-bit key concatenates, most significant
// first, the segment id of the record (rounds >= 1: the runs of records equal
// in every word so far, numbered in order) and the fields of as many of the
// next words as fit: the key order is the lexicographic order of those words
// within each segment.  The pair sort is stable, so records equal in every
// word keep their input order (they are bit-identical, so the output is
// unique).  Rounds stop when no two adjacent keys are equal or the words are
// exhausted; a final gather permutes the records.  (Lists whose words take
// few values -- the shared-prefix class -- pack many words per round: 15
// ternary words and a random one are ONE round.)
#pragma once
#include <cstdint>

namespace sr {

// per-word minimum / maximum (mm[2j] = min, mm[2j+1] = max; preset to
// INT32_MAX / INT32_MIN by the host)
__global__ void k_rec_minmax(const int32_t* __restrict__ recs, int64_t n, int words, int32_t* __restrict__ mm) {
  const int64_t total = n * words;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (stride % words == 0) {  // every thread visits one word position: private min / max
    const int j = (int)(t0 % words);
    int32_t lo = INT32_MAX, hi = INT32_MIN;
    for (int64_t t = t0; t < total; t += stride) {
      const int32_t v = recs[t];
      lo = min(lo, v);
      hi = max(hi, v);
    }
    if (t0 < total) {
      atomicMin(mm + 2 * j, lo);
      atomicMax(mm + 2 * j + 1, hi);
    }
    return;
  }
  for (int64_t t = t0; t < total; t += stride) {
    const int j = (int)(t % words);
    const int32_t v = recs[t];
    atomicMin(mm + 2 * j, v);
    atomicMax(mm + 2 * j + 1, v);
  }
}

// One round's fields: words wl[0..nw) with minima wmin[] and widths wbits[]
// (sum of the widths + seg_bits <= 64).
struct RecRound {
  int32_t nw, seg_bits, shift;  // shift = 64 - (seg_bits + the widths)
  int32_t wl[64];
  int32_t wmin[64];
  int32_t wbits[64];
};

// key of record r = idx[i] (round 0: idx = identity, written here): the
// segment id (ex[i] + flag, rounds >= 1) then the round's word fields, as an
// unsigned 64-bit value mapped to signed order (top bit flipped)
__global__ void k_rec_key(const int32_t* __restrict__ recs, int64_t n, int words, RecRound rr,
                          const uint32_t* __restrict__ ex, const int64_t* __restrict__ key_in,
                          int64_t* __restrict__ key_out, uint32_t* __restrict__ idx) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint64_t k = 0;
    int64_t r = i;
    if (ex) {  // rounds >= 1: flag recomputed from the previous keys (the scan overwrote it)
      const bool b = i > 0 && key_in[i] != key_in[i - 1];
      k = (uint64_t)ex[i] + (b ? 1u : 0u);
      r = idx[i];
    } else {
      idx[i] = (uint32_t)i;
    }
    const int32_t* rec = recs + r * words;
    for (int q = 0; q < rr.nw; q++) {
      const int b = rr.wbits[q];
      const uint64_t f = (uint64_t)((uint32_t)rec[rr.wl[q]] - (uint32_t)rr.wmin[q]);  // < 2^b
      k = (k << b) | f;
    }
    if (rr.shift < 64) k <<= rr.shift;
    else k = 0;
    key_out[i] = (int64_t)(k ^ 0x8000000000000000ull);
  }
}

// boundary flags of the sorted keys (flag[i] = key[i] != key[i-1], flag[0] = 0)
// and whether any two adjacent keys are equal (a further round is needed);
// ctl[0] |= tie, ctl[1] += the number of boundaries (segments - 1)
__global__ void k_rec_flags(const int64_t* __restrict__ key, int64_t n, uint32_t* __restrict__ flag,
                            uint32_t* __restrict__ ctl) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool tie = false;
  uint32_t nb = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const bool b = i > 0 && key[i] != key[i - 1];
    flag[i] = b ? 1u : 0u;
    nb += b;
    tie |= i > 0 && !b;
  }
  if (__any_sync(0xffffffffu, tie) && (threadIdx.x & 31) == 0) atomicOr(ctl, 1u);
  for (int o = 16; o > 0; o >>= 1) nb += __shfl_xor_sync(0xffffffffu, nb, o);
  if ((threadIdx.x & 31) == 0 && nb) atomicAdd(ctl + 1, nb);
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
