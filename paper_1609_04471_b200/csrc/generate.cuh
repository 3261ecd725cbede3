// generate.cuh -- on-device generator of the paper's input classes (SURVEY.md
// §8(f) NEXT #4; §2, lines 56-87), bit-identical to workloads/gen.py
// on the same seed so that the bench can build 1 GiB inputs on the GPU.
//
// PRNG: splitmix64 as a counter-based generator, draw i (0-based) of stream
// `seed` = mix64(seed + (i + 1) * 0x9E3779B97F4A7C15) (any
// seedable generator with a published algorithm); U[0, m) = the
// multiply-high approximation ((d >> 32) * m + (((d & 0xffffffff) * m) >> 32))
// >> 32, exactly as workloads/gen.py computes it.  Sequential constructions
// (swaps applied in draw order, Fisher-Yates shuffles, rejection sampling of
// the few-unique values) run on one thread, or one thread per independent
// block; everything else is one grid-stride pass.
#pragma once
#include <cstdint>

#include "common.cuh"

namespace sr {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;

__host__ __device__ __forceinline__ uint64_t gen_draw(uint64_t seed, uint64_t i) { return mix64(seed + (i + 1) * kGamma); }

__host__ __device__ __forceinline__ uint64_t gen_below(uint64_t d, uint64_t m) {
  const uint64_t t = (d >> 32) * m + (((d & 0xffffffffULL) * m) >> 32);
  return t >> 32;
}

template <typename K>
__host__ __device__ __forceinline__ K gen_uniform_key(uint64_t d) {
  if constexpr (sizeof(K) == 4) return (K)(int32_t)(uint32_t)(d >> 32);
  else return (K)(int64_t)d;
}

// section j of k equal sections of [0, n): bounds floor(j n / k)
__device__ __forceinline__ int64_t gen_bound(int64_t j, int64_t n, int64_t k) { return (j * n) / k; }
__device__ __forceinline__ int64_t gen_section(int64_t i, int64_t n, int64_t k) {
  int64_t j = (i * k) / n;
  while (j + 1 < k && gen_bound(j + 1, n, k) <= i) j++;
  while (j > 0 && gen_bound(j, n, k) > i) j--;
  return j;
}

// Element-wise classes (order codes: include/sr_sort.h SR_GEN_*).
template <typename K>
__global__ void k_gen_map(K* __restrict__ out, int64_t n, int order, uint64_t seed, int64_t param,
                          const K* __restrict__ table, const int64_t* __restrict__ perm) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    K v;
    switch (order) {
      case 0:  // random: uniform over the full range (G1)
        v = gen_uniform_key<K>(gen_draw(seed, i));
        break;
      case 2:  // reversed ramp (k-sharp teeth with k = 1)
        v = (K)(n - 1 - i);
        break;
      case 4: {  // few unique: a[i] = table[U[0, m)] (k-limited analogue)
        v = table[gen_below(gen_draw(seed ^ 0xF00DULL, i), (uint64_t)param)];
        break;
      }
      case 5: {  // runs of L: ramp blocks in the order perm (BASELINE configs[2]); the short last
                 // block (n % L keys, if any) sits at order position perm[nb]
        const int64_t L = param, nb = (n + L - 1) / L, shortlen = n - (nb - 1) * L, ts = perm[nb];
        int64_t t, st;
        if (i < ts * L) { t = i / L; st = t * L; }
        else if (i < ts * L + shortlen) { t = ts; st = ts * L; }
        else { t = ts + 1 + (i - ts * L - shortlen) / L; st = t * L - (L - shortlen); }
        v = (K)(perm[t] * L + (i - st));
        break;
      }
      case 6:  // ramp, the last `param` positions uniform random (BASELINE configs[2])
        v = i < n - param ? (K)i : gen_uniform_key<K>(gen_draw(seed, i - (n - param)));
        break;
      case 7: {  // k-sharp teeth: ramp, 1-based odd sections reversed
        const int64_t j = gen_section(i, n, param);
        v = (j % 2 == 0) ? (K)(gen_bound(j, n, param) + gen_bound(j + 1, n, param) - 1 - i) : (K)i;
        break;
      }
      case 8: {  // k-equal teeth: sections each a ramp 1..n/k
        const int64_t j = gen_section(i, n, param);
        v = (K)(i - gen_bound(j, n, param) + 1);
        break;
      }
      case 9: {  // k-even teeth: equal teeth with 1-based odd sections reversed
        const int64_t j = gen_section(i, n, param);
        v = (j % 2 == 0) ? (K)(gen_bound(j + 1, n, param) - i) : (K)(i - gen_bound(j, n, param) + 1);
        break;
      }
      case 11:  // all equal (k-limited with k = 0)
        v = (K)param;
        break;
      case 12: {  // extremes: MIN / MAX / 0 / -1 / 1 / MIN+1 / MAX-1
        v = table[gen_below(gen_draw(seed, i), 7)];
        break;
      }
      default:  // 1 sorted, 3 swaps, 10 distance: the ramp (the permutations follow)
        v = (K)i;
        break;
    }
    out[i] = v;
  }
}

// swaps: k random position swaps applied in draw order, p = U(draw 2j), q = U(draw 2j+1) (k-exchange)
template <typename K>
__global__ void k_gen_swaps(K* __restrict__ out, int64_t n, uint64_t seed, int64_t k) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  for (int64_t j = 0; j < k; j++) {
    const int64_t p = (int64_t)gen_below(gen_draw(seed, 2 * j), (uint64_t)n);
    const int64_t q = (int64_t)gen_below(gen_draw(seed, 2 * j + 1), (uint64_t)n);
    const K t = out[p];
    out[p] = out[q];
    out[q] = t;
  }
}

// k-distance: blocks of k+1 positions, each Fisher-Yates shuffled; the draws
// continue across blocks (block b starts at draw b k)
template <typename K>
__global__ void k_gen_distance(K* __restrict__ out, int64_t n, uint64_t seed, int64_t k) {
  const int64_t B = k + 1;
  const int64_t nblocks = (n + B - 1) / B;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nblocks; b += stride) {
    const int64_t s = b * B, len = (s + B < n ? s + B : n) - s;
    int64_t di = b * (B - 1);
    for (int64_t i = len - 1; i > 0; i--) {
      const int64_t j = (int64_t)gen_below(gen_draw(seed, di++), (uint64_t)(i + 1));
      const K t = out[s + i];
      out[s + i] = out[s + j];
      out[s + j] = t;
    }
  }
}

// runs of L: Fisher-Yates over the block order, draw (nb - 1 - i) for position
// i; perm[nb] = the order position of the last block
__global__ void k_gen_perm(int64_t* __restrict__ perm, int64_t nb, uint64_t seed) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  for (int64_t i = 0; i < nb; i++) perm[i] = i;
  for (int64_t i = nb - 1; i > 0; i--) {
    const int64_t j = (int64_t)gen_below(gen_draw(seed, nb - 1 - i), (uint64_t)(i + 1));
    const int64_t t = perm[i];
    perm[i] = perm[j];
    perm[j] = t;
  }
  for (int64_t i = 0; i < nb; i++)
    if (perm[i] == nb - 1) perm[nb] = i;
}

// few unique: the first m distinct values of the stream (rejection), draw idx = 0, 1, ...
template <typename K>
__global__ void k_gen_table(K* __restrict__ table, int64_t m, uint64_t seed) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  int64_t have = 0;
  for (uint64_t idx = 0; have < m; idx++) {
    const K v = gen_uniform_key<K>(gen_draw(seed, idx));
    bool seen = false;
    for (int64_t t = 0; t < have && !seen; t++) seen = table[t] == v;
    if (!seen) table[have++] = v;
  }
}

}  // namespace sr
