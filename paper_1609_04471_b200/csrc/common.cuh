// common.cuh -- shared device helpers for the sr_sort kernels (sm_100a only).
//
// Nothing here is shared with oracle/ (the two share no code).
#pragma once
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "sr_sort is written for sm_100a (B200) only"
#endif

// Checked build (build.py --checked: -DSR_CHECKED, libsr_sort_checked.so):
// SR_CHECK asserts an index or range on the device and traps with its source
// line on a violation (the pool does not allow compute-sanitizer; the checked
// library runs the GPU test suite instead).  No code in the normal build.
#ifdef SR_CHECKED
#define SR_CHECK(cond)                                                              \
  do {                                                                              \
    if (!(cond)) {                                                                  \
      printf("[sr checked] %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
             (int)blockIdx.x, (int)threadIdx.x);                                     \
      __trap();                                                                     \
    }                                                                               \
  } while (0)
#else
#define SR_CHECK(cond) \
  do {                 \
  } while (0)
#endif

namespace sr {

constexpr int kWarp = 32;

// ---- key traits: ascending signed order -------------------------
template <typename K> struct KeyTraits;
template <> struct KeyTraits<int32_t> {
  static __host__ __device__ __forceinline__ int32_t max_key() { return INT32_MAX; }
  static __host__ __device__ __forceinline__ int32_t min_key() { return INT32_MIN; }
  using AtomicT = int;
  static constexpr int kPadEvery = 32;   // one pad element per 128 B of smem
};
template <> struct KeyTraits<int64_t> {
  static __host__ __device__ __forceinline__ int64_t max_key() { return INT64_MAX; }
  static __host__ __device__ __forceinline__ int64_t min_key() { return INT64_MIN; }
  using AtomicT = long long;
  static constexpr int kPadEvery = 16;
};

// Padded shared-memory index: one spare slot every 128 bytes so that a warp
// reading "blocked" items (thread t, item i -> t*VT+i) hits distinct banks.
template <typename T>
__host__ __device__ __forceinline__ int pad_idx(int i) {
  return i + i / (128 / (int)sizeof(T));
}
template <typename T>
__host__ __device__ constexpr int padded_size(int n) {
  return n + n / (128 / (int)sizeof(T)) + 1;
}

// ---- counter-based jitter (splitmix64 finalizer, published generator) ------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// Stratified jittered sample position k of segment [start, start+len) with S
// strata ("jittered regular positions ... deterministic"): stratum
// k is [k*len/S, (k+1)*len/S), offset = floor(h*w / 2^64) for the k-th jitter
// draw h and stratum width w.  log2S >= 0 selects the shift form of the
// division (S a power of two).
__host__ __device__ __forceinline__ int64_t sample_position(int64_t start, int64_t len, int64_t S, int64_t k,
                                                          int log2S = -1) {
  int64_t lo, hi;
  if (log2S >= 0) {
    lo = (k * len) >> log2S;
    hi = ((k + 1) * len) >> log2S;
  } else {
    lo = (k * len) / S;
    hi = ((k + 1) * len) / S;
  }
  uint64_t w = (uint64_t)(hi - lo);
  uint64_t h = mix64((uint64_t)start + (uint64_t)(k + 1) * 0x9E3779B97F4A7C15ULL);
#ifdef __CUDA_ARCH__
  uint64_t off = __umul64hi(h, w);
#else
  uint64_t off = (uint64_t)(((unsigned __int128)h * w) >> 64);
#endif
  return start + lo + (int64_t)off;
}

// ---- warp / block scans ----------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_inclusive_sum(T v) {
#pragma unroll
  for (int o = 1; o < kWarp; o <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) >= o) v += u;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_inclusive_max(T v) {
#pragma unroll
  for (int o = 1; o < kWarp; o <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) >= o) v = v > u ? v : u;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_reduce_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_reduce_min(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) { T u = __shfl_xor_sync(0xffffffffu, v, o); v = u < v ? u : v; }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_reduce_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) { T u = __shfl_xor_sync(0xffffffffu, v, o); v = u > v ? u : v; }
  return v;
}
// 32- and 64-bit signed keys: the warp reduction instruction (redux.sync), a
// 64-bit key as its high word, then the low words of the lanes that hold it.
template <>
__device__ __forceinline__ int32_t warp_reduce_min<int32_t>(int32_t v) {
  return __reduce_min_sync(0xffffffffu, v);
}
template <>
__device__ __forceinline__ int32_t warp_reduce_max<int32_t>(int32_t v) {
  return __reduce_max_sync(0xffffffffu, v);
}
template <>
__device__ __forceinline__ int64_t warp_reduce_min<int64_t>(int64_t v) {
  const int32_t hi = __reduce_min_sync(0xffffffffu, (int32_t)(v >> 32));
  const unsigned lo = __reduce_min_sync(0xffffffffu, (int32_t)(v >> 32) == hi ? (unsigned)v : 0xffffffffu);
  return (int64_t)(((uint64_t)(uint32_t)hi << 32) | lo);
}
template <>
__device__ __forceinline__ int64_t warp_reduce_max<int64_t>(int64_t v) {
  const int32_t hi = __reduce_max_sync(0xffffffffu, (int32_t)(v >> 32));
  const unsigned lo = __reduce_max_sync(0xffffffffu, (int32_t)(v >> 32) == hi ? (unsigned)v : 0u);
  return (int64_t)(((uint64_t)(uint32_t)hi << 32) | lo);
}

// Block-wide exclusive sum. `scratch` needs NT/32 + 1 entries. Returns the
// exclusive prefix; *total receives the block sum. Contains __syncthreads().
template <int NT, typename T>
__device__ __forceinline__ T block_exclusive_sum(T v, T* scratch, T* total) {
  constexpr int NW = NT / kWarp;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T inc = warp_inclusive_sum(v);
  if (lane == 31) scratch[w] = inc;
  __syncthreads();
  if (w == 0) {
    T s = lane < NW ? scratch[lane] : T(0);
    T si = warp_inclusive_sum(s);
    if (lane < NW) scratch[lane] = si - s;
    if (lane == NW - 1) scratch[NW] = si;
  }
  __syncthreads();
  T r = scratch[w] + inc - v;
  if (total) *total = scratch[NW];
  __syncthreads();
  return r;
}

// Block-wide inclusive max (for "last break before me" scans).
template <int NT, typename T>
__device__ __forceinline__ T block_inclusive_max(T v, T* scratch, T identity) {
  constexpr int NW = NT / kWarp;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T inc = warp_inclusive_max(v);
  if (lane == 31) scratch[w] = inc;
  __syncthreads();
  if (w == 0) {
    T s = lane < NW ? scratch[lane] : identity;
    T si = warp_inclusive_max(s);
    // exclusive warp prefix
    T ex = __shfl_up_sync(0xffffffffu, si, 1);
    if (lane == 0) ex = identity;
    if (lane < NW) scratch[lane] = ex;
  }
  __syncthreads();
  T p = scratch[w];
  T r = inc > p ? inc : p;
  __syncthreads();
  return r;
}

template <int NT, typename T>
__device__ __forceinline__ T block_reduce_sum(T v, T* scratch) {
  constexpr int NW = NT / kWarp;
  T s = warp_reduce_sum(v);
  if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = s;
  __syncthreads();
  T r = 0;
#pragma unroll
  for (int i = 0; i < NW; i++) r += scratch[i];
  __syncthreads();
  return r;
}
template <int NT, typename T>
__device__ __forceinline__ T block_reduce_min(T v, T* scratch) {
  constexpr int NW = NT / kWarp;
  T s = warp_reduce_min(v);
  if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = s;
  __syncthreads();
  T r = scratch[0];
#pragma unroll
  for (int i = 1; i < NW; i++) r = scratch[i] < r ? scratch[i] : r;
  __syncthreads();
  return r;
}
template <int NT, typename T>
__device__ __forceinline__ T block_reduce_max(T v, T* scratch) {
  constexpr int NW = NT / kWarp;
  T s = warp_reduce_max(v);
  if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = s;
  __syncthreads();
  T r = scratch[0];
#pragma unroll
  for (int i = 1; i < NW; i++) r = scratch[i] > r ? scratch[i] : r;
  __syncthreads();
  return r;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace sr
