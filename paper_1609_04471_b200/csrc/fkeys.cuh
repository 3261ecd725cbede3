// fkeys.cuh -- floating-point keys (the paper's
// "random double" class, Table 3).
//
// Order: IEEE 754 totalOrder -- -NaN (larger payload first) < -inf < negative
// numbers < -0 < +0 < positive numbers < +inf < +NaN (larger payload last).
// For binary formats that order is the order of the sign-magnitude bit
// patterns, so x -> x ^ ((x >> (W-1)) & 0x7f..f) on the bits read as a signed
// W-bit integer maps it onto signed integer order (negative patterns have
// their magnitude bits flipped, positive ones are unchanged).  The map is its
// own inverse: the float sort is the integer sort bracketed by two in-place
// passes of this kernel (2 x (read + write) of the keys; values untouched, so
// stability of the pair sort carries over).  Keys equal in totalOrder are
// bit-identical, so the result is unique and comparable bit for bit.
#pragma once
#include <cstdint>

namespace sr {

template <typename I>
__global__ void k_fkey_flip(I* __restrict__ keys, int64_t n) {
  constexpr int W = 8 * (int)sizeof(I);
  const I mag = (I)(~((uint64_t)1 << (W - 1)));  // 0x7f..f
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if ((reinterpret_cast<uintptr_t>(keys) & 15) == 0) {  // 16-byte vectors
    constexpr int V = 16 / (int)sizeof(I);
    const int64_t nv = n / V;
    for (int64_t v = i; v < nv; v += stride) {
      int4 q = reinterpret_cast<int4*>(keys)[v];
      I x[V];
      memcpy(x, &q, 16);
#pragma unroll
      for (int j = 0; j < V; j++) x[j] ^= (x[j] >> (W - 1)) & mag;
      memcpy(&q, x, 16);
      reinterpret_cast<int4*>(keys)[v] = q;
    }
    for (int64_t t = nv * V + i; t < n; t += stride) keys[t] ^= (keys[t] >> (W - 1)) & mag;
  } else {
    for (int64_t t = i; t < n; t += stride) keys[t] ^= (keys[t] >> (W - 1)) & mag;
  }
}

}  // namespace sr
