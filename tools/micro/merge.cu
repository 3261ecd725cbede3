// micro-benchmark: one CTA (512 threads) merging two sorted 4096-key runs in shared
// memory with the merge-path pattern used by the resident kernel, in variants
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <typename LA, typename LB>
__device__ __forceinline__ int mp_search(LA a, int a_len, LB b, int b_len, int diag) {
  int lo = diag - b_len > 0 ? diag - b_len : 0;
  int hi = diag < a_len ? diag : a_len;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (!(b(diag - 1 - mid) < a(mid))) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <int VT>
__device__ __forceinline__ void merge_generic(const int* A, int la, const int* B, int lb, int* out) {
  for (int d0 = threadIdx.x * VT; d0 < la + lb; d0 += blockDim.x * VT) {
    int ai = mp_search([&](int i) { return A[i]; }, la, [&](int i) { return B[i]; }, lb, d0);
    int bi = d0 - ai;
#pragma unroll
    for (int i = 0; i < VT; i++) {
      if (d0 + i < la + lb) {
        const bool p = (bi >= lb) || (ai < la && !(B[bi] < A[ai]));
        out[(d0 + i) & 4095] = p ? A[ai] : B[bi];
        ai += p;
        bi += !p;
      }
    }
  }
}

// registers hold the current heads: one shared load per output
template <int VT>
__device__ __forceinline__ void merge_heads(const int* A, int la, const int* B, int lb, int* out) {
  for (int d0 = threadIdx.x * VT; d0 < la + lb; d0 += blockDim.x * VT) {
    int ai = mp_search([&](int i) { return A[i]; }, la, [&](int i) { return B[i]; }, lb, d0);
    int bi = d0 - ai;
    int a = ai < la ? A[ai] : INT32_MAX, b = bi < lb ? B[bi] : INT32_MAX;
    int r[VT];
#pragma unroll
    for (int i = 0; i < VT; i++) {
      const bool p = bi >= lb || (ai < la && !(b < a));
      r[i] = p ? a : b;
      if (p) { ai++; a = ai < la ? A[ai] : INT32_MAX; } else { bi++; b = bi < lb ? B[bi] : INT32_MAX; }
    }
#pragma unroll
    for (int i = 0; i < VT; i++)
      if (d0 + i < la + lb) out[(d0 + i) & 4095] = r[i];
  }
}

__global__ void k_bench(int variant, long long* cycles, int* sink) {
  __shared__ int A[4096], B[4096], O[4096];  // (the second half of the outputs overwrites O: timing only)
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) { A[i] = 2 * i; B[i] = 2 * i + 1; }
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < 10; rep++) {
    if (variant == 0) merge_generic<16>(A, 4096, B, 4096, O);
    else if (variant == 1) merge_generic<15>(A, 4096, B, 4096, O);
    else if (variant == 2) merge_heads<16>(A, 4096, B, 4096, O);
    else merge_heads<15>(A, 4096, B, 4096, O);
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[variant] = (t1 - t0) / 10;
  if (O[threadIdx.x] == -1) sink[0] = 1;
}

int main() {
  long long* c; int* s;
  cudaMalloc(&c, 64); cudaMalloc(&s, 64);
  for (int v = 0; v < 4; v++) { k_bench<<<1, 512>>>(v, c, s); }
  for (int v = 0; v < 4; v++) { k_bench<<<1, 512>>>(v, c, s); }
  long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
  const char* nm[4] = {"generic VT16", "generic VT15", "heads VT16", "heads VT15"};
  for (int v = 0; v < 4; v++) printf("%-14s %lld cycles per 8192-key merge (1 CTA, 512 thr)\n", nm[v], h[v]);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
