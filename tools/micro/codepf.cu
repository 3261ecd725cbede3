// Can a kernel read (and prefetch into L2) its own instruction bytes?  The
// device-side address of a __global__ function is read as data and compared
// with the cubin's encoding; then a code-heavy kernel is timed after an L2
// flush with and without a prior L2 prefetch of its code range.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define REP8(x) x x x x x x x x
#define REP64(x) REP8(REP8(x))
#define REP512(x) REP8(REP64(x))

__global__ void big(uint32_t* out, uint32_t s) {
  uint32_t a = s + threadIdx.x, b = s ^ 0x9e3779b9u;
  // ~12K straight-line instructions (no loop: every one is fetched once)
  REP512(a = a * 0x01000193u + b; b ^= a >> 7; a += b << 3;)
  REP512(a = a * 0x01000193u + b; b ^= a >> 7; a += b << 3;)
  REP512(a = a * 0x01000193u + b; b ^= a >> 7; a += b << 3;)
  REP512(a = a * 0x01000193u + b; b ^= a >> 7; a += b << 3;)
  if (a == 0x12345678u) out[0] = a + b;
}

__global__ void probe(unsigned long long* out) {
  unsigned long long a;
  asm volatile("mov.b64 %0, %1;" : "=l"(a) : "l"((const void*)big));
  out[0] = a;
  const uint32_t* q = (const uint32_t*)a;
  for (int i = 0; i < 8; i++) out[1 + i] = 0;
  (void)q;
}

__global__ void pf(const char* base, size_t bytes) {
  for (size_t o = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 128; o < bytes; o += (size_t)gridDim.x * blockDim.x * 128)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(base + o));
}
__global__ void flush(uint4* b, size_t n, uint32_t v) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = make_uint4(v, v, v, v);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64 * 8);
  probe<<<1, 1>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  printf("probe: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  unsigned long long h[9];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("big at 0x%llx, first words:", h[0]);
  for (int i = 1; i < 9; i++) printf(" %08llx", h[i]);
  printf("\n");
  uint32_t* o;
  cudaMalloc(&o, 4);
  size_t fl = (size_t)512 << 20;
  uint4* fb;
  cudaMalloc(&fb, fl);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; mode++) {
    float tot = 0;
    for (int it = 0; it < 6; it++) {
      flush<<<1184, 512>>>(fb, fl / 16, it);
      if (mode == 1) pf<<<148, 128>>>((const char*)h[0], 256 << 10);
      if (mode == 2) { big<<<148, 512>>>(o, 1); }  // warm
      cudaEventRecord(e0);
      big<<<148, 512>>>(o, it);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it) tot += ms;
    }
    printf("mode %d (%s): %.1f us\n", mode, mode == 0 ? "cold after flush" : mode == 1 ? "L2 prefetch of code" : "warm", tot / 5 * 1e3);
  }
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
