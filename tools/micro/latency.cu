// Latency micro-benchmark (one warp, and 16 warps concurrently): dependent
// shared-memory loads, dependent shuffles, dependent L2 loads, clock overhead.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(int* g, long long* out, int warps_active) {
  __shared__ int s[4096];
  const int tid = threadIdx.x, w = tid >> 5;
  for (int i = tid; i < 4096; i += blockDim.x) s[i] = (i * 17 + 5) & 4095;
  __syncthreads();
  if (w >= warps_active) return;
  int p = tid & 31;
  long long t0 = clock64();
  for (int i = 0; i < 1000; i++) p = s[p];
  long long t1 = clock64();
  int v = p;
  long long t2 = clock64();
  for (int i = 0; i < 1000; i++) v = __shfl_xor_sync(0xffffffffu, v, 1) + 1;
  long long t3 = clock64();
  int q = (tid * 64) & ((1 << 20) - 1);
  long long t4 = clock64();
  for (int i = 0; i < 200; i++) q = __ldcg(g + q);
  long long t5 = clock64();
  if (tid == 0) {
    out[0] = (t1 - t0) / 1000;
    out[1] = (t3 - t2) / 1000;
    out[2] = (t5 - t4) / 200;
    out[3] = p + v + q;
  }
}

int main() {
  int* g;
  long long* o;
  cudaMalloc(&g, 4 << 20);
  cudaMalloc(&o, 64);
  int* h = new int[1 << 20];
  for (int i = 0; i < (1 << 20); i++) h[i] = (int)(((long long)i * 7919 + 12345) % (1 << 20));
  cudaMemcpy(g, h, 4 << 20, cudaMemcpyHostToDevice);
  for (int wa : {1, 16}) {
    for (int it = 0; it < 2; it++) k_lat<<<1, 512>>>(g, o, wa);
    long long r[4];
    cudaMemcpy(r, o, 32, cudaMemcpyDeviceToHost);
    printf("%2d warps: dependent LDS %lld cycles, dependent SHFL+IADD %lld cycles, dependent L2 load %lld cycles\n", wa,
           r[0], r[1], r[2]);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
