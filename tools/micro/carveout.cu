// micro-benchmark: device time of an (almost) empty 148x512 cooperative kernel
// with 0 / 210 KB dynamic shared memory, launched after a plain elementwise
// kernel (L1-heavy carveout) -- is there a carveout-switch cost per launch?
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void k_fill(float* p, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = i;
}
__global__ void k_coop(int* c) {
  __shared__ int sm[1];
  if (threadIdx.x == 0) sm[0] = blockIdx.x;
  __syncthreads();
  cg::this_grid().sync();
  if (threadIdx.x == 0) atomicAdd(c, sm[0] & 1);
}
int main() {
  cudaStream_t s; cudaStreamCreate(&s);
  int* c; cudaMalloc(&c, 64);
  float* f; const int nf = 1 << 20; cudaMalloc(&f, nf * 4);
  cudaFuncSetAttribute(k_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1, e2; cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
  for (int smem : {0, 48 * 1024, 100 * 1024, 210 * 1024}) {
    for (int fill : {0, 1}) {
      float tot = 0; const int R = 200;
      for (int r = 0; r < R + 5; r++) {
        if (fill) k_fill<<<592, 256, 0, s>>>(f, nf);
        cudaEventRecord(e1, s);
        void* args[] = {&c};
        cudaLaunchCooperativeKernel((void*)k_coop, 148, 512, args, smem, s);
        cudaEventRecord(e2, s);
        cudaStreamSynchronize(s);
        float ms; cudaEventElapsedTime(&ms, e1, e2);
        if (r >= 5) tot += ms;
      }
      printf("smem %6d after fill %d: coop kernel %6.2f us (event to event)\n", smem, fill, tot / R * 1e3);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
