// micro-benchmark: cost of back-to-back kernels whose shared-memory footprint
// differs (L1/smem carveout reconfiguration), with and without a fixed
// max-shared carveout preference; and the cost of a cooperative grid sync.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_small(const int* g, int* p) {
  if (*g != 7) return;
  if (threadIdx.x == 0) p[blockIdx.x] = 1;
}
__global__ void k_big(const int* g, int* p) {
  extern __shared__ int sm[];
  if (*g != 7) return;
  sm[threadIdx.x] = 1;
  __syncthreads();
  if (threadIdx.x == 0) p[blockIdx.x] = sm[5];
}
__global__ void k_sync(int* p, int iters) {
  cg::grid_group grid = cg::this_grid();
  for (int i = 0; i < iters; i++) {
    if (threadIdx.x == 0) atomicAdd(p + (blockIdx.x & 15), 1);
    grid.sync();
  }
}

int main() {
  int* d;
  cudaMalloc(&d, 1 << 20);
  cudaMemset(d, 0, 1 << 20);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int big = 100 * 1024;
  cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  auto run = [&](const char* what, bool alternate, int grid) {
    for (int rep = 0; rep < 3; rep++) {
      cudaEventRecord(a, s);
      for (int i = 0; i < 100; i++) {
        if (alternate && (i & 1)) k_big<<<grid, 256, big, s>>>(d, d + 16);
        else k_small<<<grid, 256, 0, s>>>(d, d + 16);
      }
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("%-34s grid %5d: %.2f us/launch\n", what, grid, ms * 10);
    }
  };
  for (int grid : {148, 888}) {
    run("same kernel (no carveout pref)", false, grid);
    run("alternating smem (no carveout pref)", true, grid);
  }
  cudaFuncSetAttribute(k_small, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaFuncSetAttribute(k_big, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  for (int grid : {148, 888}) {
    run("same kernel (carveout 100)", false, grid);
    run("alternating smem (carveout 100)", true, grid);
  }
  // graph of the alternating chain
  {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 100; i++) {
      if (i & 1) k_big<<<888, 256, big, s>>>(d, d + 16);
      else k_small<<<888, 256, 0, s>>>(d, d + 16);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int rep = 0; rep < 3; rep++) {
      cudaEventRecord(a, s);
      cudaGraphLaunch(ge, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("graph alternating (carveout 100) grid 888: %.2f us/launch\n", ms * 10);
    }
  }
  // cooperative grid sync cost
  for (int per_sm : {1, 2, 4}) {
    int grid = 148 * per_sm;
    int iters = 100;
    void* args[] = {&d, &iters};
    for (int rep = 0; rep < 3; rep++) {
      cudaEventRecord(a, s);
      cudaLaunchCooperativeKernel((void*)k_sync, grid, 256, args, 0, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("cooperative grid %4d x 256: %.2f us per grid.sync\n", grid, ms * 10);
    }
  }
  {
    int iters = 1;
    void* args[] = {&d, &iters};
    for (int rep = 0; rep < 5; rep++) {
      cudaEventRecord(a, s);
      cudaLaunchCooperativeKernel((void*)k_sync, 148, 1024, args, 0, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 4) printf("one cooperative launch 148x1024 with 1 sync: %.2f us\n", ms * 1e3);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
