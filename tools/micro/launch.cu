// micro-benchmark: back-to-back launch cost of tiny kernels on one stream, and in a CUDA graph
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_empty(int* p) { if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1; }
__global__ void k_gate(const int* g, int* p) { if (*g != 7) return; if (threadIdx.x == 0) p[blockIdx.x] = 1; }
int main() {
  int* d; cudaMalloc(&d, 1 << 20); cudaMemset(d, 0, 1 << 20);
  cudaStream_t s; cudaStreamCreate(&s);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int grid : {1, 148, 1184}) {
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(a, s);
      for (int i = 0; i < 100; i++) k_gate<<<grid, 256, 0, s>>>(d, d + 16);
      cudaEventRecord(b, s); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("stream: grid %5d gated kernel: %.2f us/launch\n", grid, ms * 10);
    }
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 100; i++) k_gate<<<grid, 256, 0, s>>>(d, d + 16);
    cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0);
    for (int rep = 0; rep < 3; rep++) {
      cudaEventRecord(a, s); cudaGraphLaunch(ge, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("graph : grid %5d gated kernel: %.2f us/launch\n", grid, ms * 10);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
