// micro-benchmark: host cost of a cooperative launch vs a cooperative kernel
// node in an instantiated CUDA graph whose parameters are updated per launch
#include <chrono>
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
struct Args { int* p; long long pad[24]; };
__global__ void k_coop(Args a) {
  extern __shared__ int sm[];
  cg::this_grid().sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) a.p[0] += 1 + sm[0] * 0;
}
using clk = std::chrono::steady_clock;
int main() {
  cudaStream_t s; cudaStreamCreate(&s);
  Args a{}; cudaMalloc(&a.p, 64); cudaMemset(a.p, 0, 64);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int R = 300;
  auto T = [&](const char* what, auto f) {
    for (int i = 0; i < 10; i++) f();
    cudaStreamSynchronize(s);
    auto t0 = clk::now();
    for (int i = 0; i < R; i++) { f(); cudaStreamSynchronize(s); }
    auto t1 = clk::now();
    printf("%-40s %7.2f us/launch+sync\n", what, std::chrono::duration<double>(t1 - t0).count() * 1e6 / R);
  };
  T("cudaLaunchCooperativeKernel", [&] { void* args[] = {&a}; cudaLaunchCooperativeKernel((void*)k_coop, 148, 512, args, smem, s); });
  // graph
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaKernelNodeParams kp = {};
  void* args[] = {&a};
  kp.func = (void*)k_coop; kp.gridDim = dim3(148); kp.blockDim = dim3(512); kp.sharedMemBytes = smem; kp.kernelParams = args;
  cudaGraphNode_t node;
  printf("add node: %s\n", cudaGetErrorString(cudaGraphAddKernelNode(&node, g, nullptr, 0, &kp)));
  cudaLaunchAttributeValue v = {}; v.cooperative = 1;
  printf("set coop attr: %s\n", cudaGetErrorString(cudaGraphKernelNodeSetAttribute(node, cudaLaunchAttributeCooperative, &v)));
  cudaGraphExec_t ge;
  printf("instantiate: %s\n", cudaGetErrorString(cudaGraphInstantiate(&ge, g, 0)));
  T("graph launch (same params)", [&] { cudaGraphLaunch(ge, s); });
  T("graph set params + launch", [&] { a.pad[0]++; cudaGraphExecKernelNodeSetParams(ge, node, &kp); cudaGraphLaunch(ge, s); });
  int h; cudaMemcpy(&h, a.p, 4, cudaMemcpyDeviceToHost);
  printf("counter %d err=%s\n", h, cudaGetErrorString(cudaGetLastError()));
}
