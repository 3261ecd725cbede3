// micro-benchmark: host-side cost of the CUDA API calls one sr_sort call makes,
// and the event-measured cost of a call sequence shaped like the resident path
// (alloc, memset, cooperative launch, 64-B readback + sync, free) against a
// leaner one (cached workspace, in-kernel zeroing, mapped-memory completion flag).
#include <chrono>
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void k_coop(int* p, int* host_flag) {
  cg::this_grid().sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p[0] += 1;
    if (host_flag) {
      __threadfence_system();
      *(volatile int*)host_flag = p[0];
    }
  }
}
__global__ void k_plain(int* p) { if (blockIdx.x == 0 && threadIdx.x == 0) p[0] += 1; }
using clk = std::chrono::steady_clock;
static double us(clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count() * 1e6; }
int main() {
  cudaFree(0);
  cudaStream_t s;
  cudaStreamCreate(&s);
  int* d;
  cudaMalloc(&d, 1 << 20);
  cudaMemset(d, 0, 1 << 20);
  int* h;
  cudaHostAlloc(&h, 4096, cudaHostAllocMapped);
  int* hd;
  cudaHostGetDevicePointer(&hd, h, 0);
  cudaMemPool_t pool;
  cudaDeviceGetDefaultMemPool(&pool, 0);
  uint64_t thr = UINT64_MAX;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int R = 200;
  auto T = [&](const char* what, auto f) {
    for (int i = 0; i < 10; i++) f();
    cudaStreamSynchronize(s);
    auto t0 = clk::now();
    for (int i = 0; i < R; i++) f();
    auto t1 = clk::now();
    cudaStreamSynchronize(s);
    printf("%-44s %7.2f us/call (host)\n", what, us(t0, t1) / R);
  };
  T("cudaGetDevice", [&] { int dv; cudaGetDevice(&dv); });
  T("cudaPointerGetAttributes", [&] { cudaPointerAttributes at; cudaPointerGetAttributes(&at, d); });
  T("cudaMallocAsync+cudaFreeAsync 20MB", [&] { void* p; cudaMallocAsync(&p, 20 << 20, s); cudaFreeAsync(p, s); });
  T("cudaMemsetAsync 4KB", [&] { cudaMemsetAsync(d, 0, 4096, s); });
  T("kernel<<<148,512>>>", [&] { k_plain<<<148, 512, 0, s>>>(d); });
  T("cudaLaunchCooperativeKernel 148x512", [&] {
    int* nf = nullptr;
    void* args[] = {&d, &nf};
    cudaLaunchCooperativeKernel((void*)k_coop, 148, 512, args, 0, s);
  });
  T("cudaEventRecord", [&] { cudaEventRecord(a, s); });
  {
    int* hp;
    cudaHostAlloc(&hp, 4096, 0);
    T("memcpy D2H 64B + cudaStreamSynchronize", [&] {
      cudaMemcpyAsync(hp, d, 64, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
    });
    T("coop launch + D2H 64B + sync", [&] {
      int* nf = nullptr;
      void* args[] = {&d, &nf};
      cudaLaunchCooperativeKernel((void*)k_coop, 148, 512, args, 0, s);
      cudaMemcpyAsync(hp, d, 64, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
    });
    T("coop launch + spin on mapped flag", [&] {
      static int expect = 0;
      const int want = ++expect;
      *(volatile int*)h = -1;
      void* args[] = {&d, &hd};
      cudaLaunchCooperativeKernel((void*)k_coop, 148, 512, args, 0, s);
      while (*(volatile int*)h == -1) {
      }
      (void)want;
    });
    // event-measured sequences (what the bench sees)
    auto E = [&](const char* what, auto f) {
      float best = 1e9, sum = 0;
      for (int i = 0; i < 60; i++) {
        cudaStreamSynchronize(s);
        cudaEventRecord(a, s);
        f();
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (i >= 10) { sum += ms; best = ms < best ? ms : best; }
      }
      printf("%-44s %7.2f us mean  %7.2f us min (events)\n", what, sum / 50 * 1e3, best * 1e3);
    };
    E("seq: malloc+memset+coop+readback+free", [&] {
      void* p;
      cudaMallocAsync(&p, 20 << 20, s);
      cudaMemsetAsync(p, 0, 4096, s);
      int* nf = nullptr;
      void* args[] = {&d, &nf};
      cudaLaunchCooperativeKernel((void*)k_coop, 148, 512, args, 0, s);
      cudaMemcpyAsync(hp, d, 64, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      cudaFreeAsync(p, s);
    });
    E("seq: coop+readback", [&] {
      int* nf = nullptr;
      void* args[] = {&d, &nf};
      cudaLaunchCooperativeKernel((void*)k_coop, 148, 512, args, 0, s);
      cudaMemcpyAsync(hp, d, 64, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
    });
    E("seq: coop+mapped flag spin", [&] {
      *(volatile int*)h = -1;
      void* args[] = {&d, &hd};
      cudaLaunchCooperativeKernel((void*)k_coop, 148, 512, args, 0, s);
      while (*(volatile int*)h == -1) {
      }
    });
    E("seq: coop only (async)", [&] {
      int* nf = nullptr;
      void* args[] = {&d, &nf};
      cudaLaunchCooperativeKernel((void*)k_coop, 148, 512, args, 0, s);
    });
    E("seq: plain launch only (async)", [&] { k_plain<<<148, 512, 0, s>>>(d); });
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
